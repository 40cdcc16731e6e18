"""Measure the FP64 denominators on the box (MEASURED_PEAKS.json has none):
cuBLAS DGEMM (torch.matmul float64) at 8192^3, burst (best of 10) and sustained
(back to back for ~4 s), with SM clocks sampled during the sustained loop.
Writes gpurun_out/fp64_peaks.json."""
import json
import os
import subprocess
import time

import torch


def main():
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    burst = 2 * n ** 3 / best / 1e12
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw",
                            "--format=csv,noheader,nounits", "-lms", "200"],
                           stdout=subprocess.PIPE, text=True)
    t0 = time.time()
    e0 = torch.cuda.Event(True)
    e1 = torch.cuda.Event(True)
    e0.record()
    it = 0
    while time.time() - t0 < 4.0:
        for _ in range(4):
            a @ b
        it += 4
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    smi.terminate()
    out = smi.communicate()[0].strip().splitlines()
    clocks = [float(l.split(",")[0]) for l in out if l.strip()]
    sus = 2 * n ** 3 * it / (e0.elapsed_time(e1) / 1e3) / 1e12
    res = dict(dgemm_tflops_burst=burst, dgemm_tflops_sustained=sus, n=n,
               sm_mhz_median=sorted(clocks)[len(clocks) // 2] if clocks else None,
               how="torch.matmul float64 8192^3 (cuBLAS DGEMM): best of 10, and back to back ~4 s")
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(res, open("gpurun_out/fp64_peaks.json", "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
