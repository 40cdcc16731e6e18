"""Build profiles/ncu_traffic_c3.json (the bench line's roofline.traffic) from an
`ncu --set full --nvtx --nvtx-include gemm_dmma/` capture: DRAM bytes (read + write)
per covariance-GEMM CALL -- a call is one k_gemm launch, or a k_gemm launch of the
data-parallel waves followed by its k_gemm_sk stream-K tail.

usage: python tools/traffic_json.py REP.ncu-rep ROUND_TAG > profiles/ncu_traffic_c3.json
"""
import csv
import io
import json
import subprocess
import sys


def main():
    rep, tag = sys.argv[1], sys.argv[2]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
                          "launch__grid_size"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    col = {k: h.index(k) for k in ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum",
                                   "dram__bytes_write.sum", "launch__grid_size")}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1, "us": 1e-3, "ns": 1e-6}

    def val(r, k):
        return float(r[col[k]].replace(",", "")) * scale.get(units[col[k]], 1)

    calls, cur = [], None
    for r in data:
        name = r[col["Kernel Name"]]
        b = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
        ms = val(r, "gpu__time_duration.sum")
        grid = int(float(r[col["launch__grid_size"]]))
        if "k_gemm_sk" in name:
            if cur is not None:   # else: the tail of a call whose k_gemm was not captured
                cur["dram_bytes"] += b
                cur["ms"] += ms
                cur["kernels"] += f" + k_gemm_sk grid {grid}"
                calls.append(cur)
            cur = None
            continue
        if cur is not None:
            calls.append(cur)
        cur = dict(kernels=f"k_gemm grid {grid}", dram_bytes=b, ms=ms)
    # a trailing k_gemm may still lack its stream-K tail (capture ended): drop it
    # unless its grid is not a stream-K data-parallel part (grid % 296 != 0)
    if cur is not None and int(cur["kernels"].split()[-1]) % 296 != 0:
        calls.append(cur)
    per = sum(c["dram_bytes"] for c in calls) / max(1, len(calls))
    json.dump({"gemm_dmma": {
        "dram_bytes_per_launch": per,
        "per_launch": calls,
        "source": f"ncu --set full --nvtx --nvtx-include gemm_dmma/ on bench.py --steps 2 ({tag}): "
                  "dram__bytes_read.sum + dram__bytes_write.sum per covariance-GEMM call "
                  "(data-parallel k_gemm + its stream-K tail), averaged over the captured calls"}},
        sys.stdout, indent=1)


if __name__ == "__main__":
    main()
