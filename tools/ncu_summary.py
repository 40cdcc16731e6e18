"""Summarise gpurun_out ncu artefacts into profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py launches gpurun_out/launches_r01a.csv  > profiles/..._launches.txt
    python tools/ncu_summary.py full gpurun_out/prof_r01a.ncu-rep      > profiles/..._full.txt
"""
import collections
import csv
import io
import subprocess
import sys

FULL_METRICS = [
    "Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers", "l1tex__t_bytes.sum", "lts__t_bytes.sum",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) < len(h):
            continue
        name = r[ki].split("(")[0]
        name = name.replace("void ", "").split("<")[0]
        v = float(r[vi].replace(",", ""))
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    # NVTX class (the library's LaunchScope ranges) when captured with --nvtx
    ncol = next((i for i, c in enumerate(h) if "Push/Pop_Range" in c), None)
    byclass = collections.OrderedDict()
    if ncol is not None:
        for r in rows[hdr + 1:]:
            if len(r) < len(h):
                continue
            rng = r[ncol].strip()
            # '<tid>  "<default domain>:<range>:none:..."' -> <range>
            rng = rng.split('"')[1].split(":")[1] if '"' in rng else "(no range)"
            a = byclass.setdefault(rng, [0, 0.0])
            a[0] += 1
            a[1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu launch list ({path}): gpu__time_duration.sum, --clock-control none")
    print("# cold-cache, serialised per launch: compare SHARES, not absolutes")
    print(f"# {sum(v[0] for v in agg.values())} launches, {tot / 1e6:.3f} ms total")
    print(f"{'kernel':40s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:40s} {v[0]:8d} {v[1] / 1e6:10.3f} {100 * v[1] / tot:6.1f}%")
    if byclass:
        print("# by library kernel class (NVTX range)")
        for k, v in sorted(byclass.items(), key=lambda x: -x[1][1]):
            print(f"{k[:40]:40s} {v[0]:8d} {v[1] / 1e6:10.3f} {100 * v[1] / tot:6.1f}%")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print(f"# ncu --set full summary ({path})")
    for r in rows[2:]:
        for w in FULL_METRICS:
            if w in h:
                i = h.index(w)
                print(f"{w:80s} {r[i]} {units[i]}")
        print("---")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
