#!/usr/bin/env python
"""Benchmark: saddle-point A+P applies/sec (FP64) and time-to-1e-8 residual, % of roofline.

Workload (default): BASELINE.json configs[3] -- linear heat s=4096, N=127
(128 windows), p=1024, 64 RHS, P_D with the parallel-in-time L_M(4) and R_hat = R,
preconditioned MINRES; other configs via --config.

One STEP = one batched MINRES (GMRES for configs[4]) iteration over all m RHS = one
A apply + one P apply + the Krylov vector work.
value = A+P applies/s of the whole job: with N > 1 ranks (torchrun) the time
windows of ONE batch are sharded over the ranks (NCCL halos + Krylov allreduce,
scaling "strong", default --shard time) or every rank solves its own batch
(--shard batch, scaling "weak").

Timing: W warm-up steps, then exactly K steps inside ONE wf4dvar_solve call (tol
below reach; the solve's initialisation -- one extra P apply -- is inside the timed
region, which only makes the number pessimistic), bracketed by barrier + cuda
synchronize, CUDA events on the library's stream, max over ranks.  Inputs are larger
than L2 at configs[1..4] (each configs[3] vector is 604 MB).  The per-kernel-class
roofline comes from a second, instrumented pass of the same K steps.
"""
import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CELLS = {
    0: dict(shape="PD", lhat="LM", k=3, rhat="exact", solver="minres"),
    # BJ.c1: "GMRES(restart 50) with each of the paper's preconditioner variants" -- the
    # bench line takes P_D, L_M(4), R_hat = R; tools/grid.py c1 times all 60 cells
    1: dict(shape="PD", lhat="LM", k=4, rhat="exact", solver="gmres"),
    2: dict(shape="PD", lhat="LM", k=4, rhat="exact", solver="minres"),
    3: dict(shape="PD", lhat="LM", k=4, rhat="exact", solver="minres"),
    4: dict(shape="PI", lhat="LM", k=4, rhat="exact", solver="gmres"),
    # NEXT-1 workload with the paper's preconditioner choices: R_block by Algorithm 1,
    # IC(0) factors of B_RR / Q_RR (ridge 0.01)
    5: dict(shape="PD", lhat="LM", k=4, rhat="block", solver="minres", factor="ichol",
            ridge=0.01, block_tol=0.05),
}
PC_KEYS = ("shape", "lhat", "k", "rhat", "factor", "ridge", "block_tol", "pvec", "block",
           "apply_mode")


FP64_ALU_PEAK = 148 * 64 * 2 * 1.965e9 / 1e12   # TFLOP/s, FP64 DFMA pipe at max SM clock


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed Krylov iterations (default 20; GMRES: one restart cycle, 50; "
                         "GMRES step counts are rounded up to whole restart cycles so the "
                         "CGS2 cost is averaged over complete cycles)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--m", type=int, default=None, help="override the RHS batch width")
    ap.add_argument("--N", type=int, default=None,
                    help="override N (experiments: a G-way time shard of configs[3] is N+1 = 128/G)")
    ap.add_argument("--shape", default=None)
    ap.add_argument("--lhat", default=None)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--rhat", default=None)
    ap.add_argument("--block", type=int, default=None, help="R_block uniform block size")
    ap.add_argument("--apply-mode", default=None, choices=["trsm", "inverse"],
                    help="dense D_hat/R_hat blocks: triangular solves (default) or the opt-in "
                         "explicit inverses (DESIGN.md reading A32)")
    ap.add_argument("--restart", type=int, default=50)
    ap.add_argument("--solver", default=None, choices=["minres", "gmres"])
    ap.add_argument("--tts-maxit", type=int, default=2000,
                    help="cap for the time-to-1e-8 solve (0 disables it)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--shard", default="time", choices=["time", "batch"],
                    help="N > 1: 'time' = the windows of ONE batch sharded over the ranks "
                         "(NCCL halos + allreduce, strong scaling; SURVEY 8(e)); 'batch' = an "
                         "independent batch per rank (no collective, weak scaling)")
    return ap.parse_args()


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """SM clock / throttle-reason sampler running during the timed region (the recipe's
    clocks line).  NVML (nvidia-ml-py) in a thread every 20 ms; nvidia-smi writing to a
    file as the fallback (a pipe would lose its block-buffered output when the sampler
    is terminated after a sub-second timed region -- the round-1 bench lines carried no
    clock record for that reason)."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, torch, device):
        self.torch, self.device = torch, device
        self.samples, self.mx, self.reasons, self.err = [], None, set(), None
        self.proc = None

    def _nvml_handle(self):
        import pynvml as N
        N.nvmlInit()
        pr = self.torch.cuda.get_device_properties(self.device)
        want = (getattr(pr, "pci_domain_id", 0), pr.pci_bus_id, pr.pci_device_id)
        for i in range(N.nvmlDeviceGetCount()):
            h = N.nvmlDeviceGetHandleByIndex(i)
            pci = N.nvmlDeviceGetPciInfo(h)
            if (pci.domain, pci.bus, pci.device) == want:
                return N, h
        return N, N.nvmlDeviceGetHandleByIndex(self.device)

    def __enter__(self):
        import threading
        self.stop = threading.Event()
        try:
            N, h = self._nvml_handle()
            get_r = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons
            self.mx = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))

            def loop():
                while True:
                    try:
                        self.samples.append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
                        bits = int(get_r(h))
                        for bit, nm in self.REASONS.items():
                            if bits & bit:
                                self.reasons.add(nm)
                    except Exception as e:   # pragma: no cover
                        self.err = repr(e)
                    if self.stop.wait(0.02):
                        break
            self.th = threading.Thread(target=loop, daemon=True)
            self.th.start()
            self.src = "nvml"
        except Exception as e:
            self.err = repr(e)
            self.th = None
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            self.fname = os.path.join("/tmp", f"bench_clocks_{os.getpid()}.csv")
            try:
                self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                              "--format=csv,noheader,nounits", "-lms", "50",
                                              "-f", self.fname], stderr=subprocess.DEVNULL)
                self.src = "nvidia-smi"
            except Exception as e2:
                self.err += " / " + repr(e2)
        return self

    def __exit__(self, *a):
        if self.th is not None:
            time.sleep(0.03)
            self.stop.set()
            self.th.join()
        elif self.proc is not None:
            time.sleep(0.3)
            self.proc.terminate()
            self.proc.wait()
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            try:
                for l in open(self.fname):
                    f = [x.strip() for x in l.split(",")]
                    try:
                        self.samples.append(float(f[0]))
                        self.mx = float(f[1])
                    except (ValueError, IndexError):
                        continue
                    for nm, v in zip(names, f[2:6]):
                        if v.lower().startswith("active"):
                            self.reasons.add(nm)
            except OSError as e:
                self.err = repr(e)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.mx, "reasons": [],
                    "error": f"no clock samples ({self.err})"}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "source": getattr(self, "src", None)}


def measure_dgemm_peak(torch, dev):
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    del a, b
    torch.cuda.empty_cache()
    return 2 * n ** 3 / best / 1e12


def cell_of(args):
    cell = dict(CELLS[args.config])
    for key in ("shape", "lhat", "k", "rhat", "block", "apply_mode"):
        v = getattr(args, key)
        if v is not None:
            cell[key] = v
    if cell["shape"] == "PI":
        cell["solver"] = "gmres"
    if args.solver:
        cell["solver"] = args.solver
    return cell


def steps_for(args, cell):
    """Timed steps: --steps, default 20; for GMRES(m_r) whole restart cycles (>= one),
    so the CGS2 work (growing with the Arnoldi index) is averaged over full cycles."""
    k = args.steps if args.steps is not None else (args.restart if cell["solver"] == "gmres" else 20)
    if cell["solver"] == "gmres" and k % args.restart:
        k = (k // args.restart + 1) * args.restart
    return k


def workload_name(config):
    return (f"BASELINE.json configs[{config}]" if config <= 4 else
            "NEXT-1 paper heat workload (SURVEY 8(f); not a BASELINE.json config)")


def sample_problem(SC, config):
    """The oracle's bounded sample of a config: ONE RHS column and at most 16 of its
    windows (every window costs the same in the blockwise oracle, so per-apply time
    scales linearly with W)."""
    N = SC.CONFIGS[config]["N"]
    Ns = min(N, 15)
    return SC.make_problem(config, seed0=0, m=1, N=Ns), (N + 1) / (Ns + 1)


def oracle_sample(prob, cell, reps=1):
    """CPU oracle (test infrastructure) on ONE RHS column: seconds per A+P apply."""
    from oracle.saddle import Precond, Saddle
    from synth.layout import to_paper_order
    sad = Saddle(prob, col=0)
    opc = Precond(shape=cell["shape"], lhat=cell["lhat"], k=cell["k"], rhat=cell["rhat"],
                  ridge=cell.get("ridge", 0.0), factor=cell.get("factor", "chol"),
                  block_tol=cell.get("block_tol", float("inf")),
                  pvec=tuple(cell["pvec"]) if cell.get("pvec") else None)
    v = np.random.Generator(np.random.PCG64(7)).standard_normal((2 * prob.s + prob.p) * prob.W)
    sad.apply_Pinv(opc, v)          # factorisations (setup) outside the timed sample
    t0 = time.perf_counter()
    for _ in range(reps):
        sad.apply_A(sad.apply_Pinv(opc, v))
    return (time.perf_counter() - t0) / reps


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([d.get("num_threads", 1) for d in info] or [os.cpu_count()])
    except Exception:
        return os.cpu_count()


def run_reference(args):
    ws, rank, local = dist_setup()
    if rank != 0:
        return
    from synth import configs as SC
    cell = cell_of(args)
    args.steps = steps_for(args, cell)
    prob, wscale = sample_problem(SC, args.config)
    if cell["rhat"] == "block" and "pvec" not in cell and "pvec" in prob.extra:
        cell["pvec"] = prob.extra["pvec"]
    m_full = args.m or SC.CONFIGS[args.config]["m"]
    # bounded sample: one untimed warm-up apply (the oracle's factorisations), then as
    # many of the K steps as fit a ~150 s budget
    t1 = oracle_sample(prob, cell, 1)
    reps = max(1, min(args.steps, int(150.0 / max(t1, 1e-9))))
    t = oracle_sample(prob, cell, reps) * wscale
    val = 1.0 / (t * m_full)
    cores = blas_threads()
    sample = (f"{reps} timed A+P applies of the blockwise oracle on 1 of {m_full} RHS columns "
              f"and {prob.W} of {SC.CONFIGS[args.config]['N'] + 1} windows (s={prob.s}, "
              f"p={prob.p}; factorisations in an untimed warm-up apply), scaled to the full "
              f"batch and window count")
    line = dict(impl="reference", metric="saddle-point A+P applies/sec (FP64)", value=val,
                unit="A+P applies/s", n_gpus=args.gpus, steps=args.steps, warmup=args.warmup,
                ms_per_step=t * m_full * 1e3, higher_is_better=True, scaling="weak",
                vs_baseline=None, dtype="f64", data="synthetic",
                config=dict(workload=workload_name(args.config), cell=cell,
                            s=prob.s, p=prob.p, N=SC.CONFIGS[args.config]["N"], m=m_full),
                cpu_baseline=dict(value=val, unit="A+P applies/s", cores=cores, kind="oracle",
                                  sample=sample),
                e2e=dict(value=val, unit="A+P applies/s", h2d_bytes_per_step=0,
                         d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import paper_2105_06975_b200 as W
    from synth import configs as SC

    ws, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    cell = cell_of(args)
    args.steps = steps_for(args, cell)
    cfgm = SC.CONFIGS[args.config]["m"]
    m = args.m or cfgm
    time_shard = ws > 1 and args.shard == "time"
    prob = SC.make_problem(args.config, seed0=0 if time_shard else rank * m, m=m, N=args.N)
    stream = torch.cuda.Stream(device=dev)
    if cell["rhat"] == "block" and "pvec" not in cell and "pvec" in prob.extra:
        cell["pvec"] = prob.extra["pvec"]     # Algorithm 1 on the workload's block structure
    pc = {k: cell[k] for k in PC_KEYS if k in cell}
    dkw = {}
    if time_shard:
        ids = [W.nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(ids, src=0)
        dkw = dict(rank=rank, world=ws, nccl_id=ids[0])
    ctx = W.Context.from_problem(prob, pc, device=local, stream=stream.cuda_stream, **dkw)
    peak_fp64 = measure_dgemm_peak(torch, dev) if rank == 0 else None
    rhs = prob.rhs
    if time_shard:
        rhs = W.local_windows(prob.rhs, prob.s, prob.p, prob.W, m, ctx.w_begin, ctx.w_end)
    n_local = rhs.size
    b = torch.from_numpy(rhs).to(dev)
    x = torch.empty_like(b)
    solver = cell["solver"]
    kw = dict(solver=solver, tol=1e-300, restart=args.restart, mark_tol=1e-8)

    # warm-up (also allocates the Krylov workspace)
    with torch.cuda.stream(stream):
        ctx.solve(b, x, maxit=max(1, args.warmup), check_every=10 ** 6, **kw)
    torch.cuda.synchronize(dev)

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    l0 = ctx.launch_count
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with Clocks(torch, local) as clk:
        barrier()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        rep = ctx.solve(b, x, maxit=args.steps, check_every=10 ** 6, **kw)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
    launches = ctx.launch_count - l0
    secs_total = e0.elapsed_time(e1) / 1e3
    # the K steps are the K Krylov iterations: the solver's initialisation (MINRES:
    # z_1 = P^{-1} b, ~one extra P apply) is measured by the library's own events on the
    # same stream and taken out (reported as init_ms)
    secs = secs_total - max(0.0, float(rep.get("seconds_init", 0.0)))
    if ws > 1:
        t = torch.tensor([secs], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        secs = float(t.item())
    steps = args.steps
    units = 1 if time_shard else ws       # A+P applies of the whole job per step
    value = units * steps / secs

    # per-kernel-class rates: the same K steps again with the library's CUDA-event
    # instrumentation on (launches serialised on the library stream while profiling,
    # so concurrent kernels do not inflate one another's durations)
    ctx.profile_enable(True)
    ctx.solve(b, x, maxit=args.steps, check_every=10 ** 6, **kw)
    prof = ctx.profile_read()
    ctx.profile_enable(False)

    # the two operator applies alone (device buffers, CUDA events on the library stream):
    # where a step's time goes between A and P (the rest is the Krylov vector work)
    phases = {}
    if ws == 1:
        xa = torch.from_numpy(np.random.Generator(np.random.PCG64(6)).standard_normal(n_local)).to(dev)
        ya = torch.empty_like(xa)
        for name, fn in (("apply_A", ctx.apply_A), ("apply_P", ctx.apply_P)):
            with torch.cuda.stream(stream):
                fn(xa, ya)
                q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                q0.record(stream)
                for _ in range(5):
                    fn(xa, ya)
                q1.record(stream)
            torch.cuda.synchronize(dev)
            phases[name + "_ms"] = q0.elapsed_time(q1) / 5
        del xa, ya

    # end-to-end: the public API with HOST buffers (H2D + A+P + D2H every step)
    xh = torch.from_numpy(np.random.Generator(np.random.PCG64(5)).standard_normal(n_local)).pin_memory()
    yh = torch.empty(n_local, dtype=torch.float64).pin_memory()
    ctx.apply_AP_host(xh.numpy(), yh.numpy())
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        ctx.apply_AP_host(xh.numpy(), yh.numpy())
    e2e_secs = time.perf_counter() - t0
    if ws > 1:
        t = torch.tensor([e2e_secs], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_secs = float(t.item())
    e2e_val = units * args.e2e_steps / e2e_secs

    # time-to-1e-8 (one real solve; reported, capped)
    tts = None
    if args.tts_maxit > 0:
        r = ctx.solve(b, x, solver=solver, tol=1e-8, maxit=args.tts_maxit, restart=args.restart,
                      mark_tol=1e-8, check_every=10)
        tts = dict(seconds=r["seconds_to_mark"] if r["seconds_to_mark"] >= 0 else None,
                   iterations=int(r["iters_to_mark"]) if r["iters_to_mark"] >= 0 else None,
                   maxit=args.tts_maxit, reached=bool(r["seconds_to_mark"] >= 0),
                   max_relres_at_exit=float(np.max(r["relres"])),
                   median_iters=float(np.median(r["iters"])))

    if rank != 0:
        return
    # roofline of the dominant kernel class (largest share of the profiled pass)
    dom = max(prof, key=lambda k: prof[k]["ms"])
    tot_ms = sum(v["ms"] for v in prof.values())
    d = prof[dom]
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    fp64_src = ("cuBLAS DGEMM 8192^3 measured live in this run (MEASURED_PEAKS.json has no "
                "FP64 entry)")
    if dom in ("gemm_dmma", "trsm_dmma", "trsm_update_dmma"):
        achieved = d["flops"] / (d["ms"] / 1e3) / 1e12
        roof = dict(bound="tensor", achieved=achieved, peak=peak_fp64, unit="TFLOP/s",
                    frac=achieved / peak_fp64, peak_source=fp64_src)
    elif dom == "model_stencil" and prob.model == "l96":
        # matrix-free RK4 tangent/adjoint recomputation: FP64 ALU (DFMA) bound
        achieved = d["flops"] / (d["ms"] / 1e3) / 1e12
        roof = dict(bound="alu", achieved=achieved, peak=FP64_ALU_PEAK, unit="TFLOP/s",
                    frac=achieved / FP64_ALU_PEAK,
                    peak_source="derived: 148 SMs x 64 FP64 FMA/clk x 2 flops x 1.965 GHz "
                                "(DESIGN.md section 5)")
    else:
        achieved = d["bytes"] / (d["ms"] / 1e3) / 1e9
        roof = dict(bound="hbm", achieved=achieved, peak=hbm, unit="GB/s", frac=achieved / hbm,
                    peak_source="MEASURED_PEAKS.json hbm_gbs")
    roof.update(kernel=dom, launches=d["launches"],
                flops_per_launch=d["flops"] / max(d["launches"], 1),
                bytes_per_launch=d["bytes"] / max(d["launches"], 1),
                share_of_step=d["ms"] / tot_ms if tot_ms else None, traffic=None,
                how=("algorithmic bytes" if roof["bound"] == "hbm" else
                     "algorithmic flops (2MNK per GEMM, 2 per FMA otherwise)") +
                    " / CUDA-event time of the class's launches in a profiled pass of the "
                    "same K steps")
    traffic_file = os.path.join(ROOT, "profiles", f"ncu_traffic_c{args.config}.json")
    if os.path.exists(traffic_file):
        tr = json.load(open(traffic_file)).get(dom)
        if tr:
            roof["traffic"] = tr.get("dram_bytes_per_launch")
            roof["traffic_source"] = tr.get("source")
    # roofline of the whole step (BJ north_star: "the fused apply_A+apply_P step"):
    # T_roof = max(algorithmic flops / FP64 peak, algorithmic bytes / HBM peak)
    # over the whole timed solve (its initialisation included on both sides, so the
    # ratio is consistent): all algorithmic work of the instrumented pass vs the
    # measured time of the un-instrumented one
    F = sum(v["flops"] for v in prof.values())
    By = sum(v["bytes"] for v in prof.values())
    t_roof = max(F / (peak_fp64 * 1e12), By / (hbm * 1e9))
    # second, dependency-aware bound: every kernel class at its own roofline, the classes
    # back to back (a Krylov step's vector work needs the operator's output and the next
    # operator apply needs the orthogonalised vector, so the tensor-bound and the
    # HBM-bound phases cannot overlap in one batch); frac_serial >= frac
    t_roof_ser = sum(max(v["flops"] / (peak_fp64 * 1e12), v["bytes"] / (hbm * 1e9))
                     for v in prof.values())
    step_roof = dict(flops_per_step=F / steps, bytes_per_step=By / steps,
                     t_roof_ms=t_roof / steps * 1e3, t_step_ms=secs_total / steps * 1e3,
                     frac=t_roof / secs_total, profiled_pass_ms_per_step=tot_ms / steps,
                     t_roof_serial_ms=t_roof_ser / steps * 1e3,
                     frac_serial=t_roof_ser / secs_total,
                     note="per step = per timed solve / K (solver initialisation included); "
                          "t_roof = max(all flops / FP64 peak, all bytes / HBM peak) (perfect "
                          "overlap of compute and memory phases); t_roof_serial = sum over "
                          "kernel classes of max(class flops / FP64 peak, class bytes / HBM)")
    kernels = {k: dict(launches=v["launches"], ms=round(v["ms"], 3),
                       tflops=(v["flops"] / (v["ms"] / 1e3) / 1e12) if v["ms"] else None,
                       gbs=(v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] else None)
               for k, v in prof.items() if v["launches"]}
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        p1, wscale = sample_problem(SC, args.config)
        t1 = oracle_sample(p1, cell, 1) * wscale
        cpu = dict(value=1.0 / (t1 * m), unit="A+P applies/s", cores=blas_threads(), kind="oracle",
                   sample=f"one A+P apply of the blockwise oracle on 1 of {m} RHS columns and "
                          f"{p1.W} of {prob.W} windows (s={prob.s}, p={prob.p}), factorisations "
                          f"untimed, scaled to {m} columns x {prob.W} windows")
    line = dict(metric="saddle-point A+P applies/sec (FP64)", value=value, unit="A+P applies/s",
                n_gpus=ws, steps=steps, warmup=args.warmup, ms_per_step=secs / steps * 1e3,
                init_ms=(secs_total - secs) * 1e3,
                higher_is_better=True, scaling="strong" if time_shard else "weak", vs_baseline=None, dtype="f64",
                data="synthetic",
                config=dict(workload=workload_name(args.config),
                            desc=SC.CONFIGS[args.config]["desc"], cell=cell, s=prob.s, p=prob.p,
                            N=prob.N, m=m, step="one batched Krylov iteration (1 A + 1 P apply)",
                            l2="inputs larger than L2 (no flush needed)",
                            parallelism=(f"time windows sharded over {ws} ranks (NCCL one-state "
                                         f"halos + Krylov allreduce)") if time_shard else
                                        f"independent batch per rank x{ws}"),
                roofline=roof, step_roofline=step_roof, cpu_baseline=cpu,
                e2e=dict(value=e2e_val, unit="A+P applies/s", h2d_bytes_per_step=n_local * 8 * ws,
                         d2h_bytes_per_step=n_local * 8 * ws,
                         how="wf4dvar_apply_AP_host: pinned host x -> device, A+P, y -> host"),
                gpu_launches=launches, clocks=clk.summary(), time_to_1e8=tts, kernels=kernels,
                phases=phases,
                counters=dict(n_apply_A=rep["n_apply_A"], n_apply_P=rep["n_apply_P"]))
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
