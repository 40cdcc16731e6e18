#!/bin/bash
# r02aw: every shared-memory pad of k_gemm_tma made the TMA-staged coupling GEMMs
# reproducible (r02av), including 20000 B which keeps two CTAs per SM but moves the kernel's
# carve-out to the maximum.  Probe: no pad, preferred carve-out 100%; pad 20000 timing.
TAG=r02aw
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
R="env CFG=3 NREP=3 MODE=P WF4DVAR_GEMM_TMA=1 timeout 600 python tools/diag/c4_race2.py"
TAGENV="tma1" $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+carve100" WF4DVAR_TMA_CARVEOUT=100 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+carve100 (2)" WF4DVAR_TMA_CARVEOUT=100 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+pad20000 (2)" WF4DVAR_TMA_SMEM_PAD=20000 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+pad4096" WF4DVAR_TMA_SMEM_PAD=4096 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+pad80" WF4DVAR_TMA_SMEM_PAD=80 $R >> gpurun_out/race_$TAG.log 2>&1
R4="env CFG=4 NREP=4 MODE=P WF4DVAR_GEMM_TMA=1 timeout 600 python tools/diag/c4_race2.py"
TAGENV="tma1+carve100 cfg4" WF4DVAR_TMA_CARVEOUT=100 $R4 >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+pad20000 cfg4" WF4DVAR_TMA_SMEM_PAD=20000 $R4 >> gpurun_out/race_$TAG.log 2>&1
echo "race=$?" >> gpurun_out/status_$TAG
B="python bench.py --steps 20 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 600 $B > gpurun_out/bench_c3_${TAG}.log 2>&1
WF4DVAR_GEMM_TMA=1 WF4DVAR_TMA_CARVEOUT=100 timeout 600 $B > gpurun_out/bench_c3_${TAG}_tma1_carve100.log 2>&1
WF4DVAR_GEMM_TMA=1 WF4DVAR_TMA_SMEM_PAD=20000 timeout 600 $B > gpurun_out/bench_c3_${TAG}_tma1_pad20000.log 2>&1
echo "bench=$?" >> gpurun_out/status_$TAG
