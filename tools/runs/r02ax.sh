#!/bin/bash
# r02ax: is the third co-resident CTA the column-sequential heat kernel (45 KB of shared
# memory, cp.async staging)?  TMA-staged coupling GEMMs without pad, heat kernel variants
# that cannot share an SM with two k_gemm_tma CTAs (R = 32: 78 KB) or use no cp.async tile
# (thread-per-chunk form).  Also: k_trsm X loads back to scalar (r02av measured the
# vectorised form slower), c3 bench.
TAG=r02ax
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
R="env CFG=3 NREP=3 MODE=P WF4DVAR_GEMM_TMA=1 timeout 600 python tools/diag/c4_race2.py"
TAGENV="tma1+heat_seq32" WF4DVAR_HEAT_SEQ=32 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+heat_seq32 (2)" WF4DVAR_HEAT_SEQ=32 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+heat_seq0_tile0 (thread per chunk)" WF4DVAR_HEAT_SEQ=0 WF4DVAR_HEAT_TILE=0 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+heat_seq0 (warp scan)" WF4DVAR_HEAT_SEQ=0 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+heat_seqw4 (4 warps, 29 KB)" WF4DVAR_HEAT_SEQW=4 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1" $R >> gpurun_out/race_$TAG.log 2>&1
echo "race=$?" >> gpurun_out/status_$TAG
B="python bench.py --steps 20 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 600 $B > gpurun_out/bench_c3_${TAG}.log 2>&1
echo "bench=$?" >> gpurun_out/status_$TAG
