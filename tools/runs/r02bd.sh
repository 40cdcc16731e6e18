#!/bin/bash
# r02bd: producer-side device-scope fence (+ proxy fence) at the end of the panel kernel
TAG=r02bd
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
WF4DVAR_NVCC_FLAGS="-DTRSM_END_FENCE -DTMA_FENCE" python -c "from paper_2105_06975_b200 import build as b; b.build(force=True)" > gpurun_out/build_$TAG.log 2>&1
R="env CFG=3 NREP=3 MODE=P WF4DVAR_GEMM_TMA=1 timeout 600 python tools/diag/c4_race2.py"
TAGENV="tma1+trsm_end_fence+tma_fence" $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+trsm_end_fence+tma_fence (2)" $R >> gpurun_out/race_$TAG.log 2>&1
echo "race=$?" >> gpurun_out/status_$TAG
