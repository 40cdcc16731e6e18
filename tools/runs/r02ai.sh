#!/bin/bash
TAG=r02ai
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
WF4DVAR_NVCC_FLAGS="-DTRSM_PROXY_FENCE" python -c "from paper_2105_06975_b200 import build as b; b.build(force=True)" > gpurun_out/build_$TAG.log 2>&1
env CFG=4 NREP=4 MODE=P TAGENV="tma3+trsm_fence" WF4DVAR_GEMM_TMA=3 timeout 600 python tools/diag/c4_race2.py >> gpurun_out/race_$TAG.log 2>&1
env CFG=3 NREP=3 MODE=P TAGENV="tma1+trsm_fence" WF4DVAR_GEMM_TMA=1 timeout 600 python tools/diag/c4_race2.py >> gpurun_out/race_$TAG.log 2>&1
