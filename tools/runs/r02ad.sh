#!/bin/bash
TAG=r02ad
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
for f in "-DTMA_INVAL" "-DTMA_FENCE" "-DTMA_INVAL -DTMA_FENCE"; do
  WF4DVAR_NVCC_FLAGS="$f" python -c "from paper_2105_06975_b200 import build as b; b.build(force=True)" > gpurun_out/build_$TAG.log 2>&1
  env NREP=3 MODE=P TAGENV="tma1 $f" WF4DVAR_GEMM_TMA=1 timeout 600 python tools/diag/c4_race2.py >> gpurun_out/c4race2_$TAG.log 2>&1
done
