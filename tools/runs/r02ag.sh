#!/bin/bash
TAG=r02ag
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
for cfg in 3 1 4; do
  env CFG=$cfg NREP=4 MODE=PA TAGENV=default timeout 900 python tools/diag/c4_race2.py >> gpurun_out/race_$TAG.log 2>&1
done
env CFG=3 NREP=3 MODE=P TAGENV=tma1 WF4DVAR_GEMM_TMA=1 timeout 900 python tools/diag/c4_race2.py >> gpurun_out/race_$TAG.log 2>&1
