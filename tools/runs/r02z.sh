#!/bin/bash
TAG=r02z
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
env TAGENV=default timeout 600 python tools/diag/gemm_race.py >> gpurun_out/gemmrace_$TAG.log 2>&1
env TAGENV=tma0 WF4DVAR_GEMM_TMA=0 timeout 600 python tools/diag/gemm_race.py >> gpurun_out/gemmrace_$TAG.log 2>&1
for e in "TAGENV=default" "TAGENV=tma0 WF4DVAR_GEMM_TMA=0" "TAGENV=fork0 WF4DVAR_FORK=0"; do
  env NREP=4 $e timeout 600 python tools/diag/c4_race2.py >> gpurun_out/c4race2_$TAG.log 2>&1
done
