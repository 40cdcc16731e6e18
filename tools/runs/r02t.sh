#!/bin/bash
TAG=r02t
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
for env in "X=1" "WF4DVAR_HEAT_SEQ=0" "WF4DVAR_HEAT_SEQ=32" "WF4DVAR_GEMM_SK=0" "WF4DVAR_GEMM_TMA=0" "WF4DVAR_FORK=0"; do
  echo "== $env" >> gpurun_out/colindep_$TAG.log
  env $env timeout 600 python tools/diag/colindep.py 4 me >> gpurun_out/colindep_$TAG.log 2>&1
done
env X=1 timeout 600 python tools/diag/colindep.py 1 me >> gpurun_out/colindep_$TAG.log 2>&1
env X=1 timeout 600 python tools/diag/colindep.py 3 exact >> gpurun_out/colindep_$TAG.log 2>&1
