#!/bin/bash
TAG=r02aa
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
for mode in A P; do
for e in "TAGENV=default" "TAGENV=tma0 WF4DVAR_GEMM_TMA=0"; do
  env NREP=3 MODE=$mode $e timeout 600 python tools/diag/c4_race2.py >> gpurun_out/c4race2_$TAG.log 2>&1
done; done
