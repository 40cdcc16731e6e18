#!/bin/bash
TAG=r02y
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
for e in "TAGENV=default" "TAGENV=fork0 WF4DVAR_FORK=0" "TAGENV=heatscan WF4DVAR_HEAT_SEQ=0" "TAGENV=tma0 WF4DVAR_GEMM_TMA=0" "TAGENV=seq32 WF4DVAR_HEAT_SEQ=32" "TAGENV=w4 WF4DVAR_HEAT_SEQW=4" "TAGENV=prio0 WF4DVAR_AUX_PRIORITY=0" "TAGENV=sk0 WF4DVAR_GEMM_SK=0"; do
  env $e timeout 600 python tools/diag/c4_race2.py >> gpurun_out/c4race2_$TAG.log 2>&1
done
