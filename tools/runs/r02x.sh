#!/bin/bash
TAG=r02x
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
for e in "TAGENV=default" "TAGENV=fork0 WF4DVAR_FORK=0" "TAGENV=sk0 WF4DVAR_GEMM_SK=0" "TAGENV=heatscan WF4DVAR_HEAT_SEQ=0" "TAGENV=graphs0 WF4DVAR_GRAPHS=0"; do
  env $e timeout 900 python tools/diag/c4_race.py exact >> gpurun_out/c4race_$TAG.log 2>&1
done
env TAGENV=default timeout 900 python tools/diag/c4_race.py diag >> gpurun_out/c4race_$TAG.log 2>&1
