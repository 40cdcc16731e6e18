#!/bin/bash
# r02be: more repeats of the heat-kernel variants with every GEMM TMA-staged (configs[3], P)
TAG=r02be
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
R="env CFG=3 NREP=3 MODE=P WF4DVAR_GEMM_TMA=1 timeout 600 python tools/diag/c4_race2.py"
for rep in 1 2 3; do
  TAGENV="tma1+heat_seqw4 run$rep" WF4DVAR_HEAT_SEQW=4 $R >> gpurun_out/race_$TAG.log 2>&1
  TAGENV="tma1+heat_seq32 run$rep" WF4DVAR_HEAT_SEQ=32 $R >> gpurun_out/race_$TAG.log 2>&1
done
echo "race=$?" >> gpurun_out/status_$TAG
