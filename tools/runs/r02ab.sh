#!/bin/bash
TAG=r02ab
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
for e in "TAGENV=tma_not_trsm WF4DVAR_GEMM_TMA=2" "TAGENV=tma_only_trsm WF4DVAR_GEMM_TMA=3" "TAGENV=default_sk0 WF4DVAR_GEMM_SK=0" "TAGENV=default_nb WF4DVAR_TRSM_SB=2048"; do
  env NREP=3 MODE=P $e timeout 600 python tools/diag/c4_race2.py >> gpurun_out/c4race2_$TAG.log 2>&1
done
