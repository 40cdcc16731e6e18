#!/bin/bash
TAG=r02af
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
WF4DVAR_GEMM_TMA=3 timeout 600 python tools/diag/c4_race3.py > gpurun_out/c4race3_$TAG.log 2>&1
echo "== WF4DVAR_GEMM_TMA=3 WF4DVAR_GEMM_SK=0" >> gpurun_out/c4race3_$TAG.log
WF4DVAR_GEMM_TMA=3 WF4DVAR_GEMM_SK=0 timeout 600 python tools/diag/c4_race3.py >> gpurun_out/c4race3_$TAG.log 2>&1
