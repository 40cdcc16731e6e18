#!/bin/bash
# r02az: do the TMA operand loads see stale L1 lines left by an earlier in-place epilogue
# (Z = Y read through L1)?  Build with the epilogue Z loads L2-only (ld.global.cg).
TAG=r02az
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
WF4DVAR_NVCC_FLAGS="-DGEMM_Z_LDCG" python -c "from paper_2105_06975_b200 import build as b; b.build(force=True)" > gpurun_out/build_$TAG.log 2>&1
R="env CFG=3 NREP=3 MODE=P WF4DVAR_GEMM_TMA=1 timeout 600 python tools/diag/c4_race2.py"
TAGENV="tma1+z_ldcg" $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+z_ldcg (2)" $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+z_ldcg (3)" $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+z_ldcg cfg4" env CFG=4 NREP=4 MODE=P WF4DVAR_GEMM_TMA=1 timeout 600 python tools/diag/c4_race2.py >> gpurun_out/race_$TAG.log 2>&1
echo "race=$?" >> gpurun_out/status_$TAG
