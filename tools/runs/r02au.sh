#!/bin/bash
# r02au: probes of the TMA coupling-GEMM irreproducibility on configs[3] (P_D, every GEMM
# TMA-staged: fails in every run so far): tensor maps read from global memory instead of
# the parameter space; aux streams without priority; one k_gemm_tma CTA per SM; stream-K off
TAG=r02au
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
R="env CFG=3 NREP=3 MODE=P WF4DVAR_GEMM_TMA=1 timeout 600 python tools/diag/c4_race2.py"
TAGENV="tma1" $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+desc_global" WF4DVAR_TMA_DESC_GLOBAL=1 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+desc_global (2)" WF4DVAR_TMA_DESC_GLOBAL=1 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+nopriority" WF4DVAR_AUX_PRIORITY=0 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+pad40000" WF4DVAR_TMA_SMEM_PAD=40000 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+sk0" WF4DVAR_GEMM_SK=0 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+desc_global cfg4" WF4DVAR_TMA_DESC_GLOBAL=1 env CFG=4 NREP=4 MODE=P WF4DVAR_GEMM_TMA=1 timeout 600 python tools/diag/c4_race2.py >> gpurun_out/race_$TAG.log 2>&1
echo "race=$?" >> gpurun_out/status_$TAG
