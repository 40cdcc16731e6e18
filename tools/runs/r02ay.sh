#!/bin/bash
# r02ay: the triple (two k_gemm_tma CTAs + one 8-warp k_heat_iir_seq CTA) fills the SM's
# register file exactly (2 x 4 x 32 x 192 + 8 x 32 x 64 = 65536).  Probes: heat kernel
# capped at 56 registers (triple still fits, file not full) and at 72 (triple impossible).
TAG=r02ay
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
R="env CFG=3 NREP=3 MODE=P WF4DVAR_GEMM_TMA=1 timeout 600 python tools/diag/c4_race2.py"
for NR in 56 72; do
  WF4DVAR_NVCC_FLAGS="-DHEAT_SEQ_MAXNREG=$NR" python -c "from paper_2105_06975_b200 import build as b; b.build(force=True)" > gpurun_out/build_${TAG}_$NR.log 2>&1
  TAGENV="tma1+heat_maxnreg$NR" $R >> gpurun_out/race_$TAG.log 2>&1
  TAGENV="tma1+heat_maxnreg$NR (2)" $R >> gpurun_out/race_$TAG.log 2>&1
done
echo "race=$?" >> gpurun_out/status_$TAG
