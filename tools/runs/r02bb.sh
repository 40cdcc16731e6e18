#!/bin/bash
# r02bb: the new store-alignment kernel tests; more repeats of the pad-20000 probe (TMA-staged
# coupling GEMMs with the heat triple excluded) on configs[3] and [4], PA mode included
TAG=r02bb
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -rf > gpurun_out/pytest_kernels_$TAG.log 2>&1; echo "pytest_kernels=$?" >> gpurun_out/status_$TAG
for rep in 1 2 3; do
  TAGENV="tma1+pad20000 P run$rep" env CFG=3 NREP=3 MODE=P WF4DVAR_GEMM_TMA=1 WF4DVAR_TMA_SMEM_PAD=20000 timeout 600 python tools/diag/c4_race2.py >> gpurun_out/race_$TAG.log 2>&1
  TAGENV="tma1+pad20000 P run$rep" env CFG=4 NREP=4 MODE=P WF4DVAR_GEMM_TMA=1 WF4DVAR_TMA_SMEM_PAD=20000 timeout 600 python tools/diag/c4_race2.py >> gpurun_out/race_$TAG.log 2>&1
done
TAGENV="tma1+pad20000 PA" env CFG=3 NREP=3 MODE=PA WF4DVAR_GEMM_TMA=1 WF4DVAR_TMA_SMEM_PAD=20000 timeout 600 python tools/diag/c4_race2.py >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma2 (default) PA" env CFG=3 NREP=3 MODE=PA timeout 600 python tools/diag/c4_race2.py >> gpurun_out/race_$TAG.log 2>&1
echo "race=$?" >> gpurun_out/status_$TAG
