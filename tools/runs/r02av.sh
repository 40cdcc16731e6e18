#!/bin/bash
# r02av: which co-residency matters for the TMA coupling-GEMM irreproducibility (r02au: one
# k_gemm_tma CTA per SM was reproducible).  pad 35000: two k_gemm_tma CTAs no longer fit
# one SM, a k_gemm_tma CTA + a k_trsm panel CTA still do; pad 20000: everything still pairs.
# Also: vectorised Z / X loads (this build) -- kernel + parity subset, c3 bench.
TAG=r02av
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?" >> gpurun_out/status_$TAG
R="env CFG=3 NREP=3 MODE=P timeout 600 python tools/diag/c4_race2.py"
TAGENV="tma2 (default)" $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+pad35000" WF4DVAR_GEMM_TMA=1 WF4DVAR_TMA_SMEM_PAD=35000 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+pad35000 (2)" WF4DVAR_GEMM_TMA=1 WF4DVAR_TMA_SMEM_PAD=35000 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+pad20000" WF4DVAR_GEMM_TMA=1 WF4DVAR_TMA_SMEM_PAD=20000 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma1+pad40000" WF4DVAR_GEMM_TMA=1 WF4DVAR_TMA_SMEM_PAD=40000 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma3+pad35000 (coupling only)" WF4DVAR_GEMM_TMA=3 WF4DVAR_TMA_SMEM_PAD=35000 $R >> gpurun_out/race_$TAG.log 2>&1
echo "race=$?" >> gpurun_out/status_$TAG
B="python bench.py --steps 20 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 600 $B > gpurun_out/bench_c3_${TAG}.log 2>&1
WF4DVAR_GEMM_TMA=1 WF4DVAR_TMA_SMEM_PAD=35000 timeout 600 $B > gpurun_out/bench_c3_${TAG}_tma1_pad35000.log 2>&1
echo "bench=$?" >> gpurun_out/status_$TAG
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_repro.py tests/test_gpu_parity.py tests/test_gpu_edge.py -m gpu -q -x > gpurun_out/pytest_sub_$TAG.log 2>&1; echo "pytest_sub=$?" >> gpurun_out/status_$TAG
