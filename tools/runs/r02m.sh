#!/bin/bash
# r02m: fused CGS2 pass (first projection + second inner products, k_axpy_multidot):
# GMRES parity tests, c4 / c1 steps fused vs unfused.
TAG=r02m
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c1.py tests/test_gpu_c4.py tests/test_gpu_dist.py tests/test_gpu_paper_heat.py -q -rf -s -k "gmres or c1 or c4 or batched or sharded" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG
for cfg in 4 1; do
timeout 900 python bench.py --config $cfg --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c${cfg}_fused_$TAG.log 2>&1; echo "c${cfg}f=$?" >> gpurun_out/status_$TAG
WF4DVAR_CGS2_FUSED=0 timeout 900 python bench.py --config $cfg --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c${cfg}_unfused_$TAG.log 2>&1; echo "c${cfg}u=$?" >> gpurun_out/status_$TAG
done
