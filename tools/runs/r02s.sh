#!/bin/bash
# r02s: multidot grid reverted; DF determinism test; stream-K tail threshold sweep for the
# TRSM recursion's coupling GEMMs (c3 / c4).
TAG=r02s
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 1800 python -m pytest -q -rf tests/test_gpu_kernels.py tests/test_gpu_c4.py tests/test_gpu_c1.py > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG
B="python bench.py --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run() { name=$1; shift; env "$@" timeout 600 $B > gpurun_out/ab_${name}_$TAG.log 2>&1; echo "$name=$?" >> gpurun_out/status_$TAG; }
run c3 X=1
run c3_sk55 WF4DVAR_GEMM_SK_TAIL=55
run c3_sk80 WF4DVAR_GEMM_SK_TAIL=80
B="python bench.py --config 4 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run c4 X=1
run c4_sk55 WF4DVAR_GEMM_SK_TAIL=55
run c4_sk80 WF4DVAR_GEMM_SK_TAIL=80
