#!/bin/bash
# r02q: dataflow TRSM engaged (dense factors with registered triangle ranges), whole-
# triangle DF for n <= 2048, heat seq R = 16 default; reading A35 solution tests.
TAG=r02q
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?" >> gpurun_out/status_$TAG
timeout 1200 python -m pytest -q -rf -x tests/test_gpu_kernels.py > gpurun_out/pytest_kern_$TAG.log 2>&1; echo "kern=$?" >> gpurun_out/status_$TAG
B="python bench.py --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run() { name=$1; shift; env "$@" timeout 600 $B > gpurun_out/ab_${name}_$TAG.log 2>&1; echo "$name=$?" >> gpurun_out/status_$TAG; }
run c3 X=1
run c3_nodf WF4DVAR_TRSM_DF=0
run c3_whole WF4DVAR_TRSM_LEAF=0 WF4DVAR_TRSM_SB=4096
run c3_leaf1024 WF4DVAR_TRSM_LEAF=1024
run c3_leaf256 WF4DVAR_TRSM_LEAF=256
B="python bench.py --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 --N 31"
run c3_N31 X=1
run c3_N31_nodf WF4DVAR_TRSM_DF=0
B="python bench.py --config 1 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run c1 X=1
run c1_nodf WF4DVAR_TRSM_DF=0
B="python bench.py --config 1 --solver minres --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run c1m X=1
run c1m_nodf WF4DVAR_TRSM_DF=0
B="python bench.py --config 4 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run c4 X=1
run c4_nodf WF4DVAR_TRSM_DF=0
B="python bench.py --config 5 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run c5 X=1
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG
