#!/bin/bash
TAG=r02ah
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest -q -rf tests/test_gpu_repro.py > gpurun_out/pytest_repro_$TAG.log 2>&1; echo "repro=$?" >> gpurun_out/status_$TAG
run() { name=$1; shift; env "$@" timeout 600 $B > gpurun_out/ab_${name}_$TAG.log 2>&1; echo "$name=$?" >> gpurun_out/status_$TAG; }
B="python bench.py --config 4 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run c4 X=1
run c4_g16 WF4DVAR_MULTIDOT_G=16
B="python bench.py --config 1 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run c1 X=1
run c1_g16 WF4DVAR_MULTIDOT_G=16
