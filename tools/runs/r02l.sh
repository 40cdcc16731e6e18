#!/bin/bash
# r02l: warp-scan heat kernel with two columns per pass (ILP 2) at R = 64/128/256 vs the
# thread-per-chunk form; apply_A / apply_P phase times; c1 under GMRES(50).
TAG=r02l
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c3_shape.py -q -rf -s -k "apply_A or full_size or heat or c3_shaped" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG
B="python bench.py --steps 12 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 2"
run() { name=$1; shift; env "$@" timeout 600 $B > gpurun_out/sweep_${name}_$TAG.log 2>&1; echo "$name=$?" >> gpurun_out/status_$TAG; }
run h128 X=1
run h64 WF4DVAR_HEAT_TILE=64
run h256 WF4DVAR_HEAT_TILE=256
run h0 WF4DVAR_HEAT_TILE=0
timeout 900 python bench.py --config 1 > gpurun_out/bench_c1_$TAG.log 2>&1; echo "c1=$?" >> gpurun_out/status_$TAG
