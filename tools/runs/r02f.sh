#!/bin/bash
# r02f: warp-scan heat IIR with cp.async staging (parity + c3/c1 step), TRSM leaf-512
# default, configs[1] GMRES(50) grid tests against the oracle.
TAG=r02f
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
WF4DVAR_HEAT_TILE=256 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_dist.py -q -x -k "apply_A or full_size or heat or sharded or c0" > gpurun_out/pytest_heat_$TAG.log 2>&1; echo "pytest_heatscan=$?" >> gpurun_out/status_$TAG
B="python bench.py --steps 12 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run() { name=$1; shift; env "$@" timeout 600 $B > gpurun_out/sweep_${name}_$TAG.log 2>&1; echo "$name=$?" >> gpurun_out/status_$TAG; }
run default X=1
run scan256 WF4DVAR_HEAT_TILE=256
run scan128 WF4DVAR_HEAT_TILE=128
for t in 0 256 128; do
WF4DVAR_HEAT_TILE=$t timeout 600 python bench.py --config 1 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c1_h${t}_$TAG.log 2>&1; echo "c1_h$t=$?" >> gpurun_out/status_$TAG
done
timeout 1800 python -m pytest tests/test_gpu_c1.py -q -rf -s > gpurun_out/pytest_c1_$TAG.log 2>&1; echo "pytest_c1=$?" >> gpurun_out/status_$TAG
