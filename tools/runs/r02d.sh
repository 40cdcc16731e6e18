#!/bin/bash
# r02d: warp-scan heat IIR kernel (parity + c3 step), TRSM recursion leaf sweep, c4 step.
TAG=r02d
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_dist.py -q -x -k "apply_A or full_size or heat or sharded or c0" > gpurun_out/pytest_heat_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG
B="python bench.py --steps 12 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run() { name=$1; shift; env "$@" timeout 600 $B > gpurun_out/sweep_${name}_$TAG.log 2>&1; echo "$name=$?" >> gpurun_out/status_$TAG; }
run scan256 X=1
run scan128 WF4DVAR_HEAT_TILE=128
run heatold WF4DVAR_HEAT_TILE=0
run leaf256 WF4DVAR_TRSM_LEAF=256
run leaf512 WF4DVAR_TRSM_LEAF=512
run leaf768 WF4DVAR_TRSM_LEAF=768
run leaf512_old WF4DVAR_TRSM_LEAF=512 WF4DVAR_HEAT_TILE=0
for cfg in 1 2 4; do
timeout 900 python bench.py --config $cfg --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c${cfg}_$TAG.log 2>&1; echo "c$cfg=$?" >> gpurun_out/status_$TAG
WF4DVAR_HEAT_TILE=0 timeout 900 python bench.py --config $cfg --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c${cfg}_old_$TAG.log 2>&1; echo "c${cfg}old=$?" >> gpurun_out/status_$TAG
done
