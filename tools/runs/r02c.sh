#!/bin/bash
# r02c: c3 step under the TRSM-apply default: knob sweep (super-block, panel width,
# left-looking, recursion, stream-K tail threshold, fork/join), kbench, ncu of k_trsm.
TAG=r02c
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_dist.py -q -x -k "apply_A or full_size or heat or sharded" > gpurun_out/pytest_heat_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG
B="python bench.py --steps 12 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run() { name=$1; shift; env "$@" timeout 600 $B > gpurun_out/sweep_${name}_$TAG.log 2>&1; echo "$name=$?" >> gpurun_out/status_$TAG; }
run default X=1
run sb512 WF4DVAR_TRSM_SB=512
run sb2048 WF4DVAR_TRSM_SB=2048
run nb16 WF4DVAR_TRSM_NB=16
run nb64 WF4DVAR_TRSM_NB=64
run left WF4DVAR_TRSM_LEFT=1
run leaf512 WF4DVAR_TRSM_LEAF=512
run leaf1024 WF4DVAR_TRSM_LEAF=1024
run sktail60 WF4DVAR_GEMM_SK_TAIL=60
run nofork WF4DVAR_FORK=0
run inv WF4DVAR_EXPLICIT_INV=1
run heatold WF4DVAR_HEAT_TILE=0
timeout 600 python tools/kbench.py > gpurun_out/kbench_$TAG.log 2>&1; echo "kbench=$?" >> gpurun_out/status_$TAG
CMD="python bench.py --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu_launch=$?" >> gpurun_out/status_$TAG
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_trsm -s 8 -c 4 -o gpurun_out/prof_trsm_$TAG $CMD > gpurun_out/ncu_trsm_$TAG.log 2>&1; echo "ncu_trsm=$?" >> gpurun_out/status_$TAG
