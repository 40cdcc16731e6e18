#!/bin/bash
# r02v: dataflow TRSM with X staged at start and the last dependency's G block staged
# before its flag; c1 A/B; c3 leaf panel-width experiments.
TAG=r02v
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?" >> gpurun_out/status_$TAG
timeout 1200 python -m pytest -q -rf tests/test_gpu_kernels.py tests/test_gpu_c1.py -k "trsm or minres or c1_gmres50_cell" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG
run() { name=$1; shift; env "$@" timeout 600 $B > gpurun_out/ab_${name}_$TAG.log 2>&1; echo "$name=$?" >> gpurun_out/status_$TAG; }
B="python bench.py --config 1 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run c1 X=1
B="python bench.py --config 1 --solver minres --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run c1m X=1
run c1m_nodf WF4DVAR_TRSM_DF=0
B="python bench.py --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run c3_nb16 WF4DVAR_TRSM_NB=16
run c3_nb64 WF4DVAR_TRSM_NB=64
CMD1="python bench.py --config 1 --solver minres --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1_$TAG.csv $CMD1 > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "ncu=$?" >> gpurun_out/status_$TAG
