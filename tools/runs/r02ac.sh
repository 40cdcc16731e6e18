#!/bin/bash
# r02ac: TMA off for the TRSM coupling GEMMs (default 2): reproducibility, c4/c1 GMRES
# parity tests, c3/c4 step times against TMA everywhere.
TAG=r02ac
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
env NREP=3 MODE=PA TAGENV=default timeout 600 python tools/diag/c4_race2.py >> gpurun_out/c4race2_$TAG.log 2>&1
env TAGENV=default timeout 900 python tools/diag/c4_race.py exact >> gpurun_out/c4race_$TAG.log 2>&1
timeout 1500 python -m pytest -q -rf tests/test_gpu_c4.py tests/test_gpu_c1.py tests/test_gpu_kernels.py > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG
B="python bench.py --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run() { name=$1; shift; env "$@" timeout 600 $B > gpurun_out/ab_${name}_$TAG.log 2>&1; echo "$name=$?" >> gpurun_out/status_$TAG; }
run c3 X=1
run c3_tma1 WF4DVAR_GEMM_TMA=1
B="python bench.py --config 4 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run c4 X=1
