#!/bin/bash
# r02j: GMRES count check (recurrence noise envelope), D_hat^{-1} column-half split on two
# streams, host-path chunk count / copy order (e2e).
TAG=r02j
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -rf -s -k "c0_matches or host or AP" > gpurun_out/pytest_c0_$TAG.log 2>&1; echo "pytest_c0=$?" >> gpurun_out/status_$TAG
B="python bench.py --steps 12 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 4"
run() { name=$1; shift; env "$@" timeout 600 $B > gpurun_out/sweep_${name}_$TAG.log 2>&1; echo "$name=$?" >> gpurun_out/status_$TAG; }
run default X=1
run split WF4DVAR_DHAT_SPLIT=1
run hc1 WF4DVAR_HOST_CHUNKS=1
run hc2 WF4DVAR_HOST_CHUNKS=2
run x3first WF4DVAR_HOST_X3_FIRST=1
run x3first_hc2 WF4DVAR_HOST_X3_FIRST=1 WF4DVAR_HOST_CHUNKS=2
run inv WF4DVAR_EXPLICIT_INV=1
