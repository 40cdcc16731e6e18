#!/bin/bash
# r02g: full GPU suite (per-block parity, c1/c3-shape/c4 solve parity, host-path column
# chunks) + smoke + default bench (c3, with time-to-1e-8) + c4 bench.
TAG=r02g
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?" >> gpurun_out/status_$TAG
timeout 3600 python -m pytest tests -m gpu -q -rf -s > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG
timeout 900 python bench.py > gpurun_out/bench_c3_$TAG.log 2>&1; echo "bench_c3=$?" >> gpurun_out/status_$TAG
timeout 900 python bench.py --config 4 --tts-maxit 0 > gpurun_out/bench_c4_$TAG.log 2>&1; echo "bench_c4=$?" >> gpurun_out/status_$TAG
