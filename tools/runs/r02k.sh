#!/bin/bash
# r02k: full GPU suite (TMA for every BK=16 GEMM shape, host chunks = 2, GMRES true-residual
# fallback) + smoke + default bench.
TAG=r02k
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?" >> gpurun_out/status_$TAG
timeout 3600 python -m pytest tests -m gpu -q -rf -s > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG
timeout 900 python bench.py > gpurun_out/bench_c3_$TAG.log 2>&1; echo "bench_c3=$?" >> gpurun_out/status_$TAG
for cfg in 1 4; do timeout 900 python bench.py --config $cfg > gpurun_out/bench_c${cfg}_$TAG.log 2>&1; echo "c$cfg=$?" >> gpurun_out/status_$TAG; done
