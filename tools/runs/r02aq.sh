#!/bin/bash
# r02aq: verification of HEAD after the container restore (c84c808: 16-column slab
# small GEMM): smoke, bench c3 (default command) / c2 / c1 / c4, launch list of the
# default bench command, full GPU suite.
TAG=r02aq
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
nvidia-smi > gpurun_out/nvsmi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?" >> gpurun_out/status_$TAG
timeout 900 python bench.py > gpurun_out/bench_c3_$TAG.log 2>&1; echo "c3=$?" >> gpurun_out/status_$TAG
timeout 600 python bench.py --config 2 --steps 20 --tts-maxit 200 > gpurun_out/bench_c2_$TAG.log 2>&1; echo "c2=$?" >> gpurun_out/status_$TAG
timeout 600 python bench.py --config 1 > gpurun_out/bench_c1_$TAG.log 2>&1; echo "c1=$?" >> gpurun_out/status_$TAG
timeout 1200 python bench.py --config 4 --tts-maxit 300 > gpurun_out/bench_c4_$TAG.log 2>&1; echo "c4=$?" >> gpurun_out/status_$TAG
CMD="python bench.py --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --csv --log-file gpurun_out/launches_c3_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "ncu=$?" >> gpurun_out/status_$TAG
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG
