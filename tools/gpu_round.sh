#!/bin/bash
# One gpurun call: GPU tests, smoke, bench lines, ncu launch list + one full capture.
# usage (from the repo root on the box): bash tools/gpu_round.sh TAG [ncu-kernel-regex] [skip] [count] [what]
#   what: "all" (default) | "bench" (skip pytest/smoke)
TAG=${1:-r01}
KRE=${2:-k_gemm}
SKIP=${3:-60}
CNT=${4:-15}
WHAT=${5:-all}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
if [ "$WHAT" = "all" ]; then
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?" >> gpurun_out/status_$TAG
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG
fi
timeout 900 python bench.py > gpurun_out/bench_c3_$TAG.log 2>&1; echo "bench_c3=$?" >> gpurun_out/status_$TAG
timeout 600 python bench.py --config 1 > gpurun_out/bench_c1_$TAG.log 2>&1; echo "bench_c1=$?" >> gpurun_out/status_$TAG
CMD="python bench.py --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KRE -s $SKIP -c $CNT -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu=$?" >> gpurun_out/status_$TAG
