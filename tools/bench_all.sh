#!/bin/bash
# Bench lines for every BASELINE.json config (the default bench is configs[3]).
# usage on the box: bash tools/bench_all.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 300 python bench.py --config 0 --steps 50 --tts-maxit 3000 > gpurun_out/bench_c0_$TAG.log 2>&1; echo "c0=$?" >> gpurun_out/status_all_$TAG
timeout 600 python bench.py --config 1 --steps 30 > gpurun_out/bench_c1_$TAG.log 2>&1; echo "c1=$?" >> gpurun_out/status_all_$TAG
timeout 900 python bench.py --config 2 --steps 20 --tts-maxit 200 > gpurun_out/bench_c2_$TAG.log 2>&1; echo "c2=$?" >> gpurun_out/status_all_$TAG
timeout 900 python bench.py --config 3 --steps 20 > gpurun_out/bench_c3_$TAG.log 2>&1; echo "c3=$?" >> gpurun_out/status_all_$TAG
timeout 1200 python bench.py --config 4 --steps 20 --tts-maxit 300 > gpurun_out/bench_c4_$TAG.log 2>&1; echo "c4=$?" >> gpurun_out/status_all_$TAG
timeout 900 python bench.py --config 5 --steps 20 --tts-maxit 400 > gpurun_out/bench_c5_$TAG.log 2>&1; echo "c5=$?" >> gpurun_out/status_all_$TAG
