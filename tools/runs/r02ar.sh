#!/bin/bash
# r02ar: L2 eviction hints on the TMA GEMM operand streams (A evict_last, X evict_first):
# DRAM traffic per covariance product and step time, hint off / on, raster group 32 / 16 / 24
TAG=r02ar
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?" >> gpurun_out/status_$TAG
B="python bench.py --steps 20 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
for cfg in "0 0" "1 0" "1 16" "1 24" "0 16"; do
  set -- $cfg
  E="WF4DVAR_GEMM_L2HINT=$1"; [ "$2" != "0" ] && E="$E WF4DVAR_GEMM_GM=$2"
  env $E timeout 600 $B > gpurun_out/bench_c3_${TAG}_h$1_g$2.log 2>&1; echo "bench h$1 g$2=$?" >> gpurun_out/status_$TAG
done
CMD="python bench.py --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
for cfg in "0 0" "1 0" "1 16" "1 24"; do
  set -- $cfg
  E="WF4DVAR_GEMM_L2HINT=$1"; [ "$2" != "0" ] && E="$E WF4DVAR_GEMM_GM=$2"
  env $E timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "gemm_dmma/" -s 6 -c 6 -o gpurun_out/traffic_${TAG}_h$1_g$2 $CMD > gpurun_out/ncu_${TAG}_h$1_g$2.log 2>&1
  echo "ncu h$1 g$2=$?" >> gpurun_out/status_$TAG
done
