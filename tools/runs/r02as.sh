#!/bin/bash
# r02as: (1) probes of the TMA coupling-GEMM irreproducibility with the new knobs (L2
# eviction hints on the operand loads, L2 promotion of the tensor maps);
# (2) DRAM traffic of the cuBLAS DGEMM 8192^3 the bench times as its FP64 peak (comparator
# for roofline.traffic)
TAG=r02as
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
R="env CFG=4 NREP=4 MODE=P WF4DVAR_GEMM_TMA=3 timeout 600 python tools/diag/c4_race2.py"
TAGENV="tma3" $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma3+hint2" WF4DVAR_GEMM_L2HINT=2 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma3+promo0" WF4DVAR_TMA_L2PROMO=0 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma3+promo2" WF4DVAR_TMA_L2PROMO=2 $R >> gpurun_out/race_$TAG.log 2>&1
TAGENV="tma2(default)" WF4DVAR_GEMM_TMA=2 env CFG=4 NREP=4 MODE=P timeout 600 python tools/diag/c4_race2.py >> gpurun_out/race_$TAG.log 2>&1
echo "race=$?" >> gpurun_out/status_$TAG
CMD="python bench.py --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:Kernel2 -c 4 -o gpurun_out/traffic_cublas_$TAG $CMD > gpurun_out/ncu_cublas_$TAG.log 2>&1
echo "ncu=$?" >> gpurun_out/status_$TAG
