#!/bin/bash
# r02h (after the TMA GEMM): full-GMRES diagnosis on c0, c3 time-to-1e-8 for both apply
# modes, bench lines for every config, shard projections (one shard's windows of
# configs[3] at N+1 = 64/32/16), the reference arm, ncu launch list + GEMM capture
# (roofline.traffic) + heat-scan capture of the default c3 step.
TAG=r02h
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python tools/gmres_full_diag.py > gpurun_out/gmres_full_diag_$TAG.log 2>&1; echo "diag=$?" >> gpurun_out/status_$TAG
timeout 1500 python tools/tts.py --config 3 --maxit 3000 --out gpurun_out/tts_c3_$TAG.json > gpurun_out/tts_c3_$TAG.log 2>&1; echo "tts=$?" >> gpurun_out/status_$TAG
for cfg in 0 1 2 5; do
timeout 900 python bench.py --config $cfg > gpurun_out/bench_c${cfg}_$TAG.log 2>&1; echo "c$cfg=$?" >> gpurun_out/status_$TAG
done
for n in 63 31 15; do
timeout 900 python bench.py --N $n --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_N${n}_$TAG.log 2>&1; echo "N$n=$?" >> gpurun_out/status_$TAG
WF4DVAR_EXPLICIT_INV=1 timeout 900 python bench.py --N $n --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_N${n}_inv_$TAG.log 2>&1; echo "N${n}inv=$?" >> gpurun_out/status_$TAG
done
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/ref_c3_$TAG.log 2>&1; echo "ref=$?" >> gpurun_out/status_$TAG
CMD="python bench.py --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD > gpurun_out/plain_$TAG.log 2>&1; echo "plain=$?" >> gpurun_out/status_$TAG
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu_launch=$?" >> gpurun_out/status_$TAG
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "gemm_dmma/" -s 6 -c 6 -o gpurun_out/prof_gemm_$TAG $CMD > gpurun_out/ncu_gemm_$TAG.log 2>&1; echo "ncu_gemm=$?" >> gpurun_out/status_$TAG
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_heat_iir -s 20 -c 3 -o gpurun_out/prof_heat_$TAG $CMD > gpurun_out/ncu_heat_$TAG.log 2>&1; echo "ncu_heat=$?" >> gpurun_out/status_$TAG
