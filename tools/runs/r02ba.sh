#!/bin/bash
# r02ba: final verification of HEAD (16-byte pair stores, vectorised Z loads): smoke, default
# bench command, every other config, reference arm, launch list + GEMM capture of the default
# bench command, full GPU suite.
TAG=r02ba
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
nvidia-smi > gpurun_out/nvsmi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?" >> gpurun_out/status_$TAG
timeout 900 python bench.py > gpurun_out/bench_c3_$TAG.log 2>&1; echo "c3=$?" >> gpurun_out/status_$TAG
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG
timeout 300 python bench.py --config 0 --steps 50 --tts-maxit 3000 > gpurun_out/bench_c0_$TAG.log 2>&1; echo "c0=$?" >> gpurun_out/status_$TAG
timeout 600 python bench.py --config 1 > gpurun_out/bench_c1_$TAG.log 2>&1; echo "c1=$?" >> gpurun_out/status_$TAG
timeout 600 python bench.py --config 1 --solver minres --steps 30 > gpurun_out/bench_c1m_$TAG.log 2>&1; echo "c1m=$?" >> gpurun_out/status_$TAG
timeout 900 python bench.py --config 2 --steps 20 --tts-maxit 200 > gpurun_out/bench_c2_$TAG.log 2>&1; echo "c2=$?" >> gpurun_out/status_$TAG
timeout 1200 python bench.py --config 4 --tts-maxit 300 > gpurun_out/bench_c4_$TAG.log 2>&1; echo "c4=$?" >> gpurun_out/status_$TAG
timeout 900 python bench.py --config 5 --steps 20 --tts-maxit 1000 > gpurun_out/bench_c5_$TAG.log 2>&1; echo "c5=$?" >> gpurun_out/status_$TAG
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c3_$TAG.log 2>&1; echo "ref=$?" >> gpurun_out/status_$TAG
CMD="python bench.py --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --csv --log-file gpurun_out/launches_c3_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "gemm_dmma/" -s 6 -c 6 -o gpurun_out/prof_gemm_$TAG $CMD > gpurun_out/ncu_gemm_$TAG.log 2>&1
echo "ncu=$?" >> gpurun_out/status_$TAG
