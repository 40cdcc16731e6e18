#!/bin/bash
# r02n: re-verification after the container restart (HEAD b51ae50: deferred MINRES update,
# heat scan two columns per pass): smoke, full GPU suite, c3/c1/c4 bench, launch list,
# ncu --set full of the heat scan kernel on c3.
TAG=r02n
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
nvidia-smi > gpurun_out/nvsmi_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?" >> gpurun_out/status_$TAG
timeout 900 python bench.py > gpurun_out/bench_c3_$TAG.log 2>&1; echo "bench_c3=$?" >> gpurun_out/status_$TAG
WF4DVAR_MINRES_OVERLAP=0 timeout 900 python bench.py --tts-maxit 0 --no-cpu-baseline > gpurun_out/bench_c3_nodefer_$TAG.log 2>&1; echo "bench_c3nd=$?" >> gpurun_out/status_$TAG
CMD="python bench.py --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_heat -s 4 -c 3 -o gpurun_out/prof_heat_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu=$?" >> gpurun_out/status_$TAG
timeout 3000 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG
for cfg in 1 4; do timeout 900 python bench.py --config $cfg > gpurun_out/bench_c${cfg}_$TAG.log 2>&1; echo "c$cfg=$?" >> gpurun_out/status_$TAG; done
