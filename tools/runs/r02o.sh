#!/bin/bash
# r02o: MINRES overlap flag fix (active count initialised to m), heat scan kernel with
# base rows prefetched into registers, scan kernel for every size again: the r02n
# failures, smoke, c3 bench, ncu of the heat kernel.
TAG=r02o
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?" >> gpurun_out/status_$TAG
timeout 1500 python -m pytest -q -rf -s tests/test_gpu_parity.py tests/test_gpu_c1.py tests/test_gpu_c3_shape.py tests/test_gpu_dist.py tests/test_gpu_ichol.py tests/test_gpu_nccl1.py tests/test_gpu_outer.py tests/test_gpu_paper_heat.py -k "minres or gmres or solve or c1 or c3_shaped or exact_L or outer" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG
timeout 900 python bench.py --tts-maxit 0 > gpurun_out/bench_c3_$TAG.log 2>&1; echo "bench_c3=$?" >> gpurun_out/status_$TAG
CMD="python bench.py --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_heat -s 4 -c 3 -o gpurun_out/prof_heat_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu=$?" >> gpurun_out/status_$TAG
