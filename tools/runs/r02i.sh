#!/bin/bash
# r02i: 2-D TMA-staged GEMM (k_gemm_tma): kernel parity, kbench on/off, c3 step on/off,
# ncu capture of k_gemm_tma; host-path / halo-overlap / dist tests.
TAG=r02i
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_banded.py tests/test_gpu_edge.py -q -rf -x > gpurun_out/pytest_kern_$TAG.log 2>&1; echo "pytest_kern=$?" >> gpurun_out/status_$TAG
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_nccl1.py tests/test_gpu_parity.py -q -rf -k "dist or sharded or nccl or host or apply_A or AP or c0 or full_size" > gpurun_out/pytest_dist_$TAG.log 2>&1; echo "pytest_dist=$?" >> gpurun_out/status_$TAG
timeout 600 python tools/kbench.py --gemm-only > gpurun_out/kbench_tma_$TAG.log 2>&1; echo "kb_tma=$?" >> gpurun_out/status_$TAG
WF4DVAR_GEMM_TMA=0 timeout 600 python tools/kbench.py --gemm-only > gpurun_out/kbench_notma_$TAG.log 2>&1; echo "kb_notma=$?" >> gpurun_out/status_$TAG
B="python bench.py --steps 12 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 3"
timeout 600 $B > gpurun_out/sweep_tma_$TAG.log 2>&1; echo "tma=$?" >> gpurun_out/status_$TAG
WF4DVAR_GEMM_TMA=0 timeout 600 $B > gpurun_out/sweep_notma_$TAG.log 2>&1; echo "notma=$?" >> gpurun_out/status_$TAG
CMD="python bench.py --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tma -s 4 -c 3 -o gpurun_out/prof_tma_$TAG $CMD > gpurun_out/ncu_tma_$TAG.log 2>&1; echo "ncu_tma=$?" >> gpurun_out/status_$TAG
