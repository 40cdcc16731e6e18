mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01e.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_dist.py -x -q > gpurun_out/pytest_k_r01e.log 2>&1; echo "pytest_k=$?" >> gpurun_out/status_r01e
for S in 0 1; do echo "SK=$S"; WF4DVAR_GEMM_SK=$S python tools/kbench.py; done > gpurun_out/kbench_r01e.log 2>&1
for S in 0 1; do WF4DVAR_GEMM_SK=$S timeout 600 python bench.py --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_sk${S}_r01e.log 2>&1; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r01e.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r01e
