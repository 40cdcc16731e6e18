mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01x.log 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k gemm > gpurun_out/pytest_k_r01x.log 2>&1; echo "pytest_k=$?" >> gpurun_out/status_r01x
for B in 1 0; do echo "BULK=$B"; WF4DVAR_GEMM_BULK=$B timeout 300 python tools/kbench.py --gemm-only; done > gpurun_out/kbench_r01x.log 2>&1
for B in 1 0; do WF4DVAR_GEMM_BULK=$B timeout 400 python bench.py --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_bulk${B}_r01x.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x > gpurun_out/pytest_r01x.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r01x
echo done >> gpurun_out/status_r01x
