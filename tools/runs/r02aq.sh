# 16-column slabs in the small DMMA GEMM: bench c2, smoke, GEMM/L96 parity
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02aq.log 2>&1
B="python bench.py --config 2 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 300 $B > gpurun_out/bench_c2_r02aq.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02aq.log 2>&1; echo "smoke=$?" >> gpurun_out/status_r02aq
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r02aq.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r02aq
timeout 300 python bench.py --config 0 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c0_r02aq.log 2>&1
