mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01bv.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01bv.log 2>&1; echo "smoke=$?" >> gpurun_out/status_r01bv
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_banded.py tests/test_gpu_ichol.py -q > gpurun_out/pytest_r01bv.log 2>&1; echo "p=$?" >> gpurun_out/status_r01bv
timeout 300 python bench.py --config 5 --steps 30 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c5_r01bv.log 2>&1
echo done >> gpurun_out/status_r01bv
