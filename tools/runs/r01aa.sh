mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01aa.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ichol.py tests/test_gpu_kernels.py -q -x > gpurun_out/pytest_r01aa.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r01aa
timeout 900 python bench.py --config 5 --steps 20 --tts-maxit 400 > gpurun_out/bench_c5_r01aa.log 2>&1; echo "c5=$?" >> gpurun_out/status_r01aa
timeout 400 python bench.py --N 15 --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_N15_r01aa.log 2>&1
echo done >> gpurun_out/status_r01aa
