mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01v.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ichol.py tests/test_gpu_edge.py -q -x > gpurun_out/pytest_r01v.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r01v
timeout 900 python bench.py --config 5 --steps 20 --tts-maxit 400 > gpurun_out/bench_c5_r01v.log 2>&1; echo "c5=$?" >> gpurun_out/status_r01v
timeout 600 python bench.py --config 3 --shape PI --steps 5 --tts-maxit 400 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_PI_r01v.log 2>&1; echo "c3pi=$?" >> gpurun_out/status_r01v
echo done >> gpurun_out/status_r01v
