mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01af.log 2>&1
timeout 900 python -m pytest tests/test_gpu_banded.py tests/test_gpu_paper_heat.py tests/test_gpu_ichol.py tests/test_gpu_kernels.py tests/test_gpu_rblock.py -q -x > gpurun_out/pytest_banded_r01af.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r01af
timeout 600 python bench.py --config 5 --steps 20 --tts-maxit 400 > gpurun_out/bench_c5_r01af.log 2>&1; echo "c5=$?" >> gpurun_out/status_r01af
WF4DVAR_BANDED=0 timeout 600 python bench.py --config 5 --steps 20 --tts-maxit 0 --no-cpu-baseline > gpurun_out/bench_c5_dense_r01af.log 2>&1; echo "c5d=$?" >> gpurun_out/status_r01af
timeout 600 python bench.py --config 3 --steps 10 --tts-maxit 0 --no-cpu-baseline > gpurun_out/bench_c3_r01af.log 2>&1; echo "c3=$?" >> gpurun_out/status_r01af
