mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01an.log 2>&1
timeout 900 python -m pytest tests/test_gpu_banded.py tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_r01an.log 2>&1; echo "p=$?" >> gpurun_out/status_r01an
B="python bench.py --config 3 --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 300 $B > gpurun_out/c3_r01an.log 2>&1
timeout 300 $B > gpurun_out/c3b_r01an.log 2>&1
timeout 300 python bench.py --config 5 --steps 20 --tts-maxit 0 --no-cpu-baseline > gpurun_out/c5_r01an.log 2>&1
timeout 300 python bench.py --config 4 --steps 20 --tts-maxit 0 --no-cpu-baseline > gpurun_out/c4_r01an.log 2>&1
echo done >> gpurun_out/status_r01an
