mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01au.log 2>&1
timeout 900 python -m pytest tests/test_gpu_banded.py tests/test_gpu_paper_heat.py tests/test_gpu_ichol.py tests/test_gpu_rblock.py -q -x > gpurun_out/pytest_r01au.log 2>&1; echo "p=$?" >> gpurun_out/status_r01au
timeout 300 python bench.py --config 5 --steps 20 --tts-maxit 400 > gpurun_out/c5_r01au.log 2>&1
timeout 300 python bench.py --config 1 --steps 30 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c1_r01au.log 2>&1
echo done >> gpurun_out/status_r01au
