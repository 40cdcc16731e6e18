mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01av.log 2>&1
timeout 900 python -m pytest tests/test_gpu_banded.py tests/test_gpu_paper_heat.py tests/test_gpu_ichol.py tests/test_gpu_rblock.py tests/test_gpu_kernels.py -q > gpurun_out/pytest_r01av.log 2>&1; echo "p=$?" >> gpurun_out/status_r01av
echo done >> gpurun_out/status_r01av
