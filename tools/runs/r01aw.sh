mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01aw.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -k "graphs or stream_k" > gpurun_out/pytest_r01aw.log 2>&1; echo "p=$?" >> gpurun_out/status_r01aw
echo done >> gpurun_out/status_r01aw
