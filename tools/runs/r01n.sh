mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01n.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_outer.py tests/test_gpu_spectral.py -q > gpurun_out/pytest_new_r01n.log 2>&1; echo "pytest_new=$?" >> gpurun_out/status_r01n
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01n.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r01n
