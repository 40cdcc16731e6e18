mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01o.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_ichol.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_r01o.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r01o
bash tools/bench_all.sh r01o
