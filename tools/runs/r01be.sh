mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01be.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_r01be.log 2>&1; echo "p=$?" >> gpurun_out/status_r01be
echo done >> gpurun_out/status_r01be
