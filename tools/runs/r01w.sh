mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01w.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01w.log 2>&1; echo "smoke=$?" >> gpurun_out/status_r01w
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01w.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r01w
timeout 900 python bench.py --config 5 --steps 20 --tts-maxit 400 > gpurun_out/bench_c5_r01w.log 2>&1; echo "c5=$?" >> gpurun_out/status_r01w
timeout 900 python bench.py > gpurun_out/bench_c3_r01w.log 2>&1; echo "c3=$?" >> gpurun_out/status_r01w
