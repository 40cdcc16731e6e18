mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_r02aj.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02aj.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02aj.log 2>&1; echo "smoke=$?" >> gpurun_out/status_r02aj
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r02aj.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r02aj
timeout 900 python bench.py > gpurun_out/bench_c3_r02aj.log 2>&1; echo "bench_c3=$?" >> gpurun_out/status_r02aj
timeout 600 python bench.py --config 2 > gpurun_out/bench_c2_r02aj.log 2>&1; echo "bench_c2=$?" >> gpurun_out/status_r02aj
