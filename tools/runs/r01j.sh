mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01j.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01j.log 2>&1; echo "smoke=$?" >> gpurun_out/status_r01j
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r01j.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r01j
bash tools/bench_all.sh r01j
for G in 0 1; do WF4DVAR_GRAPHS=$G timeout 300 python bench.py --config 1 --steps 30 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c1_g${G}_r01j.log 2>&1; done
