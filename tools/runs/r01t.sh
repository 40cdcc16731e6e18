mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01t.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_edge.py -q -x > gpurun_out/pytest_r01t.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r01t
for S in 1 0; do WF4DVAR_HEAT_IIR_SMEM=$S timeout 400 python bench.py --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_iir${S}_r01t.log 2>&1; done
timeout 900 python bench.py --config 5 --steps 20 --tts-maxit 400 > gpurun_out/bench_c5_r01t.log 2>&1; echo "c5=$?" >> gpurun_out/status_r01t
timeout 300 python bench.py --config 1 --steps 30 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c1_r01t.log 2>&1
echo done >> gpurun_out/status_r01t
