mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01p.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_r01p.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r01p
timeout 300 python tools/kbench.py --trsm-only > gpurun_out/kbench_trsm_r01p.log 2>&1
for P in 1 0; do WF4DVAR_AUX_PRIORITY=$P timeout 400 python bench.py --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_pri${P}_r01p.log 2>&1; done
timeout 400 python bench.py --config 4 --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c4_r01p.log 2>&1
echo done >> gpurun_out/status_r01p
