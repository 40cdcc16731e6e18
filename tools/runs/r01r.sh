mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01r.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_dist.py -q -x > gpurun_out/pytest_r01r.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r01r
timeout 600 python bench.py --config 4 --steps 20 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c4_r01r.log 2>&1
for L in 0 1; do WF4DVAR_TRSM_LEFT=$L timeout 400 python bench.py --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_left${L}_r01r.log 2>&1; done
for L in 0 1; do echo "LEFT=$L"; WF4DVAR_TRSM_LEFT=$L timeout 300 python tools/kbench.py --trsm-only; done > gpurun_out/kbench_trsm_r01r.log 2>&1
echo done >> gpurun_out/status_r01r
