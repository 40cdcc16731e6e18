mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01c.log 2>&1
for L in 0 128 256 512; do echo "LEAF=$L"; WF4DVAR_TRSM_LEAF=$L python tools/kbench.py --trsm-only; done > gpurun_out/kbench_trsm_r01c.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_kernels.py -x -q > gpurun_out/pytest_dist_r01c.log 2>&1; echo "pytest_dist=$?" >> gpurun_out/status_r01c
for L in 0 256 512; do WF4DVAR_TRSM_LEAF=$L timeout 600 python bench.py --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_leaf${L}_r01c.log 2>&1; done
echo done >> gpurun_out/status_r01c
