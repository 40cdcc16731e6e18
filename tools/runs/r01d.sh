mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01d.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/pytest_dist_r01d.log 2>&1; echo "pytest_dist=$?" >> gpurun_out/status_r01d
for G in 8 16 32 64; do echo "GM=$G"; WF4DVAR_GEMM_GM=$G python tools/kbench.py --gemm-only; done > gpurun_out/kbench_gemm_r01d.log 2>&1
timeout 600 python bench.py --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_r01d.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD > gpurun_out/plain_r01d.log 2>&1 && timeout 1200 ncu --set full --clock-control none -k regex:k_gemm -s 60 -c 15 -o gpurun_out/prof_r01d $CMD > gpurun_out/ncu_full_r01d.log 2>&1
echo "ncu=$?" >> gpurun_out/status_r01d
