mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01h.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_r01h.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r01h
timeout 300 python tools/kbench.py --trsm-only > gpurun_out/kbench_trsm_r01h.log 2>&1
for H in 0 1; do WF4DVAR_HEAT_STENCIL=$H timeout 400 python bench.py --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_st${H}_r01h.log 2>&1; echo "bench_st$H=$?" >> gpurun_out/status_r01h; done
CMD="python bench.py --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD > gpurun_out/plain_r01h.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "trsm_dmma/" -s 8 -c 1 -o gpurun_out/prof_trsm_r01h $CMD > gpurun_out/ncu_trsm_r01h.log 2>&1
echo "ncu=$?" >> gpurun_out/status_r01h
