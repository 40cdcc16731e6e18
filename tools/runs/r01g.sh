mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01g.log 2>&1
for P in 1 0; do WF4DVAR_AUX_PRIORITY=$P timeout 400 python bench.py --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_pri${P}_r01g.log 2>&1; echo "bench_pri$P=$?" >> gpurun_out/status_r01g; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x > gpurun_out/pytest_r01g.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r01g
CMD="python bench.py --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD > gpurun_out/plain_r01g.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "trsm_dmma/" -s 8 -c 2 -o gpurun_out/prof_trsm_r01g $CMD > gpurun_out/ncu_trsm_r01g.log 2>&1
echo "ncu=$?" >> gpurun_out/status_r01g
