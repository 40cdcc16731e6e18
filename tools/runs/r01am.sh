mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01am.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 1200 ncu --set full --clock-control none --nvtx --nvtx-include "trsm_update_dmma/" -s 6 -c 6 -o gpurun_out/prof_tupd_r01am $CMD > gpurun_out/ncu_tupd_r01am.log 2>&1
echo "ncu=$?" >> gpurun_out/status_r01am
