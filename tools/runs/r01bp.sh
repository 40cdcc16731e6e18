mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01bp.log 2>&1
CMD="python bench.py --config 5 --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "trsm_dmma/" -s 10 -c 4 -o gpurun_out/prof_trsm_c5_r01bp $CMD > gpurun_out/ncu_trsm_c5_r01bp.log 2>&1; echo "ncu=$?" >> gpurun_out/status_r01bp
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --csv --log-file gpurun_out/launches_c5_r01bp.csv $CMD > gpurun_out/ncu_l5_r01bp.log 2>&1; echo "l=$?" >> gpurun_out/status_r01bp
