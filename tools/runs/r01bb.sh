mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01bb.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01bb.log 2>&1; echo "smoke=$?" >> gpurun_out/status_r01bb
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01bb.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r01bb
bash tools/bench_all.sh r01bb
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c3_r01bb.log 2>&1; echo "ref=$?" >> gpurun_out/status_r01bb
CMD="python bench.py --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD > gpurun_out/plain_r01bb.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --csv --log-file gpurun_out/launches_r01bb.csv $CMD > gpurun_out/ncu_launch_r01bb.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "gemm_dmma/" -s 6 -c 6 -o gpurun_out/prof_gemm_r01bb $CMD > gpurun_out/ncu_gemm_r01bb.log 2>&1
echo "ncu=$?" >> gpurun_out/status_r01bb
