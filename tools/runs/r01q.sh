mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01q.log 2>&1
CMD="python bench.py --config 4 --steps 4 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD > gpurun_out/plain_r01q.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "vector/" --nvtx-include "dot_reduce/" -s 6 -c 4 -o gpurun_out/prof_gmres_r01q $CMD > gpurun_out/ncu_r01q.log 2>&1
echo "ncu=$?" >> gpurun_out/status_r01q
