mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01k.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_nccl1.py -q -x > gpurun_out/pytest_r01k.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r01k
timeout 600 python bench.py --config 2 --steps 20 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c2_r01k.log 2>&1; echo "c2=$?" >> gpurun_out/status_r01k
CMD="python bench.py --config 4 --steps 3 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD > gpurun_out/plain_r01k.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "vector/" -s 2 -c 2 -o gpurun_out/prof_vec_r01k $CMD > gpurun_out/ncu_vec_r01k.log 2>&1
echo "ncu=$?" >> gpurun_out/status_r01k
