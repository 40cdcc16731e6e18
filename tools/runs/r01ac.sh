mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01ac.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r01ac.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r01ac
for c in 0 2; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c${c}_r01ac.log 2>&1; echo "c$c=$?" >> gpurun_out/status_r01ac
  WF4DVAR_TRSM_SMALL=0 WF4DVAR_GEMM_SMALL=0 timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --tts-maxit 0 > gpurun_out/bench_c${c}_nosmall_r01ac.log 2>&1
done
CMD="python bench.py --config 2 --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --csv --log-file gpurun_out/launches_c2_r01ac.csv $CMD > gpurun_out/ncu_launch_c2_r01ac.log 2>&1
echo "ncu=$?" >> gpurun_out/status_r01ac
