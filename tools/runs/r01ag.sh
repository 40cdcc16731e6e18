mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01ag.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k trsm > gpurun_out/pytest_trsm_default_r01ag.log 2>&1; echo "p0=$?" >> gpurun_out/status_r01ag
WF4DVAR_TRSM_INV=1 timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_inv_r01ag.log 2>&1; echo "pinv=$?" >> gpurun_out/status_r01ag
for c in 1 5 3 4; do
  WF4DVAR_TRSM_INV=1 timeout 600 python bench.py --config $c --steps 20 --tts-maxit 0 --no-cpu-baseline > gpurun_out/bench_c${c}_inv_r01ag.log 2>&1; echo "c$c=$?" >> gpurun_out/status_r01ag
  timeout 600 python bench.py --config $c --steps 20 --tts-maxit 0 --no-cpu-baseline > gpurun_out/bench_c${c}_base_r01ag.log 2>&1
done
