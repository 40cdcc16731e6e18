mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01aj.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "host_path" > gpurun_out/pytest_host_r01aj.log 2>&1; echo "p=$?" >> gpurun_out/status_r01aj
B4="python bench.py --config 4 --steps 20 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
for rep in 1 2; do
  timeout 300 $B4 > gpurun_out/c4_inv_${rep}_r01aj.log 2>&1
  WF4DVAR_TRSM_INV=0 timeout 300 $B4 > gpurun_out/c4_sub_${rep}_r01aj.log 2>&1
  WF4DVAR_AUX_PRIORITY=0 timeout 300 $B4 > gpurun_out/c4_noprio_${rep}_r01aj.log 2>&1
done
timeout 300 python bench.py --config 3 --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 3 > gpurun_out/c3_e2e_r01aj.log 2>&1
echo done >> gpurun_out/status_r01aj
