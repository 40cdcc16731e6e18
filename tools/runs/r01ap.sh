mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01ap.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x > gpurun_out/pytest_r01ap.log 2>&1; echo "p=$?" >> gpurun_out/status_r01ap
B="python bench.py --config 3 --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
for t in 30 60 80; do WF4DVAR_GEMM_SK_TAIL=$t timeout 400 $B > gpurun_out/c3_t${t}_r01ap.log 2>&1; echo "t$t=$?" >> gpurun_out/status_r01ap; done
timeout 400 python bench.py --config 4 --steps 20 --tts-maxit 0 --no-cpu-baseline > gpurun_out/c4_r01ap.log 2>&1; echo "c4=$?" >> gpurun_out/status_r01ap
echo done >> gpurun_out/status_r01ap
