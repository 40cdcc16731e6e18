# DMMA small products (K <= 64) and tile-inverse small triangles (configs[2])
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02ao.log 2>&1
B="python bench.py --config 2 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 300 $B > gpurun_out/bench_c2_r02ao_new.log 2>&1
WF4DVAR_GEMM_SMALL=1 WF4DVAR_TRSM_SMALL_INV=0 timeout 300 $B > gpurun_out/bench_c2_r02ao_old.log 2>&1
WF4DVAR_TRSM_SMALL_INV=0 timeout 300 $B > gpurun_out/bench_c2_r02ao_gemmonly.log 2>&1
CMD="python bench.py --config 2 --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launch_c2_r02ao.csv $CMD > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02ao.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r02ao
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02ao.log 2>&1; echo "smoke=$?" >> gpurun_out/status_r02ao
