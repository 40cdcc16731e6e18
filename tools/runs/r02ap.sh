# smoke / MINRES-count sensitivity to the small-kernel changes; L96 epilogue; GPU suite
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02ap.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02ap.log 2>&1; echo "smoke=$?" >> gpurun_out/status_r02ap
WF4DVAR_GEMM_SMALL=1 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02ap_gs1.log 2>&1; echo "smoke_gs1=$?" >> gpurun_out/status_r02ap
WF4DVAR_TRSM_SMALL_INV=1 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02ap_inv.log 2>&1; echo "smoke_inv=$?" >> gpurun_out/status_r02ap
B="python bench.py --config 2 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 300 $B > gpurun_out/bench_c2_r02ap.log 2>&1
WF4DVAR_TRSM_SMALL_INV=1 timeout 300 $B > gpurun_out/bench_c2_r02ap_inv.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r02ap.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r02ap
