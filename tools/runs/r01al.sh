mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01al.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k gemm > gpurun_out/pytest_gemm_r01al.log 2>&1; echo "p=$?" >> gpurun_out/status_r01al
timeout 300 python tools/kbench.py --gemm-only > gpurun_out/kb_split_r01al.json 2>&1
WF4DVAR_GEMM_SK=0 timeout 300 python tools/kbench.py --gemm-only > gpurun_out/kb_plain_r01al.json 2>&1
B="python bench.py --config 3 --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 300 $B > gpurun_out/c3_split_r01al.log 2>&1
WF4DVAR_GEMM_SK=0 timeout 300 $B > gpurun_out/c3_plain_r01al.log 2>&1
timeout 300 $B > gpurun_out/c3_split2_r01al.log 2>&1
echo done >> gpurun_out/status_r01al
