mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01ao.log 2>&1
B="python bench.py --config 3 --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
for t in 30 60 80; do WF4DVAR_GEMM_SK_TAIL=$t timeout 300 $B > gpurun_out/c3_t${t}_r01ao.log 2>&1; done
WF4DVAR_GEMM_SK_TAIL=60 timeout 300 python tools/kbench.py --gemm-only > gpurun_out/kb_t60_r01ao.json 2>&1
echo done >> gpurun_out/status_r01ao
