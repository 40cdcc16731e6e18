mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01ba.log 2>&1
timeout 900 python bench.py --config 3 --steps 10 --tts-maxit 400 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c3_tts_r01ba.log 2>&1
timeout 600 python bench.py --config 1 --steps 30 --tts-maxit 400 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c1_tts_r01ba.log 2>&1
WF4DVAR_EXPLICIT_INV=0 timeout 600 python bench.py --config 1 --steps 30 --tts-maxit 400 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c1_tts_trsm_r01ba.log 2>&1
timeout 600 python bench.py --config 4 --steps 20 --tts-maxit 300 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c4_tts_r01ba.log 2>&1
echo done >> gpurun_out/status_r01ba
