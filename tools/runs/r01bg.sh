mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01bg.log 2>&1
B="python bench.py --config 3 --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
for ti in 16 8; do WF4DVAR_HEAT_TI=$ti timeout 300 $B > gpurun_out/c3_ti${ti}_r01bg.log 2>&1; done
B1="python bench.py --config 1 --steps 30 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
for ti in 16 8; do WF4DVAR_HEAT_TI=$ti timeout 300 $B1 > gpurun_out/c1_ti${ti}_r01bg.log 2>&1; done
B0="python bench.py --config 0 --steps 50 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
for ti in 32 16 8; do WF4DVAR_HEAT_TI=$ti timeout 300 $B0 > gpurun_out/c0_ti${ti}_r01bg.log 2>&1; done
echo done >> gpurun_out/status_r01bg
