mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01bh.log 2>&1
B5="python bench.py --config 5 --steps 30 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
for ti in 32 16 8; do WF4DVAR_HEAT_EXPL_TI=$ti timeout 300 $B5 > gpurun_out/c5_ti${ti}_r01bh.log 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q -x -k "heat or parity or paper" > gpurun_out/pytest_r01bh.log 2>&1; echo "p=$?" >> gpurun_out/status_r01bh
echo done >> gpurun_out/status_r01bh
