mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01bl.log 2>&1
B4="python bench.py --config 4 --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
B3="python bench.py --config 3 --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
for r in 1 2 3; do
  timeout 300 $B4 > gpurun_out/c4_f1_${r}_r01bl.log 2>&1
  WF4DVAR_FORK=0 timeout 300 $B4 > gpurun_out/c4_f0_${r}_r01bl.log 2>&1
done
for r in 1 2; do
  timeout 300 $B3 > gpurun_out/c3_f1_${r}_r01bl.log 2>&1
  WF4DVAR_FORK=0 timeout 300 $B3 > gpurun_out/c3_f0_${r}_r01bl.log 2>&1
done
echo done >> gpurun_out/status_r01bl
