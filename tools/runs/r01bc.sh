mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01bc.log 2>&1
for N in 63 31 15; do timeout 400 python bench.py --config 3 --N $N --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_N${N}_r01bc.log 2>&1; done
echo done >> gpurun_out/status_r01bc
