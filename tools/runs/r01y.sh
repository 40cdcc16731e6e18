mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01y.log 2>&1
for N in 63 31 15; do timeout 400 python bench.py --N $N --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_N${N}_r01y.log 2>&1; done
for N in 15; do for NB in 16 32; do WF4DVAR_TRSM_NB=$NB timeout 400 python bench.py --N $N --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_N${N}_nb${NB}_r01y.log 2>&1; done; done
echo done >> gpurun_out/status_r01y
