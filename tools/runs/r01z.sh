mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01z.log 2>&1
for N in 15 31; do for SB in 256 512; do WF4DVAR_TRSM_SB=$SB timeout 400 python bench.py --N $N --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_N${N}_sb${SB}_r01z.log 2>&1; done; done
for N in 15 31; do WF4DVAR_GEMM_SK=1 timeout 400 python bench.py --N $N --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_N${N}_sk_r01z.log 2>&1; done
echo done >> gpurun_out/status_r01z
