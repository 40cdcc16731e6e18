mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01bq.log 2>&1
B5="python bench.py --config 5 --steps 30 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
for nb in 0 16 32; do WF4DVAR_TRSM_NB=$nb timeout 300 $B5 > gpurun_out/c5_nb${nb}_r01bq.log 2>&1; done
echo done >> gpurun_out/status_r01bq
