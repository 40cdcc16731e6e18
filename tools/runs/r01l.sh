mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01l.log 2>&1
B="python bench.py --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
for cfg in "SB=1024" "SB=512" "SB=2048" "LEAF=512" "LEAF=1024"; do
  k=${cfg%%=*}; v=${cfg##*=}
  if [ $k = SB ]; then env WF4DVAR_TRSM_SB=$v timeout 400 $B > gpurun_out/bench_c3_sb${v}_r01l.log 2>&1; else env WF4DVAR_TRSM_LEAF=$v timeout 400 $B > gpurun_out/bench_c3_leaf${v}_r01l.log 2>&1; fi
done
for L in 0 512 1024; do echo "LEAF=$L"; WF4DVAR_TRSM_LEAF=$L timeout 300 python tools/kbench.py --trsm-only; done > gpurun_out/kbench_trsm_r01l.log 2>&1
echo done >> gpurun_out/status_r01l
