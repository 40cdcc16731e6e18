# L96: round-1 kernel vs fused/stored-substep kernel, per-kernel durations (ncu launch list)
mkdir -p gpurun_out
CMD="python bench.py --config 2 --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
cp paper_2105_06975_b200/csrc/l96.cu /tmp/l96_new.cu
run() {
  N=$1
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02al_$N.log 2>&1
  timeout 300 python bench.py --config 2 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c2_r02al_$N.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:l96 -c 120 --csv --log-file gpurun_out/l96_launch_r02al_$N.csv $CMD > /dev/null 2>&1
}
cp tools/diag/l96_r02aj.cu paper_2105_06975_b200/csrc/l96.cu; run OLD
cp /tmp/l96_new.cu paper_2105_06975_b200/csrc/l96.cu; run NEW
WF4DVAR_NVCC_FLAGS="-DL96_ADJ_STASH=1 -DL96_MINB_A=3" run STASH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02al.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "l96 or c2" > gpurun_out/pytest_l96_r02al.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r02al
