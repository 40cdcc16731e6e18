# L96: merged ragged-chain launch; 4-lanes-per-problem variant (WF4DVAR_L96_LPP=4)
mkdir -p gpurun_out
CMD="python bench.py --config 2 --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
B="python bench.py --config 2 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02am.log 2>&1
timeout 300 $B > gpurun_out/bench_c2_r02am_L8.log 2>&1
WF4DVAR_L96_LPP=4 timeout 300 $B > gpurun_out/bench_c2_r02am_L4.log 2>&1
WF4DVAR_L96_LPP=4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:l96 -c 120 --csv --log-file gpurun_out/l96_launch_r02am_L4.csv $CMD > /dev/null 2>&1
WF4DVAR_NVCC_FLAGS="-DL96_ADJ_STASH=1 -DL96_MINB_A4=3" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02am_S.log 2>&1
WF4DVAR_L96_LPP=4 timeout 300 $B > gpurun_out/bench_c2_r02am_L4S.log 2>&1
timeout 300 $B > gpurun_out/bench_c2_r02am_L8S.log 2>&1
WF4DVAR_L96_LPP=4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:l96 -c 120 --csv --log-file gpurun_out/l96_launch_r02am_L4S.csv $CMD > /dev/null 2>&1
WF4DVAR_L96_LPP=4 timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "l96 or c2" > gpurun_out/pytest_l96_r02am_L4.log 2>&1; echo "pytest_L4=$?" >> gpurun_out/status_r02am
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02am2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_outer.py tests/test_gpu_dist.py -q -k "l96 or c2 or outer or dist" > gpurun_out/pytest_l96_r02am.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r02am
