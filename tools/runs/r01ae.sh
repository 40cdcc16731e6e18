mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01ae.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r01ae.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r01ae
timeout 600 python bench.py --config 2 --steps 20 --tts-maxit 200 > gpurun_out/bench_c2_r01ae.log 2>&1; echo "c2=$?" >> gpurun_out/status_r01ae
CMD="python bench.py --config 2 --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --csv --log-file gpurun_out/launches_c2_r01ae.csv $CMD > gpurun_out/ncu_launch_c2_r01ae.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_small|k_l96_step" -s 10 -c 6 -o gpurun_out/prof_c2_r01ae $CMD > gpurun_out/ncu_c2_r01ae.log 2>&1
echo "ncu=$?" >> gpurun_out/status_r01ae
