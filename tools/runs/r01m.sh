mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01m.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_spectral.py tests/test_gpu_paper_heat.py tests/test_gpu_rblock.py -q > gpurun_out/pytest_r01m.log 2>&1; echo "pytest_new=$?" >> gpurun_out/status_r01m
bash tools/r01l.sh
for c in 2 4; do timeout 600 python bench.py --config $c --steps 20 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c${c}_r01m.log 2>&1; done
echo done >> gpurun_out/status_r01m
