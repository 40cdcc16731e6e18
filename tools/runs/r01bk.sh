mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01bk.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "host" > gpurun_out/pytest_r01bk.log 2>&1; echo "p=$?" >> gpurun_out/status_r01bk
for r in 1 2; do timeout 400 python bench.py --config 1 --steps 30 --tts-maxit 0 --no-cpu-baseline --e2e-steps 10 > gpurun_out/c1_${r}_r01bk.log 2>&1; done
timeout 400 python bench.py --config 4 --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 3 > gpurun_out/c4_r01bk.log 2>&1
timeout 400 python bench.py --config 3 --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 3 > gpurun_out/c3_r01bk.log 2>&1
echo done >> gpurun_out/status_r01bk
