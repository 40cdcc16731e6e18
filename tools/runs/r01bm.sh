mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01bm.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01bm.log 2>&1; echo "smoke=$?" >> gpurun_out/status_r01bm
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/pytest_r01bm.log 2>&1; echo "p=$?" >> gpurun_out/status_r01bm
for c in 0 1 2 5; do timeout 400 python bench.py --config $c --steps 30 --tts-maxit 0 --no-cpu-baseline --e2e-steps 3 > gpurun_out/c${c}_r01bm.log 2>&1; done
for r in 1 2 3; do timeout 400 python bench.py --config 4 --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c4_${r}_r01bm.log 2>&1; done
echo done >> gpurun_out/status_r01bm
