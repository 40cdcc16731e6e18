mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01ar.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "solve or minres or krylov or determinism or dist" > gpurun_out/pytest_r01ar.log 2>&1; echo "p=$?" >> gpurun_out/status_r01ar
for c in 2 3 1; do timeout 300 python bench.py --config $c --steps 20 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c${c}_r01ar.log 2>&1; done
echo done >> gpurun_out/status_r01ar
