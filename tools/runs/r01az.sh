mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01az.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_r01az.log 2>&1; echo "p=$?" >> gpurun_out/status_r01az
for c in 3 1 4; do timeout 400 python bench.py --config $c --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c${c}_r01az.log 2>&1; done
for c in 3 1; do WF4DVAR_EXPLICIT_INV=0 timeout 400 python bench.py --config $c --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c${c}_trsm_r01az.log 2>&1; done
timeout 900 python bench.py --config 3 --steps 10 --tts-maxit 400 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c3_tts_r01az.log 2>&1
echo done >> gpurun_out/status_r01az
