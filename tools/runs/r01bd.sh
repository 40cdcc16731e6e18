mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01bd.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r01bd.log 2>&1; echo "p=$?" >> gpurun_out/status_r01bd
timeout 300 python tools/kbench.py --gemm-only > gpurun_out/kb_r01bd.json 2>&1
for c in 1 5 0; do timeout 400 python bench.py --config $c --steps 30 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c${c}_r01bd.log 2>&1; done
for c in 1 5; do WF4DVAR_GEMM_SPLITK=0 timeout 400 python bench.py --config $c --steps 30 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/c${c}_nosplit_r01bd.log 2>&1; done
echo done >> gpurun_out/status_r01bd
