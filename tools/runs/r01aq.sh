mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01aq.log 2>&1
for r in 1 2; do timeout 300 python bench.py --config 2 --steps 20 --tts-maxit 0 --no-cpu-baseline > gpurun_out/c2_${r}_r01aq.log 2>&1; done
timeout 600 python -m pytest tests -m gpu -q -x -k "l96 or outer or c2" > gpurun_out/pytest_l96_r01aq.log 2>&1; echo "p=$?" >> gpurun_out/status_r01aq
echo done >> gpurun_out/status_r01aq
