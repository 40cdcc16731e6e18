mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01ay.log 2>&1
timeout 1200 compute-sanitizer --tool memcheck --leak-check no python tools/sanitize_smoke.py > gpurun_out/san_mem_r01ay.log 2>&1; echo "mem=$?" >> gpurun_out/status_r01ay
timeout 1500 compute-sanitizer --tool racecheck python tools/sanitize_smoke.py > gpurun_out/san_race_r01ay.log 2>&1; echo "race=$?" >> gpurun_out/status_r01ay
echo done >> gpurun_out/status_r01ay
