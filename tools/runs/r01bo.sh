mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01bo.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01bo.log 2>&1; echo "smoke=$?" >> gpurun_out/status_r01bo
START=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_default_r01bo.log 2>&1; echo "bench=$? secs=$(( $(date +%s) - START ))" >> gpurun_out/status_r01bo
START=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/bench_defref_r01bo.log 2>&1; echo "ref=$? secs=$(( $(date +%s) - START ))" >> gpurun_out/status_r01bo
