#!/bin/bash
# r02a: per-block parity with the triangular solves as default; the smoke
# cell's iteration-count diagnosis; c3 time-to-1e-8 with triangular solves vs A32.
TAG=r02a
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_parity.py -q -rf -s > gpurun_out/pytest_parity_$TAG.log 2>&1; echo "parity=$?" >> gpurun_out/status_$TAG
timeout 600 python tools/iter_bias.py > gpurun_out/iter_bias_$TAG.log 2>&1; echo "bias=$?" >> gpurun_out/status_$TAG
timeout 600 python bench.py --tts-maxit 0 --no-cpu-baseline > gpurun_out/bench_c3_$TAG.log 2>&1; echo "bench=$?" >> gpurun_out/status_$TAG
timeout 1500 python tools/tts.py --config 3 --maxit 5000 --out gpurun_out/tts_c3_$TAG.json > gpurun_out/tts_c3_$TAG.log 2>&1; echo "tts=$?" >> gpurun_out/status_$TAG
