#!/bin/bash
# r02b: GPU suite with per-block parity (fixed kappa cache) + smoke; cell grids c1/c2/c4/c3.
TAG=r02b
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?" >> gpurun_out/status_$TAG
timeout 3000 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG
for g in c1 c2 c4; do
timeout 1200 python tools/grid.py $g --maxit 2000 --out gpurun_out/grid_${g}_$TAG.json > gpurun_out/grid_${g}_$TAG.log 2>&1; echo "grid_$g=$?" >> gpurun_out/status_$TAG
done
timeout 1800 python tools/grid.py c3 --maxit 2000 --out gpurun_out/grid_c3_$TAG.json > gpurun_out/grid_c3_$TAG.log 2>&1; echo "grid_c3=$?" >> gpurun_out/status_$TAG
