#!/bin/bash
# r02bc: reproducibility battery of the DEFAULT path (TMA staging for the covariance products
# only): 60 chained applies, 5 repeats each, P and PA modes, configs[3] and [4]
TAG=r02bc
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
for cfg in 3 4; do for mode in P PA A; do
  TAGENV="default" env CFG=$cfg NREP=5 MODE=$mode timeout 900 python tools/diag/c4_race2.py >> gpurun_out/race_$TAG.log 2>&1
done; done
echo "race=$?" >> gpurun_out/status_$TAG
