#!/bin/bash
TAG=r02u
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python tools/diag/split_overlap.py 4 50 > gpurun_out/split_c4_$TAG.log 2>&1
timeout 900 python tools/diag/split_overlap.py 3 20 > gpurun_out/split_c3_$TAG.log 2>&1
