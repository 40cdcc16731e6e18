#!/bin/bash
# r02w: c4 history diagnosis; heat thread-per-chunk for small launches (c1); L96 forward
# kernel at 3 CTAs per SM (default) vs 2 / 4.
TAG=r02w
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python tools/diag/c4_hist.py me > gpurun_out/c4hist_me_$TAG.log 2>&1
run() { name=$1; shift; env "$@" timeout 600 $B > gpurun_out/ab_${name}_$TAG.log 2>&1; echo "$name=$?" >> gpurun_out/status_$TAG; }
B="python bench.py --config 1 --solver minres --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run c1m X=1
run c1m_seqall WF4DVAR_HEAT_SEQ_MINCTA=1
B="python bench.py --config 2 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run c2_f3 X=1
WF4DVAR_NVCC_FLAGS="-DL96_MINB_F=2" python -c "from paper_2105_06975_b200 import build as b; b.build(force=True)" > gpurun_out/build2_$TAG.log 2>&1
run c2_f2 X=1
WF4DVAR_NVCC_FLAGS="-DL96_MINB_F=4" python -c "from paper_2105_06975_b200 import build as b; b.build(force=True)" > gpurun_out/build4_$TAG.log 2>&1
run c2_f4 X=1
WF4DVAR_NVCC_FLAGS="-DL96_MINB_F=3 -DL96_MINB_A=3" python -c "from paper_2105_06975_b200 import build as b; b.build(force=True)" > gpurun_out/build33_$TAG.log 2>&1
run c2_f3a3 X=1
