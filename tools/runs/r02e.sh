#!/bin/bash
# r02e: ncu captures of the HBM/ALU-bound kernels: heat IIR (thread-per-chunk and warp-scan
# forms) on c3, GMRES CGS2 multidot/multiaxpy on c4, L96 tangent/adjoint on c2.
TAG=r02e
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
C3="python bench.py --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
WF4DVAR_HEAT_TILE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_heat_iir -s 20 -c 3 -o gpurun_out/prof_heatold_$TAG $C3 > gpurun_out/ncu_heatold_$TAG.log 2>&1; echo "heatold=$?" >> gpurun_out/status_$TAG
WF4DVAR_HEAT_TILE=256 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_heat_iir -s 20 -c 3 -o gpurun_out/prof_heatscan_$TAG $C3 > gpurun_out/ncu_heatscan_$TAG.log 2>&1; echo "heatscan=$?" >> gpurun_out/status_$TAG
C4="python bench.py --config 4 --steps 50 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_multi" -s 200 -c 4 -o gpurun_out/prof_cgs2_$TAG $C4 > gpurun_out/ncu_cgs2_$TAG.log 2>&1; echo "cgs2=$?" >> gpurun_out/status_$TAG
C2="python bench.py --config 2 --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_l96 -s 20 -c 4 -o gpurun_out/prof_l96_$TAG $C2 > gpurun_out/ncu_l96_$TAG.log 2>&1; echo "l96=$?" >> gpurun_out/status_$TAG
