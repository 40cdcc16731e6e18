#!/bin/bash
# r02r: dataflow TRSM only for whole triangles with <= 1024 RHS columns (upper solves one
# dependency tile per sweep: deterministic); multidot groups dispatched per row block;
# heat seq CTA width variants; smoke, GPU suite, benches, ncu of the new kernels.
TAG=r02r
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?" >> gpurun_out/status_$TAG
timeout 1200 python -m pytest -q -rf tests/test_gpu_kernels.py > gpurun_out/pytest_kern_$TAG.log 2>&1; echo "kern=$?" >> gpurun_out/status_$TAG
B="python bench.py --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run() { name=$1; shift; env "$@" timeout 600 $B > gpurun_out/ab_${name}_$TAG.log 2>&1; echo "$name=$?" >> gpurun_out/status_$TAG; }
run c3 X=1
run c3_w4 WF4DVAR_HEAT_SEQW=4
run c3_w16 WF4DVAR_HEAT_SEQW=16
B="python bench.py --config 1 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run c1 X=1
B="python bench.py --config 1 --solver minres --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run c1m X=1
B="python bench.py --config 4 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run c4 X=1
CMD="python bench.py --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_heat_iir_seq -s 4 -c 3 -o gpurun_out/prof_heatseq_$TAG $CMD > gpurun_out/ncu_full_heat_$TAG.log 2>&1
CMD1="python bench.py --config 1 --solver minres --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_trsm_df -s 8 -c 4 -o gpurun_out/prof_trsmdf_$TAG $CMD1 > gpurun_out/ncu_full_df_$TAG.log 2>&1
echo "ncu=$?" >> gpurun_out/status_$TAG
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG
