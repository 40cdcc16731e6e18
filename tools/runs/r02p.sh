#!/bin/bash
# r02p: dataflow TRSM (k_trsm_df), column-sequential heat kernel (k_heat_iir_seq), MINRES
# overlap: iteration 1 always eager.  Full GPU suite + smoke; A/B benches.
TAG=r02p
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?" >> gpurun_out/status_$TAG
timeout 1200 python -m pytest -q -rf -x tests/test_gpu_kernels.py > gpurun_out/pytest_kern_$TAG.log 2>&1; echo "kern=$?" >> gpurun_out/status_$TAG
B="python bench.py --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run() { name=$1; shift; env "$@" timeout 600 $B > gpurun_out/ab_${name}_$TAG.log 2>&1; echo "$name=$?" >> gpurun_out/status_$TAG; }
run c3 X=1
run c3_nodf WF4DVAR_TRSM_DF=0
run c3_noseq WF4DVAR_HEAT_SEQ=0
run c3_seq16 WF4DVAR_HEAT_SEQ=16
B="python bench.py --config 1 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run c1 X=1
run c1_nodf WF4DVAR_TRSM_DF=0
B="python bench.py --config 1 --solver minres --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run c1m X=1
run c1m_nodf WF4DVAR_TRSM_DF=0
B="python bench.py --config 4 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
run c4 X=1
run c4_nodf WF4DVAR_TRSM_DF=0
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$TAG
