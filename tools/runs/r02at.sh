#!/bin/bash
# r02at: 16-byte accumulator-pair stores in the TRSM panel / dataflow kernels and the GEMM
# epilogues (whole sectors per store instruction).  Hypothesis: the TMA-staged coupling
# GEMMs read rows whose sectors were half written per instruction by the panel kernel.
# Probes: chained P applies with every GEMM TMA-staged (c4 =3 and =1, c3 =1), repeated.
TAG=r02at
mkdir -p gpurun_out
export WF4DVAR_PROBLEM_CACHE=/tmp/wfpc_$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?" >> gpurun_out/status_$TAG
for rep in 1 2 3; do
  TAGENV="tma3 run$rep" env CFG=4 NREP=4 MODE=P WF4DVAR_GEMM_TMA=3 timeout 600 python tools/diag/c4_race2.py >> gpurun_out/race_$TAG.log 2>&1
  TAGENV="tma1 run$rep" env CFG=4 NREP=4 MODE=P WF4DVAR_GEMM_TMA=1 timeout 600 python tools/diag/c4_race2.py >> gpurun_out/race_$TAG.log 2>&1
done
for rep in 1 2; do
  TAGENV="tma1 run$rep" env CFG=3 NREP=3 MODE=P WF4DVAR_GEMM_TMA=1 timeout 600 python tools/diag/c4_race2.py >> gpurun_out/race_$TAG.log 2>&1
done
TAGENV="tma2 (default)" env CFG=4 NREP=2 MODE=P timeout 600 python tools/diag/c4_race2.py >> gpurun_out/race_$TAG.log 2>&1
echo "race=$?" >> gpurun_out/status_$TAG
B="python bench.py --steps 20 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 600 $B > gpurun_out/bench_c3_${TAG}_tma2.log 2>&1
WF4DVAR_GEMM_TMA=1 timeout 600 $B > gpurun_out/bench_c3_${TAG}_tma1.log 2>&1
timeout 600 $B --config 4 --steps 50 > gpurun_out/bench_c4_${TAG}_tma2.log 2>&1
WF4DVAR_GEMM_TMA=1 timeout 600 $B --config 4 --steps 50 > gpurun_out/bench_c4_${TAG}_tma1.log 2>&1
echo "bench=$?" >> gpurun_out/status_$TAG
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_repro.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_sub_$TAG.log 2>&1; echo "pytest_sub=$?" >> gpurun_out/status_$TAG
