# L96 kernel variants on configs[2] (fused forward stages, stored substep states, adjoint stash)
mkdir -p gpurun_out
for V in "A:-DL96_ADJ_STASH=0 -DL96_MINB_A=2" "B:-DL96_ADJ_STASH=1 -DL96_MINB_A=3" "C:-DL96_ADJ_STASH=1 -DL96_MINB_A=2" "D:-DL96_ADJ_STASH=0 -DL96_MINB_A=2 -DL96_MINB_F=2"; do
  N=${V%%:*}; F=${V#*:}
  WF4DVAR_NVCC_FLAGS="$F" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02ak_$N.log 2>&1
  for i in 1 2; do
    timeout 300 python bench.py --config 2 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c2_r02ak_${N}_$i.log 2>&1
  done
done
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02ak.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "l96 or c2" > gpurun_out/pytest_l96_r02ak.log 2>&1; echo "pytest=$?" >> gpurun_out/status_r02ak
timeout 900 python -m pytest tests/test_gpu_outer.py tests/test_gpu_dist.py -q > gpurun_out/pytest_outer_r02ak.log 2>&1; echo "pytest2=$?" >> gpurun_out/status_r02ak
