# ncu --set full: L96 forward/adjoint chain kernels (configs[2]) and the GMRES multidot (configs[4])
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02an.log 2>&1
CMD="python bench.py --config 2 --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_l96_step -s 30 -c 6 -o gpurun_out/prof_l96_r02an $CMD > gpurun_out/ncu_l96_r02an.log 2>&1
echo "ncu_l96=$?" >> gpurun_out/status_r02an
CMD4="python bench.py --config 4 --steps 50 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_multidot_partial|k_multiaxpy" -s 60 -c 4 -o gpurun_out/prof_cgs2_r02an $CMD4 > gpurun_out/ncu_cgs2_r02an.log 2>&1
echo "ncu_cgs2=$?" >> gpurun_out/status_r02an
