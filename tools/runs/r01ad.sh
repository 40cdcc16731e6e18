mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01ad.log 2>&1
CMD="python bench.py --config 2 --steps 2 --warmup 3 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_small|k_trsm_small|k_l96_step" -s 10 -c 8 -o gpurun_out/prof_c2_r01ad $CMD > gpurun_out/ncu_c2_r01ad.log 2>&1
echo "ncu=$?" >> gpurun_out/status_r01ad
