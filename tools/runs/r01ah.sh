mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01ah.log 2>&1
B="python bench.py --config 3 --steps 10 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
timeout 300 $B > gpurun_out/sweep_def_r01ah.log 2>&1
WF4DVAR_GEMM_SK=1 timeout 300 $B > gpurun_out/sweep_sk_r01ah.log 2>&1
WF4DVAR_TRSM_SB=512 timeout 300 $B > gpurun_out/sweep_sb512_r01ah.log 2>&1
WF4DVAR_TRSM_SB=2048 timeout 300 $B > gpurun_out/sweep_sb2048_r01ah.log 2>&1
WF4DVAR_TRSM_LEFT=1 timeout 300 $B > gpurun_out/sweep_left_r01ah.log 2>&1
WF4DVAR_TRSM_LEAF=1024 timeout 300 $B > gpurun_out/sweep_leaf_r01ah.log 2>&1
timeout 300 $B > gpurun_out/sweep_def2_r01ah.log 2>&1
echo done > gpurun_out/status_r01ah
