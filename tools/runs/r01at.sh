mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01at.log 2>&1
B="python bench.py --config 1 --steps 30 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
for sb in 0 128 512 1024; do WF4DVAR_TRSM_SB=$sb timeout 300 $B > gpurun_out/c1_sb${sb}_r01at.log 2>&1; done
B5="python bench.py --config 5 --steps 20 --tts-maxit 0 --no-cpu-baseline --e2e-steps 1"
for sb in 0 256 1024 2048; do WF4DVAR_TRSM_SB=$sb timeout 300 $B5 > gpurun_out/c5_sb${sb}_r01at.log 2>&1; done
echo done >> gpurun_out/status_r01at
