mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01ak.log 2>&1
timeout 300 python tools/kbench.py --gemm-only > gpurun_out/kb_plain_r01ak.json 2>&1
WF4DVAR_GEMM_SK=1 timeout 300 python tools/kbench.py --gemm-only > gpurun_out/kb_sk_r01ak.json 2>&1
cat > /tmp/one.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2105_06975_b200 import _lib as L
A = torch.randn(4096, 4096, dtype=torch.float64, device="cuda")
X = torch.randn(4096, 8256, dtype=torch.float64, device="cuda")
Y = torch.empty(4096, 8256, dtype=torch.float64, device="cuda")
for _ in range(3): L.test_gemm(A, X, Y)
torch.cuda.synchronize()
PY
WF4DVAR_GEMM_SK=1 timeout 600 ncu --set full --clock-control none -k regex:"k_gemm" -s 1 -c 1 -o gpurun_out/prof_sk_r01ak python /tmp/one.py > gpurun_out/ncu_sk_r01ak.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_gemm" -s 1 -c 1 -o gpurun_out/prof_plain_r01ak python /tmp/one.py > gpurun_out/ncu_plain_r01ak.log 2>&1
echo done > gpurun_out/status_r01ak
