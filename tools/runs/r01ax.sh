mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r01ax.log 2>&1
cat > /tmp/kb1.py <<'PY'
import sys, torch, json
sys.path.insert(0, ".")
from paper_2105_06975_b200 import _lib as L
A = torch.randn(4096, 4096, dtype=torch.float64, device="cuda")
X = torch.randn(4096, 8192, dtype=torch.float64, device="cuda")
Y = torch.empty(4096, 8192, dtype=torch.float64, device="cuda")
for _ in range(2): L.test_gemm(A, X, Y)
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); L.test_gemm(A, X, Y); b.record(); torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b))
print(json.dumps(dict(tflops=2*4096*8192*4096/best/1e9)))
PY
for cfg in -1 1 3 4 5 6 7 8 9 10; do echo -n "$cfg " >> gpurun_out/cfg_r01ax.txt; WF4DVAR_GEMM_CFG=$cfg timeout 120 python /tmp/kb1.py >> gpurun_out/cfg_r01ax.txt 2>&1; done
echo done >> gpurun_out/status_r01ax
