"""fp64 GEMM throughput via torch.matmul (cuBLAS DGEMM) — roofline context for the fp64 peak."""
import json, torch
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
for _ in range(2): torch.matmul(a, b)
torch.cuda.synchronize(); best = 1e9
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(5):
    e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
print(json.dumps({"kernel": "torch_dgemm_8192", "ms": best, "tflops": 2 * 8192**3 / best / 1e9}))
