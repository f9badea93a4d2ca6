"""Comparator only: cuBLAS fp64 GEMM throughput at the MTTSP shapes (not product code)."""
import json, torch
torch.backends.cuda.matmul.allow_tf32 = False
shapes = [(25600, 25600, 400), (4096, 4096, 64), (250000, 500, 100), (500, 250000, 100), (1600, 64000, 64), (64000, 1600, 64), (8192, 8192, 8192)]
for (m, k, n) in shapes:
    a = torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"kind": "cublas_dgemm", "m": m, "k": k, "n": n, "ms": round(ms, 4), "tflops": round(2 * m * k * n / ms / 1e9, 2)}))
    del a, b, c
