"""fp64 peak calibration: cuBLAS DGEMM via torch (calibration only, never shipped on the path)."""
import json, time, torch
dev = torch.device("cuda:0")
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=dev); b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(3): torch.matmul(a, b)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    # sustained 4 s
    t0 = time.time(); cnt = 0; e0.record()
    while time.time() - t0 < 4.0:
        torch.matmul(a, b); cnt += 1
        if cnt % 4 == 0: torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize(); sus = e0.elapsed_time(e1) / cnt
    print(json.dumps({"kind": "cublas_dgemm", "n": n, "burst_tflops": 2 * n**3 / best / 1e9, "sustained_tflops": 2 * n**3 / sus / 1e9}))
x = torch.randn(1 << 27, dtype=torch.float64, device=dev); y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
torch.cuda.synchronize(); e0.record()
for _ in range(10): y.copy_(x)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"kind": "copy_f64", "gbs": 10 * 2 * x.numel() * 8 / e0.elapsed_time(e1) / 1e6}))
