"""cuBLAS ZGEMM (torch complex128 matmul) on the mode-product shapes, for
context next to the DMMA kernel (library baseline, not the product)."""
import json
import torch

for (b, m, k, n) in [(4, 512, 512, 512), (2, 512, 512, 512), (1, 256, 256, 65536), (1, 4096, 4096, 4096)]:
    A = torch.randn(b, m, k, dtype=torch.complex128, device="cuda")
    B = torch.randn(b, k, n, dtype=torch.complex128, device="cuda")
    for _ in range(3):
        C = A @ B
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        C = A @ B
    e1.record()
    torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) / 1e3 / 10
    print(json.dumps({"cublas_zgemm": [b, m, k, n], "us": dt * 1e6, "tflops": 8.0 * b * m * k * n / dt / 1e12}))
