"""Time one cuFFT Z2Z transform of a 512^3 complex128 field through the
library's plan cache (spectral.fft_dev / ifft_dev) vs torch.fft.fftn."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_02816_b200 import spectral  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
x = torch.randn((n, n, n), dtype=torch.complex128, device="cuda")
for name, fn in (("cgl fft_dev", lambda: spectral.fft_dev(x)), ("torch.fft.fftn", lambda: torch.fft.fftn(x))):
    y = fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        y = fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name}: {ms:.3f} ms per {n}^3 Z2Z ({2 * 16 * n ** 3 / ms / 1e6:.0f} GB/s of one read+write pass)")
    del y
