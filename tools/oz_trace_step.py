"""CTA-0 phase timeline of the LAST emulated-GEMM launch of a C1 integration
(in-step conditions: graph replay, PDL neighbours, warm L2).
`CGL_OZ_TRACE=1 python tools/oz_trace_step.py [scheme] [steps]`"""
import os
import sys

os.environ["CGL_OZ_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes  # noqa: E402

import torch  # noqa: E402

import paper_2403_02816_b200 as P  # noqa: E402
from paper_2403_02816_b200 import _lib, workloads as W  # noqa: E402

scheme = sys.argv[1] if len(sys.argv) > 1 else "if4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
w = W.CONFIGS["C1"]
prob = W.build_problem(w)
x0 = W.initial_state_device(w)
P.integrate(prob, scheme, (x0,), w.tau * steps, steps)
r = P.integrate(prob, scheme, (x0,), w.tau * steps, steps)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 128)()
_lib.load().cgl_oz_trace(buf)
t0 = buf[0]
names = {0: "start", 1: "setup done", 42: "end"}
for j in range(8):
    names[3 + j] = f"tile {j}: issuer got accumulator"
    names[11 + j] = f"tile {j}: MMAs issued + committed"
    names[19 + j] = f"tile {j}: epilogue sees MMAs done"
    names[27 + j] = f"tile {j}: epilogue stored"
    names[44 + j] = f"  producer: chunk {j} copy issued"
    names[52 + j] = f"  issuer: chunk {j} data ready"
for j in range(16):
    names[64 + j] = f"  issuer: chunk {j} MMAs issued"
print(f"# last GEMM launch of a C1 {scheme} run ({1e3 * r.device_seconds / steps:.4f} ms/step); tile 0 live chunks: {buf[63]}")
buf[63] = 0
for t, lab in sorted((buf[i], names.get(i, f"slot {i}")) for i in range(128) if buf[i]):
    print(f"{(t - t0) / 1e3:8.2f} us  {lab}")
