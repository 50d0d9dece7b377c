"""Phase timeline of CTA 0 of one ozgemm launch (CGL_OZ_TRACE=1)."""
import ctypes
import os
import sys

os.environ["CGL_OZ_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_02816_b200 import _lib, ozaki, workloads as W  # noqa: E402

lib = _lib.load()
w = W.CONFIGS["C1"]
prob = W.build_problem(w)
prob.operator.prepare(w.tau, (1,))
fac = prob.operator.sliced_factors(1)[0]
ins = [torch.randn(w.extents, dtype=torch.complex128, device="cuda") for _ in range(4)]
outs = [torch.empty_like(x) for x in ins]
ws = ozaki.Workspace()
for _ in range(3):
    ozaki.mode_product_oz(ins, [fac] * 4, outs, 0, ws)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 128)()
lib.cgl_oz_trace(buf)
t0 = buf[0]
persistent = True  # the persistent kernel serves every S = 8 product of the plans
names = {0: "start", 1: "setup done (barriers, TMEM alloc+zero)", 40: "epilogue: tmem full", 41: "epilogue: staged",
         42: "end"}
if persistent:
    for j in range(8):
        names[3 + j] = f"tile {j}: issuer got accumulator"
        names[11 + j] = f"tile {j}: MMAs issued + committed"
        names[19 + j] = f"tile {j}: epilogue sees MMAs done"
        names[27 + j] = f"tile {j}: epilogue stored"
        names[44 + j] = f"  producer: chunk {j} copy issued"
        names[52 + j] = f"  issuer: chunk {j} data ready"
    for j in range(16):
        names[64 + j] = f"  issuer: chunk {j} MMAs issued"
    for j in range(8):
        names[112 + j] = f"tile {j}: issuer loop top"
        names[120 + j] = f"tile {j}: issuer zero-map prefetch issued"
    for j in range(8, 16):
        names[80 + j] = f"  issuer: chunk {j} data ready"
        names[96 + j] = f"  producer: chunk {j} copy issued"
    for j in range(2):
        names[36 + 3 * j] = f"tile {j}: epilogue levels recombined"
        names[37 + 3 * j] = f"tile {j}: epilogue buffer re-zeroed + released"
        names[38 + 3 * j] = f"tile {j}: epilogue scaled"
    print("tile 0 live chunks:", buf[63])
    buf[63] = 0
else:
    names.update({44 + i: f"epilogue warp {i + 2}: levels done" for i in range(4)})
    names.update({48 + i: f"epilogue warp {i + 2}: tmem full seen" for i in range(4)})
    names.update({55 + i: f"mma chunk {i} issued" for i in range(1, 9)})
    names.update({2 + i: f"producer chunk {i}" for i in range(1, 17)})
    names.update({18 + i: f"mma chunk {i} ready" for i in range(1, 17)})
ev = sorted((buf[i], names.get(i, f"slot {i}")) for i in range(128) if buf[i])
for t, lab in ev:
    print(f"{(t - t0) / 1e3:8.2f} us  {lab}")
