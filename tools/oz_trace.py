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
buf = (ctypes.c_longlong * 64)()
lib.cgl_oz_trace(buf)
t0 = buf[0]
names = {0: "start", 1: "setup done (barriers, TMEM alloc+zero)", 40: "epilogue: tmem full", 41: "epilogue: staged",
         42: "end"}
names.update({44 + i: f"epilogue warp {i + 2}: levels done" for i in range(4)})
names.update({48 + i: f"epilogue warp {i + 2}: tmem full seen" for i in range(4)})
names.update({55 + i: f"mma chunk {i} issued" for i in range(1, 9)})
for i in range(64):
    if buf[i]:
        lab = names.get(i, f"producer chunk {i - 2}" if 3 <= i <= 18 else f"mma chunk {i - 18} ready")
        if 56 <= i <= 63:
            lab = f"mma chunk {i - 55} issued"
        print(f"{(buf[i] - t0) / 1e3:8.2f} us  {lab}")
