"""Does the emulated GEMM's speed depend on the data?  Times the if4 step's
2-field axis-0 product (E_1/2, data pre-sliced by the MID stage) on the step's
own operands after a real C1 run, and on random operands of the same shape."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_02816_b200 as P  # noqa: E402
from paper_2403_02816_b200 import _lib, ozaki, workloads as W  # noqa: E402
from fractions import Fraction  # noqa: E402

w = W.CONFIGS["C1"]
prob = W.build_problem(w)
x0 = W.initial_state_device(w)
P.integrate(prob, "if4", (x0,), w.tau * 40, 40)
plan = next(iter(prob._plans.values()))
F = plan._fs
u2, a = plan.B[2], plan.B[3]
x1, x5 = plan.B[0], plan.B[1]
fac = plan.blocks[0].sliced_factors(Fraction(1, 2))[0]
ws = plan.oz_ws


def timeit(fn, reps=40):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (3 * reps)


step = timeit(lambda: ozaki.mode_product_oz([u2[0], a[0]], [fac] * 2, [x1[0], x5[0]], 0, ws, presliced=[F[3], F[4]]))
# random operands, sliced the same way (fresh workspace)
g = torch.Generator(device="cuda").manual_seed(3)
R = [torch.randn(w.extents, dtype=torch.complex128, device="cuda", generator=g) for _ in range(2)]
O = [torch.empty_like(r) for r in R]
ws2 = ozaki.Workspace()
ozaki.mode_product_oz(R, [fac] * 2, O, 0, ws2)
Bs = [ws2.bufs[("D", k, 512)] for k in range(2)]
rnd = timeit(lambda: ozaki.mode_product_oz(R, [fac] * 2, O, 0, ws2, presliced=Bs))
# the step's operands scaled by random phases (same magnitudes, random low digits)
print(json.dumps({"step_operands_us": round(step, 2), "random_operands_us": round(rnd, 2)}))
