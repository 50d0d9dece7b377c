"""Per-pass timing of the pencil-FFT kernels (csrc/fftpass.cu) at a 3D grid
(default 512^3): each program timed as 10 back-to-back launches inside a CUDA
graph (CUDA events), achieved HBM GB/s from the pass's algorithmic bytes,
against the measured copy bandwidth; cuFFT Z2Z 3D alongside.

    python tools/fft_probe.py [n]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

from paper_2403_02816_b200 import fftpass, spectral, workloads as W  # noqa: E402
from paper_2403_02816_b200 import SCHEMES  # noqa: E402


def timed(fn, reps=10, iters=5):
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
    for _ in range(iters):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / (iters * reps)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 512
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json"))).get("hbm_gbs", 6545.9) \
        if os.path.exists(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) else 6545.9
    w = W.CONFIGS["C3"].scaled(n, 1)
    prob = W.build_problem(w)
    prob.prepare(w.tau, SCHEMES["if4"])
    from paper_2403_02816_b200.plan import PencilFourierPlan
    shape = w.extents
    x = torch.randn(shape, dtype=torch.complex128, device="cuda")
    T = x.clone()
    u = x.clone()
    g = [x.clone() for _ in range(3)]
    plan = PencilFourierPlan(prob, "if4", [x])
    plan.load_state([x], w.tau)
    plan.flag = None  # timing only: no divergence skipping on overflowing data
    N = x.numel()
    rows = []

    eager = "--ncu" in sys.argv   # one eager launch per program (for an ncu capture)

    T0 = T.clone()
    copy_dt = timed(lambda: T.copy_(T0))

    def run(name, fn, bytes_pp, fresh=False):
        """fresh: refill T from a pristine field before each launch (programs
        with data-dependent FP64 work -- g, flows -- must not run on the
        overflowed values repeated unnormalised transforms produce); the copy's
        own time is subtracted."""
        if eager:
            fn()
            torch.cuda.synchronize()
            print(name, flush=True)
            return
        if fresh:
            dt = timed(lambda: (T.copy_(T0), fn())) - copy_dt
        else:
            dt = timed(fn)
        gbs = bytes_pp * N / dt / 1e9
        rows.append(dict(name=name, us=dt * 1e6, gbs=gbs, frac=gbs / peak, bytes_pp=bytes_pp))
        print(f"{name:28s} {dt * 1e6:9.1f} us  {gbs:8.1f} GB/s  {gbs / peak:6.3f} of {peak:.0f}", flush=True)

    for axis in (2, 1, 0):
        run(f"plain fwd axis {axis}", lambda a=axis: fftpass.axis_pass(T, T, a), 32)
        run(f"plain inv axis {axis}", lambda a=axis: fftpass.axis_pass(T, T, a, inverse=True), 32)
    # realistic magnitudes: T = F(u) of a field of O(0.1) values
    T0.copy_(fftpass.fftn(0.1 * x))
    run("G axis 0 (inv, g, fwd)", lambda: plan._pass("g", 0, T, T, w.tau, scale=1.0 / N), 32, True)
    run("IF4_B1 axis 2", lambda: plan._pass("if4_b1", 2, T, T, w.tau, u=u, g_out=g[0]), 64, True)
    run("IF4_B3 axis 2", lambda: plan._pass("if4_b3", 2, T, T, w.tau, u=u, g=(g[0], None, None), g_out=g[0]), 80,
        True)
    v = u.clone()
    run("IF4_B4 axis 2", lambda: plan._pass("if4_b4", 2, T, T, w.tau, u=g[0], u_out=v), 64, True)
    y = x.clone()
    run("STR_A0 axis 0", lambda: plan._pass("str_a0", 0, T, T, w.tau, u_out=y, scale=1.0 / N), 48, True)
    run("STR_A0F axis 0 (fused flows)", lambda: plan._pass("str_a0f", 0, T, T, w.tau, u_out=y, scale=1.0 / N), 48, True)
    run("STR_MID axis 2", lambda: plan._pass("str_mid", 2, T, T, w.tau), 32, True)
    run("cuFFT Z2Z 3D fwd", lambda: spectral.fft_dev(T, inverse=False, out=T), 32)
    if not eager:
        print(json.dumps(dict(n=n, peak_gbs=peak, rows=rows)))


if __name__ == "__main__":
    main()
