"""Fixtures for the pencil-FFT Fourier plans from the REAL reference.

The stepper fixtures (make_golden.py) use grids the pencil passes do not
serve (extents < 16 or not powers of two), so these cases pin the fused
plans (plan.PencilFourierPlan: if4 and strang on 2D/3D power-of-two grids)
directly against `cglsolve.integrate` (integrators.py:241-282): smooth runs,
every divergence reason the two schemes can produce, and snapshots around a
divergence (the look-ahead flow of strang's fused end-of-step pass must not
cost the reference's last snapshot).  Same case schema as steppers.json.

    python tests/golden/make_golden_pencil.py  -> tests/golden/pencil.{json,npz}
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import CQ, _ref_problem, rc, rint  # noqa: E402

P_CUBIC = dict(alpha1=1.0, beta1=0.5, alpha2=1.0, alpha3=-1.0, beta3=1.0)
P_BLOW = dict(alpha1=1.0, beta1=0.3, alpha2=1.0, alpha3=2.0, beta3=1.0)
TWO_PI = 2.0 * np.pi


def spectral_ic(seed, shape, amp):
    return np.fft.fftn(amp * rc(np.random.default_rng(seed), shape))


def bump_ic(shape, intervals, amp, spectral=True):
    """Centred Gaussian bump (coefficient space for Fourier cases): grows
    smoothly under an explosive nonlinearity, so a divergence lands after a
    few good steps."""
    ax = [a + (b - a) * np.arange(n) / n for n, (a, b) in zip(shape, intervals)]
    d = len(shape)
    r2 = sum(((x - (a + b) / 2) ** 2).reshape([-1 if j == i else 1 for j in range(d)])
             for i, (x, (a, b)) in enumerate(zip(ax, intervals)))
    u = amp * np.exp(-r2) * (1 + 0.1j)
    return np.fft.fftn(u) if spectral else u


def cases():
    out = []
    smooth = [
        dict(name="p3_cubic16", extents=(16, 16, 16), intervals=((0.0, 2 * TWO_PI),) * 3, params=P_CUBIC,
             kind="cubic", t_final=0.2, steps=10, amp=0.5, seed=11),
        dict(name="p3_cq_16x32x32", extents=(16, 32, 32), intervals=((-3.0, 3.0), (-4.0, 4.0), (-5.0, 5.0)),
             params=CQ, kind="cubic_quintic", t_final=0.02, steps=4, amp=0.3, seed=12),
        dict(name="p2_cubic64x32", extents=(64, 32), intervals=((0.0, 20.0), (0.0, 10.0)), params=P_CUBIC,
             kind="cubic", t_final=0.1, steps=10, amp=0.5, seed=13),
        dict(name="p3_cubic16x16x128", extents=(16, 16, 128), intervals=((0.0, 4.0), (0.0, 4.0), (0.0, 32.0)),
             params=P_CUBIC, kind="cubic", t_final=0.05, steps=5, amp=0.5, seed=14),
    ]
    for b in smooth:
        ic = spectral_ic(b["seed"], b["extents"], b["amp"])
        for s in ("if4", "strang"):
            out.append(dict(b, op="fourier", scheme=s, ic=[ic], name=f"{b['name']}_{s}"))
    return out


def divergence_cases():
    """Amplitude searched so the reference diverges after a few good steps."""
    specs = [
        # exact cubic flow: y = 2 a3 |u|^2 t >= 1 ("finite-time blow-up in cubic flow")
        dict(name="div_p2_blow_strang", extents=(32, 16), intervals=((-4.0, 4.0),) * 2, params=P_BLOW,
             kind="cubic", scheme="strang", t_final=0.5, steps=10, lo=1.2, hi=2.2, want="blow-up"),
        # Lawson on an explosive nonlinearity: non-finite state
        dict(name="div_p3_nonfinite_if4", extents=(16, 16, 16), intervals=((-4.0, 4.0),) * 3, params=P_BLOW,
             kind="cubic", scheme="if4", t_final=1.0, steps=10, lo=1.6, hi=2.4, want="non-finite state"),
        # cubic-quintic strang uses one RK4 substep as the flow: non-finite RK4 flow output
        dict(name="div_p3_cq_rk4flow_strang", extents=(16, 16, 16), intervals=((-3.0, 3.0),) * 3,
             params=dict(CQ, alpha4=3.0), kind="cubic_quintic", scheme="strang", t_final=1.0, steps=10,
             lo=0.6, hi=1.1, want="RK4"),
        # FD (Kronecker) strang: the fused end-of-step kernel also runs the next
        # step's first flow, so a blow-up there must still leave the last
        # snapshot the reference takes
        dict(name="div_fd_blow_strang", op="fd", bc="dirichlet", extents=(16, 16), lengths=(8.0, 8.0),
             intervals=((-4.0, 4.0),) * 2, params=P_BLOW, kind="cubic", scheme="strang", t_final=0.5, steps=10,
             lo=1.2, hi=2.6, want="blow-up"),
    ]
    out = []
    for sp in specs:
        hit = None
        for amp in np.geomspace(sp["lo"], sp["hi"], 81):
            op = sp.get("op", "fourier")
            ic = bump_ic(sp["extents"], sp["intervals"], amp, spectral=op == "fourier")
            case = dict(sp, op=op, ic=[ic])
            res = rint.integrate(_ref_problem(case), case["scheme"], (ic,), case["t_final"], case["steps"])
            if res.diverged and 3 <= res.diverged_at <= 8 and sp["want"] in res.reason:
                hit = dict(case, amp=float(amp))
                break
        if hit is None:
            raise RuntimeError(f"no diverging amplitude for {sp['name']}")
        out.append(hit)
    return out


def main():
    arrays, meta = {}, []
    all_cases = cases() + divergence_cases()
    for i, case in enumerate(all_cases):
        snaps = []
        # every step around a divergence; one mid-run step of a smooth run
        snap_steps = (tuple(range(1, case["steps"] + 1)) if case["name"].startswith("div_")
                      else (case["steps"] // 2,))
        res = rint.integrate(_ref_problem(case), case["scheme"], tuple(case["ic"]), case["t_final"], case["steps"],
                             snapshot_steps=snap_steps, on_snapshot=lambda k, t, f: snaps.append((k, f[0].copy())))
        arrays[f"s{i}_ic0"] = case["ic"][0]
        arrays[f"s{i}_out0"] = res.fields[0]
        for k, f in snaps:
            arrays[f"s{i}_snap{k}"] = f
        m = {k: v for k, v in case.items() if k not in ("ic", "seed", "want", "lo", "hi")}
        m.update(index=i, components=1, diverged=res.diverged, diverged_at=res.diverged_at, reason=res.reason,
                 snapshot_steps=list(snap_steps), snapshots_taken=[k for k, _ in snaps])
        meta.append(m)
        print(f"  {case['name']}: diverged={res.diverged}@{res.diverged_at} {res.reason!r} snaps={len(snaps)}")
    with open(os.path.join(HERE, "pencil.json"), "w") as f:
        json.dump(meta, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "pencil.npz"), **arrays)


if __name__ == "__main__":
    main()
