"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py            # unit + stepper + config fixtures
    python tests/golden/make_golden.py --no-c1    # skip the ~3 min C1 runs

The reference package `cglsolve` (/root/reference/pkg/src) is imported
read-only and executed as-is; its outputs pin both the oracle restatement
(oracle/cgl_oracle.py, CPU tests) and the GPU path (GPU parity tests).
Inputs come from seeded generators (numpy default_rng for unit cases, the
reference's own splitmix64 `normal_tensor` for the BASELINE configs); the
2nd-order / Neumann FD matrices of the BASELINE configs are built with the
oracle's builders and handed to the reference's KroneckerOperator, which
accepts any square factors (operators.py:111-118).
"""

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(REPO, "oracle"))
sys.path.insert(0, REPO)

import cglsolve  # noqa: E402  (the reference)
from cglsolve import flows as rflows  # noqa: E402
from cglsolve import integrators as rint  # noqa: E402
from cglsolve import linalg as rlinalg  # noqa: E402
from cglsolve import operators as rops  # noqa: E402
from cglsolve import rng as rrng  # noqa: E402
from cglsolve import spectral as rspec  # noqa: E402
from cglsolve import tensors as rtens  # noqa: E402

import cgl_oracle as O  # noqa: E402

SHAPES = [(7,), (16,), (3, 5), (8, 6), (2, 9), (4, 4, 4), (3, 4, 5), (6, 2, 7), (2, 3, 2, 4), (3, 2, 2, 2)]
CUBIC = dict(alpha1=1.0, beta1=2.0, alpha2=1.0, alpha3=-1.0, beta3=0.2)
CQ = dict(alpha1=0.5, beta1=0.5, alpha2=-0.5, alpha3=2.52, beta3=1.0, alpha4=-1.0, beta4=-0.11)
COUPLED = dict(alpha1=0.125, beta1=0.5, alpha2=-0.9, alpha0=-0.4, alpha3=1.0, beta3=0.8, alpha4=-0.1,
               beta4=-0.6, alpha5=0.5)
SCHEMES = ("rk2", "rk4", "strang", "split4", "strang_3t", "split4_3t", "if2", "if4")


def rc(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def unit_fixtures():
    out = {}
    rng = np.random.default_rng(20240)
    # mode products / tucker / kron sum (tensors.py:38-85)
    for i, shape in enumerate(SHAPES):
        u = rc(rng, shape)
        out[f"mp{i}_u"] = u
        for axis, n in enumerate(shape):
            m = rc(rng, (n + 1, n))
            out[f"mp{i}_a{axis}_m"] = m
            out[f"mp{i}_a{axis}_out"] = rtens.mu_mode_product(u, m, axis)
        sq = [rc(rng, (n, n)) for n in shape]
        for axis, m in enumerate(sq):
            out[f"tk{i}_m{axis}"] = m
        out[f"tk{i}_out"] = rtens.tucker_apply(u, sq)
        out[f"ks{i}_out"] = rtens.kron_sum_apply(u, sq)
    # expm across the Pade ladder + squaring (linalg.py:75-87)
    for j, nrm in enumerate((1e-3, 0.1, 0.8, 1.9, 5.0, 40.0)):
        a = rc(rng, (9, 9))
        a *= nrm / np.linalg.norm(a, 1)
        out[f"expm{j}_a"] = a
        out[f"expm{j}_out"] = rlinalg.expm_pade(a, 1.0)
    # flows (flows.py:62-133)
    pts = np.array([1.0, 0.3 - 0.7j, -1.1 + 0.4j, 0.05j, 2.0 + 1.0j])
    out["flow_pts"] = pts
    pc, pq, pk = (cglsolve.CglParameters(**d) for d in (CUBIC, CQ, COUPLED))
    out["cubic_flow"] = rflows.cubic_flow(pts, 0.3, pc)
    out["cubic_flow_pos"] = rflows.cubic_flow(pts, 0.02, pq)
    out["quintic_flow"] = rflows.quintic_flow(pts, 0.2, pq)
    out["g_cubic"] = rflows.eval_g(rflows.NonlinearSpec("cubic", pc), (pts,))[0]
    out["g_cq"] = rflows.eval_g(rflows.NonlinearSpec("cubic_quintic", pq), (pts,))[0]
    g2 = rflows.eval_g(rflows.NonlinearSpec("coupled_cubic_quintic", pk), (pts, pts[::-1].copy()))
    out["g_coupled_0"], out["g_coupled_1"] = g2
    r2 = rflows.rk4_flow(rflows.NonlinearSpec("coupled_cubic_quintic", pk), (pts, pts[::-1].copy()), 0.1)
    out["rk4_coupled_0"], out["rk4_coupled_1"] = r2
    out["rk4_cq"] = rflows.rk4_flow(rflows.NonlinearSpec("cubic_quintic", pq), (pts,), 0.05)[0]
    # rng (rng.py:21-64)
    out["rng_uniforms"] = rrng.uniforms(2024, 64)
    out["rng_normal_5x7"] = rrng.normal_tensor(2024, (5, 7))
    out["rng_normal_odd"] = rrng.standard_normals(7, 9)
    # spectral (spectral.py:26-129)
    g = rspec.FourierGrid((8, 5, 6), ((0.0, 10.0), (-1.0, 2.0), (0.0, 2 * np.pi)))
    out["wn_8"] = g.wavenumbers(0)
    out["wn_5"] = g.wavenumbers(1)
    out["symbol_856"] = rspec.build_symbol(g, pk, 1)
    u = rc(rng, (8, 5, 6))
    out["fft_u"] = u
    out["fft_out"] = rspec.dft_forward(u)
    out["ifft_out"] = rspec.dft_inverse(u)
    # snapshot bytes (io.py:35-59): reference writer on a small 3D pair
    import tempfile
    from cglsolve import io as rio
    su, sv = rc(rng, (3, 4, 5)), rc(rng, (3, 4, 5))
    grids = [np.linspace(0.0, 1.0, 3), np.linspace(-1.0, 1.0, 4), np.arange(5.0)]
    with tempfile.TemporaryDirectory() as td:
        rio.write_snapshot(td + "/s.cgls", (su, sv), 0.75, grids)
        out["snap_bytes"] = np.frombuffer(open(td + "/s.cgls", "rb").read(), dtype=np.uint8).copy()
        out["snap_grid"] = np.frombuffer(open(td + "/s.cgls.grid.txt", "rb").read(), dtype=np.uint8).copy()
    out["snap_u"], out["snap_v"] = su, sv
    # FD matrices (operators.py:49-85)
    out["fd4_dir_9"] = rops.fd_second_derivative_dirichlet(9, 3.0)
    out["fd4_dn_10"] = rops.fd_second_derivative_dirichlet_neumann(10, 3.0)
    return out


def _ref_problem(case):
    p = cglsolve.CglParameters(**case["params"])
    spec = rflows.NonlinearSpec(case["kind"], p)
    if case["op"] == "fd":
        if case["bc"] in ("dirichlet", "dirichlet_neumann"):
            op = rops.build_fd_operator(p, case["extents"], case["lengths"], case["bc"])
        else:
            d = len(case["extents"])
            mats = [p.diffusion * O.FD_BUILDERS[case["bc"]](n, L) + (p.alpha2 / d) * np.eye(n)
                    for n, L in zip(case["extents"], case["lengths"])]
            op = rops.KroneckerOperator(mats)
    else:
        grid = rspec.FourierGrid(case["extents"], case["intervals"])
        if spec.components == 2:
            op = rops.BlockOperator([rops.build_periodic_operator(grid, p, 1),
                                     rops.build_periodic_operator(grid, p, -1)])
        else:
            op = rops.build_periodic_operator(grid, p)
    return rint.Problem(op, spec)


def stepper_cases():
    """Small problems x all 8 schemes, plus divergence cases."""
    rng = np.random.default_rng(777)
    cases = []
    base = [
        dict(name="fd2d_dir4_cubic", op="fd", bc="dirichlet", extents=(12, 10), lengths=(6.0, 5.0),
             params=CUBIC, kind="cubic", t_final=0.3, steps=6, amp=0.5),
        dict(name="fd3d_dn4_cq", op="fd", bc="dirichlet_neumann", extents=(8, 7, 9), lengths=(4.0, 3.5, 4.5),
             params=CQ, kind="cubic_quintic", t_final=0.05, steps=4, amp=0.3),
        dict(name="fd2d_neu2_cq", op="fd", bc="neumann2", extents=(9, 11), lengths=(4.0, 5.0),
             params=CQ, kind="cubic_quintic", t_final=0.05, steps=5, amp=0.3),
        dict(name="four2d_cubic", op="fourier", extents=(16, 12), intervals=((0.0, 10.0), (0.0, 8.0)),
             params=CUBIC, kind="cubic", t_final=0.2, steps=5, amp=0.5),
        dict(name="four3d_cq", op="fourier", extents=(8, 6, 10), intervals=((-3.0, 3.0),) * 3,
             params=CQ, kind="cubic_quintic", t_final=0.04, steps=4, amp=0.3),
        dict(name="four1d_coupled", op="fourier", extents=(32,), intervals=((0.0, 70.0),),
             params=COUPLED, kind="coupled_cubic_quintic", t_final=0.3, steps=5, amp=0.5),
        dict(name="four2d_coupled", op="fourier", extents=(16, 8), intervals=((0.0, 70.0), (0.0, 35.0)),
             params=COUPLED, kind="coupled_cubic_quintic", t_final=0.3, steps=5, amp=0.5),
    ]
    for b in base:
        comps = 2 if b["kind"] == "coupled_cubic_quintic" else 1
        ics = [b["amp"] * rc(rng, b["extents"]) for _ in range(comps)]
        for s in SCHEMES:
            if comps == 2 and s in ("strang_3t", "split4_3t"):
                continue
            cases.append(dict(b, scheme=s, ic=ics, name=f"{b['name']}_{s}"))
    # divergence: explicit RK far outside stability (test_integrators.py:123-132)
    u0 = (np.random.default_rng(73).standard_normal(64) / 50.0).astype(complex)
    cases.append(dict(name="div_rk4_fd1d", op="fd", bc="dirichlet", extents=(64,), lengths=(100.0,),
                      params=CUBIC, kind="cubic", scheme="rk4", t_final=12.0, steps=10, ic=[u0]))
    # divergence: cubic blow-up (alpha3 > 0, y >= 1) inside a strang flow
    u0 = 3.0 * rc(np.random.default_rng(5), (6, 7))
    pblow = dict(alpha1=1.0, beta1=0.3, alpha2=0.0, alpha3=2.0, beta3=1.0)
    cases.append(dict(name="div_blowup_strang", op="fd", bc="dirichlet", extents=(6, 7), lengths=(3.0, 3.0),
                      params=pblow, kind="cubic", scheme="strang", t_final=0.5, steps=5, ic=[u0]))
    cases.append(dict(name="div_blowup_split4_3t", op="fourier", extents=(8, 8), intervals=((0.0, 5.0),) * 2,
                      params=pblow, kind="cubic", scheme="split4_3t", t_final=0.5, steps=5,
                      ic=[np.fft.fftn(3.0 * rc(np.random.default_rng(6), (8, 8)))]))
    return cases


def run_case(case):
    prob = _ref_problem(case)
    res = rint.integrate(prob, case["scheme"], tuple(case["ic"]), case["t_final"], case["steps"])
    return res


def stepper_fixtures():
    arrays, meta = {}, []
    for i, case in enumerate(stepper_cases()):
        res = run_case(case)
        for c, u in enumerate(case["ic"]):
            arrays[f"s{i}_ic{c}"] = u
        for c, u in enumerate(res.fields):
            arrays[f"s{i}_out{c}"] = u
        m = {k: v for k, v in case.items() if k not in ("ic", "amp")}
        m.update(index=i, components=len(case["ic"]), diverged=res.diverged,
                 diverged_at=res.diverged_at, reason=res.reason)
        meta.append(m)
        print(f"  {case['name']}: diverged={res.diverged} at={res.diverged_at} {res.reason!r}")
    return arrays, meta


def config_fixtures(with_c1=True):
    from paper_2403_02816_b200 import workloads as W
    arrays, meta = {}, []

    def run(tag, w, scheme, n_steps=None):
        u0 = W.initial_state(w)
        p = cglsolve.CglParameters(**{k: getattr(w.params, k) for k in O.Params.NAMES})
        spec = rflows.NonlinearSpec(w.kind, p)
        if w.boundary == "periodic":
            grid = rspec.FourierGrid(w.extents, (w.interval,) * len(w.extents))
            prob = rint.Problem(rops.build_periodic_operator(grid, p), spec)
            x0 = rspec.dft_forward(u0)
        else:
            a, b = w.interval
            d = len(w.extents)
            mats = [p.diffusion * O.FD_BUILDERS[w.boundary](n, b - a) + (p.alpha2 / d) * np.eye(n)
                    for n in w.extents]
            prob = rint.Problem(rops.KroneckerOperator(mats), spec)
            x0 = u0
        t0 = time.perf_counter()
        res = rint.integrate(prob, scheme, (x0,), w.t_final, w.steps)
        dt = time.perf_counter() - t0
        arrays[f"{tag}_out"] = res.fields[0]
        meta.append(dict(tag=tag, workload=w.name, scheme=scheme, extents=list(w.extents), steps=w.steps,
                         tau=w.tau, diverged=res.diverged, diverged_at=res.diverged_at, reason=res.reason,
                         ref_seconds=res.seconds, wall=dt))
        print(f"  {tag}: {w.name} {scheme} diverged={res.diverged}@{res.diverged_at} "
              f"loop={res.seconds:.2f}s")

    C = W.CONFIGS
    run("C0_strang", C["C0"], "strang")
    run("C1s64_if4", C["C1"].scaled(64, 40), "if4")
    run("C1s64_rk4", C["C1"].scaled(64, 40), "rk4")
    run("C2s24_split4", C["C2"].scaled(24, 10), "split4")
    run("C3s32_if4", C["C3"].scaled(32, 10), "if4")
    run("C3s32_strang", C["C3"].scaled(32, 10), "strang")
    run("C4s24_if4", C["C4"].scaled(24, 6), "if4")
    big = {}
    if with_c1:
        for s in ("if4", "strang", "rk4"):
            run(f"C1_{s}", C["C1"], s)
            big[f"C1_{s}_out"] = arrays.pop(f"C1_{s}_out")
    return arrays, meta, big


def main():
    with_c1 = "--no-c1" not in sys.argv
    print("unit fixtures")
    np.savez_compressed(os.path.join(HERE, "unit.npz"), **unit_fixtures())
    print("stepper fixtures")
    arrs, meta = stepper_fixtures()
    np.savez_compressed(os.path.join(HERE, "steppers.npz"), **arrs)
    with open(os.path.join(HERE, "steppers.json"), "w") as f:
        json.dump(meta, f, indent=1, default=lambda o: list(o) if isinstance(o, tuple) else str(o))
    print("config fixtures")
    arrs, meta, big = config_fixtures(with_c1)
    np.savez_compressed(os.path.join(HERE, "configs.npz"), **arrs)
    for k, v in big.items():
        np.save(os.path.join(HERE, f"{k}.npy"), v)
    old = []
    path = os.path.join(HERE, "configs.json")
    if not with_c1 and os.path.exists(path):
        old = [m for m in json.load(open(path)) if m["tag"].startswith("C1_")]
    with open(path, "w") as f:
        json.dump(meta + old, f, indent=1)


if __name__ == "__main__":
    main()
