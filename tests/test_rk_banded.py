"""Fused plans added in round 2 for the schemes that stepped eagerly before.

Banded Kronecker-sum Runge-Kutta stages (csrc/rkstage.cu, plan.BandedRKPlan)
against dense products (torch) for one stage, and the graph-captured rk2 / rk4
plans against the generic dense-GEMM path (CGL_FUSED=0) for whole runs:
1..3 dimensions, both FD orders, one and two components, a blow-up.
Tolerances: one stage <= 1e-13 relative max; runs <= 1e-11 relative L2
(identical math, different summation order); divergence step / reason and
the finite mask exact.  The stepper fixtures recorded from the reference
(test_gpu_parity.test_all_stepper_cases) run through the same plan."""

import numpy as np
import pytest
import torch

from conftest import rel_l2

pytestmark = pytest.mark.gpu


def _rand(shape, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.empty(shape, dtype=torch.complex128, device="cuda")
    x.real.normal_(generator=g)
    x.imag.normal_(generator=g)
    return x


def _banded(n, b, seed):
    rng = np.random.default_rng(seed)
    m = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    i, j = np.indices((n, n))
    m[np.abs(i - j) > b] = 0.0
    return m


def _pack(m, b):
    n = m.shape[0]
    band = np.zeros((n, 2 * b + 1), dtype=complex)
    for d in range(2 * b + 1):
        off = d - b
        i0, i1 = max(0, -off), min(n, n - off)
        band[i0:i1, d] = m[np.arange(i0, i1), np.arange(i0, i1) + off]
    return torch.from_numpy(band).cuda()


@pytest.mark.parametrize("shape,hb", [((40,), (2,)), ((24, 36), (1, 2)), ((12, 20, 16), (2, 0, 3))])
@pytest.mark.parametrize("nf", [1, 2])
def test_rk_stage_matches_dense_products(shape, hb, nf):
    from paper_2403_02816_b200 import _lib
    d = len(shape)
    mats = [[_banded(shape[mu], hb[mu], 10 * c + mu) for mu in range(d)] for c in range(nf)]
    bands = [_pack(mats[c][mu], hb[mu]) for c in range(nf) for mu in range(d)]
    x = [_rand(shape, 1 + c) for c in range(nf)]
    u = [_rand(shape, 5 + c) for c in range(nf)]
    acc = [_rand(shape, 9 + c) for c in range(nf)]
    nl = _lib.Nonlinear()
    nl.alpha3, nl.beta3, nl.alpha4, nl.beta4, nl.alpha5, nl.kind = -1.0, 0.7, 0.3, -0.2, 0.5 if nf == 2 else 0.0, \
        2 if nf == 2 else 1
    # dense reference: f = sum_mu A_mu x_mu x + g(x)
    f = []
    m2 = [xc.abs() ** 2 for xc in x]
    for c in range(nf):
        k = torch.zeros_like(x[c])
        for mu in range(d):
            a = torch.from_numpy(mats[c][mu]).cuda()
            k = k + torch.movedim(torch.tensordot(a, x[c], dims=([1], [mu])), 0, mu)
        g = (nl.alpha3 + 1j * nl.beta3) * m2[c] * x[c] + (nl.alpha4 + 1j * nl.beta4) * m2[c] ** 2 * x[c]
        if nf == 2:
            g = g + nl.alpha5 * m2[1 - c] * x[c]
        f.append(k + g)
    cx, ca = 0.37, -0.21
    x_out = [torch.empty_like(t) for t in x]
    acc_out = [torch.empty_like(t) for t in x]
    flag = _lib.new_flag(0)
    pa = _lib.ptr_array
    hb_c = (_lib.c_int * d)(*hb)
    rc = _lib.load().cgl_rk_stage(_lib.stream(), d, _lib.i64_array(shape), nf, hb_c, pa(bands), _lib.ctypes.byref(nl),
                                  pa(x), pa(u), pa(acc), pa(x_out), pa(acc_out), cx, ca, 1, _lib.flag_ptr(flag),
                                  _lib.rel_pos(1))
    assert rc == 0, _lib.load().cgl_last_error()
    torch.cuda.synchronize()
    for c in range(nf):
        scale = float(f[c].abs().max())
        assert float((x_out[c] - (u[c] + cx * f[c])).abs().max()) <= 1e-13 * scale
        assert float((acc_out[c] - (acc[c] + ca * f[c])).abs().max()) <= 1e-13 * scale
    assert int(flag[0]) == -1
    # acc_in = NULL starts the combination from u; an inf in x is flagged at (step, 255)
    x[0].view(-1)[3] = float("inf")
    rc = _lib.load().cgl_rk_stage(_lib.stream(), d, _lib.i64_array(shape), nf, hb_c, pa(bands), _lib.ctypes.byref(nl),
                                  pa(x), pa(u), None, None, pa(acc_out), 0.0, ca, 1, _lib.flag_ptr(flag),
                                  _lib.rel_pos(1))
    assert rc == 0
    key = int(flag[0].item())
    assert key != -1 and key & 0xFF == _lib.NONFINITE_STATE and (key >> 8) & 0xFFFF == 255


def test_rk_stage_argument_errors():
    from paper_2403_02816_b200 import _lib
    shape = (8, 8)
    x, u = _rand(shape, 0), _rand(shape, 1)
    band = _pack(_banded(8, 1, 0), 1)
    nl = _lib.Nonlinear()
    nl.kind = 0
    pa = _lib.ptr_array
    lib = _lib.load()

    def call(hb=(1, 1), xo=None, nf=1):
        xo = [torch.empty_like(x)] if xo is None else xo
        return lib.cgl_rk_stage(_lib.stream(), 2, _lib.i64_array(shape), nf, (_lib.c_int * 2)(*hb), pa([band, band]),
                                _lib.ctypes.byref(nl), pa([x]), pa([u]), None, pa(xo), None, 1.0, 1.0, 0, None, 0)

    assert call() == 0
    assert call(hb=(9, 1)) != 0            # half-bandwidth above 8
    assert call(xo=[x]) != 0               # output aliases the stage input
    assert call(nf=2) != 0                 # two components need the coupled kind


def _problem(extents, bc, kind):
    from paper_2403_02816_b200 import BlockOperator, CglParameters, NonlinearSpec, Problem, build_fd_operator
    kw = dict(alpha1=1.0, beta1=0.5, alpha2=1.0, alpha3=-1.0, beta3=1.0)
    if kind != "cubic":
        kw.update(alpha4=-0.1, beta4=0.05)
    if kind.startswith("coupled"):
        kw.update(alpha5=0.2)
    p = CglParameters(**kw)
    spec = NonlinearSpec(kind, p)
    lengths = tuple(10.0 + i for i in range(len(extents)))
    op = build_fd_operator(p, tuple(extents), lengths, bc)
    if spec.components == 2:
        op = BlockOperator([op, build_fd_operator(p, tuple(extents), lengths, bc)])
    return Problem(op, spec)


@pytest.mark.parametrize("extents,bc,kind", [((48,), "dirichlet", "cubic"), ((40, 56), "neumann2", "cubic_quintic"),
                                              ((16, 20, 24), "dirichlet_neumann", "cubic"),
                                              ((32, 32), "dirichlet2", "coupled_cubic_quintic")])
@pytest.mark.parametrize("scheme", ["rk2", "rk4"])
def test_banded_rk_plan_matches_dense_path(extents, bc, kind, scheme, monkeypatch):
    import paper_2403_02816_b200 as P
    from paper_2403_02816_b200.plan import BandedRKPlan
    rng = np.random.default_rng(7)
    nf = 2 if kind.startswith("coupled") else 1
    ic = [0.3 * (rng.standard_normal(extents) + 1j * rng.standard_normal(extents)) for _ in range(nf)]
    steps, t_final = 40, 40 * 2e-4
    prob = _problem(extents, bc, kind)
    got = P.integrate(prob, scheme, ic, t_final, steps)
    assert any(isinstance(pl, BandedRKPlan) for pl in prob._plans.values()), "banded RK plan not used"
    monkeypatch.setenv("CGL_FUSED", "0")
    want = P.integrate(_problem(extents, bc, kind), scheme, ic, t_final, steps)
    assert not got.diverged and not want.diverged
    for a, b in zip(got.fields, want.fields):
        assert rel_l2(a, b) <= 1e-11


def test_banded_rk_blow_up_matches_dense_path(monkeypatch):
    """An unstable step size: same diverged_at / reason and the same finite
    mask as the dense path (the failed step is redone on dense products)."""
    import paper_2403_02816_b200 as P
    rng = np.random.default_rng(3)
    extents = (64, 64)
    ic = [rng.standard_normal(extents) + 1j * rng.standard_normal(extents)]
    got = P.integrate(_problem(extents, "dirichlet2", "cubic"), "rk4", ic, 2.0, 40)
    monkeypatch.setenv("CGL_FUSED", "0")
    want = P.integrate(_problem(extents, "dirichlet2", "cubic"), "rk4", ic, 2.0, 40)
    assert want.diverged and (got.diverged, got.diverged_at, got.reason) == (True, want.diverged_at, want.reason)
    assert np.array_equal(np.isfinite(got.fields[0]), np.isfinite(want.fields[0]))


def test_dense_factors_stay_on_the_gemm_path():
    from paper_2403_02816_b200 import CglParameters, KroneckerOperator, NonlinearSpec, Problem, plan
    rng = np.random.default_rng(0)
    mats = [rng.standard_normal((24, 24)) * 0.1 for _ in range(2)]
    p = CglParameters(alpha1=1.0, beta1=0.5, alpha2=1.0, alpha3=-1.0, beta3=1.0)
    prob = Problem(KroneckerOperator(mats), NonlinearSpec("cubic", p))
    assert not plan.supports(prob, "rk4")
    assert plan.half_bandwidth(np.eye(5)) == 0 and plan.half_bandwidth(np.zeros((4, 4))) == 0


@pytest.mark.parametrize("scheme", ["strang_3t", "split4_3t"])
@pytest.mark.parametrize("extents", [(40, 56), (512, 512), (16, 20, 24)])
def test_three_term_schemes_run_fused(scheme, extents, monkeypatch):
    """strang_3t / split4_3t (integrators.py:178-195) on the graph-captured FD
    plan (strang / split4 bodies, every flow a pair of exact flows, kind 3 in the
    stage kernels; 512^2 takes the INT8-emulated products) == the eager generic
    path, and a quintic blow-up is reported at the same step with the same reason."""
    import paper_2403_02816_b200 as P
    from paper_2403_02816_b200.plan import FusedPlan
    rng = np.random.default_rng(11)
    ic = [0.4 * (rng.standard_normal(extents) + 1j * rng.standard_normal(extents))]
    steps, t_final = 12, 0.06
    prob = _problem(extents, "dirichlet2", "cubic_quintic")
    got = P.integrate(prob, scheme, ic, t_final, steps)
    plans = list(prob._plans.values())
    assert plans and all(type(pl) is FusedPlan and pl.three for pl in plans), "three-term plan not used"
    # explosive quintic term: finite-time blow-up of the exact quintic flow
    big = [8.0 * ic[0]]
    from paper_2403_02816_b200 import CglParameters, NonlinearSpec, Problem, build_fd_operator
    pp = CglParameters(alpha1=1.0, beta1=0.5, alpha2=1.0, alpha3=-1.0, beta3=1.0, alpha4=0.5, beta4=0.05)
    mk = lambda: Problem(build_fd_operator(pp, tuple(extents), tuple(10.0 + i for i in range(len(extents))),  # noqa: E731
                                           "dirichlet2"), NonlinearSpec("cubic_quintic", pp))
    got_b = P.integrate(mk(), scheme, big, t_final, steps)
    monkeypatch.setenv("CGL_FUSED", "0")
    want = P.integrate(_problem(extents, "dirichlet2", "cubic_quintic"), scheme, ic, t_final, steps)
    want_b = P.integrate(mk(), scheme, big, t_final, steps)
    assert not got.diverged and not want.diverged
    assert rel_l2(got.fields[0], want.fields[0]) <= 1e-11
    assert want_b.diverged and "quintic" in want_b.reason
    assert (got_b.diverged, got_b.diverged_at, got_b.reason) == (True, want_b.diverged_at, want_b.reason)
