"""The CPU oracle (oracle/cgl_oracle.py) pinned against fixtures produced by
the real reference (tests/golden/make_golden.py).  No GPU needed."""

import numpy as np
import pytest

import cgl_oracle as O
from cases import inputs, oracle_problem
from conftest import rel_l2, rel_max

SHAPES = [(7,), (16,), (3, 5), (8, 6), (2, 9), (4, 4, 4), (3, 4, 5), (6, 2, 7), (2, 3, 2, 4), (3, 2, 2, 2)]
CUBIC = O.Params(alpha1=1.0, beta1=2.0, alpha2=1.0, alpha3=-1.0, beta3=0.2)
CQ = O.Params(alpha1=0.5, beta1=0.5, alpha2=-0.5, alpha3=2.52, beta3=1.0, alpha4=-1.0, beta4=-0.11)
COUPLED = O.Params(alpha1=0.125, beta1=0.5, alpha2=-0.9, alpha0=-0.4, alpha3=1.0, beta3=0.8, alpha4=-0.1,
                   beta4=-0.6, alpha5=0.5)


@pytest.mark.parametrize("i", range(len(SHAPES)))
def test_mode_products(unit_golden, i):
    g = unit_golden
    u = g[f"mp{i}_u"]
    for axis in range(u.ndim):
        got = O.mode_product(u, g[f"mp{i}_a{axis}_m"], axis)
        assert rel_max(got, g[f"mp{i}_a{axis}_out"]) <= 1e-13
    mats = [g[f"tk{i}_m{a}"] for a in range(u.ndim)]
    assert rel_max(O.tucker(u, mats), g[f"tk{i}_out"]) <= 1e-13
    assert rel_max(O.kron_sum(u, mats), g[f"ks{i}_out"]) <= 1e-13


def test_tucker_matches_dense_kron(unit_golden):
    g = unit_golden
    u = g["mp3_u"]
    mats = [g["tk3_m0"], g["tk3_m1"]]
    dense = np.kron(mats[1], mats[0])
    assert rel_max(O.vec(O.tucker(u, mats)), dense @ O.vec(u)) <= 1e-13
    assert rel_max(O.vec(O.kron_sum(u, mats)), O.kron_sum_dense(mats) @ O.vec(u)) <= 1e-13


@pytest.mark.parametrize("j", range(6))
def test_expm(unit_golden, j):
    g = unit_golden
    assert rel_max(O.expm(g[f"expm{j}_a"]), g[f"expm{j}_out"]) <= 1e-14


def test_flows(unit_golden):
    g = unit_golden
    pts = g["flow_pts"]
    assert rel_max(O.cubic_flow(pts, 0.3, CUBIC), g["cubic_flow"]) <= 1e-15
    assert rel_max(O.cubic_flow(pts, 0.02, CQ), g["cubic_flow_pos"]) <= 1e-15
    assert rel_max(O.quintic_flow(pts, 0.2, CQ), g["quintic_flow"]) <= 1e-15
    assert rel_max(O.eval_g("cubic", CUBIC, (pts,))[0], g["g_cubic"]) <= 1e-15
    assert rel_max(O.eval_g("cubic_quintic", CQ, (pts,))[0], g["g_cq"]) <= 1e-15
    a, b = O.eval_g("coupled_cubic_quintic", COUPLED, (pts, pts[::-1].copy()))
    assert rel_max(a, g["g_coupled_0"]) <= 1e-15 and rel_max(b, g["g_coupled_1"]) <= 1e-15
    a, b = O.rk4_flow("coupled_cubic_quintic", COUPLED, (pts, pts[::-1].copy()), 0.1)
    assert rel_max(a, g["rk4_coupled_0"]) <= 1e-15 and rel_max(b, g["rk4_coupled_1"]) <= 1e-15
    assert rel_max(O.rk4_flow("cubic_quintic", CQ, (pts,), 0.05)[0], g["rk4_cq"]) <= 1e-15


def test_blowup_raises():
    with pytest.raises(O.Diverged) as e:
        O.cubic_flow(np.array([2.0 + 1.0j]), 0.1, CQ)
    assert "blow-up" in e.value.reason


def test_rng_bitwise(unit_golden):
    g = unit_golden
    assert np.array_equal(O.uniforms(2024, 64), g["rng_uniforms"])
    assert np.array_equal(O.normal_tensor(2024, (5, 7)), g["rng_normal_5x7"])
    assert np.array_equal(O.normals(7, 9), g["rng_normal_odd"])


def test_spectral(unit_golden):
    g = unit_golden
    assert np.array_equal(O.wavenumbers(8, (0.0, 10.0)), g["wn_8"])
    assert np.array_equal(O.wavenumbers(5, (-1.0, 2.0)), g["wn_5"])
    ext, iv = (8, 5, 6), ((0.0, 10.0), (-1.0, 2.0), (0.0, 2 * np.pi))
    assert rel_max(O.symbol(ext, iv, COUPLED, 1), g["symbol_856"]) <= 1e-15


def test_fd_matrices(unit_golden):
    g = unit_golden
    assert np.array_equal(O.fd4_dirichlet(9, 3.0), g["fd4_dir_9"])
    assert np.array_equal(O.fd4_dirichlet_neumann(10, 3.0), g["fd4_dn_10"])


def test_fd2_conventions():
    a = O.fd2_dirichlet(5, 6.0)
    assert np.allclose(a * 1.0 ** 2, -2 * np.eye(5) + np.eye(5, k=1) + np.eye(5, k=-1))
    n = O.fd2_neumann(4, 3.0)  # h = 1
    assert n[0, 1] == 2.0 and n[3, 2] == 2.0 and n[1, 0] == 1.0
    # Neumann D2 annihilates constants (mass-conserving diffusion)
    assert np.allclose(n @ np.ones(4), 0.0)


def test_all_stepper_cases(stepper_golden):
    meta, arrays = stepper_golden
    for case in meta:
        ic, want = inputs(case, arrays)
        res = O.integrate(oracle_problem(case), case["scheme"], ic, case["t_final"], case["steps"])
        assert res.diverged == case["diverged"], case["name"]
        assert res.diverged_at == case["diverged_at"], case["name"]
        assert res.reason == case["reason"], case["name"]
        for got, w in zip(res.fields, want):
            fin = np.isfinite(w)
            assert np.array_equal(np.isfinite(got), fin), case["name"]
            if fin.any():
                assert rel_l2(got[fin], w[fin]) <= 1e-12, case["name"]


@pytest.mark.parametrize("tag", ["C0_strang", "C1s64_if4", "C1s64_rk4", "C2s24_split4", "C3s32_if4",
                                 "C3s32_strang", "C4s24_if4"])
def test_config_cases(config_golden, tag):
    from paper_2403_02816_b200 import workloads as W
    meta, arrays = config_golden
    m = meta[tag]
    key = m["workload"].split("-")[0]
    w = W.CONFIGS[key]
    if "@" in m["workload"]:
        w = w.scaled(m["extents"][0], m["steps"])
    u0 = W.initial_state(w)
    p = O.Params(**{k: getattr(w.params, k) for k in O.Params.NAMES})
    if w.boundary == "periodic":
        blocks = [O.FourierOp(O.symbol(w.extents, (w.interval,) * len(w.extents), p))]
        x0 = np.fft.fftn(u0)
    else:
        a, b = w.interval
        mats = [p.diffusion * O.FD_BUILDERS[w.boundary](n, b - a) + (p.alpha2 / len(w.extents)) * np.eye(n)
                for n in w.extents]
        blocks = [O.KronOp(mats)]
        x0 = u0
    res = O.integrate(O.Prob(blocks, w.kind, p), m["scheme"], (x0,), w.t_final, w.steps)
    assert res.diverged == m["diverged"]
    assert rel_l2(res.fields[0], arrays[f"{tag}_out"]) <= 1e-12
