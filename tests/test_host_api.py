"""Host-side logic that needs no GPU: parameter/spec validation, scheme
registry, grids, FD builders, bit-compatible seeded inputs, Pade setup and
the BASELINE workloads."""

from fractions import Fraction

import numpy as np
import pytest

import paper_2403_02816_b200 as P
from paper_2403_02816_b200 import linalg, operators, rng, spectral, workloads
from conftest import rel_max


def test_public_names_match_reference():
    want = {"CglParameters", "NonlinearSpec", "DivergenceError", "FourierGrid", "KroneckerOperator",
            "FourierOperator", "BlockOperator", "build_fd_operator", "build_periodic_operator", "SCHEMES",
            "Problem", "IntegrationResult", "integrate"}
    assert want <= set(P.__all__)


def test_params_validation():
    with pytest.raises(ValueError):
        P.CglParameters(alpha1=0.0)
    with pytest.raises(ValueError):
        P.CglParameters(alpha1=1.0, beta1=float("nan"))
    with pytest.raises(ValueError):
        P.CglParameters(alpha1=1.0, alpha3=float("inf"))
    p = P.CglParameters(alpha1=1.0, beta1=2.0, alpha3=-1.0, beta3=0.5, alpha4=0.1, beta4=0.2)
    assert p.diffusion == 1 + 2j and p.cubic == -1 + 0.5j and p.quintic == 0.1 + 0.2j


def test_spec_validation():
    p = P.CglParameters(alpha1=1.0, alpha4=0.1)
    with pytest.raises(ValueError):
        P.NonlinearSpec("cubic", p)
    with pytest.raises(ValueError):
        P.NonlinearSpec("quartic", p)
    with pytest.raises(TypeError):
        P.NonlinearSpec("cubic_quintic", {"alpha1": 1.0})
    with pytest.raises(ValueError):
        P.NonlinearSpec("cubic_quintic", P.CglParameters(alpha1=1.0, alpha5=0.3))
    assert P.NonlinearSpec("coupled_cubic_quintic", P.CglParameters(alpha1=1.0, alpha5=0.3)).components == 2


def test_scheme_registry():
    assert set(P.SCHEMES) == {"rk2", "rk4", "strang", "split4", "strang_3t", "split4_3t", "if2", "if4"}
    assert P.SCHEMES["if4"].fractions == (Fraction(1, 2), Fraction(1))
    assert P.SCHEMES["split4"].fractions == (Fraction(1), Fraction(1, 2))
    assert not P.SCHEMES["rk4"].uses_exponentials
    assert P.SCHEMES["split4_3t"].three_term


def test_problem_validation_no_device():
    p = P.CglParameters(alpha1=0.125, beta1=0.5, alpha2=-0.9, alpha0=-0.4, alpha3=1.0, beta3=0.8,
                        alpha4=-0.1, beta4=-0.6, alpha5=0.5)
    g = P.FourierGrid((8,), ((0.0, 70.0),))
    op = P.build_periodic_operator(g, p)
    with pytest.raises(ValueError):
        P.Problem(op, P.NonlinearSpec("coupled_cubic_quintic", p))
    blk = P.BlockOperator([P.build_periodic_operator(g, p, 1), P.build_periodic_operator(g, p, -1)])
    with pytest.raises(ValueError):
        P.Problem(blk, P.NonlinearSpec("cubic_quintic", P.CglParameters(alpha1=1.0, alpha4=0.1)))
    prob = P.Problem(blk, P.NonlinearSpec("coupled_cubic_quintic", p))
    with pytest.raises(ValueError):
        prob.prepare(0.1, P.SCHEMES["strang_3t"])
    with pytest.raises(ValueError):
        P.integrate(prob, "nope", (np.zeros(8), np.zeros(8)), 1.0, 2)
    with pytest.raises(ValueError):
        P.integrate(prob, "if4", (np.zeros(8), np.zeros(8)), 1.0, 0)


def test_fourier_grid_and_wavenumbers(unit_golden):
    g = P.FourierGrid((8, 5), ((0.0, 10.0), (-1.0, 2.0)))
    assert np.array_equal(g.wavenumbers(0), unit_golden["wn_8"])
    assert np.array_equal(g.wavenumbers(1), unit_golden["wn_5"])
    assert g.nodes(0)[1] == pytest.approx(1.25)
    with pytest.raises(ValueError):
        P.FourierGrid((1,), ((0.0, 1.0),))
    with pytest.raises(ValueError):
        P.FourierGrid((4,), ((1.0, 1.0),))


def test_symbol_matches_reference(unit_golden):
    p = P.CglParameters(alpha1=0.125, beta1=0.5, alpha2=-0.9, alpha0=-0.4, alpha3=1.0, beta3=0.8,
                        alpha4=-0.1, beta4=-0.6, alpha5=0.5)
    g = P.FourierGrid((8, 5, 6), ((0.0, 10.0), (-1.0, 2.0), (0.0, 2 * np.pi)))
    assert rel_max(spectral.build_symbol(g, p, 1), unit_golden["symbol_856"]) <= 1e-15


def test_separable_tables_factorise_the_exponential():
    p = P.CglParameters(alpha1=0.125, beta1=0.5, alpha2=-0.9, alpha0=-0.4)
    g = P.FourierGrid((8, 5, 6), ((0.0, 10.0), (-1.0, 2.0), (0.0, 2 * np.pi)))
    op = P.build_periodic_operator(g, p, -1)
    s = 0.37
    full = np.exp(s * op.symbol)
    prod = np.ones(g.shape, dtype=complex)
    for ax in range(3):
        k = g.wavenumbers(ax)
        arg = -s * p.diffusion * k ** 2
        if ax == 0:
            arg = arg + s * p.alpha2 - s * p.alpha0 * 1j * k
        prod = prod * np.exp(arg).reshape([-1 if i == ax else 1 for i in range(3)])
    assert rel_max(prod, full) <= 1e-14


def test_fd_builders_match_reference(unit_golden):
    assert np.array_equal(operators.fd_second_derivative_dirichlet(9, 3.0), unit_golden["fd4_dir_9"])
    assert np.array_equal(operators.fd_second_derivative_dirichlet_neumann(10, 3.0), unit_golden["fd4_dn_10"])
    with pytest.raises(ValueError):
        operators.fd_second_derivative_dirichlet(5, 1.0)
    with pytest.raises(ValueError):
        P.build_fd_operator(P.CglParameters(alpha1=1.0), (8,), (1.0,), "robin")


def test_fd2_builders_match_oracle():
    import cgl_oracle as O
    assert np.array_equal(operators.fd2_second_derivative_dirichlet(11, 4.0), O.fd2_dirichlet(11, 4.0))
    assert np.array_equal(operators.fd2_second_derivative_neumann(11, 4.0), O.fd2_neumann(11, 4.0))
    op = P.build_fd_operator(P.CglParameters(alpha1=1.0, beta1=0.5, alpha2=1.0), (6, 7), (2.0, 3.0), "dirichlet2")
    assert op.shape == (6, 7)
    assert op.matrices[0][0, 0] == pytest.approx((1 + 0.5j) * -2.0 / (2.0 / 7) ** 2 + 0.5)


def test_rng_bit_compatible(unit_golden):
    assert np.array_equal(rng.uniforms(2024, 64), unit_golden["rng_uniforms"])
    assert np.array_equal(rng.normal_tensor(2024, (5, 7)), unit_golden["rng_normal_5x7"])
    assert np.array_equal(rng.standard_normals(7, 9), unit_golden["rng_normal_odd"])
    with pytest.raises(ValueError):
        rng.uniforms(-1, 3)


@pytest.mark.parametrize("j", range(6))
def test_expm_pade_setup(unit_golden, j):
    got = linalg.expm_pade(unit_golden[f"expm{j}_a"])
    assert rel_max(got, unit_golden[f"expm{j}_out"]) <= 1e-14


def test_expm_validation():
    with pytest.raises(ValueError):
        linalg.expm_pade(np.ones((2, 3)))
    with pytest.raises(ValueError):
        linalg.expm_pade(np.array([[np.nan]]))
    assert np.array_equal(linalg.expm_pade(np.zeros((3, 3))), np.eye(3))


def test_workloads_are_baseline_configs():
    C = workloads.CONFIGS
    assert C["C0"].extents == (128, 128) and C["C0"].steps == 200 and C["C0"].tau == 0.01
    assert C["C1"].extents == (512, 512) and C["C1"].schemes[0] == "if4" and C["C1"].steps == 400
    assert C["C2"].boundary == "neumann2" and C["C2"].schemes == ("split4",)
    assert C["C3"].boundary == "periodic" and C["C3"].extents == (512,) * 3
    assert C["C4"].extents == (1024,) * 3 and C["C4"].tau == 0.005
    w = C["C0"]
    a = workloads.initial_state(w)
    b = workloads.initial_state(w)
    assert np.array_equal(a, b) and a.shape == (128, 128)
    x = workloads.axes(w)[0]
    assert x[0] == pytest.approx(-20.0 + 40.0 / 129.0)
    g = workloads.initial_state(C["C4"].scaled(16))
    assert g.shape == (16, 16, 16) and np.all(np.isfinite(g))


def test_snapshot_bitwise_vs_reference(unit_golden, tmp_path):
    """write_snapshot reproduces the reference writer's bytes exactly
    (io.py:35-59), and read_snapshot round-trips them."""
    from paper_2403_02816_b200 import io as cio
    g = unit_golden
    grids = [np.linspace(0.0, 1.0, 3), np.linspace(-1.0, 1.0, 4), np.arange(5.0)]
    path = tmp_path / "s.cgls"
    cio.write_snapshot(path, (g["snap_u"], g["snap_v"]), 0.75, grids)
    assert path.read_bytes() == g["snap_bytes"].tobytes()
    assert (tmp_path / "s.cgls.grid.txt").read_bytes() == g["snap_grid"].tobytes()
    (u, v), t = cio.read_snapshot(path)
    assert t == 0.75 and u.tobytes() == g["snap_u"].tobytes() and v.tobytes() == g["snap_v"].tobytes()


def test_snapshot_errors(tmp_path):
    from paper_2403_02816_b200 import io as cio
    p = tmp_path / "bad.cgls"
    p.write_bytes(b"WAT?" + b"\x00" * 64)
    with pytest.raises(ValueError, match="magic"):
        cio.read_snapshot(p)
    with pytest.raises(ValueError):
        cio.write_snapshot(tmp_path / "x.cgls", (np.zeros((2, 3)), np.zeros((3, 2))), 0.0, [range(2), range(3)])


@pytest.mark.parametrize("shape,world", [((8, 6, 4), 2), ((12, 5), 4), ((6,), 3)])
def test_sharded_snapshot_writer_matches_single_writer(tmp_path, shape, world):
    """Every rank storing its axis-0 slab through the shared file map gives the
    reference writer's bytes (io.py:35-59) -- no gather of the field."""
    from paper_2403_02816_b200 import io as cio
    rng = np.random.default_rng(1)
    fields = [rng.standard_normal(shape) + 1j * rng.standard_normal(shape) for _ in range(2)]
    grids = [np.linspace(-1.0, 1.0, n) for n in shape]
    whole, parts = tmp_path / "whole.cgls", tmp_path / "parts.cgls"
    cio.write_snapshot(whole, fields, 1.25, grids)
    p0 = shape[0] // world
    for rank in range(world):
        a, b = rank * p0, (rank + 1) * p0
        cio.write_snapshot_sharded(parts, [f[a:b] for f in fields], 1.25, grids, shape, (a, b), rank=rank,
                                   chunk_bytes=64)
    assert parts.read_bytes() == whole.read_bytes()
    assert (tmp_path / "parts.cgls.grid.txt").read_text() == (tmp_path / "whole.cgls.grid.txt").read_text()
    with pytest.raises(ValueError):
        cio.write_snapshot_sharded(parts, [fields[0]], 0.0, grids, shape, (0, p0))
