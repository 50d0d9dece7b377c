"""CPU ORACLE — test infrastructure only, never the product path.

A numpy restatement of the reference `cglsolve` hot path (arXiv 2403.02816,
`/root/reference/pkg/src/cglsolve/*`), written independently: every function
cites the reference file:line whose behaviour it restates.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py` (the `cpu_baseline` leg and
`--impl reference`) may import this module, and only as the checker / the CPU
baseline.  The shipped package `paper_2403_02816_b200` never imports it.

Parity pinning: `tests/golden/make_golden.py` imports the real reference in
the build container and records its outputs as fixtures under
`tests/golden/`; `tests/test_oracle_golden.py` checks this restatement
against every fixture (CPU, no GPU needed).  The arithmetic itself lives in
numpy (OpenBLAS zgemm via tensordot, pocketfft, LAPACK gesv) exactly as in
the reference, so the oracle reproduces the reference to rounding level.

Paths below are relative to /root/reference/pkg/src/cglsolve/.
"""

from __future__ import annotations

import math
import time
from fractions import Fraction

import numpy as np

# ---------------------------------------------------------------------------
# parameters (params.py:16-46)
# ---------------------------------------------------------------------------


class Params:
    """Coefficient bundle, restating params.py:16-46 (validation included)."""

    NAMES = ("alpha1", "beta1", "alpha2", "alpha3", "beta3", "alpha4",
             "beta4", "alpha0", "alpha5")

    def __init__(self, alpha1, beta1=0.0, alpha2=0.0, alpha3=0.0, beta3=0.0,
                 alpha4=0.0, beta4=0.0, alpha0=0.0, alpha5=0.0):
        vals = dict(alpha1=alpha1, beta1=beta1, alpha2=alpha2, alpha3=alpha3,
                    beta3=beta3, alpha4=alpha4, beta4=beta4, alpha0=alpha0,
                    alpha5=alpha5)
        for k, v in vals.items():
            if not isinstance(v, (int, float)) or not math.isfinite(v):
                raise ValueError(f"parameter {k} must be a finite real")
            setattr(self, k, float(v))
        if self.alpha1 <= 0.0:
            raise ValueError("alpha1 must be positive (parabolic diffusion)")

    diffusion = property(lambda s: complex(s.alpha1, s.beta1))  # params.py:37
    cubic = property(lambda s: complex(s.alpha3, s.beta3))      # params.py:41
    quintic = property(lambda s: complex(s.alpha4, s.beta4))    # params.py:45


# ---------------------------------------------------------------------------
# tensors.py — mode products
# ---------------------------------------------------------------------------


def mode_product(u, mat, axis):
    """tensors.py:38-59: contract `mat` (m x n_axis) with direction `axis`."""
    u = np.asarray(u)
    mat = np.asarray(mat)
    if mat.ndim != 2 or not 0 <= axis < u.ndim or mat.shape[1] != u.shape[axis]:
        raise ValueError("bad mode-product arguments")
    out = np.tensordot(mat, u, axes=(1, axis))  # one zgemm, new axis first
    return np.moveaxis(out, 0, axis)


def tucker(u, mats):
    """tensors.py:62-69: modes applied in order 0, 1, ..., d-1."""
    if len(mats) != np.ndim(u):
        raise ValueError("one factor per direction")
    for axis, m in enumerate(mats):
        u = mode_product(u, m, axis)
    return u


def kron_sum(u, mats):
    """tensors.py:72-85: sum over directions of single-mode products."""
    if len(mats) != np.ndim(u):
        raise ValueError("one factor per direction")
    acc = None
    for axis, m in enumerate(mats):
        t = mode_product(u, m, axis)
        acc = t if acc is None else acc + t
    return acc


def kron_sum_dense(mats):
    """Explicit Kronecker-sum matrix for column-major vec (tensors.py:88-112)."""
    sizes = [np.asarray(m).shape[0] for m in mats]
    total = int(np.prod(sizes))
    out = np.zeros((total, total), dtype=complex)
    for axis, m in enumerate(mats):
        f = np.eye(1)
        for k, n in enumerate(sizes):
            f = np.kron(np.asarray(m) if k == axis else np.eye(n), f)
        out += f
    return out


def vec(u):
    """tensors.py:28-30 (first index fastest)."""
    return np.asarray(u).reshape(-1, order="F")


def unvec(x, shape):
    """tensors.py:33-35."""
    return np.asarray(x).reshape(tuple(shape), order="F")


# ---------------------------------------------------------------------------
# linalg.py — Pade exponential (setup, untimed in the reference)
# ---------------------------------------------------------------------------

_PADE_THETA = ((3, 1.495585217958292e-2), (5, 2.539398330063230e-1),
               (7, 9.504178996162932e-1), (9, 2.097847961257068e0),
               (13, 5.371920351148152e0))                      # linalg.py:17-23


def _pade_coeffs(p):
    """Diagonal Pade numerator coefficients c_k = (2p-k)! p! / ((2p)! k! (p-k)!),
    normalised so that c_p = 1 (the integer tables of linalg.py:25-38)."""
    c = [Fraction(math.factorial(2 * p - k) * math.factorial(p),
                  math.factorial(k) * math.factorial(p - k)) for k in range(p + 1)]
    return [float(x / c[p]) for x in c]


def _pade(b, p):
    """linalg.py:50-72: r_p(b) = (V - U)^{-1} (V + U)."""
    c = _pade_coeffs(p)
    n = b.shape[0]
    eye = np.eye(n, dtype=complex)
    b2 = b @ b
    if p == 13:
        b4 = b2 @ b2
        b6 = b2 @ b4
        uu = b @ (b6 @ (c[13] * b6 + c[11] * b4 + c[9] * b2)
                  + c[7] * b6 + c[5] * b4 + c[3] * b2 + c[1] * eye)
        vv = (b6 @ (c[12] * b6 + c[10] * b4 + c[8] * b2)
              + c[6] * b6 + c[4] * b4 + c[2] * b2 + c[0] * eye)
    else:
        uu, vv, pw = c[1] * eye, c[0] * eye, eye
        for k in range(1, p // 2 + 1):
            pw = pw @ b2
            uu = uu + c[2 * k + 1] * pw
            vv = vv + c[2 * k] * pw
        uu = b @ uu
    return np.linalg.solve(vv - uu, vv + uu)


def expm(a, scale=1.0):
    """linalg.py:75-87: smallest Pade degree whose theta admits ||b||_1,
    else scale-and-square around degree 13."""
    b = np.asarray(a, dtype=complex) * scale
    nrm = np.linalg.norm(b, 1) if b.size else 0.0
    for p, theta in _PADE_THETA[:-1]:
        if nrm <= theta:
            return _pade(b, p)
    th13 = _PADE_THETA[-1][1]
    s = max(0, math.ceil(math.log2(nrm / th13))) if nrm > th13 else 0
    f = _pade(b / 2.0 ** s, 13)
    for _ in range(s):
        f = f @ f
    return f


# ---------------------------------------------------------------------------
# finite-difference matrices (operators.py:42-96, plus the 2nd-order
# conventions pinned in SURVEY.md §0.4 for the BASELINE configs)
# ---------------------------------------------------------------------------


def fd4_dirichlet(n, length):
    """operators.py:49-64: 4th-order D2, interior nodes, h = L/(n+1)."""
    if n < 6:
        raise ValueError("Dirichlet D2 needs at least 6 interior nodes")
    h = length / (n + 1)
    a = np.zeros((n, n))
    a[0, :5] = (-15.0, -4.0, 14.0, -6.0, 1.0)
    a[1, :4] = (16.0, -30.0, 16.0, -1.0)
    for i in range(2, n - 2):
        a[i, i - 2:i + 3] = (-1.0, 16.0, -30.0, 16.0, -1.0)
    a[n - 2, n - 4:] = (-1.0, 16.0, -30.0, 16.0)
    a[n - 1, n - 5:] = (1.0, -6.0, 14.0, -4.0, -15.0)
    return a / (12.0 * h * h)


def fd4_dirichlet_neumann(n, length):
    """operators.py:67-85: 4th-order D2 with u(0)=0, u'(L)=0, h = L/n."""
    if n < 7:
        raise ValueError("Dirichlet-Neumann D2 needs at least 7 nodes")
    h = length / n
    a = np.zeros((n, n))
    a[0, :5] = (-15.0, -4.0, 14.0, -6.0, 1.0)
    a[1, :4] = (16.0, -30.0, 16.0, -1.0)
    for i in range(2, n - 2):
        a[i, i - 2:i + 3] = (-1.0, 16.0, -30.0, 16.0, -1.0)
    a[n - 2, n - 6:] = (1.0, -6.0, 14.0, -4.0, -15.0, 10.0)
    a[n - 1, n - 5:] = (1.0, -8.0 / 3.0, -6.0, 56.0, -145.0 / 3.0)
    return a / (12.0 * h * h)


def fd2_dirichlet(n, length):
    """2nd-order central D2 on interior nodes, h = L/(n+1)."""
    h = length / (n + 1)
    a = -2.0 * np.eye(n) + np.eye(n, k=1) + np.eye(n, k=-1)
    return a / (h * h)


def fd2_neumann(n, length):
    """2nd-order D2, homogeneous Neumann on both ends by ghost mirroring:
    n nodes including both ends, h = L/(n-1); first row (-2, 2)/h^2, last
    row (2, -2)/h^2."""
    h = length / (n - 1)
    a = -2.0 * np.eye(n) + np.eye(n, k=1) + np.eye(n, k=-1)
    a[0, 1] = 2.0
    a[n - 1, n - 2] = 2.0
    return a / (h * h)


FD_BUILDERS = {"dirichlet": fd4_dirichlet,
               "dirichlet_neumann": fd4_dirichlet_neumann,
               "dirichlet2": fd2_dirichlet,
               "neumann2": fd2_neumann}


def fd_nodes(kind, n, length):
    """operators.py:88-96 plus the 2nd-order conventions (offset from a)."""
    if kind in ("dirichlet", "dirichlet2"):
        return np.arange(1, n + 1) * (length / (n + 1))
    if kind == "dirichlet_neumann":
        return np.arange(1, n + 1) * (length / n)
    if kind == "neumann2":
        return np.arange(n) * (length / (n - 1))
    raise ValueError(f"unknown boundary kind {kind!r}")


def fd_matrices(params, extents, lengths, bc):
    """operators.py:211-229: A_mu = (a1 + i b1) D2_mu + (a2/d) I."""
    d = len(extents)
    return [params.diffusion * FD_BUILDERS[bc](n, L) + (params.alpha2 / d) * np.eye(n)
            for n, L in zip(extents, lengths)]


# ---------------------------------------------------------------------------
# spectral.py
# ---------------------------------------------------------------------------


def wavenumbers(n, interval):
    """spectral.py:26-35: 0..n//2 then negatives, scaled by 2 pi/(b-a)."""
    a, b = interval
    m = np.arange(n)
    m = np.where(m > n // 2, m - n, m)
    return m * (2.0 * np.pi / (b - a))


def periodic_nodes(n, interval):
    """spectral.py:66-70: x_j = a + j (b-a)/n."""
    a, b = interval
    return a + np.arange(n) * ((b - a) / n)


def symbol(extents, intervals, params, advection_sign=0):
    """spectral.py:89-113."""
    d = len(extents)
    ksq = np.zeros(tuple(extents))
    for ax in range(d):
        k = wavenumbers(extents[ax], intervals[ax])
        sh = [1] * d
        sh[ax] = -1
        ksq = ksq + (k ** 2).reshape(sh)
    s = params.diffusion * (-ksq) + params.alpha2
    if advection_sign:
        k1 = wavenumbers(extents[0], intervals[0]).reshape([-1] + [1] * (d - 1))
        s = s + advection_sign * params.alpha0 * (1j * k1)
    return s


# ---------------------------------------------------------------------------
# flows.py
# ---------------------------------------------------------------------------

_FLOOR = 1e-14  # flows.py:29


class Diverged(Exception):
    """flows.py:32-39 (DivergenceError): reason string."""

    def __init__(self, reason):
        super().__init__(reason)
        self.reason = reason


def eval_g(kind, p, fields):
    """flows.py:62-78."""
    mods = [np.abs(u) ** 2 for u in fields]
    out = []
    for i, u in enumerate(fields):
        g = p.cubic * mods[i] * u
        if kind != "cubic":
            g = g + p.quintic * (mods[i] * mods[i]) * u
        if kind == "coupled_cubic_quintic":
            g = g + p.alpha5 * mods[1 - i] * u
        out.append(g)
    return tuple(out)


def _finite_or_raise(u, reason):
    if not np.all(np.isfinite(u)):
        raise Diverged(reason)
    return u


def cubic_flow(u, t, p):
    """flows.py:87-100: exact flow of u' = (a3 + i b3)|u|^2 u."""
    u = np.asarray(u, dtype=complex)
    m = np.abs(u) ** 2
    if abs(p.alpha3) < _FLOOR:
        return u * np.exp(1j * p.beta3 * m * t)
    y = 2.0 * p.alpha3 * m * t
    if np.any(y >= 1.0):
        raise Diverged("finite-time blow-up in cubic flow")
    c = -(p.cubic / (2.0 * p.alpha3))
    return _finite_or_raise(u * np.exp(c * np.log1p(-y)),
                            "non-finite cubic flow output")


def quintic_flow(u, t, p):
    """flows.py:103-115: exact flow of u' = (a4 + i b4)|u|^4 u."""
    u = np.asarray(u, dtype=complex)
    m4 = np.abs(u) ** 4
    if abs(p.alpha4) < _FLOOR:
        return u * np.exp(1j * p.beta4 * m4 * t)
    y = 4.0 * p.alpha4 * m4 * t
    if np.any(y >= 1.0):
        raise Diverged("finite-time blow-up in quintic flow")
    c = -(p.quintic / (4.0 * p.alpha4))
    return _finite_or_raise(u * np.exp(c * np.log1p(-y)),
                            "non-finite quintic flow output")


def rk4_flow(kind, p, fields, t):
    """flows.py:118-133: one classical RK4 step on u' = g(u)."""
    k1 = eval_g(kind, p, fields)
    k2 = eval_g(kind, p, tuple(u + 0.5 * t * k for u, k in zip(fields, k1)))
    k3 = eval_g(kind, p, tuple(u + 0.5 * t * k for u, k in zip(fields, k2)))
    k4 = eval_g(kind, p, tuple(u + t * k for u, k in zip(fields, k3)))
    out = tuple(u + (t / 6.0) * (a + 2.0 * b + 2.0 * c + d)
                for u, a, b, c, d in zip(fields, k1, k2, k3, k4))
    for u in out:
        _finite_or_raise(u, "non-finite RK4 flow output")
    return out


# ---------------------------------------------------------------------------
# operators + problem adapter (operators.py:106-208, integrators.py:62-127)
# ---------------------------------------------------------------------------


class KronOp:
    """operators.py:106-139: per-direction matrices, exp cache by Fraction."""

    fourier = False

    def __init__(self, mats):
        self.mats = [np.asarray(m, dtype=complex) for m in mats]
        self.cache = {}

    def apply(self, u):
        return kron_sum(u, self.mats)

    def prepare(self, tau, fractions):
        self.cache = {Fraction(f): [expm(m, float(Fraction(f)) * tau) for m in self.mats]
                      for f in fractions}

    def exp_apply(self, f, u):
        return tucker(u, self.cache[Fraction(f)])


class FourierOp:
    """operators.py:142-174: diagonal symbol, exp cache by Fraction."""

    fourier = True

    def __init__(self, sym):
        self.sym = np.asarray(sym)
        self.cache = {}

    def apply(self, u):
        return self.sym * u

    def prepare(self, tau, fractions):
        self.cache = {Fraction(f): np.exp(float(Fraction(f)) * tau * self.sym)
                      for f in fractions}

    def exp_apply(self, f, u):
        return self.cache[Fraction(f)] * u


# Worker threads of the n-dimensional FFTs.  1 (default, every parity use) is
# numpy's own pocketfft exactly as the reference calls it (spectral.py:79-86);
# bench.py's CPU legs set the host core count, which runs the same pocketfft
# C++ transforms through scipy.fft with the batch of 1D lines split over
# threads -- the reference algorithm with all host threads, not a different one.
FFT_WORKERS = 1


def _fftn(u):
    if FFT_WORKERS > 1:
        import scipy.fft
        return scipy.fft.fftn(u, workers=FFT_WORKERS)
    return np.fft.fftn(u)


def _ifftn(u):
    if FFT_WORKERS > 1:
        import scipy.fft
        return scipy.fft.ifftn(u, workers=FFT_WORKERS)
    return np.fft.ifftn(u)


class Prob:
    """integrators.py:62-127 (blocks = one operator per component)."""

    def __init__(self, blocks, kind, params):
        self.blocks = list(blocks)
        self.kind = kind
        self.p = params
        self.fourier = self.blocks[0].fourier

    def phys(self, fs):       # integrators.py:78-81
        return tuple(_ifftn(u) for u in fs) if self.fourier else fs

    def spec(self, fs):       # integrators.py:83-86
        return tuple(_fftn(u) for u in fs) if self.fourier else fs

    def lin(self, fs):
        return tuple(b.apply(u) for b, u in zip(self.blocks, fs))

    def expk(self, f, fs):
        return tuple(b.exp_apply(f, u) for b, u in zip(self.blocks, fs))

    def g(self, fs):
        return self.spec(eval_g(self.kind, self.p, self.phys(fs)))

    def flow(self, fs, t):   # integrators.py:103-110
        ph = self.phys(fs)
        if self.kind == "cubic":
            ph = tuple(cubic_flow(u, t, self.p) for u in ph)
        else:
            ph = rk4_flow(self.kind, self.p, ph, t)
        return self.spec(ph)

    def flow_cubic(self, fs, t):
        return self.spec(tuple(cubic_flow(u, t, self.p) for u in self.phys(fs)))

    def flow_quintic(self, fs, t):
        return self.spec(tuple(quintic_flow(u, t, self.p) for u in self.phys(fs)))


# ---------------------------------------------------------------------------
# steppers (integrators.py:130-227)
# ---------------------------------------------------------------------------

H, ONE = Fraction(1, 2), Fraction(1)

SCHEME_FRACTIONS = {"rk2": (), "rk4": (), "strang": (ONE,), "split4": (ONE, H),
                    "strang_3t": (ONE,), "split4_3t": (ONE, H), "if2": (ONE,),
                    "if4": (H, ONE)}                       # integrators.py:50-59
THREE_TERM = {"strang_3t", "split4_3t"}


def _ax(a, x, y):
    return tuple(a * p + q for p, q in zip(x, y))


def _add(x, y):
    return tuple(p + q for p, q in zip(x, y))


def _sc(a, x):
    return tuple(a * p for p in x)


def _rhs(P, u):
    return _add(P.lin(u), P.g(u))


def step_rk2(P, u, tau):               # integrators.py:146-149
    f1 = _rhs(P, u)
    f2 = _rhs(P, _ax(tau, f1, u))
    return _ax(0.5 * tau, _add(f1, f2), u)


def step_rk4(P, u, tau):               # integrators.py:152-158
    f1 = _rhs(P, u)
    f2 = _rhs(P, _ax(0.5 * tau, f1, u))
    f3 = _rhs(P, _ax(0.5 * tau, f2, u))
    f4 = _rhs(P, _ax(tau, f3, u))
    s = _add(_add(f1, _sc(2.0, f2)), _add(_sc(2.0, f3), f4))
    return _ax(tau / 6.0, s, u)


def step_strang(P, u, tau):            # integrators.py:161-164
    return P.flow(P.expk(ONE, P.flow(u, 0.5 * tau)), 0.5 * tau)


def step_split4(P, u, tau):            # integrators.py:167-175
    coarse = P.flow(P.expk(ONE, P.flow(u, 0.5 * tau)), 0.5 * tau)
    fine = P.flow(u, 0.25 * tau)
    fine = P.expk(H, fine)
    fine = P.flow(fine, 0.5 * tau)
    fine = P.expk(H, fine)
    fine = P.flow(fine, 0.25 * tau)
    return _ax(-1.0 / 3.0, coarse, _sc(4.0 / 3.0, fine))


def _strang3(P, u, tau, f):            # integrators.py:178-184
    t = float(f) * tau
    v = P.flow_quintic(u, 0.5 * t)
    v = P.flow_cubic(v, 0.5 * t)
    v = P.expk(f, v)
    v = P.flow_cubic(v, 0.5 * t)
    return P.flow_quintic(v, 0.5 * t)


def step_strang_3t(P, u, tau):         # integrators.py:187-188
    return _strang3(P, u, tau, ONE)


def step_split4_3t(P, u, tau):         # integrators.py:191-195
    coarse = _strang3(P, u, tau, ONE)
    fine = _strang3(P, _strang3(P, u, tau, H), tau, H)
    return _ax(-1.0 / 3.0, coarse, _sc(4.0 / 3.0, fine))


def step_if2(P, u, tau):               # integrators.py:198-202
    g1 = P.g(u)
    u2 = P.expk(ONE, _ax(tau, g1, u))
    out = P.expk(ONE, _ax(0.5 * tau, g1, u))
    return _ax(0.5 * tau, P.g(u2), out)


def step_if4(P, u, tau):               # integrators.py:205-215
    g1 = P.g(u)
    u2 = P.expk(H, _ax(0.5 * tau, g1, u))
    g2 = P.g(u2)
    u3 = _ax(0.5 * tau, g2, P.expk(H, u))
    g3 = P.g(u3)
    u4 = _ax(tau, P.expk(H, g3), P.expk(ONE, u))
    g4 = P.g(u4)
    out = P.expk(ONE, _ax(tau / 6.0, g1, u))
    out = _ax(tau / 3.0, P.expk(H, _add(g2, g3)), out)
    return _ax(tau / 6.0, g4, out)


STEPPERS = {"rk2": step_rk2, "rk4": step_rk4, "strang": step_strang,
            "split4": step_split4, "strang_3t": step_strang_3t,
            "split4_3t": step_split4_3t, "if2": step_if2, "if4": step_if4}


class Result:
    """integrators.py:230-238."""

    def __init__(self, fields, steps, tau, seconds, diverged=False,
                 diverged_at=0, reason=""):
        self.fields, self.steps, self.tau, self.seconds = fields, steps, tau, seconds
        self.diverged, self.diverged_at, self.reason = diverged, diverged_at, reason


def integrate(P, scheme, fields, t_final, steps, max_steps=None):
    """integrators.py:241-282.  `max_steps` (oracle-only) stops early after
    that many steps so a bounded CPU sample of a long run can be timed."""
    if scheme not in STEPPERS:
        raise ValueError(f"unknown scheme {scheme!r}")
    if steps < 1:
        raise ValueError("steps must be >= 1")
    tau = t_final / steps
    fields = tuple(np.asarray(u, dtype=complex) for u in fields)
    if scheme in THREE_TERM and P.kind == "coupled_cubic_quintic":
        raise ValueError("three-term splitting has no coupled exact flow")
    fr = SCHEME_FRACTIONS[scheme]
    if fr:
        for b in P.blocks:
            b.prepare(tau, fr)
    fn = STEPPERS[scheme]
    last = steps if max_steps is None else min(steps, max_steps)
    t0 = time.perf_counter()
    for k in range(1, last + 1):
        try:
            with np.errstate(over="ignore", invalid="ignore"):
                fields = fn(P, fields, tau)
        except Diverged as e:
            return Result(fields, steps, tau, time.perf_counter() - t0, True, k, e.reason)
        if not all(np.all(np.isfinite(u)) for u in fields):
            return Result(fields, steps, tau, time.perf_counter() - t0, True, k,
                          "non-finite state")
    return Result(fields, steps, tau, time.perf_counter() - t0)


# ---------------------------------------------------------------------------
# seeded inputs: rng.py:21-64 (splitmix64 counter stream + Box-Muller)
# ---------------------------------------------------------------------------

_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def uniforms(seed, count, start=0):
    """rng.py:21-43: value i = top 53 bits of splitmix64(seed + (i+1) g), +1, / 2^53."""
    with np.errstate(over="ignore"):
        c = np.arange(start, start + count, dtype=np.uint64)
        z = np.uint64(seed) + (c + np.uint64(1)) * _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return ((z >> np.uint64(11)).astype(np.float64) + 1.0) / float(1 << 53)


def normals(seed, count):
    """rng.py:46-57: Box-Muller on consecutive uniform pairs."""
    pairs = (count + 1) // 2
    u = uniforms(seed, 2 * pairs)
    r = np.sqrt(-2.0 * np.log(u[0::2]))
    th = 2.0 * np.pi * u[1::2]
    out = np.empty(2 * pairs)
    out[0::2] = r * np.cos(th)
    out[1::2] = r * np.sin(th)
    return out[:count]


def normal_tensor(seed, shape):
    """rng.py:60-64: filled first-index-fastest."""
    shape = tuple(int(n) for n in shape)
    return normals(seed, int(np.prod(shape))).reshape(shape, order="F")
