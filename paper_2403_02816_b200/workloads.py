"""The BASELINE.json configurations C0-C4 as concrete, seeded workloads.

Host-side setup shared by bench.py, the tests and the golden-fixture
generator: grid, boundary convention, parameters, initial state, scheme,
tau and step count.  Conventions the BASELINE text leaves open are pinned
here and recorded in DESIGN.md:
  * 2nd-order central FD; Dirichlet on interior nodes x_i = a + i h,
    h = L/(n+1); Neumann node-centred with ghost mirroring, h = L/(n-1);
  * complex noise xi_r + i xi_i with xi_r = normal_tensor(seed),
    xi_i = normal_tensor(seed + 1), seed 2024 (experiments.py:52);
  * C4's eight Gaussians drawn from uniforms(seed, 48) in the order
    (cx, cy, cz, width, phase, amplitude) per Gaussian.
No public dataset is involved: every input is synthetic and seeded.
"""

from dataclasses import dataclass

import numpy as np

from .params import CglParameters
from .rng import normal_tensor, uniforms

SEED = 2024

P_CUBIC = CglParameters(alpha1=1.0, beta1=0.5, alpha2=1.0, alpha3=-1.0, beta3=1.0)
P_CQ = CglParameters(alpha1=0.5, beta1=0.5, alpha2=-0.1, alpha3=1.0, beta3=1.0, alpha4=-0.1, beta4=-0.1)


@dataclass(frozen=True)
class Workload:
    name: str
    kind: str          # cubic / cubic_quintic
    boundary: str      # dirichlet2 / neumann2 / periodic
    params: CglParameters
    interval: tuple    # (a, b), same in every direction
    extents: tuple
    schemes: tuple     # first = headline stepper
    tau: float
    steps: int
    ic: str

    @property
    def t_final(self):
        return self.tau * self.steps

    @property
    def points(self):
        return int(np.prod(self.extents))

    def scaled(self, n, steps=None):
        """Same physics on an n^d grid (parity cases the CPU oracle can run)."""
        return Workload(self.name + f"@{n}", self.kind, self.boundary, self.params, self.interval,
                        (n,) * len(self.extents), self.schemes, self.tau,
                        self.steps if steps is None else steps, self.ic)


CONFIGS = {
    "C0": Workload("C0-2d-cubic-fd128-strang", "cubic", "dirichlet2", P_CUBIC, (-20.0, 20.0), (128, 128),
                   ("strang",), 0.01, 200, "sech_noise"),
    "C1": Workload("C1-2d-cubic-fd512", "cubic", "dirichlet2", P_CUBIC, (-20.0, 20.0), (512, 512),
                   ("if4", "rk4", "strang"), 0.005, 400, "sech_noise"),
    "C2": Workload("C2-3d-cq-neumann256-split4", "cubic_quintic", "neumann2", P_CQ, (-15.0, 15.0), (256, 256, 256),
                   ("split4",), 0.01, 100, "gauss_noise"),
    "C3": Workload("C3-3d-cubic-fourier512", "cubic", "periodic", P_CUBIC, (0.0, 16.0 * np.pi), (512, 512, 512),
                   ("if4", "strang"), 0.01, 100, "random_phase"),
    "C4": Workload("C4-3d-cq-dirichlet1024-if4", "cubic_quintic", "dirichlet2", P_CQ, (-30.0, 30.0),
                   (1024, 1024, 1024), ("if4",), 0.005, 50, "gaussians8"),
}


def axes(w):
    """Physical node coordinates per direction."""
    a, b = w.interval
    L = b - a
    out = []
    for n in w.extents:
        if w.boundary == "dirichlet2":
            out.append(a + np.arange(1, n + 1) * (L / (n + 1)))
        elif w.boundary == "neumann2":
            out.append(a + np.arange(n) * (L / (n - 1)))
        elif w.boundary == "periodic":
            out.append(a + np.arange(n) * (L / n))
        else:
            raise ValueError(w.boundary)
    return out


def _noise(shape, seed):
    return normal_tensor(seed, shape) + 1j * normal_tensor(seed + 1, shape)


def _radius2(w):
    ax = axes(w)
    r2 = np.zeros(w.extents)
    d = len(ax)
    for i, x in enumerate(ax):
        r2 = r2 + (x ** 2).reshape([-1 if j == i else 1 for j in range(d)])
    return r2


def initial_state(w, seed=SEED):
    """Physical-space u0 (numpy complex128, shape w.extents)."""
    if w.ic == "sech_noise":
        return (1.0 / np.cosh(np.sqrt(_radius2(w)))) * (1.0 + 0.01 * _noise(w.extents, seed))
    if w.ic == "gauss_noise":
        return 2.0 * np.exp(-_radius2(w) / 4.0) * (1.0 + 0.01 * _noise(w.extents, seed))
    if w.ic == "random_phase":
        return 0.1 * _noise(w.extents, seed)
    if w.ic == "gaussians8":
        a, b = w.interval
        L = b - a
        u = uniforms(seed, 48).reshape(8, 6)
        ax = axes(w)
        d = len(ax)
        out = np.zeros(w.extents, dtype=complex)
        for cx, cy, cz, wd, ph, am in u:
            centre = [a + L * (0.25 + 0.5 * c) for c in (cx, cy, cz)][:d]
            width = 1.0 + 3.0 * wd
            r2 = np.zeros(w.extents)
            for i, x in enumerate(ax):
                r2 = r2 + ((x - centre[i]) ** 2).reshape([-1 if j == i else 1 for j in range(d)])
            out += (0.5 + am) * np.exp(-r2 / (2.0 * width ** 2)) * np.exp(2j * np.pi * ph)
        return out
    raise ValueError(w.ic)


_IC_RECIPE = {"sech_noise": 0, "gauss_noise": 1, "random_phase": 2}


def initial_state_device(w, seed=SEED):
    """Device-built u0 (CUDA complex128), no N-sized host array.  The noise
    recipes run the seeded stream on the GPU (cgl_seeded_ic: uniforms
    bit-identical to the host, Box-Muller normals within a few ulp);
    gaussians8 is separable per Gaussian and assembled from 1D factors with
    the same parameters as initial_state."""
    import torch
    if w.ic in _IC_RECIPE:
        from . import _lib
        out = torch.empty(w.extents, dtype=torch.complex128, device="cuda")
        ax = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in axes(w)]
        _lib.check(_lib.load().cgl_seeded_ic(_lib.stream(), _IC_RECIPE[w.ic], seed, len(w.extents),
                                             _lib.i64_array(w.extents), _lib.ptr_array(ax), _lib.ptr(out)),
                   "cgl_seeded_ic")
        return out
    if w.ic != "gaussians8":
        return torch.from_numpy(initial_state(w, seed)).cuda()
    a, b = w.interval
    L = b - a
    u = uniforms(seed, 48).reshape(8, 6)
    ax = [torch.from_numpy(x).cuda() for x in axes(w)]
    d = len(ax)
    out = torch.zeros(w.extents, dtype=torch.complex128, device="cuda")
    for cx, cy, cz, wd, ph, am in u:
        centre = [a + L * (0.25 + 0.5 * c) for c in (cx, cy, cz)][:d]
        width = 1.0 + 3.0 * wd
        coef = (0.5 + am) * np.exp(2j * np.pi * ph)
        f = [torch.exp(-((x - c) ** 2) / (2.0 * width ** 2)) for x, c in zip(ax, centre)]
        term = f[0].to(torch.complex128) * coef
        for i in range(1, d):
            term = term.unsqueeze(-1) * f[i].reshape([1] * i + [-1])
        out += term
    return out


def fd_matrices(w):
    """Per-direction A_mu = (a1 + i b1) D2 + (a2/d) I (host numpy)."""
    from .operators import fd2_second_derivative_dirichlet, fd2_second_derivative_neumann
    build = {"dirichlet2": fd2_second_derivative_dirichlet, "neumann2": fd2_second_derivative_neumann}[w.boundary]
    a, b = w.interval
    d = len(w.extents)
    return [w.params.diffusion * build(n, b - a) + (w.params.alpha2 / d) * np.eye(n) for n in w.extents]


def build_problem(w):
    """GPU Problem for a workload (FD Kronecker form or Fourier form)."""
    from .flows import NonlinearSpec
    from .integrators import Problem
    from .operators import KroneckerOperator, build_periodic_operator
    from .spectral import FourierGrid
    spec = NonlinearSpec(w.kind, w.params)
    if w.boundary == "periodic":
        grid = FourierGrid(w.extents, (w.interval,) * len(w.extents))
        return Problem(build_periodic_operator(grid, w.params), spec)
    return Problem(KroneckerOperator(fd_matrices(w)), spec)


def state_for_problem(w, u0):
    """The integrator's state representation: coefficients for periodic
    (unnormalised forward DFT on the GPU, like experiments.py:447)."""
    if w.boundary == "periodic":
        from .spectral import dft_forward
        return dft_forward(u0)
    return u0
