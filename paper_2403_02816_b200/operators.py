"""Semidiscrete linear operators on the GPU (operator protocol of the
reference operators.py:106-208: representation / shape / apply / prepare /
exp_apply).

* KroneckerOperator — one dense matrix A_mu per direction; exp(f tau K) acts
  as a Tucker chain of the cached exp(f tau A_mu) (DMMA GEMMs).  The cache
  holds each exponential and its transpose on the device, keyed by exact
  Fraction like operators.py:123-139.
* FourierOperator — diagonal symbol in coefficient space.  When built by
  build_periodic_operator the exponential is kept FACTORISED per axis
  (exp(f tau symbol) = prod_mu e_mu[j_mu], spectral.py:101-112 is a sum of
  per-axis terms), so a multiply reads one field and tiny tables instead of
  an N-sized E tensor; an arbitrary user symbol falls back to the full
  E tensor computed on the device.
* BlockOperator — componentwise, for the coupled system.

FD matrices are host setup (numpy): the reference's 4th-order stencils
(operators.py:42-85) plus the 2nd-order central / Neumann variants the
BASELINE configs use.
"""

from fractions import Fraction

import numpy as np
import torch

from . import _lib
from ._device import to_device, to_host_if
from .linalg import expm_pade
from .spectral import build_symbol, mul_dev
from .tensors import kron_sum_dev, tucker_dev

__all__ = ["fd_second_derivative_dirichlet", "fd_second_derivative_dirichlet_neumann",
           "fd2_second_derivative_dirichlet", "fd2_second_derivative_neumann", "fd_nodes",
           "KroneckerOperator", "FourierOperator", "BlockOperator", "build_fd_operator",
           "build_periodic_operator"]

# 4th-order stencil numerators over 12 h^2 (operators.py:42-46)
_EDGE = (-15.0, -4.0, 14.0, -6.0, 1.0)
_NEXT = (16.0, -30.0, 16.0, -1.0)
_MID = (-1.0, 16.0, -30.0, 16.0, -1.0)
_NEU_PEN = (1.0, -6.0, 14.0, -4.0, -15.0, 10.0)
_NEU_LAST = (1.0, -8.0 / 3.0, -6.0, 56.0, -145.0 / 3.0)


def _interior4(n):
    a = np.zeros((n, n))
    a[0, :5] = _EDGE
    a[1, :4] = _NEXT
    for i in range(2, n - 2):
        a[i, i - 2:i + 3] = _MID
    return a


def fd_second_derivative_dirichlet(n, length):
    """4th-order D2, homogeneous Dirichlet, interior nodes h = L/(n+1)."""
    if n < 6:
        raise ValueError("Dirichlet D2 needs at least 6 interior nodes")
    h = length / (n + 1)
    a = _interior4(n)
    a[n - 2, n - 4:] = _NEXT[::-1]
    a[n - 1, n - 5:] = _EDGE[::-1]
    return a / (12.0 * h * h)


def fd_second_derivative_dirichlet_neumann(n, length):
    """4th-order D2 with u(0) = 0, u'(L) = 0, nodes i h, h = L/n."""
    if n < 7:
        raise ValueError("Dirichlet-Neumann D2 needs at least 7 nodes")
    h = length / n
    a = _interior4(n)
    a[n - 2, n - 6:] = _NEU_PEN
    a[n - 1, n - 5:] = _NEU_LAST
    return a / (12.0 * h * h)


def fd2_second_derivative_dirichlet(n, length):
    """2nd-order central D2 = tridiag(1, -2, 1)/h^2 on interior nodes,
    h = L/(n+1) (BASELINE configs 0, 1, 4)."""
    if n < 1:
        raise ValueError("need at least one interior node")
    h = length / (n + 1)
    return (-2.0 * np.eye(n) + np.eye(n, k=1) + np.eye(n, k=-1)) / (h * h)


def fd2_second_derivative_neumann(n, length):
    """2nd-order D2 with homogeneous Neumann on both ends (ghost mirroring):
    n nodes including both ends, h = L/(n-1), rows 0 and n-1 are (-2, 2) and
    (2, -2) over h^2 (BASELINE config 2)."""
    if n < 2:
        raise ValueError("Neumann D2 needs at least 2 nodes")
    h = length / (n - 1)
    a = -2.0 * np.eye(n) + np.eye(n, k=1) + np.eye(n, k=-1)
    a[0, 1] = 2.0
    a[n - 1, n - 2] = 2.0
    return a / (h * h)


_BUILDERS = {"dirichlet": fd_second_derivative_dirichlet,
             "dirichlet_neumann": fd_second_derivative_dirichlet_neumann,
             "dirichlet2": fd2_second_derivative_dirichlet,
             "neumann2": fd2_second_derivative_neumann}


def fd_nodes(kind, n, length):
    """Nodes matching the FD matrices, offset from the left end a."""
    if kind in ("dirichlet", "dirichlet2"):
        return np.arange(1, n + 1) * (length / (n + 1))
    if kind == "dirichlet_neumann":
        return np.arange(1, n + 1) * (length / n)
    if kind == "neumann2":
        return np.arange(n) * (length / (n - 1))
    raise ValueError(f"unknown boundary kind {kind!r}")


def _as_fraction(f):
    f = Fraction(f)
    if f <= 0:
        raise ValueError("step fractions must be positive")
    return f


def _check_tau(tau):
    if not np.isfinite(tau) or tau <= 0:
        raise ValueError("tau must be positive and finite")
    return float(tau)


class KroneckerOperator:
    """Kronecker sum of per-direction matrices with an exponential cache."""

    representation = "grid"

    def __init__(self, matrices):
        host = [np.asarray(m.cpu() if isinstance(m, torch.Tensor) else m, dtype=complex) for m in matrices]
        for m in host:
            if m.ndim != 2 or m.shape[0] != m.shape[1]:
                raise ValueError("per-direction factors must be square")
        self.matrices = host
        self.shape = tuple(m.shape[0] for m in host)
        self._tau = None
        self._cache = {}
        self._dev = None

    def _device_mats(self):
        if self._dev is None:
            _lib.require_cuda()
            ms = [torch.from_numpy(np.ascontiguousarray(m)).cuda() for m in self.matrices]
            self._dev = (ms, [m.transpose(0, 1).contiguous() for m in ms])
        return self._dev

    def prepare(self, tau, fractions):
        """exp(f tau A_mu) for every f (host Pade, operators.py:123-132),
        uploaded once with its transpose; identical factors computed once."""
        tau = _check_tau(tau)
        fr = [_as_fraction(f) for f in fractions]
        if tau == self._tau and set(fr) == set(self._cache):
            return  # same (tau, fractions): the cached exponentials are exact
        self._tau = tau
        self._cache = {}
        self.__dict__.pop("_oz", None)
        self.__dict__.pop("_bands", None)
        _lib.require_cuda()
        for f in fr:
            step = float(f) * self._tau
            mats, mats_t, seen = [], [], {}
            for m in self.matrices:
                key = (m.shape, m.tobytes())
                if key not in seen:
                    e = torch.from_numpy(np.ascontiguousarray(expm_pade(m, step))).cuda()
                    seen[key] = (e, e.transpose(0, 1).contiguous())
                e, et = seen[key]
                mats.append(e)
                mats_t.append(et)
            self._cache[f] = (mats, mats_t)

    def exp_factors(self, fraction):
        f = Fraction(fraction)
        if f not in self._cache:
            raise RuntimeError(f"exponential for fraction {f} not prepared; call prepare()")
        return self._cache[f]

    def sliced_factors(self, fraction):
        """INT8-tensor-core operand slices of exp(f tau A_mu) (ozaki.py), built
        once per prepared fraction and shared between identical factors."""
        f = Fraction(fraction)
        mats, _ = self.exp_factors(f)
        cache = self.__dict__.setdefault("_oz", {})
        if f not in cache:
            from .ozaki import SlicedFactor
            seen, out = {}, []
            for m in mats:
                if id(m) not in seen:
                    seen[id(m)] = SlicedFactor(m)
                out.append(seen[id(m)])
            cache[f] = out
        return cache[f]

    def tucker2d_bands(self, fraction):
        """Per-row significant bands [lo, hi] (int32 pairs, device) of each
        exp(f tau A_mu): entries >= 2^-60 of their row's largest magnitude, the
        support the cross-mode fused 2D Tucker (cgl_tucker2d) contracts."""
        f = Fraction(fraction)
        mats, _ = self.exp_factors(f)
        cache = self.__dict__.setdefault("_bands", {})
        if f not in cache:
            out = []
            for m in mats:
                a = m.abs()
                keep = a >= a.amax(dim=1, keepdim=True) * 2.0 ** -60
                n = m.shape[1]
                lo = keep.int().argmax(dim=1)
                hi = n - 1 - keep.flip(1).int().argmax(dim=1)
                out.append(torch.stack([lo, hi], dim=1).to(torch.int32).contiguous())
            cache[f] = out
        return cache[f]

    # device-level (integrator) entry points
    def apply_dev(self, u, y=None, beta=0.0, flag=None, pos=0):
        ms, mts = self._device_mats()
        return kron_sum_dev(u, ms, mts, y=y, beta=beta, flag=flag, pos=pos)

    # public protocol (host or device arrays)
    def apply(self, u):
        ud, host = to_device(u)
        self._check_shape(ud)
        return to_host_if(self.apply_dev(ud), host)

    def exp_apply(self, fraction, u):
        mats, mats_t = self.exp_factors(fraction)
        ud, host = to_device(u)
        self._check_shape(ud)
        return to_host_if(tucker_dev([ud], [mats], [mats_t])[0], host)

    def _check_shape(self, u):
        if tuple(u.shape) != self.shape:
            raise ValueError(f"field shape {tuple(u.shape)} != operator shape {self.shape}")


class FourierOperator:
    """Diagonal symbol operator on Fourier coefficient space."""

    representation = "fourier"

    def __init__(self, grid, symbol, separable=None):
        if tuple(np.shape(symbol)) != tuple(grid.shape):
            raise ValueError("symbol shape must match the grid")
        self.grid = grid
        self.symbol = np.asarray(symbol.cpu() if isinstance(symbol, torch.Tensor) else symbol)
        self.shape = grid.shape
        self._sep = separable  # (params, advection_sign) when built from CglParameters
        self._tau = None
        self._cache = {}
        self._sym_dev = None

    def symbol_dev(self):
        if self._sym_dev is None:
            self._sym_dev, _ = to_device(self.symbol)
        return self._sym_dev

    def _tables(self, s):
        """Per-axis factors of exp(s * symbol): table 0 carries exp(s alpha2)
        and the advection phase, every axis exp(-s (a1 + i b1) k_mu^2)."""
        params, sign = self._sep
        tabs = []
        for ax in range(self.grid.ndim):
            k = self.grid.wavenumbers(ax)
            arg = -s * params.diffusion * (k ** 2)
            if ax == 0:
                arg = arg + s * params.alpha2
                if sign:
                    arg = arg + s * sign * params.alpha0 * 1j * k
            tabs.append(torch.from_numpy(np.exp(arg).astype(np.complex128)).cuda())
        return tabs

    def prepare(self, tau, fractions):
        """exp(f tau symbol) per fraction (operators.py:160-167); unchanged
        (tau, fractions) keep the cached factors (and with them the step
        graphs of a plan that captured their pointers)."""
        tau = _check_tau(tau)
        fr = [_as_fraction(f) for f in fractions]
        if tau == getattr(self, "_tau", None) and set(fr) == set(getattr(self, "_cache", {})):
            return
        self._tau = tau
        self._cache = {}
        _lib.require_cuda()
        for fraction in fractions:
            f = _as_fraction(fraction)
            s = float(f) * self._tau
            if self._sep is not None and self.grid.ndim <= 4:
                self._cache[f] = ("sep", self._tables(s))
            else:
                e = torch.empty_like(self.symbol_dev())
                _lib.check(_lib.load().cgl_symbol_exp(_lib.stream(), e.numel(), s, _lib.ptr(self.symbol_dev()),
                                                      _lib.ptr(e)), "cgl_symbol_exp")
                self._cache[f] = ("full", e)

    def exp_entry(self, fraction):
        f = Fraction(fraction)
        if f not in self._cache:
            raise RuntimeError(f"exponential for fraction {f} not prepared; call prepare()")
        return self._cache[f]

    def exp_apply_dev(self, fraction, u, scale=1.0, out=None, flag=None, pos=0):
        kind, data = self.exp_entry(fraction)
        out = torch.empty_like(u) if out is None else out
        if kind == "sep":
            _lib.check(_lib.load().cgl_separable_mul(_lib.stream(), u.ndim, _lib.i64_array(u.shape),
                                                     _lib.ptr_array(data), scale, _lib.ptr(u), _lib.ptr(out),
                                                     _lib.flag_ptr(flag), pos), "cgl_separable_mul")
        else:
            mul_dev(data, u, out=out, flag=flag, pos=pos)
            if scale != 1.0:
                raise ValueError("scaled multiply needs the separable form")
        return out

    def apply_dev(self, u, flag=None, pos=0):
        return mul_dev(self.symbol_dev(), u, flag=flag, pos=pos)

    def apply(self, u):
        ud, host = to_device(u)
        return to_host_if(self.apply_dev(ud), host)

    def exp_apply(self, fraction, u):
        ud, host = to_device(u)
        return to_host_if(self.exp_apply_dev(fraction, ud), host)


class BlockOperator:
    """Block-diagonal operator for coupled systems; acts componentwise."""

    def __init__(self, blocks):
        if not blocks:
            raise ValueError("need at least one block")
        if len({b.representation for b in blocks}) != 1:
            raise ValueError("all blocks must share a representation")
        if len({b.shape for b in blocks}) != 1:
            raise ValueError("all blocks must share a shape")
        self.blocks = list(blocks)
        self.representation = blocks[0].representation
        self.shape = blocks[0].shape

    def apply(self, fields):
        self._check(fields)
        return tuple(b.apply(u) for b, u in zip(self.blocks, fields))

    def prepare(self, tau, fractions):
        for b in self.blocks:
            b.prepare(tau, fractions)

    def exp_apply(self, fraction, fields):
        self._check(fields)
        return tuple(b.exp_apply(fraction, u) for b, u in zip(self.blocks, fields))

    def _check(self, fields):
        if len(fields) != len(self.blocks):
            raise ValueError(f"expected {len(self.blocks)} components, got {len(fields)}")


def build_fd_operator(params, extents, lengths, bc):
    """A_mu = (alpha1 + i beta1) D2_mu + (alpha2/d) I (operators.py:211-229).
    bc: "dirichlet" / "dirichlet_neumann" (4th order, as the reference) or
    "dirichlet2" / "neumann2" (2nd order, BASELINE configs)."""
    if len(extents) != len(lengths):
        raise ValueError("one length per direction required")
    if bc not in _BUILDERS:
        raise ValueError(f"unknown boundary kind {bc!r}")
    d = len(extents)
    return KroneckerOperator([params.diffusion * _BUILDERS[bc](n, L) + (params.alpha2 / d) * np.eye(n)
                              for n, L in zip(extents, lengths)])


def build_periodic_operator(grid, params, advection_sign=0):
    """Fourier-form operator (operators.py:232-234), separable exponential."""
    return FourierOperator(grid, build_symbol(grid, params, advection_sign),
                           separable=(params, advection_sign))
