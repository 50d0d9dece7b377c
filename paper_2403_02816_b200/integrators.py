"""Time integrators for the semidiscrete CGL systems — GPU step engine.

Same public surface as the reference integrators.py (Scheme, SCHEMES,
Problem, IntegrationResult, integrate) and the same eight step bodies
(integrators.py:146-215), executed as sm_100a kernels on device-resident
state:

  * exp(f tau K) u: batched DMMA Tucker chains (FD) or the separable Fourier
    multiplier (periodic); independent exponentials inside a step (e.g. the
    four of Lawson-RK4 that only need u and g1) share one GEMM launch per mode;
  * g, the exact cubic/quintic flows and the RK4 substep: fused pointwise
    kernels (Fourier: sandwiched between cuFFT transforms, the 1/N of the
    inverse folded into the kernel);
  * stage combinations: one multi-term linear-combination pass.

Divergence (integrators.py:264-278) never syncs per step: every flow and the
end-of-step finiteness check min-reduce (step, call, reason) into a sticky
device key; kernels positioned after the first failure skip, so the state
buffers hold exactly the reference's returned fields; the host reads the key
every `poll` steps (and at snapshot steps) and stops early.
"""

import time
from dataclasses import dataclass
from fractions import Fraction

import torch

from . import _lib
from ._device import to_device, to_host_if
from .flows import eval_g_dev, exact_flow_dev, rk4_flow_dev
from .spectral import fft_dev, mul_dev

__all__ = ["Scheme", "SCHEMES", "Problem", "IntegrationResult", "integrate"]

_HALF = Fraction(1, 2)
_ONE = Fraction(1)


@dataclass(frozen=True)
class Scheme:
    name: str
    order: int
    fractions: tuple
    three_term: bool = False

    @property
    def uses_exponentials(self):
        return bool(self.fractions)


SCHEMES = {                                              # integrators.py:50-59
    "rk2": Scheme("rk2", 2, ()),
    "rk4": Scheme("rk4", 4, ()),
    "strang": Scheme("strang", 2, (_ONE,)),
    "split4": Scheme("split4", 4, (_ONE, _HALF)),
    "strang_3t": Scheme("strang_3t", 2, (_ONE,), three_term=True),
    "split4_3t": Scheme("split4_3t", 4, (_ONE, _HALF), three_term=True),
    "if2": Scheme("if2", 2, (_ONE,)),
    "if4": Scheme("if4", 4, (_HALF, _ONE)),
}

_COMMIT_SEQ = 254
_CHECK_SEQ = 255


class _Ctx:
    """Position bookkeeping for the sticky divergence key."""

    def __init__(self, flag):
        self.flag = flag
        self.step = 0
        self.seq = 0

    def base(self):
        return self.step << 24

    def at(self, seq):
        return (self.step << 24) | (seq << 8)

    def next_flow(self):
        p = self.at(self.seq)
        self.seq += 1
        return p


class Problem:
    """Linear operator + nonlinearity (integrators.py:62-127)."""

    def __init__(self, operator, nonlinear):
        blocks = getattr(operator, "blocks", None)
        if nonlinear.components > 1:
            if blocks is None or len(blocks) != nonlinear.components:
                raise ValueError("coupled nonlinearity needs a block operator with one block per component")
        elif blocks is not None:
            raise ValueError("scalar nonlinearity takes a plain operator")
        self.operator = operator
        self.nonlinear = nonlinear
        self.fourier = operator.representation == "fourier"
        self._blocks = list(blocks) if blocks is not None else [operator]
        self._nl = nonlinear.c_struct()
        self._ctx = None

    # -- public representation plumbing (host or device arrays) -------------
    def to_physical(self, fields):
        if not self.fourier:
            return fields
        from .spectral import dft_inverse
        return tuple(dft_inverse(u) for u in fields)

    def from_physical(self, fields):
        if not self.fourier:
            return fields
        from .spectral import dft_forward
        return tuple(dft_forward(u) for u in fields)

    def prepare(self, tau, scheme):
        if scheme.three_term and self.nonlinear.kind == "coupled_cubic_quintic":
            raise ValueError("three-term splitting has no exact flow for the coupled cross term")
        if scheme.uses_exponentials:
            self.operator.prepare(tau, scheme.fractions)

    # -- device pieces used by the steppers ----------------------------------
    @property
    def _flag(self):
        return self._ctx.flag if self._ctx else None

    def _base(self):
        return self._ctx.base() if self._ctx else 0

    def _flow_pos(self, seq=None):
        if not self._ctx:
            return 0
        if seq is None:
            return self._ctx.next_flow()
        return self._ctx.at(seq)

    def comb(self, terms):
        """sum c_i x_i componentwise; terms = [(c, fields), ...]."""
        lib = _lib.load()
        ncomp = len(terms[0][1])
        out = []
        for c in range(ncomp):
            xs = [t[1][c] for t in terms]
            o = torch.empty_like(xs[0])
            _lib.check(lib.cgl_lincomb(_lib.stream(), o.numel(), len(xs), _lib.dbl_array([t[0] for t in terms]),
                                       _lib.ptr_array(xs), _lib.ptr(o), _lib.flag_ptr(self._flag), self._base()),
                       "cgl_lincomb")
            out.append(o)
        return out

    def _phys(self, u):
        return fft_dev(u, inverse=True) if self.fourier else u

    def _spec(self, u):
        return fft_dev(u) if self.fourier else u

    def _scale(self, u):
        return 1.0 / u.numel() if self.fourier else 1.0

    def g(self, fields):
        ph = [self._phys(u) for u in fields]
        gs = eval_g_dev(self._nl, ph, scale=self._scale(fields[0]), flag=self._flag, pos=self._base())
        return [self._spec(x) for x in gs]

    def rhs(self, fields):
        """K u + g(u), the K-action accumulated onto g in the GEMM epilogue."""
        gs = self.g(fields)
        out = []
        for b, u, gc in zip(self._blocks, fields, gs):
            if self.fourier:
                ku = b.apply_dev(u, flag=self._flag, pos=self._base())
                out.append(self.comb([(1.0, [ku]), (1.0, [gc])])[0])
            else:
                out.append(b.apply_dev(u, y=gc, beta=1.0, flag=self._flag, pos=self._base()))
        return out

    def expk_multi(self, jobs):
        """[(fraction, fields), ...] -> list of fields; all FD Tucker chains of
        one call share one GEMM launch per mode."""
        if self.fourier:
            return [[b.exp_apply_dev(f, u, flag=self._flag, pos=self._base()) for b, u in zip(self._blocks, fs)]
                    for f, fs in jobs]
        from .tensors import tucker_dev
        ins, mats, mts, where = [], [], [], []
        for j, (f, fs) in enumerate(jobs):
            for c, (b, u) in enumerate(zip(self._blocks, fs)):
                m, mt = b.exp_factors(f)
                ins.append(u)
                mats.append(m)
                mts.append(mt)
                where.append((j, c))
        outs = tucker_dev(ins, mats, mts, flag=self._flag, pos=self._base())
        res = [[None] * len(fs) for _, fs in jobs]
        for (j, c), o in zip(where, outs):
            res[j][c] = o
        return res

    def expk(self, fraction, fields):
        return self.expk_multi([(fraction, fields)])[0]

    def flow(self, fields, t, seq=None):
        """Exact cubic flow for the cubic kind, one RK4 substep otherwise
        (integrators.py:103-110)."""
        if self.nonlinear.kind == "cubic":
            return self.flow_exact(fields, t, quintic=False, seq=seq)
        ph = [self._phys(u) for u in fields]
        outs = rk4_flow_dev(self._nl, ph, t, scale=self._scale(fields[0]), flag=self._flag,
                            pos=self._flow_pos(seq))
        return [self._spec(o) for o in outs]

    def flow_exact(self, fields, t, quintic, seq=None):
        out = []
        for i, u in enumerate(fields):
            pos = self._flow_pos(None if seq is None else seq + i)
            o = exact_flow_dev(self._nl, self._phys(u), t, quintic=quintic, scale=self._scale(u),
                               flag=self._flag, pos=pos)
            out.append(self._spec(o))
        return out


# ---------------------------------------------------------------------------
# step bodies (integrators.py:146-215); flow seq numbers follow the
# reference's call order so the recorded first failure is the one the
# reference would raise.
# ---------------------------------------------------------------------------

def _step_rk2(p, u, tau):
    f1 = p.rhs(u)
    f2 = p.rhs(p.comb([(1.0, u), (tau, f1)]))
    return p.comb([(1.0, u), (0.5 * tau, f1), (0.5 * tau, f2)])


def _step_rk4(p, u, tau):
    f1 = p.rhs(u)
    f2 = p.rhs(p.comb([(1.0, u), (0.5 * tau, f1)]))
    f3 = p.rhs(p.comb([(1.0, u), (0.5 * tau, f2)]))
    f4 = p.rhs(p.comb([(1.0, u), (tau, f3)]))
    t6 = tau / 6.0
    return p.comb([(1.0, u), (t6, f1), (2.0 * t6, f2), (2.0 * t6, f3), (t6, f4)])


def _step_strang(p, u, tau):
    v = p.flow(u, 0.5 * tau)
    v = p.expk(_ONE, v)
    return p.flow(v, 0.5 * tau)


def _flow_width(p):
    # calls one p.flow() makes: one per component for the exact cubic flow
    return len(p._blocks) if p.nonlinear.kind == "cubic" else 1


def _step_split4(p, u, tau):
    w = _flow_width(p)
    v = p.flow(u, 0.5 * tau, seq=0)
    f = p.flow(u, 0.25 * tau, seq=2 * w)
    v, f = p.expk_multi([(_ONE, v), (_HALF, f)])
    coarse = p.flow(v, 0.5 * tau, seq=w)
    f = p.flow(f, 0.5 * tau, seq=3 * w)
    f = p.expk(_HALF, f)
    fine = p.flow(f, 0.25 * tau, seq=4 * w)
    return p.comb([(4.0 / 3.0, fine), (-1.0 / 3.0, coarse)])


def _strang3(p, u, tau, fraction, seq0):
    n = len(p._blocks)
    t = float(fraction) * tau
    v = p.flow_exact(u, 0.5 * t, quintic=True, seq=seq0)
    v = p.flow_exact(v, 0.5 * t, quintic=False, seq=seq0 + n)
    v = p.expk(fraction, v)
    v = p.flow_exact(v, 0.5 * t, quintic=False, seq=seq0 + 2 * n)
    return p.flow_exact(v, 0.5 * t, quintic=True, seq=seq0 + 3 * n)


def _step_strang_3t(p, u, tau):
    return _strang3(p, u, tau, _ONE, 0)


def _step_split4_3t(p, u, tau):
    n4 = 4 * len(p._blocks)
    coarse = _strang3(p, u, tau, _ONE, 0)
    fine = _strang3(p, u, tau, _HALF, n4)
    fine = _strang3(p, fine, tau, _HALF, 2 * n4)
    return p.comb([(4.0 / 3.0, fine), (-1.0 / 3.0, coarse)])


def _step_if2(p, u, tau):
    g1 = p.g(u)
    u2, out = p.expk_multi([(_ONE, p.comb([(1.0, u), (tau, g1)])),
                            (_ONE, p.comb([(1.0, u), (0.5 * tau, g1)]))])
    return p.comb([(1.0, out), (0.5 * tau, p.g(u2))])


def _step_if4(p, u, tau):
    g1 = p.g(u)
    x1 = p.comb([(1.0, u), (0.5 * tau, g1)])
    x5 = p.comb([(1.0, u), (tau / 6.0, g1)])
    u2, a, b, c = p.expk_multi([(_HALF, x1), (_HALF, u), (_ONE, u), (_ONE, x5)])
    del x1, x5, g1
    g2 = p.g(u2)
    u3 = p.comb([(1.0, a), (0.5 * tau, g2)])
    del a, u2
    g3 = p.g(u3)
    s = p.comb([(1.0, g2), (1.0, g3)])
    del g2, u3
    d, e = p.expk_multi([(_HALF, g3), (_HALF, s)])
    del s, g3
    u4 = p.comb([(1.0, b), (tau, d)])
    del b, d
    g4 = p.g(u4)
    return p.comb([(1.0, c), (tau / 3.0, e), (tau / 6.0, g4)])


_STEPPERS = {"rk2": _step_rk2, "rk4": _step_rk4, "strang": _step_strang, "split4": _step_split4,
             "strang_3t": _step_strang_3t, "split4_3t": _step_split4_3t, "if2": _step_if2, "if4": _step_if4}


@dataclass
class IntegrationResult:
    fields: tuple
    steps: int
    tau: float
    seconds: float
    diverged: bool = False
    diverged_at: int = 0
    reason: str = ""
    device_seconds: float = 0.0   # CUDA-event time of the stepping loop


def _copy_into(p, src, dst, pos):
    lib = _lib.load()
    for s, d in zip(src, dst):
        _lib.check(lib.cgl_lincomb(_lib.stream(), d.numel(), 1, _lib.dbl_array([1.0]), _lib.ptr_array([s]),
                                   _lib.ptr(d), _lib.flag_ptr(p._ctx.flag), pos), "cgl_lincomb")


def _check_finite(p, fields, pos):
    _lib.check(_lib.load().cgl_check_finite(_lib.stream(), fields[0].numel(), len(fields), _lib.ptr_array(fields),
                                            _lib.flag_ptr(p._ctx.flag), pos), "cgl_check_finite")


def integrate(problem, scheme_name, fields, t_final, steps, snapshot_steps=(), on_snapshot=None, poll=16):
    """March `steps` uniform steps of the named scheme to t_final
    (integrators.py:241-282).  numpy fields in -> numpy fields out; CUDA
    tensors in -> CUDA tensors out.  `seconds` covers the stepping loop only
    (prepare excluded), measured after a device synchronise."""
    if scheme_name not in SCHEMES:
        raise ValueError(f"unknown scheme {scheme_name!r}; choose from {sorted(SCHEMES)}")
    if steps < 1:
        raise ValueError("steps must be >= 1")
    scheme = SCHEMES[scheme_name]
    tau = t_final / steps
    dev = [to_device(u) for u in fields]
    host = any(h for _, h in dev)
    if len(dev) != problem.nonlinear.components:
        raise ValueError(f"expected {problem.nonlinear.components} components, got {len(dev)}")
    problem.prepare(tau, scheme)
    step_fn = _STEPPERS[scheme_name]
    wanted = set(int(k) for k in snapshot_steps)

    from . import plan as _plan
    if _plan.supports(problem, scheme_name):
        return _integrate_fused(problem, scheme_name, [d for d, _ in dev], host, tau, steps, wanted, on_snapshot)

    flag = _lib.new_flag(1)
    state = [[d.clone() for d, _ in dev], [torch.empty_like(d) for d, _ in dev]]
    ctx = _Ctx(flag)
    problem._ctx = ctx
    key = _lib.NO_DIVERGENCE
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    try:
        torch.cuda.synchronize()
        start = time.perf_counter()
        ev0.record()
        for k in range(1, steps + 1):
            ctx.step, ctx.seq = k, 0
            new = step_fn(problem, state[(k - 1) % 2], tau)
            _copy_into(problem, new, state[k % 2], ctx.at(_COMMIT_SEQ))
            _check_finite(problem, state[k % 2], ctx.at(_CHECK_SEQ))
            del new
            if k in wanted or k % poll == 0 or k == steps:
                key = int(flag[0].item()) & ((1 << 64) - 1)
                if key != _lib.NO_DIVERGENCE:
                    break
                if k in wanted and on_snapshot is not None:
                    on_snapshot(k, k * tau, tuple(to_host_if(f.clone(), host) for f in state[k % 2]))
        ev1.record()
        torch.cuda.synchronize()
        seconds = time.perf_counter() - start
        dev_s = ev0.elapsed_time(ev1) / 1e3
    finally:
        problem._ctx = None
    if key == _lib.NO_DIVERGENCE:
        out = state[steps % 2]
        return IntegrationResult(tuple(to_host_if(f, host) for f in out), steps, tau, seconds,
                                 device_seconds=dev_s)
    k_div, reason = key >> 24, key & 0xFF
    out = state[k_div % 2] if reason == _lib.NONFINITE_STATE else state[(k_div - 1) % 2]
    return IntegrationResult(tuple(to_host_if(f, host) for f in out), steps, tau, seconds,
                             diverged=True, diverged_at=int(k_div), reason=_lib.REASONS[reason],
                             device_seconds=dev_s)


def _integrate_fused(problem, scheme_name, u0, host, tau, steps, wanted, on_snapshot):
    """Fused, graph-captured FD path (plan.py); same results contract."""
    from . import plan as _plan
    cache = problem.__dict__.setdefault("_plans", {})
    key = (scheme_name, tuple(u0[0].shape), len(u0))
    fp = cache.get(key)
    if fp is None:
        cache.clear()  # one live plan per problem bounds the device memory
        fp = cache[key] = _plan.make_plan(problem, scheme_name, u0)

    def stop(k, fields):
        if on_snapshot is not None:
            on_snapshot(k, k * tau, tuple(to_host_if(f.clone(), host) for f in fields))

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start = time.perf_counter()
    ev0.record()
    fkey = fp.run(u0, steps, tau, stop_at=wanted, on_stop=stop)
    ev1.record()
    torch.cuda.synchronize()
    seconds = time.perf_counter() - start
    dev_s = ev0.elapsed_time(ev1) / 1e3
    if fkey == _lib.NO_DIVERGENCE:
        out = fp.result(steps)
        return IntegrationResult(_detach(out, host, cache, key), steps, tau, seconds, device_seconds=dev_s)
    k_div, reason = fkey >> 24, fkey & 0xFF
    out = fp.result(k_div) if reason == _lib.NONFINITE_STATE else fp.result(k_div - 1)
    return IntegrationResult(_detach(out, host, cache, key), steps, tau, seconds,
                             diverged=True, diverged_at=int(k_div), reason=_lib.REASONS[reason],
                             device_seconds=dev_s)


def _detach(fields, host, cache, key):
    """Result fields independent of the cached plan's buffers: host copies,
    device clones, or -- when a clone does not fit (1024^3 fields) -- the
    buffers themselves, handed over by dropping the plan from the cache."""
    if host:
        return tuple(to_host_if(f, True) for f in fields)
    try:
        return tuple(f.clone() for f in fields)
    except torch.OutOfMemoryError:
        cache.pop(key, None)
        return tuple(fields)
