"""Nonlinear part of CGL: pointwise g and its flows, as fused GPU kernels.

API of the reference flows.py (NonlinearSpec, DivergenceError, eval_g,
cubic_flow, quintic_flow, rk4_flow).  The kernels (csrc/pointwise.cu)
compute |u|^2 as re^2 + im^2, keep all RK4 stages in registers (one read,
one write per component) and report blow-up / non-finite output through the
sticky device flag instead of a host-side np.any; the standalone functions
below read the flag once and raise DivergenceError like the reference.
"""

import torch

from . import _lib
from ._device import to_device, to_host_if
from .params import CglParameters

__all__ = ["NonlinearSpec", "DivergenceError", "eval_g", "cubic_flow", "quintic_flow", "rk4_flow"]

_KINDS = ("cubic", "cubic_quintic", "coupled_cubic_quintic")


class DivergenceError(RuntimeError):
    """Blow-up or NaN/Inf in a flow or a step (flows.py:32-39)."""

    def __init__(self, reason, step=None):
        self.reason = reason
        self.step = step
        where = f" at step {step}" if step is not None else ""
        super().__init__(f"{reason}{where}")


class NonlinearSpec:
    """Which nonlinear terms are active (flows.py:42-59)."""

    def __init__(self, kind, params):
        if kind not in _KINDS:
            raise ValueError(f"kind must be one of {_KINDS}, got {kind!r}")
        if not isinstance(params, CglParameters):
            raise TypeError("params must be CglParameters")
        if kind == "cubic" and (params.alpha4 != 0.0 or params.beta4 != 0.0):
            raise ValueError("cubic kind requires alpha4 = beta4 = 0")
        if kind != "coupled_cubic_quintic" and params.alpha5 != 0.0:
            raise ValueError("cross-coupling alpha5 needs the coupled kind")
        self.kind = kind
        self.params = params

    @property
    def components(self):
        return 2 if self.kind == "coupled_cubic_quintic" else 1

    def c_struct(self):
        return _lib.nonlinear_struct(self.kind, self.params)


def _struct(kind, params):
    return _lib.nonlinear_struct(kind, params)


# ---- device-level launchers (used by the integrator) -----------------------

def eval_g_dev(nl, fields, scale=1.0, outs=None, flag=None, pos=0):
    outs = [torch.empty_like(u) for u in fields] if outs is None else outs
    _lib.check(_lib.load().cgl_eval_g(_lib.stream(), fields[0].numel(), _lib.ctypes.byref(nl), len(fields),
                                      _lib.ptr_array(fields), scale, _lib.ptr_array(outs),
                                      _lib.flag_ptr(flag), pos), "cgl_eval_g")
    return outs


def exact_flow_dev(nl, u, t, quintic=False, scale=1.0, out=None, flag=None, pos=0):
    out = torch.empty_like(u) if out is None else out
    lib = _lib.load()
    fn = lib.cgl_quintic_flow if quintic else lib.cgl_cubic_flow
    _lib.check(fn(_lib.stream(), u.numel(), float(t), _lib.ctypes.byref(nl), _lib.ptr(u), scale, _lib.ptr(out),
                  _lib.flag_ptr(flag), pos), "cgl_exact_flow")
    return out


def rk4_flow_dev(nl, fields, t, scale=1.0, outs=None, flag=None, pos=0):
    outs = [torch.empty_like(u) for u in fields] if outs is None else outs
    _lib.check(_lib.load().cgl_rk4_flow(_lib.stream(), fields[0].numel(), float(t), _lib.ctypes.byref(nl),
                                        len(fields), _lib.ptr_array(fields), scale, _lib.ptr_array(outs),
                                        _lib.flag_ptr(flag), pos), "cgl_rk4_flow")
    return outs


class _OneShotFlag:
    """Device flag for the standalone API functions (not the step loop)."""

    def __init__(self):
        self.t = _lib.new_flag(0)

    def raise_if_set(self):
        key = int(self.t[0].item()) & ((1 << 64) - 1)
        if key != _lib.NO_DIVERGENCE:
            raise DivergenceError(_lib.REASONS[key & 0xFF])


# ---- public API (flows.py:62-133) ------------------------------------------

def eval_g(spec, fields):
    if len(fields) != spec.components:
        raise ValueError(f"expected {spec.components} components, got {len(fields)}")
    dev = [to_device(u) for u in fields]
    outs = eval_g_dev(spec.c_struct(), [d for d, _ in dev])
    return tuple(to_host_if(o, h) for o, (_, h) in zip(outs, dev))


def cubic_flow(u0, t, params):
    ud, host = to_device(u0)
    f = _OneShotFlag()
    out = exact_flow_dev(_struct("cubic_quintic", params), ud, t, flag=f.t)
    f.raise_if_set()
    return to_host_if(out, host)


def quintic_flow(u0, t, params):
    ud, host = to_device(u0)
    f = _OneShotFlag()
    out = exact_flow_dev(_struct("cubic_quintic", params), ud, t, quintic=True, flag=f.t)
    f.raise_if_set()
    return to_host_if(out, host)


def rk4_flow(spec, fields, t):
    if len(fields) != spec.components:
        raise ValueError(f"expected {spec.components} components, got {len(fields)}")
    dev = [to_device(u) for u in fields]
    f = _OneShotFlag()
    outs = rk4_flow_dev(spec.c_struct(), [d for d, _ in dev], t, flag=f.t)
    f.raise_if_set()
    return tuple(to_host_if(o, h) for o, (_, h) in zip(outs, dev))
