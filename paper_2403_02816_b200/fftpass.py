"""Pencil-FFT passes (csrc/fftpass.cu, C ABI `cgl_fft_pass`).

The n-dimensional transforms of the periodic path (`dft_forward` /
`dft_inverse`, reference spectral.py:79-86) as one HBM pass per axis, with
the pointwise pieces of the Fourier steppers fused into the first or last
pass (see the kernel file's header).  Grids: 2D/3D, power-of-two extents
16..512.  Passes may run in place (a CTA reads its whole tile before it
writes it).
"""

import math

import torch

from . import _lib

PROGRAMS = _lib.FFT_PROGRAMS


def supported(shape):
    shape = tuple(int(n) for n in shape)
    if len(shape) not in (2, 3):
        return False
    return bool(_lib.load().cgl_fft_pass_supported(len(shape), _lib.i64_array(shape)))


def make_ops(u=None, u_out=None, g=(None, None, None), g_out=None, tables=None, tau=0.0, scale=1.0, nl=None,
             flag=None, pos=0):
    ops = _lib.FftOps()
    ops.u = u.data_ptr() if u is not None else 0
    ops.u_out = u_out.data_ptr() if u_out is not None else 0
    for i, t in enumerate(g):
        ops.g[i] = t.data_ptr() if t is not None else 0
    ops.g_out = g_out.data_ptr() if g_out is not None else 0
    if tables is not None:
        for fr in range(2):
            for d, t in enumerate(tables[fr]):
                ops.tables[fr][d] = t.data_ptr()
    ops.tau = float(tau)
    ops.scale = float(scale)
    if nl is not None:
        ops.nl = nl
    ops.flag = flag.data_ptr() if flag is not None else 0
    ops.pos = int(pos)
    return ops


def axis_pass(src, dst, axis, inverse=False, program="plain", ops=None, shape=None):
    """One pass along `axis` of a C-contiguous complex128 CUDA field."""
    shape = tuple((src if src is not None else dst).shape) if shape is None else tuple(shape)
    _lib.check(_lib.load().cgl_fft_pass(_lib.stream(), PROGRAMS[program], len(shape), _lib.i64_array(shape),
                                        int(axis), 1 if inverse else 0, _lib.ptr(src), _lib.ptr(dst),
                                        _lib.ctypes.byref(ops) if ops is not None else None), "cgl_fft_pass")
    return dst


def fftn(x, out=None, inverse=False):
    """Unnormalised n-dimensional transform (forward = np.fft.fftn; inverse =
    N * np.fft.ifftn), one pass per axis, last axis first."""
    out = torch.empty_like(x) if out is None else out
    src = x
    for axis in reversed(range(x.ndim)):
        axis_pass(src, out, axis, inverse)
        src = out
    return out


def points(shape):
    return math.prod(shape)
