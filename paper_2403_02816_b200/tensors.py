"""Kronecker-form tensor kernels on the GPU (DMMA complex-FP64 GEMM).

Same API and conventions as the reference tensors.py:
    vec(mu_mode_product(u, m, 0)) == kron(eye(n_2), m) @ vec(u)   (column-major vec)
The shape semantics are those of numpy arrays of shape (n_1, ..., n_d); on
the device the tensors are C-contiguous complex128 (last axis fastest), so a
mu-mode product is one batched GEMM: leading axes become the batch, the
trailing axes the GEMM N dimension (cgl_mode_product, csrc/capi.cu).

numpy inputs are copied to the device and results copied back; CUDA tensors
stay on the device.  There is no CPU path.
"""

import numpy as np
import torch

from . import _lib
from ._device import matrix_to_device, to_device, to_host_if

__all__ = ["vec", "unvec", "mu_mode_product", "tucker_apply", "kron_sum_apply",
           "assemble_kron_sum"]


def vec(u):
    """Flatten first-index-fastest (tensors.py:28-30)."""
    if isinstance(u, torch.Tensor):
        return u.permute(*reversed(range(u.ndim))).reshape(-1)
    return np.asarray(u).reshape(-1, order="F")


def unvec(x, shape):
    """Inverse of vec (tensors.py:33-35)."""
    shape = tuple(shape)
    if isinstance(x, torch.Tensor):
        return x.reshape(tuple(reversed(shape))).permute(*reversed(range(len(shape)))).contiguous()
    return np.asarray(x).reshape(shape, order="F")


def _validate(u_shape, mat_shape, axis):
    if len(mat_shape) != 2:
        raise ValueError(f"factor must be a matrix, got ndim={len(mat_shape)}")
    if not 0 <= axis < len(u_shape):
        raise ValueError(f"axis {axis} out of range for order-{len(u_shape)} tensor")
    if mat_shape[1] != u_shape[axis]:
        raise ValueError(f"factor columns {mat_shape[1]} != extent {u_shape[axis]} of axis {axis}")


def mode_product_dev(u, m, mt, axis, out=None, alpha=1.0, y=None, beta=0.0, flag=None, pos=0):
    """Device-level: out = alpha * (u x_axis m) + beta * y (all CUDA tensors)."""
    shape = tuple(u.shape)
    oshape = shape[:axis] + (m.shape[0],) + shape[axis + 1:]
    if out is None:
        out = torch.empty(oshape, dtype=torch.complex128, device=u.device)
    lib = _lib.load()
    rc = lib.cgl_mode_product(_lib.stream(), len(shape), _lib.i64_array(shape), axis,
                              _lib.ptr(m), _lib.ptr(mt), m.shape[0], _lib.ptr(u), _lib.ptr(out),
                              alpha, _lib.ptr(y), beta, _lib.flag_ptr(flag), pos)
    _lib.check(rc, "cgl_mode_product")
    return out


def tucker_dev(fields, mats, mats_t, outs=None, flag=None, pos=0, work=None):
    """Device-level batched Tucker: fields[f] x_1 mats[f][0] ... x_d mats[f][d-1],
    one GEMM launch per mode for all fields (cgl_tucker).  `work`: one scratch
    field per input (allocated when None)."""
    nf = len(fields)
    shape = tuple(fields[0].shape)
    nd = len(shape)
    if outs is None:
        outs = [torch.empty_like(f) for f in fields]
    if work is None:
        work = [torch.empty_like(f) for f in fields] if nd > 1 else []
    lib = _lib.load()
    flat = [m for ms in mats for m in ms]
    flat_t = [m for ms in mats_t for m in ms]
    for i in range(0, nf, 8):
        sl = slice(i, min(nf, i + 8))
        rc = lib.cgl_tucker(_lib.stream(), nd, _lib.i64_array(shape), len(fields[sl]),
                            _lib.ptr_array(flat[sl.start * nd:sl.stop * nd]),
                            _lib.ptr_array(flat_t[sl.start * nd:sl.stop * nd]),
                            _lib.ptr_array(fields[sl]), _lib.ptr_array(outs[sl]),
                            _lib.ptr_array(work[sl]) if nd > 1 else None,
                            _lib.flag_ptr(flag), pos)
        _lib.check(rc, "cgl_tucker")
    return outs


def kron_sum_dev(u, mats, mats_t, y=None, beta=0.0, out=None, flag=None, pos=0):
    """out = sum_mu u x_mu A_mu (+ beta*y), accumulating in the GEMM epilogue."""
    out = torch.empty_like(u) if out is None else out
    for axis in range(u.ndim):
        if axis == 0:
            mode_product_dev(u, mats[0], mats_t[0], 0, out=out, y=y, beta=beta if y is not None else 0.0,
                             flag=flag, pos=pos)
        else:
            mode_product_dev(u, mats[axis], mats_t[axis], axis, out=out, y=out, beta=1.0,
                             flag=flag, pos=pos)
    return out


def mu_mode_product(u, mat, axis):
    """Apply `mat` along direction `axis` (tensors.py:38-59)."""
    u_shape = tuple(u.shape) if hasattr(u, "shape") else np.shape(u)
    mat_shape = tuple(mat.shape) if hasattr(mat, "shape") else np.shape(mat)
    _validate(u_shape, mat_shape, axis)
    ud, host = to_device(u)
    m, mt = matrix_to_device(mat)
    return to_host_if(mode_product_dev(ud, m, mt, axis), host)


def tucker_apply(u, mats):
    """u x_1 m_1 x_2 m_2 ... (tensors.py:62-69)."""
    ud, host = to_device(u)
    if len(mats) != ud.ndim:
        raise ValueError(f"need {ud.ndim} factors, got {len(mats)}")
    dev = [matrix_to_device(m) for m in mats]
    for axis, (m, _) in enumerate(dev):
        _validate(tuple(ud.shape), tuple(m.shape), axis)
        if m.shape[0] != m.shape[1]:
            # rectangular chain: apply mode by mode
            out = ud
            for ax, (mm, mmt) in enumerate(dev):
                out = mode_product_dev(out, mm, mmt, ax)
            return to_host_if(out, host)
    out = tucker_dev([ud], [[m for m, _ in dev]], [[t for _, t in dev]])[0]
    return to_host_if(out, host)


def kron_sum_apply(u, mats):
    """Action of the Kronecker sum of `mats` (tensors.py:72-85)."""
    ud, host = to_device(u)
    if len(mats) != ud.ndim:
        raise ValueError(f"need {ud.ndim} factors, got {len(mats)}")
    dev = [matrix_to_device(m) for m in mats]
    for axis, (m, _) in enumerate(dev):
        _validate(tuple(ud.shape), tuple(m.shape), axis)
        if m.shape[0] != m.shape[1]:
            raise ValueError("kron-sum factors must be square matrices")
    out = kron_sum_dev(ud, [m for m, _ in dev], [t for _, t in dev])
    return to_host_if(out, host)


def assemble_kron_sum(mats, cap=4096):
    """Explicit dense Kronecker-sum matrix (host; test/inspection helper,
    tensors.py:88-112).  Refuses more than `cap` rows."""
    sizes = []
    for m in mats:
        m = np.asarray(m)
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise ValueError("kron-sum factors must be square matrices")
        sizes.append(m.shape[0])
    total = int(np.prod(sizes))
    if total > cap:
        raise ValueError(f"refusing to assemble {total} x {total} matrix (cap={cap})")
    out = np.zeros((total, total), dtype=complex)
    for axis, m in enumerate(mats):
        f = np.eye(1)
        for k, n in enumerate(sizes):
            f = np.kron(np.asarray(m) if k == axis else np.eye(n), f)
        out += f
    return out
