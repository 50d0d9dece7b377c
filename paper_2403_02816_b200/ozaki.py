"""mu-mode products on the INT8 tensor cores (csrc/ozgemm.cu, Ozaki scheme I).

Each constant factor exp(f tau A_mu) is sliced ONCE at prepare time into
S = 8 int8 slices in both operand roles (A side for the "left" form
Out_b = E In_b, B side for the "right" form Out = In E^T of the contiguous
axis), with its block-sparsity map (the factors are numerically banded, so
whole slice blocks are exactly zero and skipped).  The data operand is
sliced per product into a reusable workspace.  Accuracy: ~1e-15 relative
per product (tools/oz_check.py; parity tests at 1e-10 after full runs).

Error model.  A product element is exact up to the truncation of its
operands at 2^-56 of their scale: the ROW maximum of E (A side) and the
COLUMN (fibre) maximum of the data (B side) -- not per element as in an FP64
GEMM.  The global relative error is unaffected (full runs against the
reference: C4 50 steps 1.3e-13 at 256^3, tests/test_full_runs.py), but an
element far below its fibre's maximum keeps fewer significant bits: on C4 at
64^3, over the points below 1e-6 of the peak, the error after 50 steps is
1.5e-8 of that band's scale (1.5e-14 of the peak) against 4e-14 for the DMMA
engine (profiles/r02_parity_full_runs.jsonl).  CGL_GEMM=dmma selects the
per-element engine where that matters.
"""

import math
import os

import torch

from . import _lib

S = 8


def geometry():
    """(A row tile, B row tile, K chunk bytes) of the compiled kernel."""
    bm, bn, kc = _lib.c_int(), _lib.c_int(), _lib.c_int()
    _lib.load().cgl_oz_geometry(_lib.ctypes.byref(bm), _lib.ctypes.byref(bn), _lib.ctypes.byref(kc))
    return bm.value, bn.value, kc.value


def enabled():
    return os.environ.get("CGL_GEMM", "oz") == "oz"


def _nbytes(rows, cols, a_mode):
    return _lib.load().cgl_oz_slice_bytes(S, rows, cols, a_mode)


def _zmap_len(rows, cols, a_mode):
    bm, bn, kc = geometry()
    rt = bm if a_mode else bn
    return ((2 * rows if a_mode else rows) + rt - 1) // rt * ((2 * cols + kc - 1) // kc)


class SlicedFactor:
    """A-operand slices (+ zero map) of one square constant factor E (n x n):
    every mode product keeps E on the A side (the last axis via Out^T = E In^T)."""

    def __init__(self, E):
        lib = _lib.load()
        n = E.shape[0]
        self.n = n
        st = _lib.stream()
        # A role: slices of E (rows i, K = k)
        self.A = torch.zeros(_nbytes(n, n, 1), dtype=torch.int8, device=E.device)
        self.Ae = torch.empty(n, dtype=torch.int32, device=E.device)
        _lib.check(lib.cgl_oz_slice(st, S, _lib.ptr(E), n, 1, n, n, 1, 0, 1, _lib.ptr(self.A), 0,
                                    _lib.ptr(self.Ae), 0), "oz_slice(E, A)")
        self.Az = torch.empty(_zmap_len(n, n, 1), dtype=torch.int8, device=E.device)
        _lib.check(lib.cgl_oz_zmap(st, S, _lib.ptr(self.A), n, n, 1, _lib.ptr(self.Az)), "oz_zmap(A)")


class Workspace:
    """Per-field data-slice buffers, grown on demand (zero-initialised once:
    the padding bytes are never written)."""

    def __init__(self):
        self.bufs = {}

    def get(self, key, nbytes, nexp, device):
        b = self.bufs.get(key)
        if b is None or b[0].numel() < nbytes or b[1].numel() < nexp:
            b = (torch.zeros(nbytes, dtype=torch.int8, device=device),
                 torch.empty(nexp, dtype=torch.int32, device=device))
            self.bufs[key] = b
        return b


def single_chunk(shape, nfields):
    """The axis-0 data slices of nfields fields fit one workspace chunk."""
    n0, Q = shape[0], math.prod(shape[1:])
    return nfields * _nbytes(Q, n0, 0) <= CHUNK_BYTES


def fits(shape, nfields):
    """Small grids (C0 128^2) are launch-latency bound: the DMMA path is faster."""
    return math.prod(shape) >= (1 << 17)


# data-slice workspace budget per field (bytes); larger products are chunked
CHUNK_BYTES = int(os.environ.get("CGL_OZ_CHUNK_BYTES", str(2 << 30)))


def _chunks(total, per_unit, nf, align=128):
    """Split `total` units (rows of Z or batches) so one chunk's slices for
    all nf fields stay under CHUNK_BYTES."""
    units = max(1, CHUNK_BYTES // max(1, per_unit * nf))
    if units < total:
        units = max(align, units // align * align)  # whole row tiles per chunk
    return [(a, min(total, a + units)) for a in range(0, total, units)]


def mode_product_oz(ins, factors, outs, axis, ws, flag=None, pos=0, presliced=None):
    """outs[f] = ins[f] x_axis E_f for square E_f (SlicedFactor), one GEMM
    launch per chunk (one chunk unless the data slices would exceed
    CHUNK_BYTES, e.g. 1024^3 fields).  presliced (first axis only): per item
    (slices, exponents) already produced (cgl_stage_slice); no slicing."""
    lib = _lib.load()
    st = _lib.stream()
    shape = tuple(ins[0].shape)
    n = shape[axis]
    P = math.prod(shape[:axis])
    Q = math.prod(shape[axis + 1:])
    nf = len(ins)
    dev = ins[0].device
    # items sharing an input tensor (u with two different factors in the if4
    # step) share its data slices: slice each distinct input once
    uniq, idx = [], []
    for x in ins:
        for k, y in enumerate(uniq):
            if y.data_ptr() == x.data_ptr() and y.shape == x.shape:
                idx.append(k)
                break
        else:
            idx.append(len(uniq))
            uniq.append(x)
    nu = len(uniq)
    Aa = _lib.ptr_array([fc.A for fc in factors])
    Ae = _lib.ptr_array([fc.Ae for fc in factors])
    Az = _lib.ptr_array([fc.Az for fc in factors])
    if Q > 1 and P > 1:
        # middle axis: per slab b, Out_b (n x Q) = E In_b; chunk over slabs
        per = _nbytes(Q, n, 0)
        for b0, b1 in _chunks(P, per, nu, align=1):
            nb = b1 - b0
            Bu, Beu = [], []
            for u in range(nu):
                buf, ex = ws.get(("D", u, n), per * nb, Q * nb, dev)
                Bu.append(buf)
                Beu.append(ex)
            Bs, Be = [Bu[k] for k in idx], [Beu[k] for k in idx]
            srcs = [x.view(-1)[b0 * n * Q:] for x in uniq]
            dsts = [o.view(-1)[b0 * n * Q:] for o in outs]
            _lib.check(lib.cgl_oz_slice_multi(st, S, nu, _lib.ptr_array(srcs), 1, Q, Q, n, nb, n * Q, 0,
                                              _lib.ptr_array(Bu), per, _lib.ptr_array(Beu), Q), "oz_slice(data, B)")
            _lib.check(lib.cgl_oz_gemm(st, S, n, Q, n, nf, Aa, Ae, Az, _lib.ptr_array(Bs), _lib.ptr_array(Be),
                                       None, _lib.ptr_array(dsts), Q, nb, 0, 0, per, Q, n * Q,
                                       _lib.flag_ptr(flag), pos), "oz_gemm(middle)")
    elif Q > 1 and presliced is not None:
        Bs, Be = [p_[0] for p_ in presliced], [p_[1] for p_ in presliced]
        _lib.check(lib.cgl_oz_gemm(st, S, n, Q, n, nf, Aa, Ae, Az, _lib.ptr_array(Bs), _lib.ptr_array(Be),
                                   None, _lib.ptr_array(outs), Q, 1, 0, 0, 0, 0, 0,
                                   _lib.flag_ptr(flag), pos), "oz_gemm(first, presliced)")
    elif Q > 1:
        # first axis (P = 1): Out (n x Q) = E In; data Z = In^T rows q; chunk over q
        per_row = _nbytes(1 << 10, n, 0) >> 10 if Q >= (1 << 10) else _nbytes(Q, n, 0) // Q
        for q0, q1 in _chunks(Q, per_row, nu):
            nq = q1 - q0
            per = _nbytes(nq, n, 0)
            Bu, Beu = [], []
            for u in range(nu):
                buf, ex = ws.get(("D", u, n), per, nq, dev)
                Bu.append(buf)
                Beu.append(ex)
            Bs, Be = [Bu[k] for k in idx], [Beu[k] for k in idx]
            srcs = [x.view(-1)[q0:] for x in uniq]
            dsts = [o.view(-1)[q0:] for o in outs]
            _lib.check(lib.cgl_oz_slice_multi(st, S, nu, _lib.ptr_array(srcs), 1, Q, nq, n, 1, 0, 0,
                                              _lib.ptr_array(Bu), 0, _lib.ptr_array(Beu), 0), "oz_slice(data, B)")
            _lib.check(lib.cgl_oz_gemm(st, S, n, nq, n, nf, Aa, Ae, Az, _lib.ptr_array(Bs), _lib.ptr_array(Be),
                                       None, _lib.ptr_array(dsts), Q, 1, 0, 0, 0, 0, 0,
                                       _lib.flag_ptr(flag), pos), "oz_gemm(first)")
    else:
        # last axis: Out (P x n) = In E^T computed as Out^T = E In^T (constant E on the
        # block-skipped A side); data Z = In rows p (K contiguous); chunk over p
        per_row = max(1, _nbytes(min(P, 1 << 10), n, 0) // min(P, 1 << 10))
        for p0, p1 in _chunks(P, per_row, nu):
            np_ = p1 - p0
            per = _nbytes(np_, n, 0)
            Bu, Beu = [], []
            for u in range(nu):
                buf, ex = ws.get(("D", u, n), per, np_, dev)
                Bu.append(buf)
                Beu.append(ex)
            Bs, Be = [Bu[k] for k in idx], [Beu[k] for k in idx]
            srcs = [x.view(-1)[p0 * n:] for x in uniq]
            dsts = [o.view(-1)[p0 * n:] for o in outs]
            _lib.check(lib.cgl_oz_slice_multi(st, S, nu, _lib.ptr_array(srcs), n, 1, np_, n, 1, 0, 0,
                                              _lib.ptr_array(Bu), 0, _lib.ptr_array(Beu), 0), "oz_slice(data, Bt)")
            _lib.check(lib.cgl_oz_gemm_t(st, S, n, np_, n, nf, Aa, Ae, Az, _lib.ptr_array(Bs), _lib.ptr_array(Be),
                                         None, _lib.ptr_array(dsts), n, 1, 0, 0, 0, 0, 0,
                                         _lib.flag_ptr(flag), pos), "oz_gemm(last axis)")
    return outs


def tucker_oz(ins, factor_sets, outs, work, ws, flag=None, pos=0, pre0=None):
    """Tucker chains of up to 8 fields, one emulated GEMM launch per mode
    (same mode order and ping-pong as cgl_tucker); `ws` is the caller's
    Workspace (per plan: captured graphs keep its pointers)."""
    nd = ins[0].ndim
    src = list(ins)
    for axis in range(nd):
        to_out = (nd - axis) % 2 == 1
        dst = outs if to_out else work
        mode_product_oz(src, [fs[axis] for fs in factor_sets], dst, axis, ws, flag=flag, pos=pos,
                        presliced=pre0 if axis == 0 else None)
        src = dst
    return outs


def executed_macs_left(factor, ntiles_n, nfields):
    """INT8 MACs one left-form launch executes (block-sparse A = factor slices,
    dense data B): sum over (row tile, chunk) of the surviving slice pairs."""
    z = factor.Az.cpu().numpy().astype(int)
    pairs = ((S + 1 - z) * (S + 2 - z) // 2) * (z <= S)
    bm, bn, kc = geometry()
    return int(pairs.sum()) * bm * bn * kc * ntiles_n * nfields


def dense_macs(M, N, K, nfields):
    """INT8 MACs of the same product without block skipping (S(S+1)/2 pairs)."""
    return (S * (S + 1) // 2) * (2 * M) * N * (2 * K) * nfields
