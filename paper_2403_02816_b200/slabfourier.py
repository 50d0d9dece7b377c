"""Slab-sharded periodic (pseudospectral) path: distributed 3D FFT with the
spectral data kept in the transposed column-block layout.

Global grid (n0, n1, n2), C order, split into axis-0 slabs of p0 = n0/P
planes.  Forward transform of a slab set:
  transforms along x2 and x1 of every local plane    (one pencil pass each, in place)
  all-to-all: slab (p0, n1 n2) -> column block (n0, m), m = n1 n2 / P
  transform along x0 of the m columns                 (one strided pencil pass, in place)
The inverse reverses the three stages.  The local transforms are the
single-GPU plan's pencil passes (csrc/fftpass.cu, one HBM pass per axis) when
the local extents are powers of two in 16..512, else batched cuFFT plans; with
the passes, F g F^-1 of a stage input (integrators.py:99-101) takes the fused
program along the contiguous axis (F_2^-1, 1/N, g, F_2 in one pass), so an
evaluation is 5 local passes and 2 exchanges instead of cuFFT's ~7 passes plus
a g kernel.  Coefficients therefore live in
(n0 x m) column blocks; the separable exp(f tau symbol) multipliers and the
Lawson stage combinations run there (cgl_stage_fourier_cols /
cgl_separable_mul_cols map a local element (k0, c) to global flat index
k0 n1 n2 + r m + c); g and the flows run on physical slabs.

One code path serves real ranks (one slab per process, NCCL all-to-all) and
P VIRTUAL ranks in one process (all slabs local, the exchange is a device
copy): the latter tests the sharded index mapping on a single GPU.
Divergence keys: one shared flag for virtual ranks; for real ranks the keys
are min-reduced before every end-of-step kernel (distributed.global_min_key).
"""

import math

import torch
import torch.distributed as dist

from . import _lib
from .distributed import global_min_key


class FftMany:
    """A cuFFT plan with advanced layout (cgl_fft_plan_many)."""

    def __init__(self, rank_n, batch, istride, idist):
        lib = _lib.load()
        h = _lib.c_ptr()
        _lib.check(lib.cgl_fft_plan_many(len(rank_n), _lib.i64_array(rank_n), batch, istride, idist, istride, idist,
                                         _lib.ctypes.byref(h)), "cgl_fft_plan_many")
        self.h = h

    def __call__(self, x, out=None, inverse=False):
        out = x if out is None else out
        _lib.check(_lib.load().cgl_fft_exec(self.h, _lib.stream(), _lib.ptr(x), _lib.ptr(out), 1 if inverse else 0),
                   "cgl_fft_exec")
        return out

    def __del__(self):
        try:
            _lib.load().cgl_fft_destroy(self.h)
        except Exception:
            pass


class SlabExchange:
    """Slab <-> column-block all-to-all over P ranks; `ranks` are the ranks
    this process holds (all P when virtual, [rank] with a process group)."""

    def __init__(self, shape, P, ranks, group=None, device="cuda"):
        n0, n1, n2 = shape
        if n0 % P or (n1 * n2) % P:
            raise ValueError(f"slab sharding needs n0={n0} and n1*n2={n1 * n2} divisible by {P}")
        self.shape, self.P, self.ranks, self.group = tuple(shape), P, list(ranks), group
        self.p0, self.m = n0 // P, (n1 * n2) // P
        self.virtual = len(self.ranks) == P and P > 1 or group is None
        if not self.virtual:
            self.send = torch.empty((P, self.p0, self.m), dtype=torch.complex128, device=device)
            self.recv = torch.empty((P, self.p0, self.m), dtype=torch.complex128, device=device)

    def to_cols(self, slabs, cols):
        P, p0, m = self.P, self.p0, self.m
        if self.virtual:
            for li, r in enumerate(self.ranks):
                src = slabs[li].reshape(p0, P, m)
                for ls, s in enumerate(self.ranks):
                    cols[ls][r * p0:(r + 1) * p0].copy_(src[:, s, :])
            return cols
        if slabs[0].is_cuda:   # row-permutation kernels (csrc/slab.cu) instead of a strided torch copy
            _lib.check(_lib.load().cgl_slab_pack(_lib.stream(), P, p0, m, _lib.ptr(slabs[0]), _lib.ptr(self.send)),
                       "cgl_slab_pack")
        else:
            self.send.copy_(slabs[0].reshape(p0, P, m).transpose(0, 1))
        dist.all_to_all_single(cols[0].view(-1), self.send.view(-1), group=self.group)
        return cols

    def to_slabs(self, cols, slabs):
        P, p0, m = self.P, self.p0, self.m
        if self.virtual:
            for li, r in enumerate(self.ranks):
                dst = slabs[li].reshape(p0, P, m)
                for ls, s in enumerate(self.ranks):
                    dst[:, s, :].copy_(cols[ls][r * p0:(r + 1) * p0])
            return slabs
        dist.all_to_all_single(self.recv.view(-1), cols[0].reshape(-1), group=self.group)
        if slabs[0].is_cuda:
            _lib.check(_lib.load().cgl_slab_unpack(_lib.stream(), P, p0, m, _lib.ptr(self.recv), _lib.ptr(slabs[0])),
                       "cgl_slab_unpack")
        else:
            slabs[0].reshape(p0, P, m).copy_(self.recv.transpose(0, 1))
        return slabs


class SlabFFT:
    """Unnormalised distributed 3D FFT: slabs (p0, n1, n2) <-> column blocks (n0, m)."""

    def __init__(self, ex):
        from . import fftpass
        n0, n1, n2 = ex.shape
        self.ex = ex
        # column block (n0, m) viewed as (n0, m / n2, n2): the pencil passes take 3D fields
        self.cshape = (n0, ex.m // n2, n2) if ex.m % n2 == 0 else None
        self.sshape = (ex.p0, n1, n2)
        self.pencil = (self.cshape is not None and fftpass.supported(self.cshape) and fftpass.supported(self.sshape))
        if not self.pencil:
            self.f2 = FftMany((n1, n2), ex.p0, 1, n1 * n2)   # planes of a slab
            self.f1 = FftMany((n0,), ex.m, ex.m, 1)          # columns of a block (stride m)

    def slab_pass(self, x, axis, inverse=False, program="plain", ops=None):
        from .fftpass import axis_pass
        axis_pass(x, x, axis, inverse=inverse, program=program, ops=ops, shape=self.sshape)

    def col_pass(self, y, inverse=False):
        from .fftpass import axis_pass
        axis_pass(y, y, 0, inverse=inverse, shape=self.cshape)

    def forward(self, slabs, cols):
        for x in slabs:
            if self.pencil:
                self.slab_pass(x, 2)
                self.slab_pass(x, 1)
            else:
                self.f2(x)
        self.ex.to_cols(slabs, cols)
        for y in cols:
            if self.pencil:
                self.col_pass(y)
            else:
                self.f1(y)
        return cols

    def inverse(self, cols, slabs, cols_scratch=None):
        """cols -> slabs (backward, no 1/N); `cols` is preserved when a
        scratch list is given."""
        work = cols
        if cols_scratch is not None:
            for a, b in zip(cols, cols_scratch):
                b.copy_(a)
            work = cols_scratch
        for y in work:
            if self.pencil:
                self.col_pass(y, inverse=True)
            else:
                self.f1(y, inverse=True)
        self.ex.to_slabs(work, slabs)
        for x in slabs:
            if self.pencil:
                self.slab_pass(x, 1, inverse=True)
                self.slab_pass(x, 2, inverse=True)
            else:
                self.f2(x, inverse=True)
        return slabs

    def g_of(self, work_cols, slabs, dst_cols, nl, scale, flag, pos):
        """dst = F g(scale F^-1 work) with the contiguous-axis transforms and g
        fused in one pass (pencil passes only); work_cols is clobbered."""
        from .fftpass import make_ops
        for y in work_cols:
            self.col_pass(y, inverse=True)
        self.ex.to_slabs(work_cols, slabs)
        ops = make_ops(nl=nl, scale=scale, flag=flag, pos=pos)
        for x in slabs:
            self.slab_pass(x, 1, inverse=True)
            self.slab_pass(x, 2, program="g", ops=ops)
            self.slab_pass(x, 1)
        self.ex.to_cols(slabs, dst_cols)
        for y in dst_cols:
            self.col_pass(y)
        return dst_cols


class ShardedFourierPlan:
    """if4 / strang on slab-sharded periodic 3D grids (scalar fields).

    if4: state = coefficients in column blocks; per step 8 distributed FFTs
    (16 all-to-alls would double-count: each FFT has ONE exchange) + 4 g
    kernels on slabs + 4 column-block stage kernels.
    strang: physical slabs between steps (F^-1 F elided as in the single-GPU
    plan): STRANG_END on slabs, forward FFT, E1 on column blocks, inverse FFT.
    """

    def __init__(self, problem, scheme, shape, P, ranks, group=None):
        if problem._blocks[0].grid.ndim != 3 or len(problem._blocks) != 1:
            raise ValueError("sharded Fourier plan: scalar 3D periodic problems")
        if scheme not in ("if4", "strang"):
            raise ValueError("sharded Fourier plan supports if4 and strang")
        self.p, self.scheme, self.shape = problem, scheme, tuple(shape)
        self.ex = SlabExchange(shape, P, ranks, group)
        self.fft = SlabFFT(self.ex)
        self.P, self.ranks, self.group = P, list(ranks), group
        self.nl = problem._nl
        self.N = math.prod(shape)
        n0, n1, n2 = shape
        p0, m = self.ex.p0, self.ex.m
        slab = lambda: [torch.empty((p0, n1, n2), dtype=torch.complex128, device="cuda") for _ in ranks]  # noqa
        cols = lambda: [torch.empty((n0, m), dtype=torch.complex128, device="cuda") for _ in ranks]  # noqa
        if scheme == "if4":
            self.U, self.Qc, self.Qs = cols(), cols(), slab()
            self.G = [cols() for _ in range(4)]
        else:
            self.Us, self.V, self.Vc = [slab(), slab()], slab(), cols()
        self.flag = _lib.new_flag(0)

    # -- helpers ------------------------------------------------------------
    def _tabs(self):
        from fractions import Fraction
        b = self.p._blocks[0]
        tabs = []
        for f in (Fraction(1, 2), Fraction(1)):
            tabs.extend((b.exp_entry(f) if f in b._cache else b.exp_entry(Fraction(1)))[1])
        self._tab_keep = tabs
        return _lib.ptr_array(tabs)

    def _col_off(self, r):
        return r * self.ex.m

    def _fstage(self, name, li, ins, outs, tau, pos):
        r = self.ranks[li]
        _lib.check(_lib.load().cgl_stage_fourier_cols(
            _lib.stream(), _lib.STAGE[name], 1, 3, _lib.i64_array(self.shape), self.ex.m, self._col_off(r),
            _lib.ctypes.byref(self.nl), tau, 1.0, self._tab_ptrs, _lib.ptr_array(ins), _lib.ptr_array(outs),
            _lib.flag_ptr(self.flag), pos), "cgl_stage_fourier_cols")

    def _g(self, slabs, pos):
        from .flows import eval_g_dev
        for x in slabs:
            eval_g_dev(self.nl, [x], scale=1.0 / self.N, outs=[x], flag=self.flag, pos=pos)

    def _reduce(self):
        if not self.ex.virtual:
            global_min_key(self.flag, self.group)

    def _gspec(self, src_cols, dst_cols, pos, clobber=False):
        """dst = F g(F^-1 src) (coefficients -> coefficients); src is preserved
        unless clobber."""
        if self.fft.pencil:
            work = src_cols
            if not clobber:
                for a, b in zip(src_cols, self.Qc):
                    b.copy_(a)
                work = self.Qc
            self.fft.g_of(work, self.Qs, dst_cols, self.nl, 1.0 / self.N, self.flag, pos)
            return
        self.fft.inverse(src_cols, self.Qs, cols_scratch=None if clobber else self.Qc)
        self._g(self.Qs, pos)
        self.fft.forward(self.Qs, dst_cols)

    # -- driver ---------------------------------------------------------------
    def run(self, u0_cols_or_slabs, steps, tau):
        """u0: list (per held rank) of coefficient column blocks (if4) or of
        physical slabs (strang); returns the flag key."""
        lib = _lib.load()
        self.flag.copy_(_lib.new_flag(0))
        self._tab_ptrs = self._tabs()
        pos = _lib.rel_pos(1)
        if self.scheme == "if4":
            for a, b in zip(self.U, u0_cols_or_slabs):
                a.copy_(b)
            G1, G2, G3, G4 = self.G
            for k in range(1, steps + 1):
                self._gspec(self.U, G1, pos)
                for name, gin, gout in (("fif4_s1", G1, G2), ("fif4_s2", G2, G3), ("fif4_s3", G3, G4)):
                    for li in range(len(self.ranks)):
                        self._fstage(name, li, [self.U[li], gin[li]], [self.Qc[li]], tau, pos)
                    # Qc holds the next stage input: F g F^-1 Qc -> gout (Qc may be clobbered)
                    self._gspec(self.Qc, gout, pos, clobber=True)
                self._reduce()
                for li in range(len(self.ranks)):
                    self._fstage("fif4_s4", li, [self.U[li], G1[li], G2[li], G3[li], G4[li]], [self.U[li]], tau, pos)
                _lib.flag_advance(self.flag, 1)
        else:
            for a, b in zip(self.Us[0], u0_cols_or_slabs):
                a.copy_(b)
            for li, x in enumerate(self.Us[0]):
                _lib.check(lib.cgl_stage(_lib.stream(), _lib.STAGE["flow1"], 1, x.numel(), _lib.ctypes.byref(self.nl),
                                         tau, 1.0, _lib.ptr_array([x]), _lib.ptr_array([self.V[li]]),
                                         _lib.flag_ptr(self.flag), pos), "cgl_stage(flow1)")
            b = self.p._blocks[0]
            from fractions import Fraction
            e1 = b.exp_entry(Fraction(1))[1]
            for k in range(1, steps + 1):
                self.fft.forward(self.V, [self.Vc[li] for li in range(len(self.ranks))])
                for li, y in enumerate(self.Vc):
                    _lib.check(lib.cgl_separable_mul_cols(_lib.stream(), 3, _lib.i64_array(self.shape), self.ex.m,
                                                          self._col_off(self.ranks[li]), _lib.ptr_array(e1), 1.0,
                                                          _lib.ptr(y), _lib.ptr(y), _lib.flag_ptr(self.flag), pos),
                               "cgl_separable_mul_cols")
                self.fft.inverse(self.Vc, self.V)
                self._reduce()
                out = self.Us[k % 2]
                for li in range(len(self.ranks)):
                    _lib.check(lib.cgl_stage(_lib.stream(), _lib.STAGE["strang_end"], 1, self.V[li].numel(),
                                             _lib.ctypes.byref(self.nl), tau, 1.0 / self.N,
                                             _lib.ptr_array([self.V[li]]), _lib.ptr_array([out[li], self.V[li]]),
                                             _lib.flag_ptr(self.flag), pos), "cgl_stage(strang_end)")
                _lib.flag_advance(self.flag, 1)
        self._reduce()
        torch.cuda.synchronize()
        return int(self.flag[0].item()) & ((1 << 64) - 1)

    def result_cols(self, k):
        """Coefficients after step k in the column-block layout (per held rank)."""
        if self.scheme == "if4":
            return self.U
        out = [torch.empty_like(c) for c in (self.Vc if hasattr(self, "Vc") else [])]
        tmp = [x.clone() for x in self.Us[k % 2]]
        self.fft.forward(tmp, out)
        return out


def split_global(x, P, layout):
    """Global (n0, n1, n2) tensor -> per-rank slabs ("slabs") or coefficient
    column blocks ("cols")."""
    n0, n1, n2 = x.shape
    p0, m = n0 // P, (n1 * n2) // P
    if layout == "slabs":
        return [x[r * p0:(r + 1) * p0].contiguous() for r in range(P)]
    flat = x.reshape(n0, n1 * n2)
    return [flat[:, r * m:(r + 1) * m].contiguous() for r in range(P)]


def gather_cols(cols, shape):
    n0, n1, n2 = shape
    return torch.cat(cols, dim=1).reshape(n0, n1, n2)
