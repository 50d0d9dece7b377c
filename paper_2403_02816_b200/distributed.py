"""Axis-0 slab sharding of the finite-difference path across ranks.

One process per GPU (torch.distributed; NCCL on B200s, gloo for the CPU
tests).  A 3D field of global shape (n0, n1, n2), C order, is split into
contiguous slabs of n0/P planes along axis 0 (the slowest axis).  Every
pointwise stage and the mu-mode products along axes 1..d-1 are local; the
axis-0 product needs whole axis-0 fibres and is done by one all-to-all
transpose each way:

  to_columns:   (p0, n1*n2) slab  --pack-->  [P][p0][m]  --all_to_all-->  (n0, m)
                (rank r receives every rank's planes of its column block r,
                 stacked in source order = the global axis-0 order)
  local GEMM:   Out (n0, m) = E0 (n0 x n0) * Cols (n0, m)       (DMMA, left form)
  from_columns: rows of slab s are contiguous in Out -> all_to_all -> unpack
                into (p0, P, m) = (p0, n1*n2)

The per-rank send volume per transpose is 16 N (P-1)/P^2 bytes (an
all-gather / reduce-scatter formulation would move P/2 times more).

Divergence: each rank keeps its own sticky key; before every end-of-step
kernel the keys are min-reduced across ranks (sign-flipped so the signed
NCCL/gloo MIN orders them as unsigned), so every rank skips exactly the
kernels the reference's single process would not have run, and all ranks
return the same (diverged_at, reason).
"""

import math

import torch
import torch.distributed as dist

from . import _lib
from .plan import FusedPlan
from .tensors import mode_product_dev

_SIGN = -(1 << 63)


class SlabLayout:
    """Slab partition of a global shape along axis 0 over `world` ranks."""

    def __init__(self, shape, world):
        self.shape = tuple(int(n) for n in shape)
        self.world = int(world)
        n0 = self.shape[0]
        rest = int(math.prod(self.shape[1:])) if len(self.shape) > 1 else 1
        if n0 % self.world or rest % self.world:
            raise ValueError(f"axis-0 slab sharding needs n0={n0} and prod(n1..)={rest} divisible by {self.world}")
        self.n0, self.rest = n0, rest
        self.p0 = n0 // self.world          # planes per rank
        self.m = rest // self.world         # columns per rank after the transpose

    def local_shape(self):
        return (self.p0,) + self.shape[1:]

    def bounds(self, rank):
        return rank * self.p0, (rank + 1) * self.p0


class Transposer:
    """Send/receive buffers and the pack -> all-to-all -> unpack sequence of
    the axis-0 transposes.  CUDA tensors use the library's row-permutation
    kernels (cgl_slab_pack / cgl_slab_unpack, csrc/slab.cu) and NCCL through
    torch.distributed; `cgl_slab_transpose` is the same sequence behind the C
    ABI for a caller that owns an ncclComm_t.  CPU tensors (the gloo
    world-size-2 tests of this layout code) move with torch copies."""

    def __init__(self, layout, group=None, device=None, dtype=torch.complex128, nbuf=1):
        self.L = layout
        self.group = group
        P, p0, m = layout.world, layout.p0, layout.m
        self.send = [torch.empty((P, p0, m), dtype=dtype, device=device) for _ in range(nbuf)]
        self.recv = [torch.empty((P, p0, m), dtype=dtype, device=device) for _ in range(nbuf)]
        self.cols_out = [torch.empty((layout.n0, m), dtype=dtype, device=device) for _ in range(nbuf)]

    def _a2a(self, out, inp, async_op=False):
        if self.L.world == 1:
            out.copy_(inp)
            return None
        return dist.all_to_all_single(out.view(-1), inp.reshape(-1), group=self.group, async_op=async_op)

    def _pack(self, local, send):
        P, p0, m = self.L.world, self.L.p0, self.L.m
        if local.is_cuda:
            _lib.check(_lib.load().cgl_slab_pack(_lib.stream(), P, p0, m, _lib.ptr(local), _lib.ptr(send)),
                       "cgl_slab_pack")
        else:
            send.copy_(local.reshape(p0, P, m).transpose(0, 1))

    def _unpack(self, recv, local_out):
        P, p0, m = self.L.world, self.L.p0, self.L.m
        if recv.is_cuda:
            _lib.check(_lib.load().cgl_slab_unpack(_lib.stream(), P, p0, m, _lib.ptr(recv), _lib.ptr(local_out)),
                       "cgl_slab_unpack")
        else:
            local_out.reshape(p0, P, m).copy_(recv.transpose(0, 1))

    def to_columns(self, local, k=0, async_op=False):
        """(p0, ...) slab -> (n0, m) column block of this rank (buffer set k);
        with async_op the all-to-all's work handle is returned alongside."""
        self._pack(local, self.send[k])
        w = self._a2a(self.recv[k], self.send[k], async_op)
        cols = self.recv[k].view(self.L.n0, self.L.m)
        return (cols, w) if async_op else cols

    def from_columns(self, cols, local_out, k=0):
        """(n0, m) column block -> (p0, ...) slab (written into local_out)."""
        self._a2a(self.recv[k], cols)
        self._unpack(self.recv[k], local_out)
        return local_out

    def from_columns_start(self, cols, k=0):
        return self._a2a(self.send[k], cols, async_op=True)

    def from_columns_finish(self, local_out, k=0):
        self._unpack(self.send[k], local_out)
        return local_out


def mode0_sharded(local_in, mat, mat_t, local_out, tr, gemm=None, flag=None, pos=0):
    """Axis-0 mu-mode product of a slab-sharded field (DMMA / host callback;
    the step plans use ShardedPlan's INT8-emulated products)."""
    cols = tr.to_columns(local_in)
    if gemm is None:
        mode_product_dev(cols, mat, mat_t, 0, out=tr.cols_out[0], flag=flag, pos=pos)
    else:
        tr.cols_out[0].copy_(gemm(mat, cols))
    return tr.from_columns(tr.cols_out[0], local_out)


def tucker_sharded(local_in, mats, mats_t, out, work, tr, gemm=None, local=None, flag=None, pos=0):
    """in x_0 M_0 x_1 M_1 ... on a slab: axis 0 through the transposes, the
    rest local (same mode order as tensors.py:62-69).  `gemm`/`local` replace
    the DMMA kernels (CPU multi-rank tests only)."""
    d = local_in.ndim
    cur = local_in
    for axis in range(d):
        dst = out if (d - axis) % 2 == 1 else work
        if axis == 0:
            mode0_sharded(cur, mats[0], mats_t[0], dst, tr, gemm=gemm, flag=flag, pos=pos)
        elif local is not None:
            dst.copy_(local(cur, mats[axis], axis))
        else:
            mode_product_dev(cur, mats[axis], mats_t[axis], axis, out=dst, flag=flag, pos=pos)
        cur = dst
    return out


def tucker_sharded_oz(items, tr, ws, flag=None, pos=0):
    """Tucker chains of several fields of a slab-sharded grid on the INT8
    tensor cores (ozaki.py), the transposes overlapped with the products:
    every field's slab -> column all-to-all is started first; field j's
    axis-0 product runs while field j+1's columns are still in flight, and its
    return all-to-all while field j+1's product runs; the local axes of field
    j follow once its slab is back.  items: [(in, factors, out, work)]
    (factors = sliced E_0 (global n0 x n0), E_1, ...); buffer set j of `tr`
    belongs to item j."""
    from .ozaki import mode_product_oz
    started = [tr.to_columns(x, k=j, async_op=True) for j, (x, _, _, _) in enumerate(items)]
    back = []
    for j, ((x, facs, out, work), (cols, w)) in enumerate(zip(items, started)):
        if w is not None:
            w.wait()
        mode_product_oz([cols], [facs[0]], [tr.cols_out[j]], 0, ws, flag=flag, pos=pos)
        back.append(tr.from_columns_start(tr.cols_out[j], k=j))
    for j, ((x, facs, out, work), w) in enumerate(zip(items, back)):
        if w is not None:
            w.wait()
        d = x.ndim
        tr.from_columns_finish(out if d % 2 == 1 else work, k=j)
        cur = out if d % 2 == 1 else work
        for axis in range(1, d):
            dst = out if (d - axis) % 2 == 1 else work
            mode_product_oz([cur], [facs[axis]], [dst], axis, ws, flag=flag, pos=pos)
            cur = dst
    return [it[2] for it in items]


def global_min_key(flag, group=None):
    """Min-reduce the sticky divergence key over ranks (unsigned order)."""
    k = flag[0:1]
    t = torch.bitwise_xor(k, _SIGN)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    k.copy_(torch.bitwise_xor(t, _SIGN))


class ShardedPlan(FusedPlan):
    """FusedPlan on the local slab: Tuckers through the axis-0 transposes on
    the INT8 tensor cores (tucker_sharded_oz: all-to-alls overlapped with the
    products), a cross-rank key reduction before every end-of-step kernel,
    eager launches (NCCL collectives are not graph-captured).  Grids below the
    emulated engine's size threshold use the DMMA products."""

    CHUNK = 1 << 30  # never graph-capture
    FUSE_STAGE_SLICE = False  # stage outputs stay FP64: the slabs travel before they are sliced

    def __init__(self, problem, scheme_name, like, layout, group=None):
        super().__init__(problem, scheme_name, like)
        from . import ozaki
        self.layout = layout
        self.group = group
        self.use_oz = ozaki.enabled() and ozaki.fits(layout.shape, 1)
        # buffer sets: one per field of the widest Tucker job list (if4: 2, split4: 2)
        self.tr = Transposer(layout, group, device=like[0].device, nbuf=2 * self.nf)
        if not self.W:
            self.W = [torch.empty_like(like[0]) for _ in range(2 * self.nf)]
        while len(self.W) < 2 * self.nf:
            self.W.append(torch.empty_like(like[0]))

    def _tucker(self, jobs, flag, pre0=None):
        if self.use_oz:
            items = []
            for f, fin, fout in jobs:
                for c in range(self.nf):
                    items.append((fin[c], self.blocks[c].sliced_factors(f), fout[c], self.W[len(items)]))
            for i in range(0, len(items), len(self.tr.send)):
                tucker_sharded_oz(items[i:i + len(self.tr.send)], self.tr, self.oz_ws, flag=flag, pos=self._pos)
            return
        for f, fin, fout in jobs:
            for c in range(self.nf):
                m, mt = self.blocks[c].exp_factors(f)
                tucker_sharded(fin[c], m, mt, fout[c], self.W[c], self.tr, flag=flag, pos=self._pos)

    def _before_end(self, flag):
        global_min_key(flag, self.group)

    def _graph(self, k0, count, flag, tau):
        raise RuntimeError("sharded plans run eagerly")

    def run(self, u0, steps, tau, stop_at=(), on_stop=None, poll_chunks=1):
        flag = self.flag
        flag.copy_(self._flag0)
        self._k_base = 0
        self._pos = _lib.rel_pos(1)
        self.load_state(u0, tau)
        self.prologue(flag, tau)
        for k in range(1, steps + 1):
            self.step(k, flag, tau)
            _lib.flag_advance(flag, 1)
            self._k_base += 1
            if k in stop_at or k == steps or k % 16 == 0:
                global_min_key(flag, self.group)
                key = int(flag[0].item()) & ((1 << 64) - 1)
                if key != _lib.NO_DIVERGENCE and (key >> 24) <= steps:
                    if (key >> 24) > k and k in stop_at and on_stop is not None:
                        on_stop(k, self.result(k))
                    return key
                if k in stop_at and on_stop is not None:
                    on_stop(k, self.result(k))
        return _lib.NO_DIVERGENCE


def integrate_sharded(problem, scheme_name, local_fields, t_final, steps, layout, group=None,
                      snapshot_steps=(), snapshot_path=None, grids=None):
    """Slab-sharded counterpart of integrate() for FD problems built on the
    LOCAL slab's operator (the axis-0 factor is the global n0 x n0 matrix).
    Returns (local result fields, diverged_at, reason, device_seconds).
    snapshot_steps + snapshot_path (a format string taking the step, e.g.
    "run_{:05d}.cgls") + grids (global node coordinates per direction): every
    rank stores its slab of those steps into the one snapshot file
    (io.write_snapshot_sharded; no gather)."""
    from .integrators import SCHEMES
    if scheme_name not in ("if4", "strang", "split4", "if2"):
        raise ValueError(f"sharded path supports if4/strang/split4/if2, not {scheme_name!r}")
    tau = t_final / steps
    problem.prepare(tau, SCHEMES[scheme_name])
    plan = ShardedPlan(problem, scheme_name, list(local_fields), layout, group)
    rank = dist.get_rank(group) if dist.is_available() and dist.is_initialized() else 0
    on_stop = None
    if snapshot_path is not None and snapshot_steps:
        if grids is None:
            raise ValueError("snapshots need the global node coordinates (grids)")
        from .io import write_snapshot_sharded
        barrier = (lambda: dist.barrier(group)) if dist.is_available() and dist.is_initialized() else None

        def on_stop(k, fields):
            write_snapshot_sharded(snapshot_path.format(k), fields, k * tau, grids, layout.shape,
                                   layout.bounds(rank), rank=rank, barrier=barrier)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record()
    key = plan.run(list(local_fields), steps, tau, stop_at=tuple(snapshot_steps), on_stop=on_stop)
    ev1.record()
    torch.cuda.synchronize()
    dev_s = ev0.elapsed_time(ev1) / 1e3
    if key == _lib.NO_DIVERGENCE:
        return plan.result(steps), 0, "", dev_s
    k_div, reason = key >> 24, key & 0xFF
    out = plan.result(k_div) if reason == _lib.NONFINITE_STATE else plan.result(k_div - 1)
    return out, int(k_div), _lib.REASONS[reason], dev_s


def tucker_slabs(slabs, mats, mats_t, ex, flag=None, pos=0):
    """Tucker chain of an axis-0 slab-sharded 3D field held as a list of the
    local slabs (one per held rank; all P with virtual ranks), using the
    slab <-> column-block exchange of slabfourier.SlabExchange: the axis-0
    product runs on the (n0 x m) column blocks, the others on the slabs."""
    n0 = ex.shape[0]
    cols = [torch.empty((n0, ex.m), dtype=torch.complex128, device=s.device) for s in slabs]
    ex.to_cols(slabs, cols)
    outc = [mode_product_dev(c, mats[0], mats_t[0], 0, flag=flag, pos=pos) for c in cols]
    tmp = [torch.empty_like(s) for s in slabs]
    ex.to_slabs(outc, tmp)
    out = []
    for t in tmp:
        for axis in range(1, t.ndim):
            t = mode_product_dev(t, mats[axis], mats_t[axis], axis, flag=flag, pos=pos)
        out.append(t)
    return out


def tucker_slabs_oz(slabs, factors, ex, ws, flag=None, pos=0):
    """tucker_slabs on the INT8 tensor cores (ozaki.py): the axis-0 product
    of each column block is the unsharded first-axis product restricted to
    those columns -- the data slices carry one exponent per column and the
    K = n0 sum runs in the same order -- so the result is bit-identical to the
    unsharded chain for any rank count."""
    from .ozaki import mode_product_oz
    n0 = ex.shape[0]
    cols = [torch.empty((n0, ex.m), dtype=torch.complex128, device=s.device) for s in slabs]
    ex.to_cols(slabs, cols)
    outc = [torch.empty_like(c) for c in cols]
    for c, o in zip(cols, outc):
        mode_product_oz([c], [factors[0]], [o], 0, ws, flag=flag, pos=pos)
    tmp = [torch.empty_like(s) for s in slabs]
    ex.to_slabs(outc, tmp)
    out = []
    for t in tmp:
        for axis in range(1, t.ndim):
            o = torch.empty_like(t)
            mode_product_oz([t], [factors[axis]], [o], axis, ws, flag=flag, pos=pos)
            t = o
        out.append(t)
    return out
