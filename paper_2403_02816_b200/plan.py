"""Fused, graph-captured step plans for the Kronecker (finite-difference) path.

A plan owns persistent device buffers for one (problem, scheme, tau) and
runs each time step as a handful of launches: batched DMMA Tucker chains
for every exp(f tau K) the step needs (integrators.py:146-215) and ONE
fused stage kernel between consecutive Tucker groups (csrc/stages.cu).
Steps are captured into CUDA graphs in chunks, so the host issues one graph
launch per chunk; kernel positions for the divergence key come from the
device step counter in the flag record, which the end-of-step kernel
advances, so a captured chunk replays unchanged.

Per-step launch structure (d = number of dimensions, one GEMM per mode):
  if4     d GEMM (4 Tuckers)  + MID + d GEMM (2 Tuckers) + END      = 2d + 2
  strang  d GEMM (1 Tucker)   + END                                  = d + 1
  split4  d GEMM (2 Tuckers)  + MID + d GEMM (1 Tucker) + END        = 2d + 2
  if2     d GEMM (2 Tuckers)  + END                                  = d + 1
"""

import os

import math

import torch

from . import _lib
from .operators import KroneckerOperator
from .tensors import tucker_dev

FUSED_SCHEMES = ("if4", "strang", "split4", "if2", "strang_3t", "split4_3t")
# three-term schemes run the strang / split4 bodies with every flow a pair of
# exact flows (integrators.py:178-195): nonlinearity kind 3 in the stage kernels
THREE_TERM = {"strang_3t": "strang", "split4_3t": "split4"}
KIND_THREE_TERM = 3


def fused_enabled():
    return os.environ.get("CGL_FUSED", "1") != "0"


FOURIER_SCHEMES = ("if4", "strang")
RK_SCHEMES = ("rk2", "rk4")
RK_MAX_BAND = 8


def supports(problem, scheme_name):
    if not fused_enabled():
        return False
    if problem.fourier:
        from .operators import FourierOperator
        return (scheme_name in FOURIER_SCHEMES and len(problem._blocks[0].shape) <= 3
                and all(isinstance(b, FourierOperator) and b._sep is not None for b in problem._blocks))
    if scheme_name in RK_SCHEMES:
        return BandedRKPlan.applies(problem, scheme_name)
    if scheme_name in THREE_TERM and len(problem._blocks) != 1:
        return False
    return scheme_name in FUSED_SCHEMES and all(isinstance(b, KroneckerOperator) for b in problem._blocks)


def make_plan(problem, scheme_name, like):
    if problem.fourier:
        if PencilFourierPlan.applies(problem, scheme_name, like):
            return PencilFourierPlan(problem, scheme_name, like)
        return FourierPlan(problem, scheme_name, like)
    if scheme_name in RK_SCHEMES:
        return BandedRKPlan(problem, scheme_name, like)
    return FusedPlan(problem, scheme_name, like)


class FusedPlan:
    CHUNK = 16
    FUSE_STAGE_SLICE = True  # if4 stages emit the next axis-0 data slices (cgl_stage_slice)

    def __init__(self, problem, scheme_name, like):
        from fractions import Fraction
        self.p = problem
        self.three = scheme_name in THREE_TERM
        scheme_name = THREE_TERM.get(scheme_name, scheme_name)
        self.scheme = scheme_name
        self.nf = len(like)
        self.n = like[0].numel()
        self.nl = problem._nl
        if self.three:
            self.nl = _lib.Nonlinear.from_buffer_copy(problem._nl)
            self.nl.kind = KIND_THREE_TERM
        self.blocks = problem._blocks
        self.half, self.one = Fraction(1, 2), Fraction(1)
        mk = lambda: [torch.empty_like(like[0]) for _ in range(self.nf)]  # noqa: E731
        nstate = 2 if scheme_name in ("strang", "split4") else 1
        nbuf = {"if4": 6, "strang": 2, "split4": 4, "if2": 4}[scheme_name]
        nwork = {"if4": 4, "strang": 1, "split4": 2, "if2": 2}[scheme_name]
        # Lean mode for fields that do not fit batched: Tucker jobs run one at a
        # time through a single scratch field (if4 on 1024^3: 8 x 17.2 GB).
        field_bytes = 16 * self.n * self.nf
        free, _ = torch.cuda.mem_get_info()
        self.lean = (nstate + nbuf + nwork) * field_bytes > 0.85 * free
        if self.lean:
            nwork = 1
        self.U = [mk() for _ in range(nstate)]
        self.B = [mk() for _ in range(nbuf)]
        self.W = [t for _ in range(nwork) for t in mk()] if like[0].ndim > 1 else []
        self.graphs = {}
        self.shape = tuple(like[0].shape)
        self.use_oz = None
        from .ozaki import Workspace
        self.oz_ws = Workspace()
        self.flag = _lib.new_flag(0)   # baked into the captured graphs; reset per run
        self._pos = _lib.rel_pos(1)
        self._k_base = 0               # host copy of the flag's step base
        self._flag0 = self.flag.clone()
        self.graph_launches = {}       # cgl kernels inside each captured graph
        self.replayed_launches = 0     # cgl kernels launched by graph replays (not seen by the C counter)

    # -- launch helpers --------------------------------------------------------
    def _fused_slices(self):
        """Workspace slots for cgl_stage_slice outputs when the fused if4 path
        applies (INT8-emulated products, single component, one slice chunk,
        not lean), else None.  Slots 0-2: END's X1, u, X5; 3-4: MID's g3, s."""
        if getattr(self, "_fs", False) is not False:
            return self._fs
        self._fs = None
        import os
        from . import ozaki
        if self.use_oz is None:
            self.use_oz = ozaki.enabled() and ozaki.fits(self.shape, 4 * self.nf)
        if (self.FUSE_STAGE_SLICE and self.scheme in ("if4", "strang", "split4") and self.use_oz and not self.lean
                and self.nf == 1 and not self.three
                and len(self.shape) >= 2 and self.shape[0] <= 1024 and self.nl.kind != 2
                and ozaki.single_chunk(self.shape, 4) and os.environ.get("CGL_FUSE_STAGE", "1") != "0"):
            n0, Q = self.shape[0], math.prod(self.shape[1:])
            per = _lib.load().cgl_oz_slice_bytes(ozaki.S, Q, n0, 0)
            dev = self.U[0][0].device
            nslots = {"if4": 5, "strang": 1, "split4": 3}[self.scheme]
            self._fs = [self.oz_ws.get(("F", j, n0), per, Q, dev) for j in range(nslots)]
        return self._fs

    def _stage_slice(self, name, ins, outs, slots, flag, tau):
        lib = _lib.load()
        fin = [t for fs in ins for t in fs]
        fout = [t for fs in outs for t in fs]
        n0, Q = self.shape[0], math.prod(self.shape[1:])
        _lib.check(lib.cgl_stage_slice(_lib.stream(), _lib.STAGE[name], n0, Q, _lib.ctypes.byref(self.nl), tau, 1.0,
                                       _lib.ptr_array(fin), _lib.ptr_array(fout) if fout else None,
                                       _lib.flag_ptr(flag), self._pos, _lib.ptr_array([t[0] for t in slots]),
                                       _lib.ptr_array([t[1] for t in slots])), "cgl_stage_slice")

    def _end_stage(self, name, ins, out, slots, flag, tau):
        """The end-of-step stage+slicing program of step k."""
        self._stage_slice(name, ins, [[out]] if out is not None else [], slots, flag, tau)

    def _if4_form(self):
        """if4 step form: "quad" (default: [A, G] = E1/2 [u, g1], four half-step
        Tuckers of two fields by the semigroup property and linearity) or "ref"
        (CGL_IF4_FORM=ref: the reference's own six Tuckers, integrators.py:
        205-215 literally -- the cross-check of the quad form in the tests and
        in tools/parity_report.py)."""
        f = os.environ.get("CGL_IF4_FORM", "quad")
        if f not in ("quad", "ref"):
            raise ValueError(f"CGL_IF4_FORM must be quad or ref, not {f!r}")
        return f

    def _ensure_oz(self):
        from . import ozaki
        if self.use_oz is None:
            self.use_oz = ozaki.enabled() and ozaki.fits(self.shape, 4 * self.nf)
        return self.use_oz

    def _tucker(self, jobs, flag, pre0=None):
        """jobs: [(fraction, in_fields, out_fields)] -> one GEMM launch per mode
        (lean mode: one job at a time through the single scratch field).
        Products run on the INT8 tensor cores (ozaki.py) unless CGL_GEMM=dmma
        or the data-slice workspace would not fit; else on the DMMA kernel.
        pre0: per job (slices, exponents) of its axis-0 data, already made by
        cgl_stage_slice (fused if4 path)."""
        if self.lean and len(jobs) > 1:
            for j in jobs:
                self._tucker([j], flag)
            return
        from . import ozaki
        if self.use_oz is None:
            self.use_oz = ozaki.enabled() and ozaki.fits(self.shape, 4 * self.nf)
        if self.use_oz:
            ins, outs, facs = [], [], []
            for f, fin, fout in jobs:
                for c in range(self.nf):
                    ins.append(fin[c])
                    outs.append(fout[c])
                    facs.append(self.blocks[c].sliced_factors(f))
            work = self.W[:len(ins)] if self.W else None
            for i in range(0, len(ins), 8):
                sl = slice(i, i + 8)
                ozaki.tucker_oz(ins[sl], facs[sl], outs[sl], work[sl] if work else None, self.oz_ws, flag=flag,
                                pos=self._pos, pre0=pre0[sl] if pre0 is not None else None)
            return
        assert pre0 is None, "pre-sliced operands need the INT8-emulated products"
        if self._tucker2d_ok():
            self._tucker2d(jobs, flag)
            return
        ins, outs, mats, mts = [], [], [], []
        for f, fin, fout in jobs:
            for c in range(self.nf):
                m, mt = self.blocks[c].exp_factors(f)
                ins.append(fin[c])
                outs.append(fout[c])
                mats.append(m)
                mts.append(mt)
        work = self.W[:len(ins)] if self.W else None
        tucker_dev(ins, mats, mts, outs=outs, flag=flag, pos=self._pos, work=work)

    def _tucker2d_ok(self):
        """Cross-mode fused 2D Tucker (cgl_tucker2d, one launch per Tucker
        group) for the small 2D grids the DMMA products serve."""
        if getattr(self, "_t2d", None) is None:
            self._t2d = (len(self.shape) == 2 and self.shape[1] <= 1024 and self.shape[0] <= 1024
                         and not self.use_oz and all(isinstance(b, KroneckerOperator) for b in self.blocks)
                         and type(self) is FusedPlan and os.environ.get("CGL_TUCKER2D", "1") != "0")
        return self._t2d

    def _tucker2d(self, jobs, flag, program=0, tau=0.0, out2=None):
        lib = _lib.load()
        items = []
        for f, fin, fout in jobs:
            for c in range(self.nf):
                (m0, m1), (_, m1t) = self.blocks[c].exp_factors(f)
                b0, b1 = self.blocks[c].tucker2d_bands(f)
                items.append((fin[c], fout[c], m0, m1t, b0, b1))
        for i in range(0, len(items), 8):
            it = items[i:i + 8]
            outs = [x[1] for x in it] + ([out2] if out2 is not None else [])
            _lib.check(lib.cgl_tucker2d(_lib.stream(), program, len(it), self.shape[0], self.shape[1],
                                        _lib.ptr_array([x[0] for x in it]), _lib.ptr_array(outs),
                                        _lib.ptr_array([x[2] for x in it]), _lib.ptr_array([x[3] for x in it]),
                                        _lib.ptr_array([x[4] for x in it]), _lib.ptr_array([x[5] for x in it]),
                                        _lib.ctypes.byref(self.nl), tau, _lib.flag_ptr(flag), self._pos),
                       "cgl_tucker2d")

    def _stage(self, name, ins, outs, flag, tau):
        lib = _lib.load()
        fin = [t for fs in ins for t in fs]
        fout = [t for fs in outs for t in fs]
        _lib.check(lib.cgl_stage(_lib.stream(), _lib.STAGE[name], self.nf, self.n, _lib.ctypes.byref(self.nl),
                                 tau, 1.0, _lib.ptr_array(fin), _lib.ptr_array(fout), _lib.flag_ptr(flag),
                                 self._pos), "cgl_stage")

    def _before_end(self, flag):
        """Hook before each end-of-step kernel (cross-rank key reduction)."""

    # -- scheme bodies -----------------------------------------------------------
    def state_after(self, k):
        return self.U[k % len(self.U)]

    def result(self, k):
        """Fields in the operator's representation after step k."""
        return self.state_after(k)

    def load_state(self, u0, tau):
        for c in range(self.nf):
            self.U[0][c].copy_(u0[c])

    def prologue(self, flag, tau):
        u, B = self.U[0], self.B
        if self.scheme == "if4" and self._if4_form() == "quad":
            from .flows import eval_g_dev
            eval_g_dev(self.nl, u, outs=B[1], flag=flag, pos=self._pos)   # g1 = g(u0)
        elif self.scheme == "if4":
            self._stage("if4_pre", [u], [B[0], B[1]], flag, tau)          # X1, X5
        elif self.scheme == "if2":
            self._stage("if2_pre", [u], [B[0], B[1]], flag, tau)          # X, Y
        elif self.scheme == "strang":
            self._stage("flow1", [u], [B[0]], flag, tau)                  # v
        elif self.scheme == "split4":
            self._stage("flow2", [u], [B[0], B[1]], flag, tau)            # v, f

    def step(self, k, flag, tau):
        """One time step k (1-based); input state_after(k-1), output state_after(k)."""
        self._pos = _lib.rel_pos(k - self._k_base)
        B, H, O = self.B, self.half, self.one
        if self.scheme == "if4" and self._fused_slices() is not None and self._if4_form() == "quad":
            # [A, G] = E1/2 [u, g1] (E1/2 X1 = A + t/2 G, E1/2 X5 = A + t/6 G by
            # linearity); MIDQ -> p, r sliced; [u4, q] = E1/2 [p, r]; ENDQ -> u, g1'
            # sliced (F0, F1).  Four half-step Tuckers per step.
            u = self.U[0]
            g1, A, G = B[1], B[2], B[3]
            F = self._fs
            self._tucker([(H, u, A), (H, g1, G)], flag, pre0=None if k == 1 else [F[0], F[1]])
            self._stage_slice("if4_midq", [A, G], [], [F[3], F[4]], flag, tau)
            self._tucker([(H, A, B[4]), (H, G, B[5])], flag, pre0=[F[3], F[4]])   # u4 -> B4, q -> B5
            self._before_end(flag)
            self._stage_slice("if4_endq", [B[4], B[5]], [u], [F[0], F[1]], flag, tau)
        elif self.scheme == "if4" and self._fused_slices() is not None:
            # reference form: X1, u, X5 (after step k-1) and g3, s reach their products
            # only as slices made by the fused stage kernels; step 1 slices the prologue's X1, X5
            u = self.U[0]
            x1, x5, u2, a, b, c = B
            F = self._fs
            self._tucker([(H, x1, u2), (H, u, a), (O, u, b), (O, x5, c)], flag,
                         pre0=None if k == 1 else [F[0], F[1], F[1], F[2]])
            self._stage_slice("if4_mid", [u2, a], [], [F[3], F[4]], flag, tau)
            self._tucker([(H, u2, x1), (H, a, x5)], flag, pre0=[F[3], F[4]])
            self._before_end(flag)
            self._end_stage("if4_end", [b, c, x1, x5], u[0], [F[0], F[1], F[2]], flag, tau)
        elif self.scheme == "if4" and self._if4_form() == "quad":
            u = self.U[0]
            g1, A, G, u4, q = B[1], B[2], B[3], B[4], B[5]
            self._tucker([(H, u, A), (H, g1, G)], flag)
            self._stage("if4_midq", [A, G], [A, G], flag, tau)             # p -> A, r -> G
            self._tucker([(H, A, u4), (H, G, q)], flag)
            self._before_end(flag)
            self._stage("if4_endq", [u4, q], [u, g1], flag, tau)
        elif self.scheme == "if4":
            u = self.U[0]
            x1, x5, u2, a, b, c = B
            self._tucker([(H, x1, u2), (H, u, a), (O, u, b), (O, x5, c)], flag)
            self._stage("if4_mid", [u2, a], [u2, a], flag, tau)          # g3 -> u2, s -> a
            self._tucker([(H, u2, x1), (H, a, x5)], flag)                 # d -> x1, e -> x5
            self._before_end(flag)
            self._stage("if4_end", [b, c, x1, x5], [u, x1, x5], flag, tau)
        elif self.scheme == "if2":
            u = self.U[0]
            x, y, u2, o = B
            self._tucker([(O, x, u2), (O, y, o)], flag)
            self._before_end(flag)
            self._stage("if2_end", [u2, o], [u, x, y], flag, tau)
        elif self.scheme == "strang" and self._fused_slices() is not None:
            # v (= flow of the previous state) reaches its product only as slices
            v, w = B
            F = self._fs
            self._tucker([(O, v, w)], flag, pre0=None if k == 1 else [F[0]])
            self._before_end(flag)
            self._end_stage("strang_end", [w], self.state_after(k)[0], [F[0]], flag, tau)
        elif self.scheme == "split4" and self._fused_slices() is not None:
            # v, f of each step and the fine-path f after its first half step
            # reach their products only as slices (slots 0, 1 and 2)
            v, f, v2, f2 = B
            F = self._fs
            self._tucker([(O, v, v2), (H, f, f2)], flag, pre0=None if k == 1 else [F[0], F[1]])
            self._stage_slice("split4_mid", [v2, f2], [v2], [F[2]], flag, tau)   # coarse c -> v2 (FP64)
            self._tucker([(H, f2, v)], flag, pre0=[F[2]])                        # f3 -> v
            self._before_end(flag)
            self._end_stage("split4_end", [v, v2], self.state_after(k)[0], [F[0], F[1]], flag, tau)
        elif self.scheme == "strang" and self.nf == 1 and self.nl.kind != 2 and not self.three \
                and self._ensure_oz() is False and self._tucker2d_ok():
            # one launch per step: Tucker + flow, check, next step's flow (cgl_tucker2d);
            # v ping-pongs between B[0] and B[1] (every output row reads a band of input rows)
            v_in, v_out = B[(k - 1) % 2], B[k % 2]
            self._tucker2d([(O, v_in, [self.state_after(k)[0]])], flag, program=1, tau=tau, out2=v_out[0])
        elif self.scheme == "strang":
            v, w = B
            self._tucker([(O, v, w)], flag)
            self._before_end(flag)
            self._stage("strang_end", [w], [self.state_after(k), v], flag, tau)
        elif self.scheme == "split4":
            v, f, v2, f2 = B
            self._tucker([(O, v, v2), (H, f, f2)], flag)
            self._stage("split4_mid", [v2, f2], [v2, f2], flag, tau)      # coarse c -> v2, f -> f2
            self._tucker([(H, f2, v)], flag)                              # f3 -> v
            self._before_end(flag)
            self._stage("split4_end", [v, v2], [self.state_after(k), v, f], flag, tau)

    # -- driver ------------------------------------------------------------------
    def _graph(self, k0, count, flag, tau):
        key = (k0 % len(self.U), count)
        g = self.graphs.get(key)
        if g is None:
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            lib = _lib.load()
            n0 = lib.cgl_launch_count()
            # no garbage collection while capturing: a finaliser that frees device
            # memory (e.g. a cuFFT plan) would invalidate the capture
            import gc
            gc.collect()
            was = gc.isenabled()
            gc.disable()
            try:
                with torch.cuda.stream(s):
                    with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
                        for j in range(count):
                            self.step(k0 + j, flag, tau)
                        _lib.flag_advance(flag, count)
            finally:
                if was:
                    gc.enable()
            torch.cuda.current_stream().wait_stream(s)
            self.graph_launches[key] = lib.cgl_launch_count() - n0
            self.graphs[key] = g
        self.replayed_launches += self.graph_launches[key]
        return g

    def run(self, u0, steps, tau, stop_at=(), on_stop=None, poll_chunks=1):
        """Advance `steps` steps from u0; returns the flag key (int)."""
        flag = self.flag
        flag.copy_(self._flag0)
        self._k_base = 0
        self._pos = _lib.rel_pos(1)
        # captured graphs bake tau and the prepared operator factors (pointers):
        # drop them when either changed since the capture (a re-prepared
        # operator rebuilds its cache dict; holding the old dicts keeps their
        # identities unique)
        sig = (float(tau), [b._cache for b in self.blocks])
        old = getattr(self, "_graph_sig", None)
        if old is None or old[0] != sig[0] or any(x is not y for x, y in zip(old[1], sig[1])):
            self.graphs.clear()
            self.graph_launches.clear()
        self._graph_sig = sig
        self.load_state(u0, tau)
        self.prologue(flag, tau)
        stops = sorted(set(int(s) for s in stop_at if 1 <= int(s) <= steps))
        k = 1
        pins = [torch.empty(1, dtype=torch.int64, pin_memory=True) for _ in range(2)]
        pending = None  # (event, pinned) of the last asynchronous flag read
        eager_first = True
        nchunk = 0

        def diverged(v):
            key = int(v) & ((1 << 64) - 1)
            return key if key != _lib.NO_DIVERGENCE and (key >> 24) <= steps else None

        while k <= steps:
            nxt = next((s for s in stops if s >= k), steps)
            count = min(self.CHUNK, nxt - k + 1)
            if eager_first:
                count = 1  # step 1 (its products slice the prologue's fields) runs eagerly
            if eager_first:
                for j in range(count):
                    self.step(k + j, flag, tau)
                _lib.flag_advance(flag, count)
                eager_first = False
            else:
                self._graph(k, count, flag, tau).replay()
            self._k_base += count
            k += count
            nchunk += 1
            if (k - 1) in stops or k > steps:
                torch.cuda.current_stream().synchronize()
                key = diverged(flag[0].item())
                if key is not None:
                    # the end-of-step pass of step k-1 also runs step k's first
                    # flow: a divergence there (key step k) leaves step k-1
                    # complete, and the reference snapshots it before failing
                    if (key >> 24) > k - 1 and (k - 1) in stops and on_stop is not None:
                        on_stop(k - 1, self.result(k - 1))
                    return key
                if (k - 1) in stops and on_stop is not None:
                    on_stop(k - 1, self.result(k - 1))
                pending = None
                continue
            # non-blocking divergence poll: read the previous chunk's copy if it landed
            if pending is not None and pending[0].query():
                key = diverged(pending[1].item())
                pending = None
                if key is not None:
                    torch.cuda.current_stream().synchronize()
                    return diverged(flag[0].item())
            if pending is None and nchunk % max(1, poll_chunks) == 0:
                pin = pins[nchunk % 2]
                pin.copy_(flag[:1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record()
                pending = (ev, pin)
        return _lib.NO_DIVERGENCE


class FourierPlan(FusedPlan):
    """Fused periodic (pseudospectral) plans: cuFFT Z2Z + spectral stage
    kernels with the separable exp(f tau symbol) evaluated in-kernel.

    if4: state kept in coefficient space; per step 8 FFTs (4 g evaluations
    as F g F^-1, integrators.py:99-101) + 4 g kernels (1/N folded) + 4
    spectral stage kernels (FIF4_S1..S4).
    strang: the state is kept in PHYSICAL space between steps: the
    reference's F^-1(F(.)) pair at each step boundary is elided (identical
    math, rounding-level difference), leaving per step one fused pointwise
    kernel (flow t/2 of step k, finiteness check, flow t/2 of step k+1),
    one FFT, the separable E1 multiply and one inverse FFT.  Coefficients are
    formed once at the end (and at snapshot steps).  cuFFT never writes a
    state buffer, so divergence semantics are preserved.
    """

    def __init__(self, problem, scheme_name, like):
        from fractions import Fraction
        self.p = problem
        self.scheme = scheme_name
        self.nf = len(like)
        self.shape = tuple(like[0].shape)
        self.n = like[0].numel()
        self.nl = problem._nl
        self.blocks = problem._blocks
        self.half, self.one = Fraction(1, 2), Fraction(1)
        mk = lambda: [torch.empty_like(like[0]) for _ in range(self.nf)]  # noqa: E731
        if scheme_name == "if4":
            self.U = [mk()]
            self.B = [mk() for _ in range(5)]      # Q, G1, G2, G3, G4
        else:
            self.U = [mk(), mk()]                  # physical state ping-pong
            self.B = [mk()]                        # Q (v / spectral scratch)
        self.graphs = {}
        self.flag = _lib.new_flag(0)
        self._pos = _lib.rel_pos(1)
        self._k_base = 0
        self._flag0 = self.flag.clone()
        self.graph_launches = {}
        self.replayed_launches = 0
        self.W = []

    def _tables(self):
        # [fraction slot (1/2, 1)][component][axis]
        tabs = []
        for f in (self.half, self.one):
            for b in self.blocks:
                kind, data = b.exp_entry(f) if f in b._cache else ("sep", None)
                if data is None:
                    data = b.exp_entry(self.one)[1]  # strang prepares only f = 1; slot unused
                tabs.extend(data)
        return tabs

    def _fft(self, fields_in, fields_out, inverse):
        from .spectral import fft_dev
        for a, b in zip(fields_in, fields_out):
            fft_dev(a, inverse=inverse, out=b)

    def _g(self, fields, scale):
        from .flows import eval_g_dev
        eval_g_dev(self.nl, fields, scale=scale, outs=fields, flag=self.flag, pos=self._pos)

    def _fstage(self, name, ins, outs, tau, scale=1.0):
        lib = _lib.load()
        fin = [t for fs in ins for t in fs]
        fout = [t for fs in outs for t in fs]
        tabs = self._tab_ptrs
        _lib.check(lib.cgl_stage_fourier(_lib.stream(), _lib.STAGE[name], self.nf, len(self.shape),
                                         _lib.i64_array(self.shape), _lib.ctypes.byref(self.nl), tau, scale,
                                         tabs, _lib.ptr_array(fin), _lib.ptr_array(fout),
                                         _lib.flag_ptr(self.flag), self._pos), "cgl_stage_fourier")

    def _pstage(self, name, ins, outs, tau, scale):
        lib = _lib.load()
        fin = [t for fs in ins for t in fs]
        fout = [t for fs in outs for t in fs]
        _lib.check(lib.cgl_stage(_lib.stream(), _lib.STAGE[name], self.nf, self.n, _lib.ctypes.byref(self.nl),
                                 tau, scale, _lib.ptr_array(fin), _lib.ptr_array(fout), _lib.flag_ptr(self.flag),
                                 self._pos), "cgl_stage")

    def _mul_e1(self, fields):
        lib = _lib.load()
        for b, x in zip(self.blocks, fields):
            _, tabs = b.exp_entry(self.one)
            _lib.check(lib.cgl_separable_mul(_lib.stream(), x.ndim, _lib.i64_array(x.shape), _lib.ptr_array(tabs),
                                             1.0, _lib.ptr(x), _lib.ptr(x), _lib.flag_ptr(self.flag),
                                             self._pos), "cgl_separable_mul")

    def load_state(self, u0, tau):
        self._tab_list = self._tables()
        self._tab_ptrs = _lib.ptr_array(self._tab_list)
        if self.scheme == "if4":
            for c in range(self.nf):
                self.U[0][c].copy_(u0[c])
        else:
            # physical state p0 = F^-1 u0 = ifftn(u0) (spectral.py:84-86)
            from .spectral import scale_dev
            self._fft(u0, self.U[0], inverse=True)
            for x in self.U[0]:
                scale_dev(x, 1.0 / self.n, out=x)
        self._scale0 = 1.0

    def prologue(self, flag, tau):
        if self.scheme == "strang":
            # v = flow(p0 / N, t/2) at seq 0 of step 1
            self._pstage("flow1", [self.U[0]], [self.B[0]], tau, self._scale0)

    def step(self, k, flag, tau):
        self._pos = _lib.rel_pos(k - self._k_base)
        inv_n = 1.0 / self.n
        if self.scheme == "if4":
            u = self.U[0]
            q, g1, g2, g3, g4 = self.B
            self._fft(u, q, inverse=True)
            self._g(q, inv_n)
            self._fft(q, g1, inverse=False)
            for name, gin, gout in (("fif4_s1", g1, g2), ("fif4_s2", g2, g3), ("fif4_s3", g3, g4)):
                self._fstage(name, [u, gin], [q], tau)
                self._fft(q, q, inverse=True)
                self._g(q, inv_n)
                self._fft(q, gout, inverse=False)
            self._fstage("fif4_s4", [u, g1, g2, g3, g4], [u], tau)
        else:
            v = self.B[0]
            self._fft(v, v, inverse=False)
            self._mul_e1(v)
            self._fft(v, v, inverse=True)
            # out_k = flow(w / N, t/2) [seq w], check, v' = flow(out_k, t/2) [step k+1, seq 0]
            self._pstage("strang_end", [v], [self.state_after(k), v], tau, inv_n)

    def result(self, k):
        if self.scheme == "if4":
            return self.U[0]
        out = [torch.empty_like(x) for x in self.U[0]]
        self._fft(self.state_after(k), out, inverse=False)
        return out


class PencilFourierPlan(FourierPlan):
    """if4 / strang on power-of-two periodic grids (2D/3D, extents 16..512)
    with the fused pencil-FFT passes (csrc/fftpass.cu) instead of cuFFT plus
    separate pointwise kernels.  One pass per axis per transform; every
    pointwise piece rides in a pass (3D, axes 0/1/2, axis 2 contiguous):

    if4 (state u in coefficient space, scratch T, g1..g3):
      prologue  IF4_START  T = F2^-1 u
      eval i    G1^-1, G0 (F0^-1, /N, g, F0), G1      (2D: G0 only)
                B_i: g_i = F2 T; next stage input q -> T = F2^-1 q; the combination
                u' = E1 (u + t/6 g1) + t/3 E1/2 (g2 + g3) + t/6 g4 accumulates term by term
                in one field (B4 adds the last, checks, stores u; T = F2^-1 u starts the
                next step)
      16 passes per 3D step: 672 B/pt of HBM traffic (cuFFT + stage kernels: ~1.1 KB/pt).
    strang (state in physical space, ping-pong U; the reference's F^-1 F at
    each step boundary elided exactly as FourierPlan):
      prologue  STR_START  T = F0 flow(u0 / N, t/2)
      step k    F1, STR_MID (F2, E1, F2^-1), F1^-1,
                STR_A0: w = F0^-1 T / N; u_k = flow(w, t/2) (checked, stored);
                T = F0 flow(u_k, t/2) of step k + 1
      4 passes per 3D step: 144 B/pt.  For the exact cubic flow the two flows at a step
      boundary are one flow(., t) by the semigroup property (STR_A0F: one log1p / sincos /
      rsqrt per point instead of two; the reference's checks decided as it decides them):
      the stored field is then w, and the state flow(w, t/2) is formed when it is asked for.
    Divergence keys and positions are those of the stage kernels (same
    programs, same flag record), so diverged_at / reason are unchanged.
    """

    def __init__(self, problem, scheme_name, like):
        from fractions import Fraction
        self.p = problem
        self.scheme = scheme_name
        self.nf = len(like)
        self.shape = tuple(like[0].shape)
        self.n = like[0].numel()
        self.nl = problem._nl
        self.blocks = problem._blocks
        self.half, self.one = Fraction(1, 2), Fraction(1)
        mk = lambda: torch.empty_like(like[0])  # noqa: E731
        self.T = mk()
        if scheme_name == "if4":
            self.U = [[mk()]]
            self.G = [mk()]   # the accumulated Lawson combination (B1 starts it, B4 finishes it)
        else:
            self.U = [[mk()], [mk()]]
        self.graphs = {}
        self.flag = _lib.new_flag(0)
        self._pos = _lib.rel_pos(1)
        self._k_base = 0
        self._flag0 = self.flag.clone()
        self.graph_launches = {}
        self.replayed_launches = 0
        self.W = []

    @staticmethod
    def applies(problem, scheme_name, like):
        from . import fftpass
        return (scheme_name in ("if4", "strang") and len(like) == 1 and problem._nl.kind != 2
                and fftpass.supported(like[0].shape))

    def _ops(self, tau, **kw):
        from .fftpass import make_ops
        return make_ops(tables=self._tabs, tau=tau, nl=self.nl, flag=self.flag, pos=self._pos, **kw)

    def _pass(self, prog, axis, src, dst, tau, inverse=False, **kw):
        from .fftpass import axis_pass
        axis_pass(src, dst, axis, inverse=inverse, program=prog, ops=self._ops(tau, **kw), shape=self.shape)

    def load_state(self, u0, tau):
        from .fftpass import fftn
        tabs = self._tables()   # [fraction (1/2, 1)][axis] for the single component
        d = len(self.shape)
        self._tab_keep = tabs
        self._tabs = [tabs[0:d], tabs[d:2 * d]]
        self._tau = float(tau)
        if self.scheme == "if4":
            self.U[0][0].copy_(u0[0])
        else:
            fftn(u0[0], out=self.U[0][0], inverse=True)   # physical p0 * N (1/N folded into STR_START)

    def prologue(self, flag, tau):
        last = len(self.shape) - 1
        if self.scheme == "if4":
            self._pass("if4_start", last, None, self.T, tau, u=self.U[0][0])
        else:
            self._pass("str_start", 0, None, self.T, tau, u=self.U[0][0], scale=1.0 / self.n)

    def step(self, k, flag, tau):
        self._pos = _lib.rel_pos(k - self._k_base)
        d = len(self.shape)
        last = d - 1
        T = self.T
        inv_n = 1.0 / self.n
        if self.scheme == "if4":
            u = self.U[0][0]
            acc = self.G[0]
            for prog in ("if4_b1", "if4_b2", "if4_b3", "if4_b4"):
                if d == 3:
                    self._pass("plain", 1, T, T, tau, inverse=True)
                self._pass("g", 0, T, T, tau, scale=inv_n)
                if d == 3:
                    self._pass("plain", 1, T, T, tau)
                if prog == "if4_b1":
                    self._pass(prog, last, T, T, tau, u=u, g_out=acc)
                elif prog == "if4_b4":
                    self._pass(prog, last, T, T, tau, u=acc, u_out=u)
                else:
                    self._pass(prog, last, T, T, tau, u=u, g=(acc, None, None), g_out=acc)
        else:
            out = self.U[k % 2][0]
            if d == 3:
                self._pass("plain", 1, T, T, tau)
            self._pass("str_mid", last, T, T, tau)
            if d == 3:
                self._pass("plain", 1, T, T, tau, inverse=True)
            self._before_end(flag)
            self._pass("str_a0f" if self._fused_boundary() else "str_a0", 0, T, T, tau, u_out=out, scale=inv_n)

    def _fused_boundary(self):
        return self.nl.kind == 0

    def result(self, k):
        from .fftpass import fftn
        if self.scheme == "if4":
            return self.U[0]
        state = self.U[k % 2][0]
        if k == 0:
            return [fftn(state) * (1.0 / self.n)]   # load_state left N x the physical input in U[0]
        if self._fused_boundary():
            # U holds w of step k: the state is flow(w, t/2) (same device function as the
            # step kernels; no divergence bookkeeping: step k's checks ran in its pass)
            w, state = state, torch.empty_like(state)
            _lib.check(_lib.load().cgl_stage(_lib.stream(), _lib.STAGE["flow1"], 1, w.numel(),
                                             _lib.ctypes.byref(self.nl), self._tau, 1.0, _lib.ptr_array([w]),
                                             _lib.ptr_array([state]), None, 0), "cgl_stage(flow1)")
        return [fftn(state)]


def half_bandwidth(m):
    """max |i - j| over the exactly non-zero entries of a square host matrix."""
    import numpy as np
    i, j = np.nonzero(m)
    return int(np.abs(i - j).max()) if i.size else 0


class BandedRKPlan(FusedPlan):
    """rk2 / rk4 (integrators.py:146-158) on Kronecker-sum operators whose
    per-direction factors are banded (half-bandwidth <= 8: every FD operator of
    operators.py:40-113), graph-captured, one `cgl_rk_stage` launch per stage:
    f_i = K x_i + g(x_i) as a (2 b + 1)-point contraction per direction, the next
    stage input and the running combination u + tau sum b_i f_i in the same
    pass.  rk4: 4 launches per step (reference: 4 x (d dense products + g +
    sums) + a 5-term combination).  1..3 dimensions, 1 or 2 components (one
    operator per component).  The new state is checked finite at (step, 255)
    like every other plan; the state ping-pongs, so a diverged run returns the
    reference's post-step fields."""

    def __init__(self, problem, scheme_name, like):
        import numpy as np
        self.p = problem
        self.scheme = scheme_name
        self.nf = len(like)
        self.shape = tuple(like[0].shape)
        self.n = like[0].numel()
        self.nl = problem._nl
        self.blocks = problem._blocks
        mk = lambda: [torch.empty_like(like[0]) for _ in range(self.nf)]  # noqa: E731
        self.U = [mk(), mk()]
        self.X = [mk(), mk()]
        self.ACC = mk()
        self.W = []
        d = len(self.shape)
        # one half-bandwidth per direction (the widest component), bands packed to it
        self.hb = [max(half_bandwidth(b.matrices[mu]) for b in self.blocks) for mu in range(d)]
        self.bands = []
        for b in self.blocks:
            for mu in range(d):
                m, hb, n = b.matrices[mu], self.hb[mu], self.shape[mu]
                band = np.zeros((n, 2 * hb + 1), dtype=complex)
                for dd in range(2 * hb + 1):
                    off = dd - hb
                    i0, i1 = max(0, -off), min(n, n - off)
                    band[i0:i1, dd] = m[np.arange(i0, i1), np.arange(i0, i1) + off]
                self.bands.append(torch.from_numpy(band).to(like[0].device))
        self._hb_c = (_lib.c_int * d)(*self.hb)
        self.graphs = {}
        self.flag = _lib.new_flag(0)
        self._pos = _lib.rel_pos(1)
        self._k_base = 0
        self._flag0 = self.flag.clone()
        self.graph_launches = {}
        self.replayed_launches = 0

    @staticmethod
    def applies(problem, scheme_name):
        if scheme_name not in RK_SCHEMES or problem.fourier:
            return False
        if not all(isinstance(b, KroneckerOperator) for b in problem._blocks):
            return False
        if len(problem._blocks[0].shape) > 3 or any(b.shape != problem._blocks[0].shape for b in problem._blocks):
            return False
        return all(half_bandwidth(m) <= RK_MAX_BAND for b in problem._blocks for m in b.matrices)

    def load_state(self, u0, tau):
        self._tau = float(tau)
        super().load_state(u0, tau)

    def result(self, k):
        """State after step k.  A step that ended non-finite is redone from its
        (intact) input on the dense-product path: a dense product turns one
        inf into NaNs along whole fibres (0 x inf), the banded contraction only
        next to it, and the reference returns the former."""
        key = int(self.flag[0].item()) & ((1 << 64) - 1)
        if key != _lib.NO_DIVERGENCE and (key >> 24) == k and (key & 0xFF) == _lib.NONFINITE_STATE:
            from .integrators import _STEPPERS
            ctx, self.p._ctx = self.p._ctx, None
            try:
                return list(_STEPPERS[self.scheme](self.p, self.U[(k - 1) % 2], self._tau))
            finally:
                self.p._ctx = ctx
        return self.U[k % 2]

    def _rk(self, x, u, acc_in, x_out, acc_out, cx, ca, check):
        pa = _lib.ptr_array
        _lib.check(_lib.load().cgl_rk_stage(
            _lib.stream(), len(self.shape), _lib.i64_array(self.shape), self.nf, self._hb_c, pa(self.bands),
            _lib.ctypes.byref(self.nl), pa(x), pa(u), pa(acc_in) if acc_in is not None else None,
            pa(x_out) if x_out is not None else None, pa(acc_out) if acc_out is not None else None,
            float(cx), float(ca), 1 if check else 0, _lib.flag_ptr(self.flag), self._pos), "cgl_rk_stage")

    def prologue(self, flag, tau):
        pass

    def step(self, k, flag, tau):
        self._pos = _lib.rel_pos(k - self._k_base)
        u, out = self.U[(k - 1) % 2], self.U[k % 2]
        X0, X1, A = self.X[0], self.X[1], self.ACC
        if self.scheme == "rk2":
            self._rk(u, u, None, X0, A, tau, 0.5 * tau, False)          # x1 = u + t f1; acc = u + t/2 f1
            self._before_end(flag)
            self._rk(X0, u, A, None, out, 0.0, 0.5 * tau, True)         # out = acc + t/2 f2
        else:
            t6 = tau / 6.0
            self._rk(u, u, None, X0, A, 0.5 * tau, t6, False)           # x1 = u + t/2 f1; acc = u + t/6 f1
            self._rk(X0, u, A, X1, A, 0.5 * tau, 2.0 * t6, False)       # x2 = u + t/2 f2; acc += t/3 f2
            self._rk(X1, u, A, X0, A, tau, 2.0 * t6, False)             # x3 = u + t f3;   acc += t/3 f3
            self._before_end(flag)
            self._rk(X0, u, A, None, out, 0.0, t6, True)                # out = acc + t/6 f4
