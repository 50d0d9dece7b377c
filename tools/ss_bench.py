"""Isolated per-launch times of the C1 if4 step kernels: each kernel launched
`reps` times back to back inside one captured CUDA graph (PDL between
consecutive launches as in the step), inputs L2-resident.

    python tools/ss_bench.py            -> one JSON line per kernel
"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_02816_b200 import _lib, ozaki, workloads as W  # noqa: E402

lib = _lib.load()
w = W.CONFIGS["C1"]
prob = W.build_problem(w)
prob.operator.prepare(w.tau / 2, (1,))
fac = prob.operator.sliced_factors(1)[0]
shape = w.extents
n0, Q = shape[0], math.prod(shape[1:])
g = torch.Generator(device="cuda").manual_seed(1)
F = [0.3 * torch.randn(shape, dtype=torch.complex128, device="cuda", generator=g) for _ in range(4)]
O = [torch.empty_like(x) for x in F]
ws = ozaki.Workspace()
per = lib.cgl_oz_slice_bytes(ozaki.S, Q, n0, 0)
slots = [ws.get(("F", j, n0), per, Q, F[0].device) for j in range(3)]
flag = _lib.new_flag(0)
nl = prob._nl
reps = int(os.environ.get("REPS", "40"))


def stage_slice(prog, ins, outs, nsl):
    _lib.check(lib.cgl_stage_slice(_lib.stream(), _lib.STAGE[prog], n0, Q, _lib.ctypes.byref(nl), w.tau, 1.0,
                                   _lib.ptr_array(ins), _lib.ptr_array(outs) if outs else None,
                                   _lib.flag_ptr(flag), _lib.rel_pos(1),
                                   _lib.ptr_array([t[0] for t in slots[:nsl]]),
                                   _lib.ptr_array([t[1] for t in slots[:nsl]])), "stage_slice")


def slice_last(nf):
    bufs = [ws.get(("D", u, n0), per, Q, F[0].device) for u in range(nf)]
    _lib.check(lib.cgl_oz_slice_multi(_lib.stream(), ozaki.S, nf, _lib.ptr_array(F[:nf]), n0, 1, Q, n0, 1, 0, 0,
                                      _lib.ptr_array([b[0] for b in bufs]), 0,
                                      _lib.ptr_array([b[1] for b in bufs]), 0), "slice")


def gemm0(nf):
    ozaki.mode_product_oz(F[:nf], [fac] * nf, O[:nf], 0, ws, flag=flag, pos=_lib.rel_pos(1),
                          presliced=[slots[0]] * nf)


def gemm1(nf):
    ozaki.mode_product_oz(F[:nf], [fac] * nf, O[:nf], 1, ws, flag=flag, pos=_lib.rel_pos(1))


cases = {
    "stage_slice_mid": lambda: stage_slice("if4_mid", F[:2], [], 2),
    "stage_slice_end": lambda: stage_slice("if4_end", F[:4], [O[0]], 3),
    "stage_slice_midq": lambda: stage_slice("if4_midq", F[:2], [], 2),
    "stage_slice_endq": lambda: stage_slice("if4_endq", F[:2], [O[0]], 2),
    "stage_slice_strang_end": lambda: stage_slice("strang_end", F[:1], [O[0]], 1),
    "stage_slice_split4_mid": lambda: stage_slice("split4_mid", F[:2], [O[0]], 1),
    "stage_slice_split4_end": lambda: stage_slice("split4_end", F[:2], [O[0]], 2),
    "slice_last_1f": lambda: slice_last(1),
    "slice_last_4f": lambda: slice_last(4),
    "slice_last_2f": lambda: slice_last(2),
    "gemm0_4f": lambda: gemm0(4),
    "gemm0_2f": lambda: gemm0(2),
    "gemm1_4f_incl_slice": lambda: gemm1(4),
}
# EVICT=MB: write a buffer of that size before every launch (L2 pressure as in the step)
evict_mb = int(os.environ.get("EVICT", "0"))
if evict_mb:
    ebuf = torch.empty(evict_mb << 20, dtype=torch.uint8, device="cuda")
    for k in list(cases):
        f0 = cases[k]
        cases[k] = (lambda f0: (lambda: (ebuf.fill_(1), f0())))(f0)
only = sys.argv[1:] or list(cases)
s = torch.cuda.Stream()
for name in only:
    fn = cases[name]
    fn()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (5 * reps)
    print(json.dumps({"kernel": name, "us_per_launch": round(us, 2), "reps": reps,
                      "pdl": os.environ.get("CGL_PDL", "1")}), flush=True)
