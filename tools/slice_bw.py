"""HBM bandwidth of the data-slicing and fused stage+slicing kernels on C2-sized
fields (256^3 complex128, 268 MB per field: not L2-resident).
`python tools/slice_bw.py` -> one line per case: us per launch, achieved GB/s
(algorithmic bytes: 16 B read + 16 B written per complex point and field, plus the
stage programs' extra operands), fraction of MEASURED_PEAKS HBM."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2403_02816_b200 import _lib, ozaki, workloads as W  # noqa: E402

lib = _lib.load()
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
hbm = peaks.get("hbm_gbs", peaks.get("hbm_copy_gbs", 6540.5))
n = 256
shape = (n, n, n)
N = n ** 3
g = torch.Generator(device="cuda").manual_seed(1)
F = [0.3 * torch.randn(shape, dtype=torch.complex128, device="cuda", generator=g) for _ in range(4)]
out = torch.empty_like(F[0])
flag = _lib.new_flag(0)
prob = W.build_problem(W.CONFIGS["C2"])
nl = prob._nl


def buf(rows, K, batch=1):
    per = lib.cgl_oz_slice_bytes(ozaki.S, rows, K, 0)
    return (torch.zeros(per * batch, dtype=torch.int8, device="cuda"),
            torch.empty(rows * batch, dtype=torch.int32, device="cuda"), per)


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


cases = []
# last axis: rows = n*n, K = n (contiguous)
b_last = buf(n * n, n)
cases.append(("slice last axis (1 field)", 32 * N, lambda: _lib.check(lib.cgl_oz_slice_multi(
    _lib.stream(), ozaki.S, 1, _lib.ptr_array(F[:1]), n, 1, n * n, n, 1, 0, 0, _lib.ptr_array([b_last[0]]), 0,
    _lib.ptr_array([b_last[1]]), 0), "s")))
# middle axis: batch n slabs of (n x n): element (r = q, k) at k*n + r
b_mid = buf(n, n, n)
cases.append(("slice middle axis (1 field)", 32 * N, lambda: _lib.check(lib.cgl_oz_slice_multi(
    _lib.stream(), ozaki.S, 1, _lib.ptr_array(F[:1]), 1, n, n, n, n, n * n, 0, _lib.ptr_array([b_mid[0]]),
    b_mid[2], _lib.ptr_array([b_mid[1]]), n), "s")))
# first axis: rows = n*n (q), K = n, element (q, k) at k*n*n + q
b_first = buf(n * n, n)
cases.append(("slice first axis (1 field)", 32 * N, lambda: _lib.check(lib.cgl_oz_slice_multi(
    _lib.stream(), ozaki.S, 1, _lib.ptr_array(F[:1]), 1, n * n, n * n, n, 1, 0, 0, _lib.ptr_array([b_first[0]]), 0,
    _lib.ptr_array([b_first[1]]), 0), "s")))
slots = [buf(n * n, n) for _ in range(3)]


def stage(prog, nin, nsl, fp):
    return lambda: _lib.check(lib.cgl_stage_slice(
        _lib.stream(), _lib.STAGE[prog], n, n * n, _lib.ctypes.byref(nl), 0.01, 1.0, _lib.ptr_array(F[:nin]),
        _lib.ptr_array([out]) if fp else None, _lib.flag_ptr(flag), _lib.rel_pos(1),
        _lib.ptr_array([t[0] for t in slots[:nsl]]), _lib.ptr_array([t[1] for t in slots[:nsl]])), "ss")


for prog, nin, nsl, fp in (("if4_mid", 2, 2, 0), ("if4_end", 4, 3, 1), ("split4_mid", 2, 1, 1),
                           ("split4_end", 2, 2, 1)):
    cases.append((f"stage+slice {prog}", 16 * N * (nin + nsl + fp), stage(prog, nin, nsl, fp)))

for name, nbytes, fn in cases:
    us = timeit(fn)
    gbs = nbytes / (us * 1e-6) / 1e9
    print(json.dumps({"case": name, "us": round(us, 1), "GB_per_s": round(gbs), "frac_hbm": round(gbs / hbm, 3)}),
          flush=True)
