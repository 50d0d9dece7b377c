"""Validate + time the INT8-tensor-core emulated complex GEMM (ozgemm) against
torch complex128 matmul.  `python tools/oz_check.py [S]`."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_02816_b200 import _lib  # noqa: E402

lib = _lib.load()
S = int(sys.argv[1]) if len(sys.argv) > 1 else 8


def slices(Z, rows, cols, sr, sc, a_mode, S, batch=1, bs=0):
    nb = lib.cgl_oz_slice_bytes(S, rows, cols, a_mode)
    out = torch.zeros(batch * nb, dtype=torch.int8, device="cuda")
    ex = torch.zeros(batch * rows, dtype=torch.int32, device="cuda")
    _lib.check(lib.cgl_oz_slice(_lib.stream(), S, _lib.ptr(Z), sr, sc, rows, cols, batch, bs, a_mode, _lib.ptr(out),
                                nb, _lib.ptr(ex), rows), "oz_slice")
    return out, ex, nb


def zmap(sl, rows, cols, a_mode, S):
    from paper_2403_02816_b200 import ozaki
    z = torch.zeros(ozaki._zmap_len(rows, cols, a_mode), dtype=torch.int8, device="cuda")
    _lib.check(lib.cgl_oz_zmap(_lib.stream(), S, _lib.ptr(sl), rows, cols, a_mode, _lib.ptr(z)), "zmap")
    return z


def run(A, B, S, nitems=1, reps=0, sparse_a=False, sparse_b=False):
    M, K = A.shape
    N = B.shape[1]
    As, Ae, _ = slices(A, M, K, K, 1, 1, S)
    Bs, Be, _ = slices(B, N, K, 1, N, 0, S)   # Z = B^T: Z(r=j, c=k) = B[k, j] at k*N + j
    Az = zmap(As, M, K, 1, S) if sparse_a else None
    Bz = zmap(Bs, N, K, 0, S) if sparse_b else None
    Cs = [torch.empty(M, N, dtype=torch.complex128, device="cuda") for _ in range(nitems)]

    def go():
        _lib.check(lib.cgl_oz_gemm(_lib.stream(), S, M, N, K, nitems, _lib.ptr_array([As] * nitems),
                                   _lib.ptr_array([Ae] * nitems), _lib.ptr_array([Az] * nitems) if Az is not None
                                   else None, _lib.ptr_array([Bs] * nitems), _lib.ptr_array([Be] * nitems),
                                   _lib.ptr_array([Bz] * nitems) if Bz is not None else None,
                                   _lib.ptr_array(Cs), N, 1, 0, 0, 0, 0, 0, None, 0),
                   "oz_gemm")
    go()
    torch.cuda.synchronize()
    dt = None
    if reps:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            go()
        e1.record()
        torch.cuda.synchronize()
        dt = e0.elapsed_time(e1) / 1e3 / reps
    return Cs[0], dt


g = torch.Generator(device="cuda").manual_seed(0)
# 1. mechanics: small integers, S = 1 is exact
for (M, K, N) in [(64, 32, 64), (100, 70, 90), (512, 512, 512)]:
    A = torch.complex(torch.randint(-100, 101, (M, K), generator=g, device="cuda").double(),
                      torch.randint(-100, 101, (M, K), generator=g, device="cuda").double())
    B = torch.complex(torch.randint(-100, 101, (K, N), generator=g, device="cuda").double(),
                      torch.randint(-100, 101, (K, N), generator=g, device="cuda").double())
    A[:, 0] = 127 + 0j
    B[0, :] = 127 + 0j
    C, _ = run(A, B, 1)
    want = A @ B
    print(json.dumps({"case": "int-exact S=1", "shape": [M, K, N],
                      "max_abs_err": (C - want).abs().max().item()}), flush=True)
# 2. accuracy + speed with random doubles
for (M, K, N, nf) in [(512, 512, 512, 1), (512, 512, 512, 4), (256, 256, 65536, 1)]:
    A = torch.randn(M, K, dtype=torch.complex128, device="cuda", generator=g)
    B = torch.randn(K, N, dtype=torch.complex128, device="cuda", generator=g)
    C, dt = run(A, B, S, nitems=nf, reps=10)
    want = A @ B
    err = ((C - want).abs().max() / want.abs().max()).item()
    print(json.dumps({"case": f"random S={S}", "shape": [M, K, N], "fields": nf, "rel_max_err": err,
                      "us": dt * 1e6, "equiv_tflops": 8.0 * M * K * N * nf / dt / 1e12}), flush=True)

# 3. the C1 exponential factor (banded in the sliced representation): left and right forms
from paper_2403_02816_b200 import workloads as W  # noqa: E402
w = W.CONFIGS["C1"]
op = W.build_problem(w).operator
op.prepare(w.tau, (0.5, 1))
E = op.exp_factors(1)[0][0]
U = torch.randn(512, 512, dtype=torch.complex128, device="cuda", generator=g)
for nf in (1, 4):
    C, dt = run(E, U, S, nitems=nf, reps=10, sparse_a=True)
    want = E @ U
    err = ((C - want).abs().max() / want.abs().max()).item()
    print(json.dumps({"case": f"E-left sparse S={S}", "fields": nf, "rel_max_err": err, "us": dt * 1e6,
                      "equiv_tflops": 8.0 * 512 ** 3 * nf / dt / 1e12}), flush=True)
    Et = E.t().contiguous()
    C, dt = run(U, Et, S, nitems=nf, reps=10, sparse_b=True)
    want = U @ Et
    err = ((C - want).abs().max() / want.abs().max()).item()
    print(json.dumps({"case": f"E-right sparse S={S}", "fields": nf, "rel_max_err": err, "us": dt * 1e6,
                      "equiv_tflops": 8.0 * 512 ** 3 * nf / dt / 1e12}), flush=True)
