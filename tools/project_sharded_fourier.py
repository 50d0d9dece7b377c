"""Projected per-rank step time of the slab-sharded Fourier path (the bench
headline C3: 512^3, if4) at P ranks, on ONE GPU: the rank-local work of rank 0
of a P-way axis-0 split -- column passes, pack / unpack kernels, slab passes
with the fused g pass, column-block stage kernels -- with each all-to-all
replaced by a device copy of the same buffer.  The exchange is modelled
separately: per rank and 3D transform 16 N (P-1)/P^2 bytes over NVLink 5 at
900 GB/s per direction, 8 transforms per if4 step (nothing overlaps them in
the current plan).

    python tools/project_sharded_fourier.py [P ...] [--steps S] [--cufft]

--cufft: the round-1 form of the local transforms (batched cuFFT plans + a
separate g kernel) for comparison.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

from paper_2403_02816_b200 import SCHEMES, _lib, slabfourier as SF, workloads as W  # noqa: E402

NVLINK_GBS = 900.0


class LoopbackExchange(SF.SlabExchange):
    """Pack / unpack kernels as at P > 1, the all-to-all a same-size device copy."""

    def __init__(self, shape, P):
        super().__init__(shape, P, [0], group=None)
        self.virtual = False
        self.send = torch.empty((P, self.p0, self.m), dtype=torch.complex128, device="cuda")
        self.recv = torch.empty((P, self.p0, self.m), dtype=torch.complex128, device="cuda")

    def to_cols(self, slabs, cols):
        P, p0, m = self.P, self.p0, self.m
        _lib.check(_lib.load().cgl_slab_pack(_lib.stream(), P, p0, m, _lib.ptr(slabs[0]), _lib.ptr(self.send)), "pack")
        cols[0].view(-1).copy_(self.send.view(-1))
        return cols

    def to_slabs(self, cols, slabs):
        P, p0, m = self.P, self.p0, self.m
        self.recv.view(-1).copy_(cols[0].reshape(-1))
        _lib.check(_lib.load().cgl_slab_unpack(_lib.stream(), P, p0, m, _lib.ptr(self.recv), _lib.ptr(slabs[0])),
                   "unpack")
        return slabs


def main():
    argv = sys.argv[1:]
    steps = 10
    if "--steps" in argv:
        i = argv.index("--steps")
        steps = int(argv[i + 1])
        argv = argv[:i] + argv[i + 2:]
    cufft = "--cufft" in argv
    ranks = [int(a) for a in argv if a.isdigit()] or [1, 2, 4, 8]
    w = W.CONFIGS["C3"]
    n = w.points
    out = []
    for P in ranks:
        prob = W.build_problem(w)
        prob.prepare(w.tau, SCHEMES["if4"])
        plan = SF.ShardedFourierPlan(prob, "if4", w.extents, P, [0], None)
        plan.ex = LoopbackExchange(w.extents, P)
        plan.fft.ex = plan.ex
        if cufft:
            n0, n1, n2 = w.extents
            plan.fft.pencil = False
            plan.fft.f2 = SF.FftMany((n1, n2), plan.ex.p0, 1, n1 * n2)
            plan.fft.f1 = SF.FftMany((n0,), plan.ex.m, plan.ex.m, 1)
        g = torch.Generator(device="cuda").manual_seed(0)
        x = torch.empty((w.extents[0], plan.ex.m), dtype=torch.complex128, device="cuda")
        x.real.normal_(generator=g)
        x.imag.normal_(generator=g)
        x *= 1e-3   # small coefficients: the run must not diverge
        plan.run([x], 2, w.tau)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        key = plan.run([x], steps, w.tau)
        e1.record()
        torch.cuda.synchronize()
        local_ms = e0.elapsed_time(e1) / steps
        bytes_per = 16.0 * n * (P - 1) / P ** 2
        comm_ms = 8 * bytes_per / (NVLINK_GBS * 1e9) * 1e3
        rec = dict(P=P, pencil=bool(plan.fft.pencil), diverged=key != (1 << 64) - 1, local_ms_per_step=local_ms,
                   comm_ms_per_step=comm_ms, projected_ms_serial=local_ms + comm_ms,
                   bytes_per_exchange=bytes_per)
        print(json.dumps(rec), flush=True)
        out.append(rec)
        del plan, prob, x
        torch.cuda.empty_cache()
    base = next((r["projected_ms_serial"] for r in out if r["P"] == 1), None)
    if base:
        print(json.dumps({"summary": [dict(P=r["P"], speedup_vs_sharded_P1=base / r["projected_ms_serial"])
                                      for r in out]}))


if __name__ == "__main__":
    main()
