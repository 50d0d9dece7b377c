"""Projected per-rank step time of the slab-sharded FD path at P ranks, on ONE
GPU (the driver's pool has no multi-GPU box): the rank-local work of rank 0
of a P-way axis-0 split of C4 (1024^3, if4, quad form) -- its slab's stage
kernels and local-axis products, the pack/unpack kernels, the axis-0 products
on its (n0 x m) column block -- with each NCCL all-to-all replaced by a
device copy of the same buffer (loopback).  The exchange itself is modelled
separately: per rank and transpose 16 N (P-1)/P^2 bytes over NVLink 5 at
900 GB/s per direction, once per transpose (2 per Tucker per field),
optionally overlapped with the products (tucker_sharded_oz).

    python tools/project_sharded.py [P ...] [--steps S]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

from paper_2403_02816_b200 import SCHEMES, distributed as D, workloads as W  # noqa: E402

NVLINK_GBS = 900.0


class LoopbackTransposer(D.Transposer):
    """All-to-all replaced by a same-size device copy (rank-local projection)."""

    def _a2a(self, out, inp, async_op=False):
        out.view(-1).copy_(inp.reshape(-1))
        return None


def main():
    argv = sys.argv[1:]
    steps = 4
    if "--steps" in argv:
        i = argv.index("--steps")
        steps = int(argv[i + 1])
        argv = argv[:i] + argv[i + 2:]
    ranks = [int(a) for a in argv if a.isdigit()] or [1, 4, 8]
    if len(ranks) > 1:
        # one process per rank count: every case gets the whole HBM
        import subprocess
        recs = []
        for P in ranks:
            res = subprocess.run([sys.executable, __file__, str(P), "--steps", str(steps)], capture_output=True,
                                 text=True)
            print(res.stdout, end="", flush=True)
            if res.returncode:
                print(json.dumps(dict(P=P, error=res.stderr.strip().splitlines()[-1:])), flush=True)
                continue
            recs.append(json.loads(res.stdout.strip().splitlines()[-1]))
        base = next((r["local_ms_per_step"] for r in recs if r["P"] == 1), None)
        if base:
            print(json.dumps({"summary": [dict(P=r["P"], speedup_serial=base / r["projected_ms_serial"],
                                               speedup_pipelined=base / r["projected_ms_pipelined"],
                                               speedup_overlapped=base / r["projected_ms_overlapped"],
                                               projected_ms_pipelined=r["projected_ms_pipelined"])
                                          for r in recs]}))
        return
    w = W.CONFIGS["C4"]
    n0, n1, n2 = w.extents
    out = []
    import paper_2403_02816_b200 as PK
    for P in ranks:
        if P == 1:
            # baseline: the single-GPU fused plan (lean 1024^3 buffers)
            prob = W.build_problem(w)
            u0 = W.initial_state_device(w)
            r = PK.integrate(prob, "if4", (u0,), w.tau * steps, steps)
            rec = dict(P=1, local_ms_per_step=r.device_seconds / steps * 1e3, comm_ms_per_step=0.0)
            rec["projected_ms_serial"] = rec["projected_ms_overlapped"] = rec["local_ms_per_step"]
            rec["projected_ms_pipelined"] = rec["local_ms_per_step"]
            print(json.dumps(rec), flush=True)
            out.append(rec)
            del prob, u0, r
            torch.cuda.empty_cache()
            continue
        L = D.SlabLayout(w.extents, P)
        prob = W.build_problem(w)
        u0 = W.initial_state_device(w)[: L.p0].contiguous()
        prob.prepare(w.tau, SCHEMES["if4"])
        plan = D.ShardedPlan(prob, "if4", [u0], L, None)
        plan.tr = LoopbackTransposer(L, None, device=u0.device, nbuf=2)
        plan.run([u0], 1, w.tau)  # warm (slicing workspaces, factors)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.run([u0], steps, w.tau)
        e1.record()
        torch.cuda.synchronize()
        local_ms = e0.elapsed_time(e1) / steps
        # quad if4: 2 Tucker groups x 2 fields per step, 2 transposes per field chain
        transposes = 2 * 2 * 2
        bytes_per = 16 * n0 * n1 * n2 * (P - 1) / P ** 2
        t_one = bytes_per / (NVLINK_GBS * 1e9) * 1e3
        comm_ms = transposes * t_one
        # tucker_sharded_oz: per group only the first field's slab->column
        # exchange has nothing to overlap with (the others run under products)
        exposed_ms = 2 * t_one
        rec = dict(P=P, local_ms_per_step=local_ms, comm_ms_per_step=comm_ms,
                   projected_ms_serial=local_ms + comm_ms, projected_ms_pipelined=local_ms + exposed_ms,
                   projected_ms_overlapped=max(local_ms, comm_ms),
                   slab=list(L.local_shape()), bytes_per_transpose=bytes_per)
        print(json.dumps(rec), flush=True)
        out.append(rec)
        del plan, prob, u0
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
