"""World-size-2 gloo tests (CPU) of the slab-sharded path's host logic:
axis-0 transposes, the sharded mode product / Tucker chain, and the
cross-rank divergence-key reduction.  The DMMA kernels are replaced by
torch CPU contractions here (they need a GPU); the data movement, slab
layout and reduction code is the code the GPU path runs."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import REPO

SHAPE = (8, 6, 4)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _global():
    g = torch.Generator().manual_seed(5)
    re = torch.randn(SHAPE, generator=g, dtype=torch.float64)
    im = torch.randn(SHAPE, generator=g, dtype=torch.float64)
    mats = [torch.complex(torch.randn(n, n, generator=g, dtype=torch.float64),
                          torch.randn(n, n, generator=g, dtype=torch.float64)) for n in SHAPE]
    return torch.complex(re, im), mats


def _mode(u, m, axis):
    return torch.movedim(torch.tensordot(m, u, dims=([1], [axis])), 0, axis)


def _worker(rank, world, port, q, tmpdir=None):
    import sys
    sys.path.insert(0, REPO)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2403_02816_b200.distributed import (SlabLayout, Transposer, global_min_key, mode0_sharded,
                                                       tucker_sharded)
        u, mats = _global()
        L = SlabLayout(SHAPE, world)
        a, b = L.bounds(rank)
        local = u[a:b].contiguous()
        tr = Transposer(L)
        res = {}
        cols = tr.to_columns(local).clone()
        flat = u.reshape(SHAPE[0], -1)
        res["cols"] = torch.equal(cols, flat[:, rank * L.m:(rank + 1) * L.m])
        back = torch.empty_like(local)
        tr.from_columns(cols, back)
        res["roundtrip"] = torch.equal(back, local)
        out = torch.empty_like(local)
        mode0_sharded(local, mats[0], None, out, tr, gemm=lambda m, x: m @ x)
        want = _mode(u, mats[0], 0)[a:b]
        res["mode0"] = float((out - want).abs().max() / want.abs().max())
        work = torch.empty_like(local)
        tucker_sharded(local, mats, [None] * 3, out, work, tr, gemm=lambda m, x: m @ x, local=_mode)
        t = u
        for ax, m in enumerate(mats):
            t = _mode(t, m, ax)
        res["tucker"] = float((out - t[a:b]).abs().max() / t.abs().max())
        # divergence keys: rank 1 diverged at (step 3, seq 1), rank 0 clean (all ones)
        flag = torch.zeros(3, dtype=torch.int64)
        flag[0] = -1 if rank == 0 else (3 << 24) | (1 << 8) | 4
        global_min_key(flag)
        res["key"] = int(flag[0].item())
        # both diverged: the earlier (step, seq) wins even against a larger unsigned value
        flag[0] = ((7 << 24) | 5) if rank == 0 else (0x7F << 56)
        global_min_key(flag)
        res["key2"] = int(flag[0].item())
        # slab-sharded Fourier exchange (real ranks): slab -> column block -> slab
        from paper_2403_02816_b200.slabfourier import SlabExchange
        ex = SlabExchange(SHAPE, world, [rank], group=dist.group.WORLD, device="cpu")
        cols = [torch.empty((SHAPE[0], ex.m), dtype=torch.complex128)]
        ex.to_cols([local], cols)
        res["fcols"] = torch.equal(cols[0], flat[:, rank * ex.m:(rank + 1) * ex.m])
        back2 = [torch.empty_like(local)]
        ex.to_slabs(cols, back2)
        res["froundtrip"] = torch.equal(back2[0], local)
        # sharded snapshot: both ranks store their slab into one file concurrently
        from paper_2403_02816_b200 import io as cio
        grids = [np.linspace(0.0, 1.0, n) for n in SHAPE]
        path = os.path.join(tmpdir, "sharded.cgls")
        cio.write_snapshot_sharded(path, [local.numpy()], 0.5, grids, SHAPE, (a, b), rank=rank, barrier=dist.barrier)
        if rank == 0:
            ref = os.path.join(tmpdir, "whole.cgls")
            cio.write_snapshot(ref, [u.numpy()], 0.5, grids)
            res["snapshot"] = open(path, "rb").read() == open(ref, "rb").read()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_slab_sharded_path_gloo(world, tmp_path):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, res in results.items():
        assert res["cols"] and res["roundtrip"], (rank, res)
        assert res["fcols"] and res["froundtrip"], (rank, res)
        assert res["mode0"] <= 1e-14 and res["tucker"] <= 1e-14, (rank, res)
        assert res["key"] == (3 << 24) | (1 << 8) | 4
        assert res["key2"] == (7 << 24) | 5
    assert results[0]["snapshot"]


def test_slab_layout_validation():
    from paper_2403_02816_b200.distributed import SlabLayout
    L = SlabLayout((1024, 1024, 1024), 8)
    assert L.local_shape() == (128, 1024, 1024) and L.m == 131072
    assert L.bounds(3) == (384, 512)
    with pytest.raises(ValueError):
        SlabLayout((10, 4, 4), 4)
