"""World-size-2 gloo tests (CPU) for the multi-GPU path's host logic: the sample
partition the engine uses, the linearity that makes a sharded solve exact
(sum of per-shard gradients/objectives over one sample set == the full
quantities, kernels.py:33-72, sampling.py:191-196), and the id broadcast that
bootstraps the engine's NCCL communicator."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ogcp_oracle as O
from paper_2110_14514_b200.distributed import _broadcast_bytes, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # id broadcast (what init_sharded_solves does with the NCCL unique id)
        payload = bytes(range(128)) if rank == 0 else b""
        got = _broadcast_bytes(payload, rank)
        assert got == bytes(range(128))

        rng = np.random.default_rng(4)
        dims = (30, 20, 10)
        lin = rng.choice(int(np.prod(dims)), size=500, replace=False)
        subs0 = np.array(np.unravel_index(lin, dims)).T
        vals = rng.integers(1, 4, size=lin.size).astype(float)
        X = O.Slice(dims, subs0, vals)
        R = 4
        A = [rng.uniform(0.1, 1.0, (d, R)) for d in dims]
        s = rng.uniform(0.5, 1.5, R)
        smp = O.draw(X, 700, 900, O.keyed_rng(3, 7, 3, 0, 0))
        subs = np.concatenate([smp.nz_subs0, smp.zero_subs0])
        x = np.concatenate([smp.nz_vals, np.zeros(smp.q)])
        scale = np.concatenate([np.full(smp.p, smp.nz_scale), np.full(smp.q, smp.zero_scale)])
        y = scale * O.loss_df("poisson", x, O.model_at(A, s, subs))
        f = scale * O.loss_f("poisson", x, O.model_at(A, s, subs))
        lo, hi = shard_range(len(y), rank, world)
        part = [O.mttkrp(subs[lo:hi], y[lo:hi], dims, A, k) * s for k in range(3)]
        gw = O.weight_grad(subs[lo:hi], y[lo:hi], A)
        fo = np.array([f[lo:hi].sum()])
        tensors = [torch.from_numpy(np.ascontiguousarray(t)) for t in part + [gw, fo]]
        for t in tensors:
            dist.all_reduce(t)
        full = [O.mttkrp(subs, y, dims, A, k) * s for k in range(3)] + [O.weight_grad(subs, y, A),
                                                                          np.array([f.sum()])]
        ok = all(np.allclose(t.numpy(), w, rtol=1e-12, atol=1e-12) for t, w in zip(tensors, full))
        out[rank] = 1 if ok else 0
    finally:
        dist.destroy_process_group()


def test_shard_partition_covers_samples():
    for total in (0, 1, 7, 1000, 1 << 24):
        for world in (1, 2, 3, 8):
            ranges = [shard_range(total, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))


def test_sharded_gradient_sum_equals_full_gloo():
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert dict(out) == {0: 1, 1: 1}
