"""Vectorised planted-model slice generator on the GPU (bench/test input only).

Follows the recipe of the reference generator gen_poisson
(pkg/src/ogcp/synthetic.py:80-171): per-mode column distributions with a
boosted minority of entries, a component mixture, per-mode inverse-CDF draws of
event coordinates, and cell counts as values.  The reference's dict loop cannot
reach 1e8 nonzeros per slice, so this version draws events with
torch on the device and merges them with a sort; entries are stored in
ascending linear order like the reference's (synthetic.py:160-165).
"""

from __future__ import annotations

import math

import numpy as np


def planted_factors(dims, rank, seed, boost=25.0, frac=0.08):
    """_dominant_stochastic_factors (synthetic.py:89-103) + mixture weights, host fp64."""
    rng = np.random.default_rng(seed)
    factors = []
    for d in dims:
        a = rng.uniform(0.05, 0.4, size=(d, rank))
        n_dom = max(1, int(np.ceil(frac * d)))
        for j in range(rank):
            dom = rng.choice(d, size=n_dom, replace=False)
            a[dom, j] *= boost
        factors.append(a / a.sum(axis=0, keepdims=True))
    mix = rng.uniform(0.5, 1.5, size=rank)
    return factors, mix / mix.sum()


def gen_slice(dims, nnz, rank, kind="poisson", seed=42, factors=None, mix=None):
    """Return (SparseTensor on the GPU, factors, mixture, total events).

    Draws events from the planted model until at least ``nnz`` distinct cells
    are hit, keeps the ``nnz`` smallest linear keys' cells with their counts
    (Bernoulli: value 1)."""
    import torch
    from .tensor import SparseTensor
    if factors is None:
        factors, mix = planted_factors(dims, rank, seed)
    dev = "cuda"
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed) * 7919 + 17)
    d = len(dims)
    # flattened per-component CDFs: component j occupies [j, j+1)
    cdfs = []
    for a in factors:
        c = np.cumsum(a, axis=0)
        c[-1, :] = 1.0
        flat = (c.T + np.arange(rank)[:, None]).reshape(-1)
        cdfs.append(torch.from_numpy(flat).to(dev))
    mix_t = torch.from_numpy(np.asarray(mix, dtype=np.float64)).to(dev)
    strides = [1] * d
    for k in range(d - 2, -1, -1):
        strides[k] = strides[k + 1] * dims[k + 1]
    keys = []
    total_events = 0
    uniq = None
    n_events = int(nnz * 1.05) + 1024
    for _ in range(10):
        comp = torch.multinomial(mix_t, n_events, replacement=True, generator=g)
        lin = torch.zeros(n_events, dtype=torch.int64, device=dev)
        for k in range(d):
            u = torch.rand(n_events, dtype=torch.float64, device=dev, generator=g)
            pos = torch.searchsorted(cdfs[k], comp.to(torch.float64) + u)
            coord = torch.clamp(pos - comp * dims[k], 0, dims[k] - 1)
            lin += coord * strides[k]
            del u, pos, coord
        del comp
        keys.append(lin)
        total_events += n_events
        allk = torch.cat(keys)
        uniq, counts = torch.unique(allk, return_counts=True)
        del allk
        if uniq.numel() >= nnz:
            break
        n_events = int((nnz - uniq.numel()) * 1.2) + 1024
    if uniq.numel() > nnz:
        keep = torch.randperm(uniq.numel(), generator=g, device=dev)[:nnz].sort().values
        uniq, counts = uniq[keep], counts[keep]
    del keys
    subs = torch.empty((uniq.numel(), d), dtype=torch.int32, device=dev)
    rem = uniq.clone()
    for k in range(d):
        subs[:, k] = (rem // strides[k]).to(torch.int32)
        rem = rem % strides[k]
    vals = counts.to(torch.float32) if kind == "poisson" else torch.ones_like(counts, dtype=torch.float32)
    del rem, uniq, counts
    X = SparseTensor.from_device(tuple(dims), subs, vals)
    return X, factors, mix, total_events
