"""Baseline infrastructure: numpy planted-model slice generator for the reference arm.

NOT part of the product.  bench.py's ``--impl reference`` leg builds the c3/c4
slice with this module so that arm imports neither ``paper_2110_14514_b200``
nor any repo shared object.  Same recipe as the product-side GPU generator
(paper_2110_14514_b200/synthetic.py, itself following gen_poisson,
/root/reference/pkg/src/ogcp/synthetic.py:80-171): the planted factors and
mixture come from the same numpy seed (bit-identical), events pick a component
by the mixture and one coordinate per mode from that component's column
distribution, cells are merged with their counts as values and a random
``nnz`` of the distinct cells kept (ascending linear order).  The event draws use numpy's Generator instead of
torch's CUDA generator, so the slice is statistically identical to the GPU
arm's, not bit-identical.

Per-mode coordinates are drawn by counts (one multinomial per component over
the rows, expanded in row order) and randomly permuted within the component:
the same law as inverse-CDF draws, without a 1e8-query binary search.
"""

from __future__ import annotations

import numpy as np


def planted_factors(dims, rank, seed, boost=25.0, frac=0.08):
    """_dominant_stochastic_factors (synthetic.py:80-94) + mixture weights (:111-112)."""
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


def _events(rng, n, factors, mix, strides):
    comp_counts = rng.multinomial(n, mix)
    lin = np.zeros(n, dtype=np.int64)
    for k, a in enumerate(factors):
        off = 0
        for j, cj in enumerate(comp_counts):
            if cj == 0:
                continue
            p = a[:, j] / a[:, j].sum()
            rows = np.repeat(np.arange(a.shape[0], dtype=np.int64), rng.multinomial(cj, p))
            rng.shuffle(rows)
            lin[off:off + cj] += rows * strides[k]
            off += cj
    return lin, int(n)


def gen_slice_np(dims, nnz, rank, kind="poisson", seed=42):
    """Return (subs0 int32[nnz, d] in ascending linear order, vals f64[nnz], factors, mix, events)."""
    dims = tuple(int(d) for d in dims)
    factors, mix = planted_factors(dims, rank, seed)
    rng = np.random.default_rng(int(seed) * 7919 + 17)
    d = len(dims)
    strides = np.ones(d, dtype=np.int64)
    for k in range(d - 2, -1, -1):
        strides[k] = strides[k + 1] * dims[k + 1]
    keys, total = [], 0
    n_events = int(nnz * 1.05) + 1024
    uniq = counts = None
    for _ in range(10):
        lin, n = _events(rng, n_events, factors, mix, strides)
        keys.append(lin)
        total += n
        uniq, counts = np.unique(np.concatenate(keys), return_counts=True)
        if uniq.size >= nnz:
            break
        n_events = int((nnz - uniq.size) * 1.2) + 1024
    if uniq.size > nnz:
        keep = np.sort(rng.choice(uniq.size, size=nnz, replace=False))
        uniq, counts = uniq[keep], counts[keep]
    subs = np.empty((uniq.size, d), dtype=np.int64)
    rem = uniq
    for k in range(d):
        subs[:, k] = rem // strides[k]
        rem = rem % strides[k]
    vals = counts.astype(np.float64) if kind == "poisson" else np.ones(uniq.size)
    return subs, vals, factors, mix, total
