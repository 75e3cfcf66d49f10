"""Test infrastructure: numpy restatement of the reference's synthetic generators.

NOT part of the product.  Only tests/ (and scripts that build fixtures) import
this module.  It regenerates, bit for bit, the data tensors of BASELINE configs
c1 and c2 on a box where /root/reference does not exist, so the long-stream
parity tests can run the engine on exactly the reference's input.  Pinned by a
SHA-256 of (subs0, vals) recorded from the reference's own output
(scripts/make_stream_golden.py -> tests/golden/stream_*.npz "data_sha256").

Follows /root/reference/pkg/src/ogcp/synthetic.py:
  gen_gaussian  :49-77   (U(0,1) factors, unit weights, einsum densify, N(0, noise))
  _dominant_stochastic_factors :80-94
  gen_poisson   :97-155  (calibrated event draws, counts as values; the dict merge
                          at :131-132 is restated as np.unique over all rounds)
  _draw_events  :158-171
"""

from __future__ import annotations

import hashlib

import numpy as np

_TINY = 1e-300


def _strides(dims):
    # tensor.py:33-38 -- mode 0 most significant
    out = np.ones(len(dims), dtype=np.int64)
    for k in range(len(dims) - 2, -1, -1):
        out[k] = out[k + 1] * dims[k + 1]
    return out


def gen_gaussian(dims, rank, noise=0.2, seed=0):
    """synthetic.py:49-77.  Returns (subs0 int64[n,d], vals f64[n], truth factors)."""
    dims = tuple(int(d) for d in dims)
    rng = np.random.default_rng(seed)
    factors = [rng.uniform(size=(d, rank)) for d in dims]
    letters = [chr(ord("a") + k) for k in range(len(dims))]
    script = ",".join(f"{c}r" for c in letters) + ",r->" + "".join(letters)
    dense = np.einsum(script, *factors, np.ones(rank))          # KTensor.full, tensor.py:268-279
    if noise > 0:
        dense = dense + rng.normal(0.0, noise, size=dims)
    flat = dense.ravel()
    zero_hits = flat == 0.0
    if zero_hits.any():
        model = np.einsum(script, *factors, np.ones(rank)).ravel()
        flat[zero_hits] = _TINY * np.where(model[zero_hits] < 0, -1.0, 1.0)
    subs0 = np.indices(dims).reshape(len(dims), -1).T
    return np.ascontiguousarray(subs0, dtype=np.int64), flat, factors


def _dominant_factors(rng, dims, rank, boost=25.0, frac=0.08):
    factors = []
    for d in dims:
        a = rng.uniform(0.05, 0.4, size=(d, rank))
        n_dom = max(1, int(np.ceil(frac * d)))
        for j in range(rank):
            dom = rng.choice(d, size=n_dom, replace=False)
            a[dom, j] *= boost
        factors.append(a / a.sum(axis=0, keepdims=True))
    return factors


def _draw_events(rng, n, mix, cdfs, strides):
    comp = rng.choice(mix.size, size=n, p=mix)
    lin = np.zeros(n, dtype=np.int64)
    for k, cdf in enumerate(cdfs):
        u = rng.random(n)
        coords = np.empty(n, dtype=np.int64)
        for j in range(mix.size):
            sel = comp == j
            if sel.any():
                coords[sel] = np.searchsorted(cdf[:, j], u[sel])
        np.minimum(coords, cdf.shape[0] - 1, out=coords)
        lin += coords * strides[k]
    return lin


def gen_poisson(dims, rank, density=0.032, seed=0):
    """synthetic.py:97-155 (density < 1 path).  Returns (subs0, vals, truth factors, truth weights)."""
    dims = tuple(int(d) for d in dims)
    omega = int(np.prod(dims))
    rng = np.random.default_rng(seed)
    factors = _dominant_factors(rng, dims, rank)
    mix = rng.uniform(0.5, 1.5, size=rank)
    mix = mix / mix.sum()
    cdfs = [np.cumsum(a, axis=0) for a in factors]
    strides = _strides(dims)
    n_events = max(1, int(-omega * np.log1p(-density)))
    keys = np.empty(0, np.int64)
    cnts = np.empty(0, np.int64)
    total_events = 0
    target = density * omega
    goal = 0.77 * target
    for _ in range(10):
        lin = _draw_events(rng, n_events, mix, cdfs, strides)
        u, c = np.unique(lin, return_counts=True)
        allk = np.concatenate([keys, u])
        allc = np.concatenate([cnts, c])
        keys, inv = np.unique(allk, return_inverse=True)
        cnts = np.bincount(inv, weights=allc, minlength=keys.size).astype(np.int64)
        total_events += n_events
        achieved = keys.size
        if achieved >= goal or achieved == omega:
            break
        gap = (target - achieved) / max(achieved, 1)
        n_events = max(1, int(total_events * min(gap, 1.0)))
    else:
        raise ValueError("could not reach density")
    vals = cnts.astype(np.float64)
    subs0 = np.empty((keys.size, len(dims)), dtype=np.int64)
    rem = keys.copy()
    for k, s in enumerate(strides):
        subs0[:, k] = rem // s
        rem = rem % s
    return subs0, vals, factors, total_events * mix


def data_sha256(subs0, vals) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(subs0, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(vals, dtype=np.float64).tobytes())
    return h.hexdigest()


def slice_of(subs0, vals, t):
    """slice_view(t) (tensor.py:179-190): 1-based t along the last mode, last coordinate dropped."""
    mask = subs0[:, -1] == t - 1
    return np.ascontiguousarray(subs0[mask, :-1]), np.ascontiguousarray(vals[mask])


def leading(subs0, vals, n):
    """leading_block(X, n) (io.py:165-173)."""
    mask = subs0[:, -1] < n
    return np.ascontiguousarray(subs0[mask]), np.ascontiguousarray(vals[mask])
