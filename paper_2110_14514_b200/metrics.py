"""Per-slice reconstruction losses on the GPU (reference: pkg/src/ogcp/metrics.py).

Exact mode sums f over every cell of the box with the K6 cell kernel plus a
nonzero correction pass; sampled mode is the stratified objective estimate on
the keyed sample set.  Both divide by ||X||^2 like the reference.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .exceptions import DataError


@dataclass
class SliceMetrics:
    """Per-slice diagnostics recorded by the streaming driver (metrics.py:16-25)."""

    t: int
    local_loss_sampled: float
    local_loss_exact: float
    epochs_weights: int
    epochs_factors: int
    wall_ms: float


@dataclass
class LocalLoss:
    """Loss total divided by ||X||_F^2; unnormalized when the slice is empty (metrics.py:28-33)."""

    value: float
    normalized: bool


def local_loss(X, model, loss, *, mode: str = "exact", p: Optional[int] = None, q: Optional[int] = None,
               rng=None, max_rejects: Optional[int] = None, max_elements: int = 50_000_000) -> LocalLoss:
    """Reconstruction loss of one slice against its model (metrics.py:36-70).

    ``model`` is a KTensor, or a (weights, DeviceModel) pair from the driver."""
    from .sampling import RngKey
    from .tensor import DeviceModel, KTensor
    if isinstance(model, KTensor):
        weights, dm = model.weights, DeviceModel.from_numpy(model.factors)
        if X.dims != model.dims:
            raise DataError(f"dims differ: {X.dims} vs {model.dims}")
    else:
        weights, dm = model
        if X.dims != dm.dims:
            raise DataError(f"dims differ: {X.dims} vs {dm.dims}")
    w, wp = _lib.f64arr(weights)
    out = C.c_double()
    norm = C.c_int32()
    if mode == "exact":
        _lib.check(_lib.lib().ogcp_local_loss(_lib.ctx(), X._handle, C.byref(dm.c()), wp, C.byref(loss._c()), 0, 0,
                                               0, 0, None, 0, -1, int(max_elements), C.byref(out), C.byref(norm)))
    elif mode == "sampled":
        if rng is None:
            raise DataError("sampled local loss needs an rng")
        if not isinstance(rng, RngKey):
            raise TypeError("pass a generator made by rng_at(seed, *key)")
        rng._consume()
        key, kp = _lib.i64arr(list(rng.key) or [0])
        _lib.check(_lib.lib().ogcp_local_loss(
            _lib.ctx(), X._handle, C.byref(dm.c()), wp, C.byref(loss._c()), 1, -1 if p is None else int(p),
            0 if q is None else int(q), rng.seed, kp, len(rng.key), -1 if max_rejects is None else int(max_rejects),
            int(max_elements), C.byref(out), C.byref(norm)))
    else:
        raise DataError(f"unknown local loss mode {mode!r}")
    return LocalLoss(float(out.value), bool(norm.value))


def global_loss(slices: Sequence, factors: Sequence[np.ndarray], weights_log: Sequence[np.ndarray], loss) -> float:
    """Average exact local loss of [[s_t; final factors]] over the stream (metrics.py:73-92)."""
    from .tensor import KTensor
    if len(weights_log) < len(slices):
        raise DataError(f"{len(slices)} slices but only {len(weights_log)} weight vectors recorded")
    if not slices:
        raise DataError("global loss over an empty stream is undefined")
    total = 0.0
    for t, X_t in enumerate(slices, start=1):
        total += local_loss(X_t, KTensor(weights_log[t - 1], factors), loss, mode="exact").value
    return total / len(slices)


def congruence_score(M1, M2) -> float:
    """Component-matched similarity of two K-tensors in [-1, 1] (metrics.py:95-148).

    Per-mode cosines come from the GPU Gram kernel (cross Gram over the column
    norms from the self Grams); the norms and signs are absorbed into the
    weights and components are paired greedily by descending signed cosine
    product, as in the reference."""
    from .kernels import gram
    if M1.dims != M2.dims:
        raise DataError(f"dims differ: {M1.dims} vs {M2.dims}")
    R1, R2 = M1.rank, M2.rank
    Rm = max(R1, R2)
    pad = lambda a: np.hstack([a, np.zeros((a.shape[0], Rm - a.shape[1]))])
    lam1, lam2 = np.array(M1.weights, dtype=np.float64), np.array(M2.weights, dtype=np.float64)
    cos = np.ones((R1, R2))
    for a, b in zip(M1.factors, M2.factors):
        A, B = pad(a), pad(b)
        n1 = np.sqrt(np.maximum(np.diag(gram([A])), 0.0))[:R1]
        n2 = np.sqrt(np.maximum(np.diag(gram([B])), 0.0))[:R2]
        cross = gram([B], other_factors=[A])[:R1, :R2]
        cos *= cross / np.outer(np.where(n1 > 0, n1, 1.0), np.where(n2 > 0, n2, 1.0))
        lam1, lam2 = lam1 * n1, lam2 * n2
    cos *= np.where(lam1 < 0, -1.0, 1.0)[:, None] * np.where(lam2 < 0, -1.0, 1.0)[None, :]
    lam1, lam2 = np.abs(lam1), np.abs(lam2)
    n_pairs = min(R1, R2)
    masked, total = cos.copy(), 0.0
    for _ in range(n_pairs):
        i, j = np.unravel_index(np.argmax(masked), masked.shape)
        top = max(lam1[i], lam2[j])
        if top > 0:
            total += (1.0 - abs(lam1[i] - lam2[j]) / top) * cos[i, j]
        masked[i, :] = -np.inf
        masked[:, j] = -np.inf
    return total / n_pairs
