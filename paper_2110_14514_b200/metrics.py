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
