"""Stream feed over a (d+1)-way tensor (reference: pkg/src/ogcp/io.py:157-173).

Only the slice feed is here: ``stream_slices`` and ``leading_block`` hand
last-mode slices / the warm-start block to the engine, each re-ingested on the
GPU (validation + membership hash, tensor.py).  The reference's FROSTT/TNS text
readers and writers are file IO outside the per-slice hot path.
"""

from __future__ import annotations

from typing import Iterator

from .exceptions import DataError
from .tensor import SparseTensor


def stream_slices(X: SparseTensor) -> Iterator[SparseTensor]:
    """Yield last-mode slices of a (d+1)-way tensor in arrival order."""
    if X.ndim < 2:
        raise DataError("streaming requires a tensor with at least 2 modes")
    for t in range(1, X.dims[-1] + 1):
        yield X.slice_view(t)


def leading_block(X: SparseTensor, n: int) -> SparseTensor:
    """First ``n`` last-mode slices as one tensor (the warm-start block)."""
    if X.ndim < 2:
        raise DataError("a block needs a tensor with at least 2 modes")
    if not 1 <= n <= X.dims[-1]:
        raise DataError(f"block size {n} out of range 1..{X.dims[-1]}")
    mask = X.subs0[:, -1] < n
    return SparseTensor.from_zero_based(X.dims[:-1] + (n,), X.subs0[mask], X.vals[mask])
