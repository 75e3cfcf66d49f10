"""Loss family selection (reference: pkg/src/ogcp/losses.py:24-82).

The loss value and derivative are evaluated inside the fused sample kernels
(csrc/compute.cu: dloss/floss); this module carries the choice of loss, its
epsilon and lower bound across the C ABI.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .exceptions import DataError

KINDS = ("gaussian", "poisson", "bernoulli")


@dataclass(frozen=True)
class LossFunction:
    """One member of the GCP loss family (losses.py:27-43)."""

    kind: str
    eps: float = 1e-10

    def __post_init__(self):
        if self.kind not in KINDS:
            raise DataError(f"unknown loss {self.kind!r}; choose from {KINDS}")
        if not self.eps > 0:
            raise DataError("eps must be positive")

    @property
    def lower_bound(self) -> float:
        """Lower bound for factor/weight entries: 0 unless gaussian (losses.py:40-43)."""
        return -np.inf if self.kind == "gaussian" else 0.0

    def _c(self):
        from ._lib import LOSS_KINDS, LossC
        return LossC(LOSS_KINDS[self.kind], float(self.eps))


def make_loss(kind: str, eps: float = 1e-10) -> LossFunction:
    return LossFunction(kind=kind, eps=eps)
