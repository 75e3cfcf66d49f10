"""Stratified sampling and estimators on the GPU (reference: pkg/src/ogcp/sampling.py).

``draw_samples`` runs the K1 sampler (csrc/sampler.cu): the same keyed PCG64
stream as the reference (``rng_at``), so the drawn nonzero ordinals and zero
coordinates are bit-identical to ``numpy``'s.  ``estimate_objective`` runs the
K6 objective kernel (+ Gram-based history and regularizers) on the device.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .exceptions import DataError, SamplingError
from .losses import LossFunction
from .tensor import DeviceModel, SparseTensor

# Phase tags for rng_at keys (sampling.py:27-36).
PHASE_INIT = 0
PHASE_WEIGHT_GRAD = 1
PHASE_WEIGHT_OBJ = 2
PHASE_FACTOR_GRAD = 3
PHASE_FACTOR_OBJ = 4
PHASE_WINDOW = 5
PHASE_METRICS = 6
PHASE_STATIC_GRAD = 7
PHASE_STATIC_OBJ = 8
PHASE_RESTART_EVAL = 9


class RngKey:
    """A keyed generator handle, ``rng_at(seed, *key)`` (sampling.py:39-42).

    The engine derives the PCG64 stream from (seed, key) itself; host-side
    scalar draws (reservoir window) use the engine's host restatement.  Every
    draw replays the keyed stream from its start, so a handle serves exactly one
    draw (the reference makes a fresh rng_at per draw: sampling.py:39-42,
    solvers.py:227-345, streaming.py:51); a second use raises instead of
    silently repeating the first draw's values."""

    def __init__(self, seed: int, key: tuple):
        self.seed = int(seed)
        self.key = tuple(int(k) for k in key)
        self._used = False

    def _consume(self):
        if self._used:
            raise SamplingError(f"{self!r} was already drawn from; keyed streams replay from their start, "
                                "so make a fresh rng_at(seed, *key) for every draw")
        self._used = True

    def integers(self, low, high=None, size=None):
        self._consume()
        if high is None:
            low, high = 0, low
        if size is None:
            return int(low + _lib.rng_integers(self.seed, self.key, [high - low], 1)[0])
        n = int(np.prod(size))
        return low + _lib.rng_integers(self.seed, self.key, [high - low], n).reshape(size)

    def __repr__(self):
        return f"rng_at({self.seed}, *{self.key})"


def rng_at(seed: int, *key: int) -> RngKey:
    return RngKey(seed, key)


@dataclass(frozen=True)
class SamplerConfig:
    """Stratified draw counts; ``None`` nonzero counts mean "all of eta" (sampling.py:45-68)."""

    grad_nonzeros: Optional[int] = 1000
    grad_zeros: int = 1000
    obj_nonzeros: Optional[int] = 10000
    obj_zeros: int = 10000
    seed: int = 0
    max_rejects: Optional[int] = None
    # Extension (not in the reference): semi-stratified estimator --
    # q cells drawn uniformly from the whole box (no rejection), nonzero draws
    # corrected by -g(0, m).  See oracle/ogcp_oracle.py draw_semi for the restatement.
    semi_stratified: bool = False

    def __post_init__(self):
        for name in ("grad_nonzeros", "grad_zeros", "obj_nonzeros", "obj_zeros"):
            v = getattr(self, name)
            if v is not None and v < 0:
                raise DataError(f"{name} must be >= 0, got {v}")
        if self.max_rejects is not None and self.max_rejects <= 0:
            raise DataError("max_rejects must be positive")

    def gradient_counts(self, X: SparseTensor) -> tuple:
        return resolve_counts(self.grad_nonzeros, self.grad_zeros, X)

    def objective_counts(self, X: SparseTensor) -> tuple:
        return resolve_counts(self.obj_nonzeros, self.obj_zeros, X)

    def _c(self):
        neg = lambda v: -1 if v is None else int(v)
        return _lib.SamplerC(neg(self.grad_nonzeros), int(self.grad_zeros), neg(self.obj_nonzeros),
                             int(self.obj_zeros), int(self.seed), neg(self.max_rejects),
                             int(bool(self.semi_stratified)))


def resolve_counts(nonzeros: Optional[int], zeros: int, X: SparseTensor) -> tuple:
    """Concrete (p, q) for one slice: None -> eta, empty slice -> p = 0 (sampling.py:71-77)."""
    p = X.nnz if nonzeros is None else int(nonzeros)
    if X.nnz == 0:
        p = 0
    return p, int(zeros)


class SampleSet:
    """One stratified draw held on the device (sampling.py:80-105)."""

    def __init__(self, X: SparseTensor, ordinals, zero_subs):
        self._X = X
        self.ord_dev = ordinals      # torch int32 [p]
        self.zero_dev = zero_subs    # torch int32 [q, d]
        self.eta = X.nnz
        self.omega = X.num_cells

    @property
    def p(self) -> int:
        return int(self.ord_dev.shape[0])

    @property
    def q(self) -> int:
        return int(self.zero_dev.shape[0])

    @property
    def nz_scale(self) -> float:
        return self.eta / self.p if self.p else 0.0

    @property
    def zero_scale(self) -> float:
        return (self.omega - self.eta) / self.q if self.q else 0.0

    @property
    def nz_ordinals(self) -> np.ndarray:
        return self.ord_dev.cpu().numpy().astype(np.int64)

    @property
    def nz_subs0(self) -> np.ndarray:
        return self._X.subs0[self.nz_ordinals]

    @property
    def nz_vals(self) -> np.ndarray:
        return self._X.vals[self.nz_ordinals]

    @property
    def zero_subs0(self) -> np.ndarray:
        return self.zero_dev.cpu().numpy().astype(np.int64).reshape(-1, self._X.ndim)


def _key_of(rng) -> RngKey:
    if isinstance(rng, RngKey):
        rng._consume()
        return rng
    raise TypeError("pass a generator made by rng_at(seed, *key); the engine replays that keyed stream")


def draw_samples(X: SparseTensor, p: int, q: int, rng, max_rejects: Optional[int] = None,
                 semi_stratified: bool = False) -> SampleSet:
    """Draw p nonzeros and q zeros uniformly with replacement (sampling.py:108-153).

    semi_stratified (extension): the q cells are drawn uniformly from the whole box
    without rejection (oracle/ogcp_oracle.py draw_semi)."""
    import torch
    k = _key_of(rng)
    ords = torch.empty(max(int(p), 0), dtype=torch.int32, device="cuda")
    zs = torch.empty((max(int(q), 0), X.ndim), dtype=torch.int32, device="cuda")
    key, kp = _lib.i64arr(list(k.key) or [0])
    _lib.check(_lib.lib().ogcp_draw_samples_ex(_lib.ctx(), X._handle, k.seed, kp, len(k.key), int(p), int(q),
                                                -1 if max_rejects is None else int(max_rejects),
                                                1 if semi_stratified else 0,
                                                C.c_void_p(ords.data_ptr() if p else None),
                                                C.c_void_p(zs.data_ptr() if q else None)))
    s = SampleSet(X, ords, zs)
    s.semi_stratified = bool(semi_stratified)
    return s


def sampled_gradient_tensor(X: SparseTensor, factors: Sequence[np.ndarray], weights: np.ndarray,
                            loss: LossFunction, p: int, q: int, rng, max_rejects: Optional[int] = None
                            ) -> SparseTensor:
    """Sparse stratified approximation of the dense gradient tensor Y (sampling.py:209-239).

    Draws on the GPU sampler (bit-exact), evaluates scale * f'(x, m) per draw in fp64 and
    merges repeated coordinates exactly like np.unique + np.bincount (parity form; the
    solves never materialise Y)."""
    import torch
    s = draw_samples(X, p, q, rng, max_rejects)
    n = s.p + s.q
    d = X.ndim
    model = factors if isinstance(factors, DeviceModel) else DeviceModel.from_numpy(factors)
    coords = torch.empty((max(n, 1), d), dtype=torch.int32, device="cuda")
    vals = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
    w, wp = _lib.f64arr(weights)
    nu = C.c_int64(0)
    _lib.check(_lib.lib().ogcp_gradient_tensor(
        _lib.ctx(), X._handle, C.c_void_p(s.ord_dev.data_ptr() if s.p else None), s.p,
        C.c_void_p(s.zero_dev.data_ptr() if s.q else None), s.q, C.byref(model.c()), wp, C.byref(loss._c()),
        C.c_void_p(coords.data_ptr()), C.c_void_p(vals.data_ptr()), C.byref(nu)))
    k = int(nu.value)
    return SparseTensor.from_zero_based(X.dims, coords[:k].cpu().numpy().astype(np.int64),
                                        vals[:k].cpu().numpy(), allow_zero_values=True)


def segment_layout(Y: SparseTensor, mode: int) -> tuple:
    """(perm, offsets) of mode ``mode``: the stable argsort of Y's mode coordinates and the
    row offsets (cumsum of bincount) that a sort-by-row MTTKRP walks."""
    import torch
    coords = torch.from_numpy(np.ascontiguousarray(Y.subs0, dtype=np.int32)).cuda()
    n = Y.nnz
    dim = Y.dims[mode]
    perm = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    offs = torch.empty(dim + 1, dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().ogcp_segment_layout(_lib.ctx(), C.c_void_p(coords.data_ptr()), n, Y.ndim, int(mode), dim,
                                               C.c_void_p(perm.data_ptr()), C.c_void_p(offs.data_ptr())))
    return perm[:n].cpu().numpy().astype(np.int64), offs.cpu().numpy()


def _window_arrays(window, rank):
    ids = np.array([int(h) for h, _ in window] or [0], dtype=np.int64)
    ws = np.vstack([np.asarray(s, dtype=np.float64) for _, s in window]) if len(window) \
        else np.zeros((1, rank))
    return np.ascontiguousarray(ids), np.ascontiguousarray(ws)


def estimate_objective(X: SparseTensor, factors: Sequence[np.ndarray], weights: np.ndarray, loss: LossFunction,
                       samples: SampleSet, *, old_factors: Optional[Sequence[np.ndarray]] = None,
                       window: Sequence = (), hist_weight: float = 0.0, hist_decay: float = 1.0, t: int = 0,
                       reg_factors: float = 0.0, reg_weights: float = 0.0) -> float:
    """Stratified estimate of the streaming objective (sampling.py:177-206)."""
    if hist_weight and len(window) and old_factors is None:
        raise DataError("history terms require the previous-step factors")
    M = factors if isinstance(factors, DeviceModel) else DeviceModel.from_numpy(factors)
    O = None
    if old_factors is not None:
        O = old_factors if isinstance(old_factors, DeviceModel) else DeviceModel.from_numpy(old_factors)
    w, wp = _lib.f64arr(weights)
    ids, ws = _window_arrays(window, M.rank)
    out = C.c_double()
    op = O.ptrs() if O is not None else None
    _lib.check(_lib.lib().ogcp_estimate_objective(
        _lib.ctx(), X._handle, C.c_void_p(samples.ord_dev.data_ptr() if samples.p else None), samples.p,
        C.c_void_p(samples.zero_dev.data_ptr() if samples.q else None), samples.q, C.byref(M.c()),
        C.cast(op, C.POINTER(C.c_void_p)) if op is not None else None, wp, C.byref(loss._c()),
        ws.ctypes.data_as(_lib.c_f64p), ids.ctypes.data_as(_lib.c_i64p), len(window), float(hist_weight),
        float(hist_decay), int(t), float(reg_factors), float(reg_weights), C.byref(out)))
    return float(out.value)

