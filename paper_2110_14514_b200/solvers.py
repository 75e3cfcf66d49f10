"""GCP-SGD subsolvers on the GPU (reference: pkg/src/ogcp/solvers.py).

``solve_weights`` and ``solve_factors`` hand the whole epoch loop to the native
runtime (``ogcp_solve_weights`` / ``ogcp_solve_factors``, csrc/engine.cu): every
iteration (draw -> fused eval/scatter -> Gram history -> fused Adam) is
enqueued on the CUDA stream and the host synchronises once per epoch for the
objective gate.  The numpy-facing signatures are the reference's.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .adam import Adam
from .exceptions import DataError
from .losses import LossFunction
from .sampling import SamplerConfig, _window_arrays
from .tensor import DeviceModel, KTensor, SparseTensor

TEMPORAL_SOLVERS = ("sgd", "least-squares")
GRADIENT_MODES = ("sampled", "dense-gaussian")


@dataclass(frozen=True)
class SolverConfig:
    """Epoch-loop, regularization, history and Adam settings (solvers.py:40-91)."""

    tol_weights: float = 0.0
    tol_factors: float = 0.0
    max_epochs_weights: int = 20
    max_epochs_factors: int = 5
    iters_weights: int = 100
    iters_factors: int = 100
    reg_factors: float = 0.0
    reg_weights: float = 0.0
    hist_weight: float = 0.0
    hist_decay: float = 1.0
    temporal_solver: str = "sgd"
    gradient_mode: str = "sampled"
    warm_start_weights: bool = False
    rate_weights: float = 0.1
    rate_factors: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    rate_decay: float = 0.1
    lower_bound: Optional[float] = None
    samples: SamplerConfig = SamplerConfig()

    def __post_init__(self):
        if self.tol_weights < 0 or self.tol_factors < 0:
            raise DataError("tolerances must be >= 0")
        if min(self.max_epochs_weights, self.max_epochs_factors, self.iters_weights, self.iters_factors) < 1:
            raise DataError("epoch and iteration counts must be >= 1")
        if not 0.0 < self.hist_decay <= 1.0:
            raise DataError("hist_decay must lie in (0, 1]")
        if min(self.reg_factors, self.reg_weights, self.hist_weight) < 0:
            raise DataError("regularization and history weights must be >= 0")
        if self.temporal_solver not in TEMPORAL_SOLVERS:
            raise DataError(f"temporal_solver must be one of {TEMPORAL_SOLVERS}")
        if self.gradient_mode not in GRADIENT_MODES:
            raise DataError(f"gradient_mode must be one of {GRADIENT_MODES}")

    def bound_for(self, loss: LossFunction) -> float:
        return loss.lower_bound if self.lower_bound is None else self.lower_bound

    def make_adam(self, rate: float, loss: LossFunction) -> Adam:
        return Adam(rate, self.beta1, self.beta2, self.adam_eps, self.bound_for(loss), self.rate_decay)

    def _c(self, loss: LossFunction):
        return _lib.SolverC(self.tol_weights, self.tol_factors, self.max_epochs_weights, self.max_epochs_factors,
                            self.iters_weights, self.iters_factors, self.reg_factors, self.reg_weights,
                            self.hist_weight, self.hist_decay, int(bool(self.warm_start_weights)),
                            self.rate_weights, self.rate_factors, self.beta1, self.beta2, self.adam_eps,
                            self.rate_decay, float(self.bound_for(loss)), self.samples._c(),
                            GRADIENT_MODES.index(self.gradient_mode), TEMPORAL_SOLVERS.index(self.temporal_solver))


@dataclass
class EpochTrace:
    """Objective estimates at epoch boundaries; index 0 is the entry value (solvers.py:94-100)."""

    objective: list = field(default_factory=list)
    epochs: int = 0
    rejections: int = 0


@dataclass
class WeightSolve:
    weights: np.ndarray
    trace: EpochTrace


@dataclass
class FactorSolve:
    factors: list
    iteration: int
    trace: EpochTrace


class _Trace:
    def __init__(self, n):
        self.buf = np.zeros(n + 1)
        self.c = _lib.TraceC(self.buf.ctypes.data_as(_lib.c_f64p), 0, 0, 0)

    def result(self):
        return EpochTrace(list(self.buf[: self.c.n_objective]), int(self.c.epochs), int(self.c.rejections))


def _check_gradient_mode(cfg: SolverConfig, loss: LossFunction):
    if cfg.gradient_mode == "dense-gaussian" and loss.kind != "gaussian":
        raise DataError("gradient_mode 'dense-gaussian' requires gaussian loss")


def solve_weights_device(X: SparseTensor, model: DeviceModel, loss: LossFunction, cfg: SolverConfig, t: int,
                         s_init: Optional[np.ndarray]) -> WeightSolve:
    """Temporal-row solve on device-resident factors (engine entry)."""
    _check_gradient_mode(cfg, loss)
    R = model.rank
    s_out = np.zeros(R)
    si = None
    if s_init is not None and cfg.warm_start_weights:
        si = np.ascontiguousarray(np.asarray(s_init, dtype=np.float64))
        if si.shape != (R,):
            raise DataError("s_init must match the model rank")
    tr = _Trace(cfg.max_epochs_weights)
    _lib.check(_lib.lib().ogcp_solve_weights(
        _lib.ctx(), X._handle, C.byref(cfg._c(loss)), C.byref(loss._c()), int(t), C.byref(model.c()),
        si.ctypes.data_as(_lib.c_f64p) if si is not None else None, s_out.ctypes.data_as(_lib.c_f64p),
        C.byref(tr.c)))
    return WeightSolve(s_out, tr.result())


def solve_weights(X: SparseTensor, factors: Sequence[np.ndarray], loss: LossFunction, cfg: SolverConfig,
                  t: int = 0, s_init: Optional[np.ndarray] = None) -> WeightSolve:
    """Temporal-weight GCP-SGD solve with the factors held fixed (solvers.py:197-268)."""
    model = factors if isinstance(factors, DeviceModel) else DeviceModel.from_numpy(factors)
    return solve_weights_device(X, model, loss, cfg, t, s_init)


def solve_factors_device(X: SparseTensor, model: DeviceModel, weights: np.ndarray, old: Optional[DeviceModel],
                         window: Sequence, cfg: SolverConfig, loss: LossFunction, adam: Adam, iteration: int,
                         t: int):
    """Factor solve updating ``model`` in place on the device; returns (iteration, trace)."""
    _check_gradient_mode(cfg, loss)
    if cfg.hist_weight and len(window) and old is None:
        raise DataError("history terms require the previous-step factors")
    w, wp = _lib.f64arr(weights)
    ids, ws = _window_arrays(window, model.rank)
    it = C.c_int64(int(iteration))
    tr = _Trace(cfg.max_epochs_factors)
    st = adam.c()
    op = old.ptrs() if old is not None else None
    _lib.check(_lib.lib().ogcp_solve_factors(
        _lib.ctx(), X._handle, C.byref(cfg._c(loss)), C.byref(loss._c()), int(t), C.byref(model.c()),
        C.cast(op, C.POINTER(C.c_void_p)) if op is not None else None, wp, ws.ctypes.data_as(_lib.c_f64p),
        ids.ctypes.data_as(_lib.c_i64p), len(window), C.byref(st), C.byref(it), C.byref(tr.c)))
    adam.rate = float(st.rate)
    return int(it.value), tr.result()


def solve_factors(X: SparseTensor, factors: Sequence[np.ndarray], weights: np.ndarray,
                  old_factors: Sequence[np.ndarray], window: Sequence, cfg: SolverConfig, loss: LossFunction,
                  adam: Adam, iteration: int, t: int = 0) -> FactorSolve:
    """Factor-matrix GCP-SGD solve with the temporal weights fixed (solvers.py:290-368)."""
    model = DeviceModel.from_numpy(factors)
    old = DeviceModel.from_numpy(old_factors) if old_factors is not None else None
    if adam._buf is None or len(adam._buf["u"]) != len(model.tensors):
        raise DataError("variable/gradient structure does not match init")
    it, tr = solve_factors_device(X, model, weights, old, window, cfg, loss, adam, iteration, t)
    return FactorSolve(model.to_numpy(), it, tr)


def factor_gradients(Y: SparseTensor, factors: Sequence[np.ndarray], weights: np.ndarray, *,
                     old_factors: Optional[Sequence[np.ndarray]] = None, window: Sequence = (),
                     hist_weight: float = 0.0, hist_decay: float = 1.0, t: int = 0,
                     reg_factors: float = 0.0) -> list:
    """Full factor-gradient assembly from a gradient tensor Y (solvers.py:127-142):
    G_k = mttkrp(Y, k) diag(s) + lambda A_k + history."""
    import torch
    model = factors if isinstance(factors, DeviceModel) else DeviceModel.from_numpy(factors)
    old = None
    if old_factors is not None:
        old = old_factors if isinstance(old_factors, DeviceModel) else DeviceModel.from_numpy(old_factors)
    if hist_weight and len(window) and old is None:
        raise DataError("history terms require the previous-step factors")
    grads = DeviceModel.zeros_like(model)
    w, wp = _lib.f64arr(weights)
    ids, ws = _window_arrays(window, model.rank)
    ords = torch.arange(Y.nnz, dtype=torch.int32, device="cuda")
    op = old.ptrs() if old is not None else None
    gp = grads.ptrs()
    ident = _lib.LossC(3, 1e-10)
    _lib.check(_lib.lib().ogcp_factor_gradients(
        _lib.ctx(), Y._handle, C.c_void_p(ords.data_ptr() if Y.nnz else None), Y.nnz, None, 0,
        C.byref(model.c()), C.cast(op, C.POINTER(C.c_void_p)) if op is not None else None, wp, C.byref(ident),
        ws.ctypes.data_as(_lib.c_f64p), ids.ctypes.data_as(_lib.c_i64p), len(window), float(hist_weight),
        float(hist_decay), int(t), float(reg_factors), C.cast(gp, C.POINTER(C.c_void_p))))
    return grads.to_numpy()


@dataclass
class StaticSolve:
    model: KTensor
    trace: EpochTrace


def _host_generator(seed: int, *key: int) -> np.random.Generator:
    """Host numpy stream for initial values, rng_at(seed, *key) (sampling.py:39-42)."""
    return np.random.default_rng(np.random.SeedSequence(int(seed), spawn_key=tuple(int(k) for k in key)))


def solve_static_device(X: SparseTensor, model: DeviceModel, weights: np.ndarray, loss: LossFunction,
                        cfg: SolverConfig, *, max_epochs: int, iters: int, rate: float, tol: float,
                        seed_key: int = 0):
    """Static fit updating ``model`` in place on the device; returns (weights, trace)."""
    _check_gradient_mode(cfg, loss)
    w = np.ascontiguousarray(np.array(weights, dtype=np.float64))
    if w.shape != (model.rank,):
        raise DataError("weights must match the model rank")
    adam = cfg.make_adam(rate, loss)
    adam.init_device(model.dims, model.rank)
    st = adam.c()
    tr = _Trace(max_epochs)
    _lib.check(_lib.lib().ogcp_solve_static(
        _lib.ctx(), X._handle, C.byref(cfg._c(loss)), C.byref(loss._c()), int(seed_key), C.byref(model.c()),
        w.ctypes.data_as(_lib.c_f64p), C.byref(st), int(max_epochs), int(iters), float(tol), C.byref(tr.c)))
    return w, tr.result()


def solve_static(X: SparseTensor, rank: int, loss: LossFunction, cfg: SolverConfig, init: Optional[KTensor] = None,
                 *, max_epochs: Optional[int] = None, iters_per_epoch: Optional[int] = None,
                 rate: Optional[float] = None, tol: Optional[float] = None, restarts: int = 1,
                 seed_key: int = 0) -> StaticSolve:
    """Static GCP-SGD fit of weights and all factor matrices jointly (solvers.py:371-493).

    Initialization is uniform(0, 1) keyed (seed, seed_key, PHASE_INIT) unless
    given; with ``restarts`` > 1 the candidate with the lowest objective on the
    shared (seed, seed_key, PHASE_RESTART_EVAL) sample set is returned."""
    from .sampling import PHASE_INIT, PHASE_RESTART_EVAL, draw_samples, estimate_objective, rng_at
    if restarts > 1:
        if init is not None:
            raise DataError("restarts > 1 and an explicit init conflict")
        cands = [solve_static(X, rank, loss, cfg, max_epochs=max_epochs, iters_per_epoch=iters_per_epoch,
                              rate=rate, tol=tol, seed_key=seed_key + r) for r in range(restarts)]
        if cfg.gradient_mode == "dense-gaussian":
            from .kernels import gaussian_sum_sq_residual
            scores = [gaussian_sum_sq_residual(X, c.model.factors, c.model.weights) for c in cands]
            return cands[int(np.argmin(scores))]
        p_eval, q_eval = cfg.samples.objective_counts(X)
        ev = draw_samples(X, p_eval, q_eval, rng_at(cfg.samples.seed, seed_key, PHASE_RESTART_EVAL),
                          cfg.samples.max_rejects)
        scores = [estimate_objective(X, c.model.factors, c.model.weights, loss, ev, reg_factors=cfg.reg_factors,
                                     reg_weights=cfg.reg_weights) for c in cands]
        return cands[int(np.argmin(scores))]
    _check_gradient_mode(cfg, loss)
    max_epochs = cfg.max_epochs_factors if max_epochs is None else max_epochs
    iters = cfg.iters_factors if iters_per_epoch is None else iters_per_epoch
    rate = cfg.rate_factors if rate is None else rate
    tol = cfg.tol_factors if tol is None else tol
    if init is None:
        g0 = _host_generator(cfg.samples.seed, seed_key, PHASE_INIT)
        factors = [g0.uniform(size=(d, rank)) for d in X.dims]
        weights = g0.uniform(size=rank)
    else:
        if init.dims != X.dims or init.rank != rank:
            raise DataError("init model does not match tensor dims/rank")
        factors, weights = list(init.factors), np.array(init.weights)
    model = DeviceModel.from_numpy(factors)
    w, trace = solve_static_device(X, model, weights, loss, cfg, max_epochs=max_epochs, iters=iters, rate=rate,
                                   tol=tol, seed_key=seed_key)
    return StaticSolve(KTensor(w, model.to_numpy()), trace)


def solve_weights_least_squares_device(X: SparseTensor, model: DeviceModel, reg_weights: float = 0.0) -> np.ndarray:
    """Gaussian least-squares temporal row on device-resident factors (engine entry)."""
    out = np.zeros(model.rank)
    _lib.check(_lib.lib().ogcp_solve_weights_ls(_lib.ctx(), X._handle, C.byref(model.c()), float(reg_weights),
                                                 out.ctypes.data_as(_lib.c_f64p)))
    return out


def solve_weights_least_squares(X: SparseTensor, factors: Sequence[np.ndarray], reg_weights: float = 0.0) -> np.ndarray:
    """Single Gaussian least-squares solve for the temporal weights (solvers.py:271-288):
    (hadamard_k Gram_k + mu I) s = Z' vec(X), implicit zeros as zero residuals."""
    model = factors if isinstance(factors, DeviceModel) else DeviceModel.from_numpy(factors)
    return solve_weights_least_squares_device(X, model, reg_weights)


def _dense_gradients(X, factors, weights, want_factors, want_weights, old_factors=None, window=(),
                     hist_weight=0.0, hist_decay=1.0, t=0, reg_factors=0.0, reg_weights=0.0):
    model = factors if isinstance(factors, DeviceModel) else DeviceModel.from_numpy(factors)
    if len(model.dims) != X.ndim or tuple(model.dims) != tuple(X.dims):
        raise DataError("factor shapes do not match the tensor")
    old = None
    if old_factors is not None:
        old = old_factors if isinstance(old_factors, DeviceModel) else DeviceModel.from_numpy(old_factors)
    if hist_weight and len(window) and old is None:
        raise DataError("history terms require the previous-step factors")
    w, wp = _lib.f64arr(weights)
    ids, ws = _window_arrays(window, model.rank)
    grads = DeviceModel.zeros_like(model) if want_factors else None
    gw = np.zeros(model.rank) if want_weights else None
    op = old.ptrs() if old is not None else None
    gp = grads.ptrs() if grads is not None else None
    _lib.check(_lib.lib().ogcp_dense_gaussian_gradients(
        _lib.ctx(), X._handle, C.byref(model.c()), C.cast(op, C.POINTER(C.c_void_p)) if op is not None else None,
        wp, ws.ctypes.data_as(_lib.c_f64p), ids.ctypes.data_as(_lib.c_i64p), len(window), float(hist_weight),
        float(hist_decay), int(t), float(reg_factors), float(reg_weights),
        C.cast(gp, C.POINTER(C.c_void_p)) if gp is not None else None,
        gw.ctypes.data_as(_lib.c_f64p) if gw is not None else None))
    return (grads.to_numpy() if grads is not None else None), gw


def dense_gaussian_factor_gradients(X: SparseTensor, factors: Sequence[np.ndarray], weights: np.ndarray, *,
                                    old_factors=None, window: Sequence = (), hist_weight: float = 0.0,
                                    hist_decay: float = 1.0, t: int = 0, reg_factors: float = 0.0) -> list:
    """Exact Gaussian factor gradients plus regularization/history terms (solvers.py:145-156)."""
    g, _ = _dense_gradients(X, factors, weights, True, False, old_factors, window, hist_weight, hist_decay, t,
                            reg_factors)
    return g


def dense_gaussian_weight_gradient(X: SparseTensor, factors: Sequence[np.ndarray], weights: np.ndarray,
                                   reg_weights: float = 0.0) -> np.ndarray:
    """2 (Gamma s - Z' vec(X)) + mu s (solvers.py:182-185)."""
    _, gw = _dense_gradients(X, factors, weights, False, True, reg_weights=reg_weights)
    return gw
