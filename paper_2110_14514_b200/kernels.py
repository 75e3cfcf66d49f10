"""Multilinear primitives on the GPU (reference: pkg/src/ogcp/kernels.py).

MTTKRP and the weight gradient of a given sparse tensor Y run the fused
sample kernels in gradient-tensor mode (y = stored value, ``OGCP_IDENTITY``);
Grams run the K4 Gram kernel with fp64 accumulation.
"""

from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .exceptions import DataError
from .tensor import DeviceModel, KTensor, SparseTensor


def _check_factor_shapes(Y: SparseTensor, factors):
    if len(factors) != Y.ndim:
        raise DataError(f"tensor has {Y.ndim} modes but {len(factors)} factors given")
    for k, a in enumerate(factors):
        if a.shape[0] != Y.dims[k]:
            raise DataError(f"factor {k} has {a.shape[0]} rows, tensor dim is {Y.dims[k]}")


def _gradient_tensor_pass(Y: SparseTensor, factors, want_grads: bool, want_gw: bool):
    import torch
    model = DeviceModel.from_numpy(factors)
    grads = DeviceModel.zeros_like(model) if want_grads else None
    gw = torch.zeros(model.rank, dtype=torch.float64, device="cuda") if want_gw else None
    ones, op = _lib.f64arr(np.ones(model.rank))
    ords = torch.arange(Y.nnz, dtype=torch.int32, device="cuda")
    gp = grads.ptrs() if grads is not None else None
    _lib.check(_lib.lib().ogcp_sampled_gradient(
        _lib.ctx(), Y._handle, C.c_void_p(ords.data_ptr() if Y.nnz else None), Y.nnz, None, 0, C.byref(model.c()),
        op, C.byref(_lib.LossC(3, 1e-10)), C.cast(gp, C.POINTER(C.c_void_p)) if gp is not None else None,
        C.c_void_p(gw.data_ptr()) if gw is not None else None))
    return grads, gw


def sampled_mttkrp(Y: SparseTensor, factors: Sequence[np.ndarray], mode: int) -> np.ndarray:
    """Mode-``mode`` MTTKRP of a sparse tensor with the factor list (kernels.py:33-56)."""
    _check_factor_shapes(Y, factors)
    if not 0 <= mode < Y.ndim:
        raise IndexError(f"mode {mode} out of range for {Y.ndim}-way tensor")
    grads, _ = _gradient_tensor_pass(Y, factors, True, False)
    return grads.to_numpy()[mode]


def weight_gradient_mttkrp(Y: SparseTensor, factors: Sequence[np.ndarray]) -> np.ndarray:
    """Z' vec(Y) over stored entries (kernels.py:59-72)."""
    _check_factor_shapes(Y, factors)
    _, gw = _gradient_tensor_pass(Y, factors, False, True)
    return gw.cpu().numpy()


def gram(factors: Sequence[np.ndarray], mode: Optional[int] = None,
         other_factors: Optional[Sequence[np.ndarray]] = None) -> np.ndarray:
    """Hadamard product of per-mode Grams B_m'A_m, skipping ``mode`` (kernels.py:75-98)."""
    others = factors if other_factors is None else other_factors
    if len(others) != len(factors):
        raise DataError("factor lists must have the same number of modes")
    for m, (b, a) in enumerate(zip(others, factors)):
        if b.shape[0] != a.shape[0]:
            raise DataError(f"mode {m}: row counts differ ({b.shape[0]} vs {a.shape[0]})")
    model = DeviceModel.from_numpy(factors)
    other = DeviceModel.from_numpy(others) if other_factors is not None else None
    out = np.zeros((model.rank, model.rank))
    op = other.ptrs() if other is not None else None
    _lib.check(_lib.lib().ogcp_gram(_lib.ctx(), C.byref(model.c()),
                                    C.cast(op, C.POINTER(C.c_void_p)) if op is not None else None,
                                    -1 if mode is None else int(mode), out.ctypes.data_as(_lib.c_f64p)))
    return out


def ktensor_inner(M1: KTensor, M2: KTensor) -> float:
    """<M1, M2> = s1' (hadamard_k A1(k)'A2(k)) s2 (kernels.py:101-106)."""
    if M1.dims != M2.dims:
        raise DataError(f"dims differ: {M1.dims} vs {M2.dims}")
    g = gram(M2.factors, other_factors=M1.factors)
    return float(M1.weights @ g @ M2.weights)


def history_penalty(M_old: KTensor, M_new: KTensor) -> float:
    """||M_old - M_new||_F^2 clamped at 0 (kernels.py:109-114)."""
    val = ktensor_inner(M_old, M_old) - 2.0 * ktensor_inner(M_old, M_new) + ktensor_inner(M_new, M_new)
    return max(val, 0.0)


def gaussian_sum_sq_residual(X: SparseTensor, factors: Sequence[np.ndarray], weights: np.ndarray) -> float:
    """Exact sum over all cells of (x - m)^2 = ||X||^2 - 2 <X, M> + ||M||^2 (kernels.py:135-146)."""
    _check_factor_shapes(X, factors)
    model = factors if isinstance(factors, DeviceModel) else DeviceModel.from_numpy(factors)
    w, wp = _lib.f64arr(weights)
    out = C.c_double()
    _lib.check(_lib.lib().ogcp_gaussian_residual(_lib.ctx(), X._handle, C.byref(model.c()), wp, C.byref(out)))
    return float(out.value)


def dense_gaussian_mttkrp_gradient(X: SparseTensor, factors: Sequence[np.ndarray], weights: np.ndarray,
                                   mode: int) -> np.ndarray:
    """Exact Gaussian gradient dF/dA(mode) = 2 (A diag(s) Gram diag(s) - mttkrp(X) diag(s)) (kernels.py:117-132)."""
    from .solvers import dense_gaussian_factor_gradients
    _check_factor_shapes(X, factors)
    if not 0 <= mode < X.ndim:
        raise IndexError(f"mode {mode} out of range for {X.ndim}-way tensor")
    return dense_gaussian_factor_gradients(X, factors, weights)[mode]
