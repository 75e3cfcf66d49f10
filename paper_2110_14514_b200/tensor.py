"""Device-resident sparse slices and CP models (reference: pkg/src/ogcp/tensor.py).

``SparseTensor`` keeps the reference constructor semantics (1-based public
coordinates, validation of bounds / finiteness / stored zeros / duplicates,
entries kept in the given order) but validation, the AoS record layout and
the membership hash are built on the GPU by the K0 ingest kernel
(csrc/ingest.cu) through ``ogcp_slice_create``.  Host copies of the entry
arrays are kept (or fetched lazily) for the attributes the reference exposes.

``DeviceModel`` holds factor matrices as row-major float32 [I_k x ldr] CUDA
tensors whose padding columns are zero -- the layout every kernel reads.
"""

from __future__ import annotations

import ctypes as C
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _lib
from .exceptions import DataError

_MAX_LINEAR = 2**63 - 1


def _check_dims(dims: Sequence[int]) -> tuple:
    dims = tuple(int(d) for d in dims)
    if len(dims) == 0 or any(d <= 0 for d in dims):
        raise DataError(f"dims must be positive integers, got {dims}")
    total = 1
    for d in dims:
        total *= d
    if total > _MAX_LINEAR:
        raise DataError(f"index space of size prod{dims} exceeds 2**63-1; cannot linearize")
    return dims


def linear_strides(dims: Sequence[int]) -> np.ndarray:
    """Mixed-radix strides, mode 0 most significant (tensor.py:33-38)."""
    strides = np.ones(len(dims), dtype=np.int64)
    for k in range(len(dims) - 2, -1, -1):
        strides[k] = strides[k + 1] * dims[k + 1]
    return strides


class SparseTensor:
    """A d-way sparse COO tensor whose validated copy lives in GPU memory."""

    def __init__(self, dims, subs, vals, allow_zero_values: bool = False):
        dims = _check_dims(dims)
        subs = np.asarray(subs, dtype=np.int64)
        if subs.size == 0:
            subs = subs.reshape(0, len(dims))
        if subs.ndim != 2 or subs.shape[1] != len(dims):
            raise DataError(f"subs must have shape (n, {len(dims)}), got {subs.shape}")
        self._init_host(dims, subs - 1, np.asarray(vals, dtype=np.float64), allow_zero_values)

    @classmethod
    def from_zero_based(cls, dims, subs0, vals, allow_zero_values: bool = False) -> "SparseTensor":
        self = cls.__new__(cls)
        dims = _check_dims(dims)
        subs0 = np.ascontiguousarray(subs0, dtype=np.int64)
        if subs0.size == 0:
            subs0 = subs0.reshape(0, len(dims))
        self._init_host(dims, subs0, np.asarray(vals, dtype=np.float64), allow_zero_values)
        return self

    @classmethod
    def from_device(cls, dims, subs0, vals, allow_zero_values: bool = False) -> "SparseTensor":
        """Construct from CUDA tensors: int32 [n, d] 0-based coordinates, float32 [n] values."""
        import torch
        self = cls.__new__(cls)
        dims = _check_dims(dims)
        self._handle = None
        subs0 = subs0.to(torch.int32).contiguous()
        vals = vals.to(torch.float32).contiguous()
        if vals.ndim != 1 or vals.shape[0] != subs0.shape[0]:
            raise DataError("vals must be a vector matching the entry count")
        self.dims = dims
        self._subs0_host = None
        self._vals_host = None
        self._dev_keep = (subs0, vals)
        d, dp = _lib.i64arr(dims)
        h = C.c_void_p()
        _lib.check(_lib.lib().ogcp_slice_create_i32(_lib.ctx(), len(dims), dp, int(vals.shape[0]),
                                                     C.c_void_p(subs0.data_ptr()), C.c_void_p(vals.data_ptr()),
                                                     int(bool(allow_zero_values)), C.byref(h)))
        self._handle = h
        self._dev_keep = None
        self._nnz = int(vals.shape[0])
        self._fetch = (subs0, vals)
        return self

    def _init_host(self, dims, subs0, vals, allow_zero_values):
        import torch
        self._handle = None
        if vals.ndim != 1 or vals.shape[0] != subs0.shape[0]:
            raise DataError("vals must be a vector matching the entry count")
        self.dims = dims
        # read-only views: the caller's own arrays stay writable
        self._subs0_host = subs0.view()
        self._vals_host = vals.view()
        self._nnz = int(vals.shape[0])
        self._fetch = None
        dev = torch.cuda.current_device() if torch.cuda.is_available() else None
        if dev is None:
            raise RuntimeError("paper_2110_14514_b200 needs a CUDA device (B200, sm_100a); there is no CPU path")
        s_dev = torch.from_numpy(np.ascontiguousarray(subs0)).to("cuda")
        v_dev = torch.from_numpy(np.ascontiguousarray(vals)).to("cuda")
        d, dp = _lib.i64arr(dims)
        h = C.c_void_p()
        _lib.check(_lib.lib().ogcp_slice_create(_lib.ctx(), len(dims), dp, self._nnz, C.c_void_p(s_dev.data_ptr()),
                                                 C.c_void_p(v_dev.data_ptr()), int(bool(allow_zero_values)),
                                                 C.byref(h)))
        self._handle = h
        self._subs0_host.flags.writeable = False
        self._vals_host.flags.writeable = False

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                _lib.lib().ogcp_slice_destroy(h)
            except Exception:
                pass
            self._handle = None

    # -- reference attributes ------------------------------------------------
    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def nnz(self) -> int:
        return self._nnz

    @property
    def num_cells(self) -> int:
        total = 1
        for d in self.dims:
            total *= d
        return total

    def _materialize(self):
        if self._subs0_host is None:
            subs0, vals = self._fetch
            self._subs0_host = subs0.cpu().numpy().astype(np.int64)
            self._vals_host = vals.cpu().numpy().astype(np.float64)
            self._subs0_host.flags.writeable = False
            self._vals_host.flags.writeable = False
            self._fetch = None

    @property
    def subs0(self) -> np.ndarray:
        self._materialize()
        return self._subs0_host

    @property
    def vals(self) -> np.ndarray:
        self._materialize()
        return self._vals_host

    @property
    def frobenius_sq(self) -> float:
        f = C.c_double()
        _lib.check(_lib.lib().ogcp_slice_info(self._handle, None, None, C.byref(f)))
        return float(f.value)

    def subs(self) -> np.ndarray:
        return self.subs0 + 1

    def linearize(self, subs0: np.ndarray) -> np.ndarray:
        return np.asarray(subs0, dtype=np.int64) @ linear_strides(self.dims)

    def contains(self, subs0: np.ndarray) -> np.ndarray:
        """Membership of 0-based coordinates via the device hash (tensor.py:163-169)."""
        import torch
        subs0 = np.ascontiguousarray(np.asarray(subs0, dtype=np.int64).reshape(-1, self.ndim))
        if subs0.shape[0] == 0:
            return np.zeros(0, dtype=bool)
        s = torch.from_numpy(subs0).cuda()
        hit = torch.empty(subs0.shape[0], dtype=torch.uint8, device="cuda")
        _lib.check(_lib.lib().ogcp_slice_contains(_lib.ctx(), self._handle, C.c_void_p(s.data_ptr()),
                                                   subs0.shape[0], C.c_void_p(hit.data_ptr())))
        return hit.cpu().numpy().astype(bool)

    def slice_view(self, t: int) -> "SparseTensor":
        """Hyperslice at last-mode index t (1-based), last coordinate dropped (tensor.py:179-190)."""
        if self.ndim < 2:
            raise IndexError("slice_view requires a tensor with at least 2 modes")
        if not 1 <= t <= self.dims[-1]:
            raise IndexError(f"slice index {t} out of range 1..{self.dims[-1]}")
        mask = self.subs0[:, -1] == t - 1
        return SparseTensor.from_zero_based(self.dims[:-1], self.subs0[mask, :-1], self.vals[mask])

    def dense(self) -> np.ndarray:
        out = np.zeros(self.dims)
        if self.nnz:
            out[tuple(self.subs0.T)] = self.vals
        return out

    def __repr__(self) -> str:
        return f"SparseTensor(dims={self.dims}, nnz={self.nnz})"


class KTensor:
    """Kruskal tensor container (tensor.py:214-282); host arrays, immutable."""

    __slots__ = ("weights", "factors")

    def __init__(self, weights, factors: Iterable[np.ndarray]):
        self.weights = np.array(weights, dtype=np.float64)
        self.factors = [np.array(a, dtype=np.float64) for a in factors]
        if self.weights.ndim != 1:
            raise DataError("weights must be a vector")
        rank = self.weights.shape[0]
        for k, a in enumerate(self.factors):
            if a.ndim != 2 or a.shape[1] != rank:
                raise DataError(f"factor {k} must have shape (I_{k + 1}, {rank}), got {a.shape}")
            if a.size and not np.isfinite(a).all():
                raise DataError(f"factor {k} contains non-finite entries")
        if self.weights.size and not np.isfinite(self.weights).all():
            raise DataError("weights contain non-finite entries")
        self.weights.flags.writeable = False
        for a in self.factors:
            a.flags.writeable = False

    @property
    def rank(self) -> int:
        return self.weights.shape[0]

    @property
    def ndim(self) -> int:
        return len(self.factors)

    @property
    def dims(self) -> tuple:
        return tuple(a.shape[0] for a in self.factors)

    def __repr__(self) -> str:
        return f"KTensor(dims={self.dims}, rank={self.rank})"


class DeviceModel:
    """Factor matrices as padded float32 CUDA tensors [I_k x ldr] (engine layout)."""

    def __init__(self, tensors, rank: int):
        self.tensors = list(tensors)
        self.rank = int(rank)
        self.ldr = _lib.padded_rank(self.rank)
        self.dims = tuple(int(t.shape[0]) for t in self.tensors)
        self._keep = None

    @classmethod
    def from_numpy(cls, factors: Sequence[np.ndarray]) -> "DeviceModel":
        import torch
        factors = [np.asarray(a, dtype=np.float64) for a in factors]
        rank = factors[0].shape[1]
        ldr = _lib.padded_rank(rank)
        ts = []
        for a in factors:
            t = torch.zeros((a.shape[0], ldr), dtype=torch.float32, device="cuda")
            t[:, :rank] = torch.from_numpy(a.astype(np.float32)).cuda()
            ts.append(t)
        return cls(ts, rank)

    @classmethod
    def zeros_like(cls, other: "DeviceModel") -> "DeviceModel":
        import torch
        return cls([torch.zeros_like(t) for t in other.tensors], other.rank)

    def clone(self) -> "DeviceModel":
        return DeviceModel([t.clone() for t in self.tensors], self.rank)

    def copy_(self, other: "DeviceModel"):
        for a, b in zip(self.tensors, other.tensors):
            a.copy_(b)

    def to_numpy(self):
        return [t[:, :self.rank].double().cpu().numpy() for t in self.tensors]

    def ptrs(self):
        return _lib.ptr_array(self.tensors)

    def c(self):
        d, dp = _lib.i64arr(self.dims)
        p = self.ptrs()
        m = _lib.ModelC(len(self.tensors), self.rank, self.ldr, dp, C.cast(p, C.POINTER(C.c_void_p)))
        self._keep = (d, p)
        return m

