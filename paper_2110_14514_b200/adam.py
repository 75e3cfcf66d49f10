"""Adam stepper with device-resident moments (reference: pkg/src/ogcp/adam.py).

Moments u, v and the epoch snapshots u_o, v_o, a_o live on the GPU in the
engine's padded layout; ``step`` runs the fused K5 kernel (clamp + isfinite
included) and ``update`` the accept/reject copies, both through the C ABI.
The numpy-facing ``step``/``update`` keep the reference signatures.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .exceptions import DataError


def _as_list(a):
    return (True, [a]) if isinstance(a, np.ndarray) else (False, list(a))


class Adam:
    """One stepper per solver; mutated single-threaded (adam.py:20-37)."""

    def __init__(self, rate: float, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                 lower_bound: float = -np.inf, rate_decay: float = 0.1):
        if rate <= 0:
            raise DataError("learning rate must be positive")
        if not 0.0 < rate_decay < 1.0:
            raise DataError("rate_decay must lie in (0, 1)")
        self.rate = float(rate)
        self.beta1 = float(beta1)
        self.beta2 = float(beta2)
        self.eps = float(eps)
        self.lower_bound = float(lower_bound)
        self.rate_decay = float(rate_decay)
        self._buf = None        # dict name -> list of CUDA tensors [rows x ldr]
        self._shapes = None     # per-part (rows, cols, original shape)
        self._single = False
        self._keep = None

    # -- device layout -------------------------------------------------------
    def init_device(self, dims, rank):
        """Zero moments for a model of the given mode sizes and rank (engine layout)."""
        import torch
        ldr = _lib.padded_rank(rank)
        self._shapes = [(int(d), int(rank), (int(d), int(rank))) for d in dims]
        self._buf = {n: [torch.zeros((int(d), ldr), dtype=torch.float32, device="cuda") for d in dims]
                     for n in ("u", "v", "u_o", "v_o", "a_o")}
        self._single = False

    def c(self):
        arrs = {n: _lib.ptr_array(ts) for n, ts in self._buf.items()}
        cp = lambda n: C.cast(arrs[n], C.POINTER(C.c_void_p))
        st = _lib.AdamC(cp("u"), cp("v"), cp("u_o"), cp("v_o"), cp("a_o"), self.rate)
        self._keep = arrs
        return st

    # -- reference API ---------------------------------------------------------
    def init(self, a):
        """Zero all moment buffers and snapshots with the shape of ``a`` (adam.py:39-46)."""
        import torch
        self._single, parts = _as_list(a)
        self._shapes = []
        self._buf = {n: [] for n in ("u", "v", "u_o", "v_o", "a_o")}
        for x in parts:
            x = np.asarray(x)
            rows, cols = (x.shape[0], x.shape[1]) if x.ndim == 2 else (x.size, 1)
            ldr = _lib.padded_rank(cols)
            self._shapes.append((rows, cols, x.shape))
            for n in self._buf:
                self._buf[n].append(torch.zeros((rows, ldr), dtype=torch.float32, device="cuda"))

    def _part_model(self, k, tensor):
        from .tensor import DeviceModel
        m = DeviceModel([tensor], self._shapes[k][1])
        return m

    def _upload(self, k, x):
        import torch
        rows, cols, _ = self._shapes[k]
        t = torch.zeros((rows, _lib.padded_rank(cols)), dtype=torch.float32, device="cuda")
        t[:, :cols] = torch.from_numpy(np.asarray(x, dtype=np.float32).reshape(rows, cols)).cuda()
        return t

    def _download(self, k, t):
        rows, cols, shape = self._shapes[k]
        return t[:, :cols].double().cpu().numpy().reshape(shape)

    def _part_state(self, k):
        arrs = {n: _lib.ptr_array([self._buf[n][k]]) for n in self._buf}
        cp = lambda n: C.cast(arrs[n], C.POINTER(C.c_void_p))
        return _lib.AdamC(cp("u"), cp("v"), cp("u_o"), cp("v_o"), cp("a_o"), self.rate), arrs

    def step(self, a, g, step_count: int):
        """One bias-corrected Adam step; ``step_count`` is 1-based (adam.py:51-81)."""
        if step_count < 1:
            raise DataError("step_count is 1-based and must be >= 1")
        _, a_parts = _as_list(a)
        _, g_parts = _as_list(g)
        if self._buf is None or len(a_parts) != len(self._shapes) or len(g_parts) != len(self._shapes):
            raise DataError("variable/gradient structure does not match init")
        out = []
        for k, (a_k, g_k) in enumerate(zip(a_parts, g_parts)):
            a_k, g_k = np.asarray(a_k), np.asarray(g_k)
            if a_k.shape != g_k.shape or a_k.shape != self._shapes[k][2]:
                raise DataError(f"shape mismatch: variable {a_k.shape}, gradient {g_k.shape}")
            at, gt = self._upload(k, a_k), self._upload(k, g_k)
            m = self._part_model(k, at)
            gp = _lib.ptr_array([gt])
            st, keep = self._part_state(k)
            _lib.check(_lib.lib().ogcp_adam_step(_lib.ctx(), C.byref(m.c()), C.cast(gp, C.POINTER(C.c_void_p)),
                                                  C.byref(st), self.beta1, self.beta2, self.eps, self.lower_bound,
                                                  int(step_count)))
            out.append(self._download(k, at))
        return out[0] if self._single else out

    def update(self, a, passed: bool):
        """Accept (snapshot) or reject (restore and decay rate) an epoch (adam.py:83-94)."""
        _, a_parts = _as_list(a)
        out = []
        for k, a_k in enumerate(a_parts):
            at = self._upload(k, a_k)
            m = self._part_model(k, at)
            st, keep = self._part_state(k)
            _lib.check(_lib.lib().ogcp_adam_update(_lib.ctx(), C.byref(m.c()), C.byref(st), int(bool(passed)),
                                                    self.rate_decay))
            out.append(self._download(k, at))
        if not passed:
            self.rate *= self.rate_decay
        return out[0] if self._single else out

    def state_arrays(self) -> dict:
        """Moment buffers and snapshots for checkpointing (adam.py:96-101)."""
        return {n: [self._download(k, t) for k, t in enumerate(ts)] for n, ts in self._buf.items()}

    def load_state_arrays(self, arrays: dict, single: bool):
        self._single = single
        parts = arrays["u"]
        self._shapes = []
        self._buf = {n: [] for n in ("u", "v", "u_o", "v_o", "a_o")}
        for x in parts:
            x = np.asarray(x)
            rows, cols = (x.shape[0], x.shape[1]) if x.ndim == 2 else (x.size, 1)
            self._shapes.append((rows, cols, x.shape))
        for n in self._buf:
            self._buf[n] = [self._upload(k, x) for k, x in enumerate(arrays[n])]
