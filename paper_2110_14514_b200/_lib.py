"""ctypes binding of libogcp_b200.so (the C ABI in include/ogcp_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a).  Importing the package does not need a GPU; the first call that
needs the device creates the engine context on torch's current CUDA device
and stream.  There is no CPU fallback: a missing library or device raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .exceptions import DataError, DivergenceError, OgcpError, SamplingError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OGCP_LIB", os.path.join(_HERE, "libogcp_b200.so"))

OK, E_INTERNAL, E_USAGE, E_DATA, E_DIVERGENCE, E_SAMPLING, E_CUDA = range(7)
LOSS_KINDS = {"gaussian": 0, "poisson": 1, "bernoulli": 2}

c_i64p = C.POINTER(C.c_int64)
c_f64p = C.POINTER(C.c_double)


class LossC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("eps", C.c_double)]


class SamplerC(C.Structure):
    _fields_ = [("grad_nonzeros", C.c_int64), ("grad_zeros", C.c_int64), ("obj_nonzeros", C.c_int64),
                ("obj_zeros", C.c_int64), ("seed", C.c_uint64), ("max_rejects", C.c_int64),
                ("semi_stratified", C.c_int32)]


class SolverC(C.Structure):
    _fields_ = [("tol_weights", C.c_double), ("tol_factors", C.c_double),
                ("max_epochs_weights", C.c_int32), ("max_epochs_factors", C.c_int32),
                ("iters_weights", C.c_int32), ("iters_factors", C.c_int32),
                ("reg_factors", C.c_double), ("reg_weights", C.c_double), ("hist_weight", C.c_double),
                ("hist_decay", C.c_double), ("warm_start_weights", C.c_int32),
                ("rate_weights", C.c_double), ("rate_factors", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("adam_eps", C.c_double), ("rate_decay", C.c_double),
                ("lower_bound", C.c_double), ("samples", SamplerC), ("gradient_mode", C.c_int32),
                ("temporal_solver", C.c_int32)]


class ModelC(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("rank", C.c_int32), ("ldr", C.c_int32), ("dims", c_i64p),
                ("factors", C.POINTER(C.c_void_p))]


class AdamC(C.Structure):
    _fields_ = [("u", C.POINTER(C.c_void_p)), ("v", C.POINTER(C.c_void_p)), ("u_o", C.POINTER(C.c_void_p)),
                ("v_o", C.POINTER(C.c_void_p)), ("a_o", C.POINTER(C.c_void_p)), ("rate", C.c_double)]


class TraceC(C.Structure):
    _fields_ = [("objective", c_f64p), ("n_objective", C.c_int32), ("epochs", C.c_int32),
                ("rejections", C.c_int32)]


_SIGS = {
    "ogcp_abi_version": (C.c_int, []),
    "ogcp_last_error": (C.c_char_p, []),
    "ogcp_padded_rank": (C.c_int32, [C.c_int32]),
    "ogcp_rng_state": (C.c_int, [C.c_uint64, c_i64p, C.c_int32, C.POINTER(C.c_uint64)]),
    "ogcp_rng_integers": (C.c_int, [C.c_uint64, c_i64p, C.c_int32, c_i64p, C.c_int32, C.c_int64, c_i64p]),
    "ogcp_ctx_create": (C.c_int, [C.c_int32, C.c_void_p, C.POINTER(C.c_void_p)]),
    "ogcp_ctx_destroy": (C.c_int, [C.c_void_p]),
    "ogcp_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ogcp_ctx_launches": (C.c_int64, [C.c_void_p]),
    "ogcp_ctx_profile_enable": (C.c_int, [C.c_void_p, C.c_int32]),
    "ogcp_ctx_profile_read": (C.c_int, [C.c_void_p, C.c_int32, c_i64p, c_f64p]),
    "ogcp_ctx_profile_reset": (C.c_int, [C.c_void_p]),
    "ogcp_ctx_set_option": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64]),
    "ogcp_sampled_gradient_ex": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                           C.POINTER(ModelC), c_f64p, C.POINTER(LossC), C.c_int32,
                                           C.POINTER(C.c_void_p), C.c_void_p]),
    "ogcp_gradient_tensor": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                       C.POINTER(ModelC), c_f64p, C.POINTER(LossC), C.c_void_p, C.c_void_p,
                                       c_i64p]),
    "ogcp_segment_layout": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int64,
                                      C.c_void_p, C.c_void_p]),
    "ogcp_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "ogcp_ctx_init_comm": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8), C.c_int32, C.c_int32]),
    "ogcp_slice_create": (C.c_int, [C.c_void_p, C.c_int32, c_i64p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int32,
                                    C.POINTER(C.c_void_p)]),
    "ogcp_slice_create_i32": (C.c_int, [C.c_void_p, C.c_int32, c_i64p, C.c_int64, C.c_void_p, C.c_void_p,
                                        C.c_int32, C.POINTER(C.c_void_p)]),
    "ogcp_slice_destroy": (C.c_int, [C.c_void_p]),
    "ogcp_slice_info": (C.c_int, [C.c_void_p, c_i64p, c_i64p, c_f64p]),
    "ogcp_slice_contains": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "ogcp_draw_samples": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, c_i64p, C.c_int32, C.c_int64, C.c_int64,
                                    C.c_int64, C.c_void_p, C.c_void_p]),
    "ogcp_draw_samples_ex": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, c_i64p, C.c_int32, C.c_int64,
                                       C.c_int64, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]),
    "ogcp_sampled_gradient": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                        C.POINTER(ModelC), c_f64p, C.POINTER(LossC), C.POINTER(C.c_void_p),
                                        C.c_void_p]),
    "ogcp_factor_gradients": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                        C.POINTER(ModelC), C.POINTER(C.c_void_p), c_f64p, C.POINTER(LossC),
                                        c_f64p, c_i64p, C.c_int32, C.c_double, C.c_double, C.c_int64, C.c_double,
                                        C.POINTER(C.c_void_p)]),
    "ogcp_estimate_objective": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                          C.POINTER(ModelC), C.POINTER(C.c_void_p), c_f64p, C.POINTER(LossC),
                                          c_f64p, c_i64p, C.c_int32, C.c_double, C.c_double, C.c_int64,
                                          C.c_double, C.c_double, c_f64p]),
    "ogcp_gram": (C.c_int, [C.c_void_p, C.POINTER(ModelC), C.POINTER(C.c_void_p), C.c_int32, c_f64p]),
    "ogcp_adam_step": (C.c_int, [C.c_void_p, C.POINTER(ModelC), C.POINTER(C.c_void_p), C.POINTER(AdamC),
                                 C.c_double, C.c_double, C.c_double, C.c_double, C.c_int64]),
    "ogcp_adam_update": (C.c_int, [C.c_void_p, C.POINTER(ModelC), C.POINTER(AdamC), C.c_int32, C.c_double]),
    "ogcp_solve_weights": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(SolverC), C.POINTER(LossC), C.c_int64,
                                     C.POINTER(ModelC), c_f64p, c_f64p, C.POINTER(TraceC)]),
    "ogcp_solve_factors": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(SolverC), C.POINTER(LossC), C.c_int64,
                                     C.POINTER(ModelC), C.POINTER(C.c_void_p), c_f64p, c_f64p, c_i64p, C.c_int32,
                                     C.POINTER(AdamC), c_i64p, C.POINTER(TraceC)]),
    "ogcp_solve_static": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(SolverC), C.POINTER(LossC), C.c_int64,
                                    C.POINTER(ModelC), c_f64p, C.POINTER(AdamC), C.c_int32, C.c_int32, C.c_double,
                                    C.POINTER(TraceC)]),
    "ogcp_solve_weights_ls": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(ModelC), C.c_double, c_f64p]),
    "ogcp_gaussian_residual": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(ModelC), c_f64p, c_f64p]),
    "ogcp_dense_gaussian_gradients": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(ModelC), C.POINTER(C.c_void_p),
                                                c_f64p, c_f64p, c_i64p, C.c_int32, C.c_double, C.c_double,
                                                C.c_int64, C.c_double, C.c_double, C.POINTER(C.c_void_p), c_f64p]),
    "ogcp_comm_selftest": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    "ogcp_debug_solve_draw": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, c_i64p, C.c_int32, C.c_int64, C.c_int64,
                                        C.c_int64, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, c_i64p, C.c_int64,
                                        C.c_void_p, c_i64p]),
    "ogcp_local_loss": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(ModelC), c_f64p, C.POINTER(LossC), C.c_int32,
                                  C.c_int64, C.c_int64, C.c_uint64, c_i64p, C.c_int32, C.c_int64, C.c_int64, c_f64p,
                                  C.POINTER(C.c_int32)]),
}

_lib = None
_lock = threading.Lock()
_ctxs = {}


def lib():
    """Load the engine library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
                h = C.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    fn = getattr(h, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = h
    return _lib


def check(status):
    """Map an ABI status code onto the reference exception hierarchy."""
    if status == OK:
        return
    msg = lib().ogcp_last_error().decode(errors="replace")
    if status == E_SAMPLING:
        raise SamplingError(msg)
    if status == E_DATA:
        raise DataError(msg)
    if status == E_DIVERGENCE:
        raise DivergenceError(msg)
    if status == E_USAGE:
        raise ValueError(msg)
    raise OgcpError(f"engine error {status}: {msg}")


def ctx():
    """Engine context for torch's current CUDA device, bound to its current stream."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2110_14514_b200 needs a CUDA device (B200, sm_100a); there is no CPU path")
    dev = torch.cuda.current_device()
    stream = torch.cuda.current_stream(dev).cuda_stream
    L = lib()
    c = _ctxs.get(dev)
    if c is None:
        h = C.c_void_p()
        check(L.ogcp_ctx_create(dev, C.c_void_p(stream), C.byref(h)))
        c = _ctxs[dev] = h
    else:
        check(L.ogcp_ctx_set_stream(c, C.c_void_p(stream)))
    return c


def launches():
    """Kernels launched so far by this process's engine contexts."""
    return sum(int(lib().ogcp_ctx_launches(c)) for c in _ctxs.values())


def padded_rank(rank: int) -> int:
    return int(lib().ogcp_padded_rank(int(rank)))


def i64arr(values):
    a = np.ascontiguousarray(np.asarray(values, dtype=np.int64))
    return a, a.ctypes.data_as(c_i64p)


def f64arr(values):
    a = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
    return a, a.ctypes.data_as(c_f64p)


def ptr_array(tensors):
    arr = (C.c_void_p * max(len(tensors), 1))()
    for i, t in enumerate(tensors):
        arr[i] = None if t is None else t.data_ptr()
    return arr


def rng_state(seed, key):
    k, kp = i64arr(list(key) or [0])
    out = (C.c_uint64 * 4)()
    check(lib().ogcp_rng_state(int(seed), kp, len(key), out))
    return tuple(int(v) for v in out)


def rng_integers(seed, key, highs, n):
    """Host restatement of Generator.integers(0, highs) on the keyed stream."""
    k, kp = i64arr(list(key) or [0])
    h, hp = i64arr(highs)
    out = np.empty(int(n), dtype=np.int64)
    check(lib().ogcp_rng_integers(int(seed), kp, len(key), hp, len(h), int(n), out.ctypes.data_as(c_i64p)))
    return out


def set_merge_draws(on: bool):
    """Engine option OGCP_OPT_MERGE_DRAWS for the current device's context."""
    check(lib().ogcp_ctx_set_option(ctx(), 1, int(bool(on))))


def set_buckets(value):
    """Engine option OGCP_OPT_BUCKETS: False/0 off, True/1 auto, k > 1 force k buckets."""
    check(lib().ogcp_ctx_set_option(ctx(), 3, int(value)))


def set_shard_sim(rank: int, world: int, timing: bool = False):
    """OGCP_OPT_SHARD_SIM: run this context as rank `rank` of `world` without a communicator
    (tests); `timing`: collectives replaced by stand-in kernels of their modeled duration and
    sharded draws run for this rank only (projections; results inexact)."""
    check(lib().ogcp_ctx_set_option(ctx(), 4, int(rank) | (int(world) << 16) | (int(bool(timing)) << 32)))


def debug_solve_draw(X, seed: int, key, p, q: int, ldr: int, max_rejects=None):
    """(ordinals, multiplicities, zero rows) of the gradient sample set a solve iteration evaluates here."""
    p = -1 if p is None else int(p)
    cap_nz = max(X.nnz, 1)
    ords = np.zeros(cap_nz, np.int32)
    cnts = np.zeros(cap_nz, np.uint8)
    zeros = np.zeros((max(q, 1), X.ndim), np.int32)
    nn, nz = C.c_int64(), C.c_int64()
    k = np.ascontiguousarray(np.asarray(key, np.int64))
    check(lib().ogcp_debug_solve_draw(ctx(), X._handle, int(seed), k.ctypes.data_as(c_i64p), len(k), p, int(q),
                                      -1 if max_rejects is None else int(max_rejects), int(ldr), cap_nz,
                                      ords.ctypes.data, cnts.ctypes.data, C.byref(nn), max(q, 1), zeros.ctypes.data,
                                      C.byref(nz)))
    return ords[:nn.value].astype(np.int64), cnts[:nn.value].astype(np.int64), zeros[:nz.value].astype(np.int64)


def set_shard_draws(on):
    """Engine option OGCP_OPT_SHARD_DRAWS: multi-GPU merged draws sharded by RNG word range
    (0: every rank replays the whole stream)."""
    check(lib().ogcp_ctx_set_option(ctx(), 11, int(bool(on))))


def set_sort_zeros(mode):
    """Engine option OGCP_OPT_SORT_ZEROS: zero rows of bucketed merged draws in walk order
    (0 off, 1 / True by (bucket, mode-0 row), 2 by bucket only)."""
    check(lib().ogcp_ctx_set_option(ctx(), 5, int(mode)))


def set_lean_walks(on: bool):
    """Engine option OGCP_OPT_LEAN_WALKS: specialised 3-way walk kernels for merged sets."""
    check(lib().ogcp_ctx_set_option(ctx(), 6, int(bool(on))))


def set_tma_walks(on: bool, wgrad: bool = False, a2_resident: bool = False):
    """Engine option OGCP_OPT_TMA_WALKS: TMA-fed warp-specialised walks for merged 3-way sets
    (the K3 walk; `wgrad` also the weight-gradient walk; `a2_resident` keeps a small mode-2
    factor in shared memory)."""
    check(lib().ogcp_ctx_set_option(ctx(), 7, int(bool(on)) | (2 if wgrad else 0) | (4 if a2_resident else 0)))


def set_walk_impl(impl: str):
    """Select the sample-walk kernels for merged 3-way sets: "tma" (default: TMA K3 walk,
    generic weight walk), "tma-a2" (mode-2 factor resident in shared memory), "tma-all" (both
    walks TMA-fed), "lean" or "generic"."""
    set_tma_walks(impl in ("tma", "tma-all", "tma-a2"), wgrad=impl == "tma-all", a2_resident=impl == "tma-a2")
    set_lean_walks(impl == "lean")


def set_batch_draws(on: bool):
    """Engine option OGCP_OPT_BATCH_DRAWS: small draws of a solver epoch made at its start."""
    check(lib().ogcp_ctx_set_option(ctx(), 8, int(bool(on))))


def set_umma_gram(on: bool):
    """Engine option OGCP_OPT_UMMA_GRAM: ldr 64 / 128 Grams on tcgen05 / TMEM."""
    check(lib().ogcp_ctx_set_option(ctx(), 9, int(bool(on))))


def set_deterministic(on: bool):
    """Engine option OGCP_OPT_DETERMINISTIC: fixed-order (bitwise reproducible) K3 for small models."""
    check(lib().ogcp_ctx_set_option(ctx(), 10, int(bool(on))))


def set_split_scatter(on: bool):
    """Engine option OGCP_OPT_SPLIT_SCATTER for the current device's context."""
    check(lib().ogcp_ctx_set_option(ctx(), 2, int(bool(on))))
