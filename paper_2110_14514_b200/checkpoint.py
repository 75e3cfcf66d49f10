"""Stream checkpoints in the reference's .npz schema (pkg/src/ogcp/streaming.py:218-278).

Checkpoints move between the two implementations: the engine writes and reads
exactly the reference's keys.  Device state (factors, previous-step factors,
factor-Adam moments) is brought to the host in float64 on save and uploaded to
the engine layout on load.
"""

from __future__ import annotations

import json

import numpy as np

from .exceptions import DataError
from .metrics import SliceMetrics
from .tensor import DeviceModel

CHECKPOINT_VERSION = 1
_MOMENTS = ("u", "v", "u_o", "v_o", "a_o")
_METRIC_FIELDS = ("t", "local_loss_sampled", "local_loss_exact", "epochs_weights", "epochs_factors", "wall_ms")


def _stack_rows(rows, width):
    return np.vstack(rows) if rows else np.empty((0, width))


def save_checkpoint(state, path) -> None:
    """Versioned binary snapshot sufficient to resume exactly under the same config."""
    R = state.rank
    header = dict(version=CHECKPOINT_VERSION, t=state.t, iteration=state.iteration, ndim=len(state.dims), rank=R,
                  window_capacity=state.window.capacity, adam_rate=state.adam_factors.rate)
    out = {"header": np.frombuffer(json.dumps(header).encode(), dtype=np.uint8)}
    out.update({f"factor_{k}": a for k, a in enumerate(state.factors)})
    out.update({f"old_factor_{k}": a for k, a in enumerate(state.old_factors)})
    out["window_ids"] = np.asarray(state.window.step_ids(), dtype=np.int64)
    out["window_weights"] = _stack_rows([row for _, row in state.window.entries], R)
    out["weights_log"] = _stack_rows(state.weights_log, R)
    out["metrics"] = np.array([[getattr(m, f) for f in _METRIC_FIELDS] for m in state.metrics])
    for moment, parts in state.adam_factors.state_arrays().items():
        out.update({f"adam_{moment}_{k}": a for k, a in enumerate(parts)})
    np.savez(path, **out)


def load_checkpoint(path, loss, cfg):
    """Rebuild a StreamState from :func:`save_checkpoint` output (either implementation's)."""
    import torch

    from .streaming import HistoryWindow, StreamState
    with np.load(path) as z:
        header = json.loads(bytes(z["header"]).decode())
        if header["version"] != CHECKPOINT_VERSION:
            raise DataError(f"checkpoint version {header['version']} not supported")
        modes = range(header["ndim"])
        factors = DeviceModel.from_numpy([np.array(z[f"factor_{k}"]) for k in modes])
        old = DeviceModel.from_numpy([np.array(z[f"old_factor_{k}"]) for k in modes])
        window = HistoryWindow(capacity=header["window_capacity"],
                               entries=[(int(h), np.array(row)) for h, row in zip(z["window_ids"],
                                                                                   z["window_weights"])])
        adam = cfg.make_adam(header["adam_rate"], loss)
        adam.init_device(factors.dims, factors.rank)
        for moment in _MOMENTS:
            for k in modes:
                host = torch.from_numpy(np.asarray(z[f"adam_{moment}_{k}"], dtype=np.float32))
                adam._buf[moment][k][:, :factors.rank].copy_(host.cuda())
        weights_log = [np.array(r) for r in z["weights_log"]]
        ints = {"t", "epochs_weights", "epochs_factors"}
        metrics = [SliceMetrics(**{f: (int(v) if f in ints else v) for f, v in zip(_METRIC_FIELDS, r)})
                   for r in z["metrics"]]
    return StreamState(factors, old, window, adam, iteration=header["iteration"], t=header["t"],
                       weights_log=weights_log, metrics=metrics)
