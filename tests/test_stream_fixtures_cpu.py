"""CPU checks of the long-stream fixtures (no GPU).

* oracle/synthetic_ref.py regenerates the c1 / c2 data tensors bit for bit (the
  SHA-256 the reference's own generator produced, scripts/make_stream_golden.py).
* The reference-written checkpoints carry the reference's schema
  (streaming.py:218-246) and are mutually consistent with the per-slice record.
* Engine-written checkpoints (tests/golden/engine_ckpt_*.npz, produced on a B200
  by tests/test_gpu_streams.py with OGCP_ENGINE_CKPT_OUT) load in the reference's
  own load_checkpoint and resume the reference stream (checkpoint interop,
  engine -> reference); that part runs where /root/reference exists.
"""

import glob
import json
import os
import sys

import numpy as np
import pytest

from oracle import synthetic_ref as SR

REF_SRC = "/root/reference/pkg/src"


def _fixture(golden_dir, name):
    return np.load(os.path.join(golden_dir, f"stream_{name}.npz"))


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_restated_generator_matches_reference_sha(golden_dir, name):
    g = _fixture(golden_dir, name)
    dims = tuple(int(d) for d in g["dims"])
    if name == "c1":
        subs0, vals, _ = SR.gen_gaussian(dims, int(g["rank"]), noise=0.2, seed=int(g["seed"]))
    else:
        subs0, vals, _, _ = SR.gen_poisson(dims, int(g["rank"]), density=0.016, seed=int(g["seed"]))
    assert vals.size == int(g["nnz"])
    assert SR.data_sha256(subs0, vals) == str(g["data_sha256"])


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_reference_checkpoints_consistent(golden_dir, name):
    g = _fixture(golden_dir, name)
    paths = sorted(glob.glob(os.path.join(golden_dir, f"stream_{name}_ckpt_*.npz")))
    assert len(paths) >= 2
    for p in paths:
        z = np.load(p)
        h = json.loads(bytes(z["header"]).decode())
        assert h["version"] == 1 and h["rank"] == int(g["rank"]) and h["ndim"] == 3
        t = h["t"]
        assert z["weights_log"].shape == (t, int(g["rank"]))
        if t >= int(g["t_first"]):  # its temporal rows are the per-slice record's
            k = t - int(g["t_first"]) + 1
            np.testing.assert_array_equal(z["weights_log"][-k:], g["weights"][:k])


def _ref():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference tree not present (build container only)")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import ogcp
    return ogcp


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_engine_checkpoint_resumes_in_reference(golden_dir, name):
    paths = sorted(glob.glob(os.path.join(golden_dir, f"engine_ckpt_{name}_*.npz")))
    if not paths:
        pytest.skip("no engine-written checkpoint committed yet")
    ogcp = _ref()
    from ogcp import load_checkpoint, process_slice, make_loss, SamplerConfig, SolverConfig
    g = _fixture(golden_dir, name)
    if name == "c1":
        cfg = SolverConfig(max_epochs_weights=20, max_epochs_factors=5, iters_weights=100, iters_factors=100,
                           rate_weights=10.0, rate_factors=1e-4, hist_weight=1.0, hist_decay=1.0,
                           samples=SamplerConfig(grad_nonzeros=10000, grad_zeros=0, obj_nonzeros=10000,
                                                 obj_zeros=0, seed=7))
        loss = make_loss("gaussian", 1e-10)
        subs0, vals, _ = SR.gen_gaussian(tuple(int(d) for d in g["dims"]), int(g["rank"]), 0.2, int(g["seed"]))
    else:
        cfg = SolverConfig(max_epochs_weights=5, max_epochs_factors=5, iters_weights=100, iters_factors=100,
                           rate_weights=0.1, rate_factors=1e-3, hist_weight=10.0, hist_decay=1.0, rate_decay=0.1,
                           warm_start_weights=True,
                           samples=SamplerConfig(grad_nonzeros=None, grad_zeros=1000, obj_nonzeros=None,
                                                 obj_zeros=10000, seed=7))
        loss = make_loss("poisson", 1e-10)
        subs0, vals, _, _ = SR.gen_poisson(tuple(int(d) for d in g["dims"]), int(g["rank"]), 0.016, int(g["seed"]))
    state = load_checkpoint(paths[-1], loss, cfg)     # the reference's own reader
    t = state.t + 1
    s, v = SR.slice_of(subs0, vals, t)
    X = ogcp.SparseTensor.from_zero_based(tuple(int(d) for d in g["dims"][:-1]), s, v)
    m = process_slice(state, X, loss, cfg, exact_loss=True)
    ref = g["metrics"][g["metrics"][:, 0] == t]
    assert ref.shape[0] == 1
    assert abs(m.local_loss_exact - ref[0, 2]) <= 1e-3 * abs(ref[0, 2])
