"""Long-stream golden fixtures at BASELINE configs c1 / c2, from the REFERENCE itself.

Build container only (/root/reference does not exist on the GPU box).  Runs the
reference package ``ogcp`` through its own public API -- gen_gaussian /
gen_poisson, warm_start, process_slice, save_checkpoint -- exactly as the
reference's acceptance criteria 6/7 do (pkg/tests/test_acceptance.py:252-330)
but at the BASELINE shapes, and writes:

  tests/golden/stream_<cfg>.npz          per-slice metrics, temporal rows, epoch
                                         traces, data SHA-256, final factors
  tests/golden/stream_<cfg>_ckpt_<t>.npz reference-written checkpoints
                                         (streaming.py:218-246) after warm start
                                         and at intermediate slices

The GPU test (tests/test_gpu_streams.py) regenerates the data with
oracle/synthetic_ref.py (checked against data_sha256), loads the reference
checkpoint into the engine and runs the same stream.

  python scripts/make_stream_golden.py c1      # ~20 min on 1 core
  python scripts/make_stream_golden.py c2      # ~25 min on 1 core
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def configs(ogcp):
    from ogcp import SamplerConfig, SolverConfig
    c1 = dict(
        kind="gaussian", dims=(30, 40, 50, 100), rank=5, seed=42, noise=0.2, loss=("gaussian", 1e-10),
        # preset synthetic-gaussian (cli.py:39-42) at R = 5; sampler seed 7 (test_acceptance.py:265)
        cfg=SolverConfig(max_epochs_weights=20, max_epochs_factors=5, iters_weights=100, iters_factors=100,
                         rate_weights=10.0, rate_factors=1e-4, hist_weight=1.0, hist_decay=1.0,
                         samples=SamplerConfig(grad_nonzeros=10000, grad_zeros=0, obj_nonzeros=10000,
                                               obj_zeros=0, seed=7)),
        warm=10, hist=50, warm_kw=dict(max_epochs=60, iters_per_epoch=50, rate=0.02),
        stream=90, ckpt_every=30)
    c2 = dict(
        kind="poisson", dims=(32, 77, 24, 5000), rank=10, seed=42, density=0.016, loss=("poisson", 1e-10),
        # chicago-binary schedule (cli.py:51-54) with Poisson loss, R = 10
        cfg=SolverConfig(max_epochs_weights=5, max_epochs_factors=5, iters_weights=100, iters_factors=100,
                         rate_weights=0.1, rate_factors=1e-3, hist_weight=10.0, hist_decay=1.0,
                         rate_decay=0.1, warm_start_weights=True,
                         samples=SamplerConfig(grad_nonzeros=None, grad_zeros=1000, obj_nonzeros=None,
                                               obj_zeros=10000, seed=7)),
        warm=20, hist=500, warm_kw=dict(max_epochs=50),
        stream=500, ckpt_every=100)
    return dict(c1=c1, c2=c2)


def main(name):
    sys.path.insert(0, REF)
    import ogcp
    from ogcp import make_loss, process_slice, save_checkpoint, warm_start
    from ogcp.io import leading_block
    from ogcp.synthetic import SyntheticSpec, gen_gaussian, gen_poisson
    from oracle.synthetic_ref import data_sha256

    c = configs(ogcp)[name]
    t0 = time.time()
    if c["kind"] == "gaussian":
        X, truth = gen_gaussian(SyntheticSpec("gaussian", dims=c["dims"], rank=c["rank"], noise=c["noise"],
                                              seed=c["seed"]))
    else:
        X, truth = gen_poisson(SyntheticSpec("poisson", dims=c["dims"], rank=c["rank"], density=c["density"],
                                             seed=c["seed"]))
    print(f"{name}: data {X.dims} nnz={X.nnz} in {time.time() - t0:.1f}s", flush=True)
    loss = make_loss(*c["loss"])
    cfg = c["cfg"]
    state = warm_start(leading_block(X, c["warm"]), c["rank"], loss, cfg, history_capacity=c["hist"],
                       **c["warm_kw"])
    save_checkpoint(state, os.path.join(OUT, f"stream_{name}_ckpt_{state.t:04d}.npz"))
    print(f"{name}: warm start done t={state.t} ({time.time() - t0:.1f}s)", flush=True)
    rows = []
    traces_w, traces_f = [], []
    weights = []
    t_first = state.t + 1
    for t in range(t_first, t_first + c["stream"]):
        m = process_slice(state, X.slice_view(t), loss, cfg, exact_loss=True)
        rows.append([m.t, m.local_loss_sampled, m.local_loss_exact, m.epochs_weights, m.epochs_factors])
        _, wt, ft = state.trace_log[-1]
        traces_w.append(np.asarray(wt, dtype=np.float64))
        traces_f.append(np.asarray(ft, dtype=np.float64))
        weights.append(np.array(state.weights_log[-1]))
        if (t - t_first + 1) % c["ckpt_every"] == 0 or t == t_first + c["stream"] - 1:
            save_checkpoint(state, os.path.join(OUT, f"stream_{name}_ckpt_{t:04d}.npz"))
        if (t - t_first) % 10 == 0:
            print(f"{name}: t={t} exact={m.local_loss_exact:.6g} ep={m.epochs_weights}/{m.epochs_factors} "
                  f"({time.time() - t0:.0f}s)", flush=True)
    off_w = np.cumsum([0] + [len(a) for a in traces_w])
    off_f = np.cumsum([0] + [len(a) for a in traces_f])
    np.savez_compressed(
        os.path.join(OUT, f"stream_{name}.npz"),
        dims=np.array(c["dims"]), rank=np.array(c["rank"]), seed=np.array(c["seed"]),
        data_sha256=np.array(data_sha256(X.subs0, X.vals)), nnz=np.array(X.nnz),
        warm=np.array(c["warm"]), t_first=np.array(t_first), metrics=np.array(rows),
        weights=np.array(weights), trace_w=np.concatenate(traces_w), trace_w_off=off_w,
        trace_f=np.concatenate(traces_f), trace_f_off=off_f,
        **{f"factor_{k}": a for k, a in enumerate(state.factors)},
        truth_weights=np.asarray(truth.weights), **{f"truth_{k}": a for k, a in enumerate(truth.factors)},
        ref_seconds=np.array(time.time() - t0))
    print(f"{name}: done in {time.time() - t0:.0f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1])
