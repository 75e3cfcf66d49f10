"""Slices/s of small streaming configs (BASELINE configs[0] c1 and configs[1] c2).

    python scripts/stream_bench.py [--config c1|c2] [--slices N]

c1: dense Gaussian 30x40x50 per slice, R = 5, preset synthetic-gaussian schedule
    (kappa_w = 20, kappa_f = 5, tau = 100, p = p' = 10000, q = q' = 0, H = 50).
c2: Chicago-shaped Poisson 32x77x24 per slice, ~906 nnz/slice, R = 10, chicago-binary
    schedule with Poisson loss (kappa = 5/5, tau = 100, p = p' = all, q = 1000,
    q' = 10000, w = 10, H = 500, warm weights).
These are latency-bound (microseconds of work per iteration); reported beside the
c4 throughput line, not as the headline.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def planted(dims, rank, seed, kind):
    rng = np.random.default_rng(seed)
    if kind == "gaussian":
        A = [rng.uniform(size=(d, rank)) for d in dims]
        dense = np.einsum("ir,jr,kr,tr->ijkt", *A) + rng.normal(0.0, 0.2, size=dims)
        dense[dense == 0] = 1e-300
        subs0 = np.indices(dims).reshape(len(dims), -1).T
        return subs0, dense.ravel(), A[:-1]
    # sparse Poisson counts at ~1.6% density
    cells = int(np.prod(dims))
    lin = np.unique(rng.integers(0, cells, size=int(cells * 0.0162)))
    subs0 = np.array(np.unravel_index(lin, dims)).T
    vals = rng.poisson(1.0, size=lin.size).astype(float) + 1.0
    A = [rng.uniform(0.05, 1.0, size=(d, rank)) for d in dims[:-1]]
    return subs0, vals, A


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=("c1", "c2"))
    ap.add_argument("--slices", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--profile", action="store_true", help="also report per-kernel-class device ms per slice")
    args = ap.parse_args()
    import torch
    import paper_2110_14514_b200 as P

    if args.config == "c1":
        dims, R, kind = (30, 40, 50, args.slices + args.warmup + 1), 5, "gaussian"
        cfg = P.SolverConfig(max_epochs_weights=20, max_epochs_factors=5, rate_weights=10.0, rate_factors=1e-4,
                             hist_weight=1.0, samples=P.SamplerConfig(10000, 0, 10000, 0, seed=7))
        H = 50
    else:
        dims, R, kind = (32, 77, 24, args.slices + args.warmup + 1), 10, "poisson"
        cfg = P.SolverConfig(max_epochs_weights=5, max_epochs_factors=5, rate_weights=0.1, rate_factors=1e-3,
                             hist_weight=10.0, warm_start_weights=True,
                             samples=P.SamplerConfig(None, 1000, None, 10000, seed=7))
        H = 500
    subs0, vals, A = planted(dims, R, 42, kind)
    loss = P.make_loss(kind)
    st = P.fresh_state(dims[:-1], R, loss, cfg, factors=A)
    st.window = P.HistoryWindow(capacity=H)
    rng = np.random.default_rng(3)
    for h in range(1, 21):
        s_h = rng.uniform(0.5, 1.5, R) * (vals.sum() / dims[-1] / R if kind == "poisson" else 1.0)
        st.weights_log.append(s_h)
        st.window.observe(h, s_h, P.rng_at(7, h, 5))
    st.t = 20
    slices = []
    for t in range(dims[-1]):
        m = subs0[:, -1] == t
        slices.append(P.SparseTensor.from_zero_based(dims[:-1], subs0[m, :-1], vals[m]))
    for X in slices[: args.warmup]:
        P.process_slice(st, X, loss, cfg, exact_loss=False)
    torch.cuda.synchronize()
    if args.profile:
        P._lib.lib().ogcp_ctx_profile_reset(P._lib.ctx())
        P._lib.lib().ogcp_ctx_profile_enable(P._lib.ctx(), 1)
    t0 = time.perf_counter()
    for X in slices[args.warmup: args.warmup + args.slices]:
        P.process_slice(st, X, loss, cfg, exact_loss=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    iters = sum(r.epochs_weights * cfg.iters_weights + r.epochs_factors * cfg.iters_factors
                for r in st.metrics[-args.slices:])
    line = {"config": args.config, "slices_per_s": args.slices / dt, "ms_per_slice": 1e3 * dt / args.slices,
            "us_per_iteration": 1e6 * dt / max(iters, 1), "launches": P._lib.launches()}
    if args.profile:
        import ctypes as C
        prof = {}
        for cls, name in enumerate(["draw", "sgrad", "wgrad", "objective", "gram", "update"]):
            n, tms = C.c_int64(), C.c_double()
            P._lib.lib().ogcp_ctx_profile_read(P._lib.ctx(), cls, C.byref(n), C.byref(tms))
            prof[name] = round(tms.value / args.slices, 2)
        line["device_ms_per_slice"] = prof
    print(json.dumps(line))


if __name__ == "__main__":
    main()
