"""Throughput of the §8(d) configs beside the c4 headline (one B200, slice resident).

    python scripts/config_bench.py c3 [--semi]       # Bernoulli 100Kx100Kx1K, 1e7 nnz, R=16
    python scripts/config_bench.py c5 --rank 64     # Poisson 100Kx100Kx1K, 1e7 nnz, H=500, w=10, theta=0.99

c3: kappa 5/5, tau 100, rate_w 0.1, rate_f 1e-3, w 10, H 50, p = q = 2^21, p' = q' = 2^22
    (stratified = the reference's estimator; --semi = the semi-stratified extension).
c5: the c3 Poisson variant with H = 500 (window pre-filled), w = 10, theta = 0.99, p = q = 2^21.
One JSON line: entries/s over the timed slices (weight + factor iterations x (p+q)),
ms per slice, per-class kernel ms per slice and the K4 (Gram) + K5 share.
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2110_14514_b200 as P  # noqa: E402
from paper_2110_14514_b200 import _lib  # noqa: E402
from paper_2110_14514_b200.synthetic import gen_slice  # noqa: E402

DIMS = (100_000, 100_000, 1_000)
NNZ = 10_000_000


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=("c3", "c5"))
    ap.add_argument("--semi", action="store_true")
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--slices", type=int, default=2)
    args = ap.parse_args()
    if os.environ.get("OGCP_BUCKETS") == "0":
        _lib.set_buckets(False)
    if os.environ.get("OGCP_UMMA") == "0":  # A/B knob: mma.sync Grams instead of tcgen05 / TMEM
        _lib.set_umma_gram(False)
    kind = "bernoulli" if args.config == "c3" else "poisson"
    R = 16 if args.config == "c3" else args.rank
    H = 50 if args.config == "c3" else 500
    X, factors, mix, total = gen_slice(DIMS, NNZ, R, kind, seed=42)
    p = q = 1 << 21
    cfg = P.SolverConfig(max_epochs_weights=5, max_epochs_factors=5, iters_weights=100, iters_factors=100,
                         rate_weights=0.1, rate_factors=1e-3, hist_weight=10.0,
                         hist_decay=0.99 if args.config == "c5" else 1.0, warm_start_weights=True,
                         samples=P.SamplerConfig(p, q, 1 << 22, 1 << 22, seed=7, semi_stratified=args.semi))
    loss = P.make_loss(kind)
    rng = np.random.default_rng(11)
    init = [a * (1.0 + 0.05 * rng.uniform(-1, 1, a.shape)) for a in factors]
    st = P.fresh_state(DIMS, R, loss, cfg, factors=init)
    st.window = P.HistoryWindow(capacity=H)
    w = (total * np.asarray(mix)) if kind == "poisson" else np.asarray(mix) * 0.5
    for h in range(1, H + 1):
        s_h = w * (1.0 + 0.05 * rng.uniform(-1, 1, w.shape))
        st.weights_log.append(s_h)
        st.window.observe(h, s_h, P.rng_at(cfg.samples.seed, h, 5))
    st.t = H
    P.process_slice(st, X, loss, cfg, exact_loss=False)  # warm-up
    torch.cuda.synchronize()
    L, ctx = _lib.lib(), _lib.ctx()
    L.ogcp_ctx_profile_reset(ctx)
    L.ogcp_ctx_profile_enable(ctx, 1)
    t_first = st.t
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.slices):
        P.process_slice(st, X, loss, cfg, exact_loss=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    prof = {}
    for cls, name in enumerate(["draw", "sgrad", "wgrad", "objective", "gram", "update"]):
        n, tms = C.c_int64(), C.c_double()
        L.ogcp_ctx_profile_read(ctx, cls, C.byref(n), C.byref(tms))
        prof[name] = round(tms.value / args.slices, 2)
    L.ogcp_ctx_profile_enable(ctx, 0)
    iters = sum(m.epochs_weights * cfg.iters_weights + m.epochs_factors * cfg.iters_factors
                for m in st.metrics if m.t > t_first)
    print(json.dumps({"config": args.config + ("-semi" if args.semi else ""), "rank": R, "H": H,
                      "entries_per_s": iters * (p + q) / (ms / 1000.0), "ms_per_slice": ms / args.slices,
                      "iterations_per_slice": iters / args.slices, "kernel_ms_per_slice": prof,
                      "gram_k5_share": (prof["gram"] + prof["update"]) / (ms / args.slices)}), flush=True)


if __name__ == "__main__":
    main()
