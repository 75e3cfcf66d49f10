"""Slices/s of the small streaming configs on their reference streams (BASELINE configs[0] c1,
configs[1] c2), resumed from the reference's own warm-start checkpoint.

    python scripts/stream_bench.py [--config c1|c2] [--slices N] [--warmup W] [--profile]

c1: gen_gaussian 30x40x50 per slice, R = 5, synthetic-gaussian preset (kappa_w = 20, kappa_f = 5,
    tau = 100, p = p' = 10000, q = q' = 0, H = 50).
c2: gen_poisson 32x77x24 per slice (~906 nnz), R = 10, chicago-binary schedule with Poisson loss
    (kappa 5/5, tau = 100, p = p' = all, q = 1000, q' = 10000, w = 10, H = 500, warm weights).
The data is regenerated bit-exactly (oracle/synthetic_ref.py, pinned by the reference's SHA-256)
and the per-slice fits are compared with the reference's (tests/golden/stream_<cfg>.npz), so the
timing is of the same stream the parity test checks.  Latency-bound: microseconds of work per
iteration; reported beside the c4 throughput line, not as the headline.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=("c1", "c2"))
    ap.add_argument("--slices", type=int, default=0, help="timed slices (0: the rest of the stream)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--profile", action="store_true", help="also report per-kernel-class device ms per slice")
    args = ap.parse_args()
    import torch
    import paper_2110_14514_b200 as P
    from test_gpu_streams import stream_config, stream_data, ckpt_path
    if os.environ.get("OGCP_DET") == "1":  # fixed-order (bitwise reproducible) factor-gradient scatter
        P._lib.set_deterministic(True)
    golden = os.path.join(ROOT, "tests", "golden")
    g = np.load(os.path.join(golden, f"stream_{args.config}.npz"))
    cfg, loss = stream_config(args.config)
    dims, subs0, vals = stream_data(g)
    from oracle.synthetic_ref import slice_of
    t0s = int(g["t_first"]) - 1
    st = P.load_checkpoint(ckpt_path(golden, args.config, t0s), loss, cfg)
    n_all = int(g["metrics"].shape[0])
    n = args.slices or (n_all - args.warmup)
    slices = []
    for t in range(t0s + 1, t0s + args.warmup + n + 1):
        s, v = slice_of(subs0, vals, t)
        slices.append(P.SparseTensor.from_zero_based(dims[:-1], s, v))
    for X in slices[: args.warmup]:
        P.process_slice(st, X, loss, cfg, exact_loss=False)
    torch.cuda.synchronize()
    if args.profile:
        P._lib.lib().ogcp_ctx_profile_reset(P._lib.ctx())
        P._lib.lib().ogcp_ctx_profile_enable(P._lib.ctx(), 1)
    l0 = P._lib.launches()
    t0 = time.perf_counter()
    rows = [P.process_slice(st, X, loss, cfg, exact_loss=False) for X in slices[args.warmup:]]
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    iters = sum(r.epochs_weights * cfg.iters_weights + r.epochs_factors * cfg.iters_factors for r in rows)
    ref = g["metrics"]
    ours = np.array([[r.t, r.local_loss_sampled] for r in rows])
    sel = ref[np.isin(ref[:, 0], ours[:, 0])]
    rel = np.abs(ours[:, 1] - sel[:, 1]) / np.abs(sel[:, 1])
    line = {"config": args.config, "slices": n, "slices_per_s": n / dt, "ms_per_slice": 1e3 * dt / n,
            "us_per_iteration": 1e6 * dt / max(iters, 1), "launches_per_iteration": (P._lib.launches() - l0) / max(iters, 1),
            "max_rel_sampled_fit_vs_reference": float(rel.max()),
            "reference_s_per_slice": float(g["ref_seconds"]) / n_all}
    if args.profile:
        import ctypes as C
        prof = {}
        for cls, name in enumerate(["draw", "sgrad", "wgrad", "objective", "gram", "update"]):
            nb, tms = C.c_int64(), C.c_double()
            P._lib.lib().ogcp_ctx_profile_read(P._lib.ctx(), cls, C.byref(nb), C.byref(tms))
            prof[name] = round(tms.value / n, 3)
        line["bracket_ms_per_slice"] = prof
    print(json.dumps(line))


if __name__ == "__main__":
    main()
