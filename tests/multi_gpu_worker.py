"""Worker of tests/test_gpu_multi.py (launched by torchrun, one process per GPU).

Runs the same short stream on every rank with the engine's NCCL communicator
(word-range sharded merged draws, reduce-scatter / all-gather row updates) and
writes this rank's final factors, weights and per-slice fits to OUT/rank<r>.npz.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_14514_b200 as P  # noqa: E402
from paper_2110_14514_b200 import distributed as PD  # noqa: E402


def stream(seed=3):
    rng = np.random.default_rng(seed)
    dims = (6000, 2500, 40)  # mode 0 past the small-model size: owner-computes row updates
    T = 4
    subs, vals = [], []
    for t in range(T):
        lin = rng.choice(int(np.prod(dims)), size=150_000, replace=False)
        s = np.array(np.unravel_index(np.sort(lin), dims)).T
        subs.append(np.column_stack([s, np.full(len(s), t)]))
        vals.append(rng.integers(1, 5, size=len(s)).astype(float))
    return dims + (T,), np.concatenate(subs), np.concatenate(vals)


def main(out, world_expected):
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world_expected > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        PD.init_sharded_solves()
    dims, subs0, vals = stream()
    X = P.SparseTensor.from_zero_based(dims, subs0, vals)
    loss = P.make_loss("poisson")
    cfg = P.SolverConfig(max_epochs_weights=2, iters_weights=10, max_epochs_factors=2, iters_factors=10,
                         rate_factors=1e-3, samples=P.SamplerConfig(None, 20000, 20000, 20000, seed=7))
    slices = list(P.stream_slices(X))
    st = P.warm_start(P.leading_block(X, 1), 8, loss, cfg, 5)
    rows = P.run_stream(st, slices[1:], loss, cfg, exact_loss=False)
    fits = np.array([r.local_loss_sampled for r in rows])
    np.savez(os.path.join(out, f"rank{rank}.npz"), *[np.asarray(f) for f in st.factors],
             weights=np.asarray(st.weights_log[-1]), fits=fits)
    if world_expected > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
