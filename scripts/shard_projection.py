"""Per-rank work of an N-GPU c4 solve, projected on one GPU (not a multi-GPU measurement).

The context runs in shard-simulation mode (OGCP_OPT_SHARD_SIM): the solves execute
exactly rank 0's share of a world-N solve -- its own ordinal range of the merged
draws, its share of the zero rows, the replicated draw words / Grams / K5 -- with
the NCCL collectives skipped (so the iterates differ from a real run; the work per
kernel does not).  The printed step time therefore excludes the per-iteration
all-reduces (factor gradients 256 MB fp32, R-vector and scalar fp64).

    python scripts/shard_projection.py [N ...]
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2110_14514_b200 as P  # noqa: E402
from paper_2110_14514_b200 import _lib  # noqa: E402
from paper_2110_14514_b200.synthetic import gen_slice  # noqa: E402


def main(worlds):
    X, factors, mix, total = gen_slice(bench.DIMS, bench.NNZ, bench.RANK, "poisson", seed=42)
    cfg = bench.make_cfg(P)
    loss = P.make_loss("poisson")
    L, ctx = _lib.lib(), _lib.ctx()
    for world in worlds:
        st = bench.make_state(P, X, factors, mix, total, cfg, loss, seed=11)
        _lib.set_shard_sim(0, world)
        for _ in range(2):
            P.process_slice(st, X, loss, cfg, exact_loss=False)
        torch.cuda.synchronize()
        L.ogcp_ctx_profile_reset(ctx)
        L.ogcp_ctx_profile_enable(ctx, 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(2):
            P.process_slice(st, X, loss, cfg, exact_loss=False)
        e1.record()
        torch.cuda.synchronize()
        prof = {}
        for cls, name in enumerate(["draw", "sgrad", "wgrad", "objective", "gram", "update"]):
            n, tms = C.c_int64(), C.c_double()
            L.ogcp_ctx_profile_read(ctx, cls, C.byref(n), C.byref(tms))
            prof[name] = round(tms.value / 2, 1)
        L.ogcp_ctx_profile_enable(ctx, 0)
        _lib.set_shard_sim(0, 1)
        print(f"N={world}: rank-0 step {e0.elapsed_time(e1) / 2:.0f} ms (collectives excluded); "
              f"per-step ms by kernel class {prof}", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 4, 8])
