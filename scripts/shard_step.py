"""One c4 slice as rank 0 of a world-N solve in shard-simulation timing mode, for an ncu
launch list of the per-rank work (the measured step is bracketed by cudaProfilerStart/Stop):

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv ... python scripts/shard_step.py N
"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2110_14514_b200 as P  # noqa: E402
from paper_2110_14514_b200 import _lib  # noqa: E402
from paper_2110_14514_b200.synthetic import gen_slice  # noqa: E402


def main(world):
    X, factors, mix, total = gen_slice(bench.DIMS, bench.NNZ, bench.RANK, "poisson", seed=42)
    cfg = bench.make_cfg(P)
    loss = P.make_loss("poisson")
    st = bench.make_state(P, X, factors, mix, total, cfg, loss, seed=11)
    _lib.set_shard_sim(0, world, timing=True)
    for _ in range(2):
        P.process_slice(st, X, loss, cfg, exact_loss=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.cudart().cudaProfilerStart()
    e0.record()
    P.process_slice(st, X, loss, cfg, exact_loss=False)
    e1.record()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print(f"world {world}: step {e0.elapsed_time(e1):.1f} ms", flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 8)
