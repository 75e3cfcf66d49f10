"""Per-rank work of an N-GPU c4 solve, projected on one GPU (NOT a multi-GPU measurement).

The context runs in timing shard simulation (OGCP_OPT_SHARD_SIM with the timing bit):
it executes exactly rank 0's share of a world-N solve -- its own ordinal range of the
merged draws, its zero rows, its owned rows of K5 / the Grams -- and every NCCL
collective is replaced in stream order by a stand-in kernel that holds 24 SMs (what an
NCCL ring / NVLS kernel holds) for the collective's modeled time: LAT_US plus the ring
bytes per rank at BUS_GBS (all-reduce 2 (N-1)/N of the buffer, reduce-scatter and
all-gather (N-1)/N of the full buffer).  The step is then timed on the device, so the
side-stream draws overlap the collectives (and compete with the walks) as they would.
Two draw designs:
* replicated: every rank generates every RNG word and probes every zero candidate
  (OGCP_OPT_SHARD_DRAWS 0);
* word-range sharded (the default): rank 0 generates its 1/N of the words; the other
  ranks' slots of the draw's all-gathers are stood in by its own.
Reported beside each: the stand-ins' total modeled time per step (no overlap).

    python scripts/shard_projection.py [N ...]  > profiles/r02_shard_projection.txt
"""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2110_14514_b200 as P  # noqa: E402
from paper_2110_14514_b200 import _lib  # noqa: E402
from paper_2110_14514_b200.synthetic import gen_slice  # noqa: E402

BUS_GBS = 700.0   # assumed NCCL ring/NVLS bus bandwidth per GPU on NVSwitch (NVLink 5: 900 GB/s per direction)
LAT_US = 15.0     # small-collective latency


def collectives_ms(world, sharded_draw, ldr=32):
    """The additive model's per-step collective time (ms)."""
    if world == 1:
        return 0.0
    rows = sum(bench.DIMS)
    grad = rows * ldr * 4 * (world - 1) / world / (BUS_GBS * 1e9) * 1e3  # one RS or AG, ms
    per_factor = 2 * grad + LAT_US / 1e3  # RS + AG of the rows + Gram all-reduce
    per_weight = LAT_US / 1e3
    per_draw = 0.0
    if sharded_draw:  # counters RS (eta / 2 bytes) + map / record all-gathers
        per_draw = bench.NNZ / 2 * (world - 1) / world / (BUS_GBS * 1e9) * 1e3 + 3 * LAT_US / 1e3
    return 100 * per_factor + 100 * per_weight + 200 * per_draw + 4 * LAT_US / 1e3


def measure(P, X, factors, mix, total, cfg, loss, world, shard_draws, timing):
    L, ctx = _lib.lib(), _lib.ctx()
    st = bench.make_state(P, X, factors, mix, total, cfg, loss, seed=11)
    _lib.set_shard_sim(0, world, timing=timing)
    _lib.set_shard_draws(shard_draws)
    try:
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
    finally:
        _lib.set_shard_sim(0, 1)
        _lib.set_shard_draws(1)
    del st
    torch.cuda.empty_cache()
    return e0.elapsed_time(e1) / 2, prof


def main(worlds):
    X, factors, mix, total = gen_slice(bench.DIMS, bench.NNZ, bench.RANK, "poisson", seed=42)
    cfg = bench.make_cfg(P)
    loss = P.make_loss("poisson")
    base = None
    for world in worlds:
        row = {"N": world}
        for tag, mode in (("replicated_draw", 0), ("sharded_draw", 1)):
            if world == 1 and mode:
                continue
            step, prof = measure(P, X, factors, mix, total, cfg, loss, world, mode, timing=True)
            base = base or step
            ent = {"step_ms": round(step, 1), "speedup": round(base / step, 2), "per_step_bracket_ms": prof}
            if world > 1:  # what the stand-ins add up to if none of them overlapped anything
                ent["collectives_ms_modeled_serial"] = round(collectives_ms(world, mode != 0), 1)
            row[tag] = ent
        print(json.dumps(row), flush=True)
    print(json.dumps({"assumptions": {"bus_gbs": BUS_GBS, "small_collective_latency_us": LAT_US,
                                      "note": "projection: rank 0's kernels measured on one B200 in timing shard "
                                              "simulation, every collective a 24-SM stand-in kernel of its modeled "
                                              "time in stream order (sharded draws: the other ranks' all-gather "
                                              "slots stood in by rank 0's own)"}}))


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 4, 8])
