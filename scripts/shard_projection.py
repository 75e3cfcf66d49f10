"""Per-rank work of an N-GPU c4 solve, projected on one GPU (NOT a multi-GPU measurement).

1. Measured: the context runs in shard-simulation mode (OGCP_OPT_SHARD_SIM) and
   executes exactly rank 0's share of a world-N solve -- its own ordinal range of the
   merged draws, its share of the zero rows, its owned rows of K5 / the Grams, and
   the draw words / probes every rank repeats -- with the NCCL collectives skipped.
2. Modeled: the per-step collectives of the real run, from their bytes at a stated
   NVLink bus bandwidth: per factor iteration one in-place reduce-scatter + one
   all-gather of every mode's factor rows (sum_k I_k * ldr * 4 bytes, (N-1)/N of it
   per rank each way) and a 2 d R^2 fp64 Gram all-reduce; per weight iteration an
   R-vector all-reduce; per objective one fp64 -- latency-bound ones at LAT_US.
3. Modeled: the same with the draw sharded by word range:
   the write and probe passes (measured per launch at N = 1 from the launch list,
   SHARDABLE_MS) divided by N, plus a reduce-scatter of 8-bit ordinal counters
   (eta bytes) and a tiny all-gather of miss counts per draw.

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
# per-draw c4 kernel time that word-range sharding divides by N (r02 launch list, ms):
# k_draw_write<1> 0.483 + k_draw_write<3> 0.218 + k_zero_hits 0.320
SHARDABLE_MS = 1.021


def collectives_ms(world, ldr=32):
    if world == 1:
        return 0.0
    rows = sum(bench.DIMS)
    grad = rows * ldr * 4 * (world - 1) / world / (BUS_GBS * 1e9) * 1e3  # one RS or AG, ms
    per_factor = 2 * grad + LAT_US / 1e3  # RS + AG of the rows + Gram all-reduce
    per_weight = LAT_US / 1e3
    return 100 * per_factor + 100 * per_weight + 4 * LAT_US / 1e3


def sharded_draw_saving_ms(world):
    if world == 1:
        return 0.0
    eta = bench.NNZ
    rs = eta * (world - 1) / world / (BUS_GBS * 1e9) * 1e3  # 8-bit counters to the ordinal owners
    per_draw = SHARDABLE_MS * (1 - 1 / world) - rs - LAT_US / 1e3
    return 200 * per_draw  # one draw per weight and per factor iteration


def main(worlds):
    X, factors, mix, total = gen_slice(bench.DIMS, bench.NNZ, bench.RANK, "poisson", seed=42)
    cfg = bench.make_cfg(P)
    loss = P.make_loss("poisson")
    L, ctx = _lib.lib(), _lib.ctx()
    base = None
    rows = []
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
        step = e0.elapsed_time(e1) / 2
        coll = collectives_ms(world)
        now = step + coll
        sharded = max(now - sharded_draw_saving_ms(world), 0.0)
        base = base or now
        row = {"N": world, "rank0_step_ms_measured": round(step, 1), "collectives_ms_modeled": round(coll, 1),
               "step_ms_current_design": round(now, 1), "speedup_current": round(base / now, 2),
               "step_ms_with_sharded_draw": round(sharded, 1), "speedup_with_sharded_draw": round(base / sharded, 2),
               "per_step_bracket_ms": prof}
        rows.append(row)
        print(json.dumps(row), flush=True)
    print(json.dumps({"assumptions": {"bus_gbs": BUS_GBS, "small_collective_latency_us": LAT_US,
                                      "shardable_draw_ms_per_draw": SHARDABLE_MS,
                                      "note": "projection: rank-0 kernels measured on one B200 in shard-simulation "
                                              "mode; collectives and the sharded draw modeled from bytes"}}))


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 4, 8])
