"""Per-step breakdown of the c4 e2e loop: ingest, solve, per-kernel-class device ms, traces."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench
import paper_2110_14514_b200 as P
from paper_2110_14514_b200 import _lib
from paper_2110_14514_b200.synthetic import gen_slice

X, factors, mix, total = gen_slice(bench.DIMS, bench.NNZ, bench.RANK, "poisson", seed=42)
cfg = bench.make_cfg(P)
loss = P.make_loss("poisson")
st = bench.make_state(P, X, factors, mix, total, cfg, loss, seed=11)
P.process_slice(st, X, loss, cfg, exact_loss=False)
subs_pin = torch.from_numpy(np.array(X.subs0)).pin_memory()
vals_pin = torch.from_numpy(np.array(X.vals)).pin_memory()
s_np, v_np = subs_pin.numpy(), vals_pin.numpy()
L, ctx = _lib.lib(), _lib.ctx()
L.ogcp_ctx_profile_enable(ctx, 1)
for it in range(6):
    L.ogcp_ctx_profile_reset(ctx)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Xh = P.SparseTensor.from_zero_based(bench.DIMS, s_np, v_np) if it % 2 == 0 else X
    t1 = time.perf_counter()
    row = P.process_slice(st, Xh, loss, cfg, exact_loss=False)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    prof = {}
    for cls, name in enumerate(["draw", "sgrad", "wgrad", "objective", "gram", "update"]):
        n, tms = C.c_int64(), C.c_double()
        L.ogcp_ctx_profile_read(ctx, cls, C.byref(n), C.byref(tms))
        prof[name] = (int(n.value), round(tms.value, 1))
    tr = st.trace_log[-1]
    print(f"{'new' if it % 2 == 0 else 'same'} slice: ingest {1e3*(t1-t0):.0f} ms solve {1e3*(t2-t1):.0f} ms "
          f"prof {prof} wtrace {[round(v, 1) for v in tr[1]]} ftrace {[round(v, 1) for v in tr[2]]}", flush=True)
    if it % 2 == 0:
        del Xh
