import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import bench
import paper_2110_14514_b200 as P
from paper_2110_14514_b200.synthetic import gen_slice
X, factors, mix, total = gen_slice(bench.DIMS, bench.NNZ, bench.RANK, "poisson", seed=42)
cfg = bench.make_cfg(P); loss = P.make_loss("poisson")
st = bench.make_state(P, X, factors, mix, total, cfg, loss, seed=11)
s_np = np.array(X.subs0); v_np = np.array(X.vals)
for i in range(8):
    Xh = P.SparseTensor.from_zero_based(bench.DIMS, s_np, v_np)
    P.process_slice(st, Xh, loss, cfg, exact_loss=False)
    del Xh
    torch.cuda.synchronize()
    free, tot = torch.cuda.mem_get_info()
    print(f"slice {i}: device used {(tot - free) / 2**30:.2f} GiB", flush=True)
