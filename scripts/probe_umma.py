"""Probe the tcgen05 Gram against numpy on small single-mode models."""
import numpy as np
import paper_2110_14514_b200 as P
from paper_2110_14514_b200 import _lib

rng = np.random.default_rng(0)
for R, rows in [(128, 32), (128, 64), (128, 300), (64, 32), (64, 100), (40, 40)]:
    A = rng.uniform(-1, 1, (rows, R))
    for umma in (True, False):
        _lib.set_umma_gram(umma)
        g = P.gram([A], None)
        want = A.T @ A
        err = np.linalg.norm(g - want) / np.linalg.norm(want)
        print(R, rows, "umma" if umma else "mma.sync", f"rel err {err:.3e}", "g[0,:4]", np.round(g[0, :4], 3),
              "want", np.round(want[0, :4], 3), flush=True)
_lib.set_umma_gram(True)
