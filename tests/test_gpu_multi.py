"""Multi-GPU solves with real NCCL (needs >= 2 GPUs; skipped otherwise -- every
box of this build has one, so the shard partition itself is covered in one
process by tests/test_gpu_shard.py and tests/test_gpu_c4_draw.py).

Two ranks run the same stream with the engine's communicators (word-range sharded
merged draws, reduce-scatter / all-gather owner-computes row updates): the ranks'
factors must be bitwise identical, and the per-slice fits must match the
single-GPU run of the same stream (sample sums in another order: 1e-4)."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(tmp, world):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    if world == 1:
        cmd = [sys.executable, os.path.join(HERE, "multi_gpu_worker.py"), str(tmp), "1"]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", "29533",
               os.path.join(HERE, "multi_gpu_worker.py"), str(tmp), str(world)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_two_gpu_stream_matches_single_gpu(tmp_path):
    one, two = tmp_path / "one", tmp_path / "two"
    one.mkdir()
    two.mkdir()
    _run(one, 1)
    _run(two, 2)
    a, b, s = np.load(two / "rank0.npz"), np.load(two / "rank1.npz"), np.load(one / "rank0.npz")
    for k in a.files:
        np.testing.assert_array_equal(a[k], b[k])  # every rank ends with the same model
    np.testing.assert_allclose(a["fits"], s["fits"], rtol=1e-4)
