"""CPU-only checks: host RNG restatement, C-ABI exports, host-side logic."""

import re
import os

import numpy as np
import pytest

from paper_2110_14514_b200 import _lib
from paper_2110_14514_b200.sampling import SamplerConfig, rng_at
from paper_2110_14514_b200.solvers import SolverConfig
from paper_2110_14514_b200.streaming import HistoryWindow
from paper_2110_14514_b200.exceptions import DataError
from oracle import ogcp_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "ogcp_b200.h")).read()
    names = set(re.findall(r"\b(ogcp_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 20
    lib = _lib.lib()
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.ogcp_abi_version() == 2


@pytest.mark.parametrize("seed,key,highs,n", [
    (0, (3,), [10], 50), (7, (4, 3, 0, 1), [1000000, 1000000, 1000], 999), (123456789012, (5000000000, 2), [77], 40),
    (1, (2, 1), [9, 4], 101), (5, (1, 1, 7, 99), [100000000], 3001), (11, (), [2**31 - 1], 64),
])
def test_host_rng_matches_numpy(seed, key, highs, n):
    g = O.keyed_rng(seed, *key)
    hi = np.array(highs)
    want = np.concatenate([g.integers(0, hi) for _ in range((n + len(hi) - 1) // len(hi))])[:n] \
        if len(hi) > 1 else g.integers(0, hi[0], size=n)
    got = _lib.rng_integers(seed, key, highs, n)
    np.testing.assert_array_equal(got, want)


def test_rng_state_matches_numpy_pcg64():
    for seed, key in [(0, ()), (7, (3, 1, 0, 5)), (2**40 + 3, (1, 2**33))]:
        st = _lib.rng_state(seed, key)
        bg = np.random.PCG64(np.random.SeedSequence(seed, spawn_key=key))
        s = bg.state["state"]
        assert (st[0] << 64 | st[1]) == s["state"]
        assert (st[2] << 64 | st[3]) == s["inc"]


def test_window_reservoir_matches_oracle():
    win = HistoryWindow(capacity=3)
    st = O.StreamOracle([], [], None, capacity=3)
    for t in range(1, 40):
        s = np.full(2, float(t))
        win.observe(t, s, rng_at(9, t, 5))
        O.window_observe(st, t, s, 9)
    assert win.step_ids() == [h for h, _ in st.window]


def test_config_validation_mirrors_reference():
    with pytest.raises(DataError):
        SamplerConfig(grad_zeros=-1)
    with pytest.raises(DataError):
        SolverConfig(hist_decay=0.0)
    with pytest.raises(DataError):
        SolverConfig(iters_factors=0)
    c = SolverConfig(samples=SamplerConfig(None, 5, None, 7, seed=3))
    cc = c._c(__import__("paper_2110_14514_b200").make_loss("poisson"))
    assert cc.samples.grad_nonzeros == -1 and cc.samples.obj_zeros == 7 and cc.lower_bound == 0.0


def test_rng_handle_is_single_use():
    """A keyed handle replays its stream from the start, so a second draw from it raises
    instead of silently repeating the first one (reference: fresh rng_at per draw)."""
    from paper_2110_14514_b200.exceptions import SamplingError
    g = rng_at(3, 1, 5)
    first = g.integers(1, 10)
    assert 1 <= first < 10
    with pytest.raises(SamplingError):
        g.integers(1, 10)
    assert rng_at(3, 1, 5).integers(1, 10) == first
