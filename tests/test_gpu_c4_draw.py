"""Sampler parity at the bench scale (BASELINE configs[3]): the
1M x 1M x 1K planted Poisson slice with 1e8 nonzeros, p = "all" (eta = 1e8 draws
with replacement) and q = 2^24 zeros, keyed like a factor-solve iteration.

* The engine's draw (ogcp_draw_samples) equals numpy's keyed stream bit for bit:
  ordinals = rng.integers(0, eta, p) (sampling.py:125) and the zero rows of the
  batched rejection loop (sampling.py:133-150) against the stored set.
* The merged (count) form the solve evaluates -- the ordinal histogram, permuted
  into the row-bucketed walk -- equals np.bincount of those ordinals, entry for
  entry, with the same accepted zero rows (sampled_gradient_tensor's merge,
  sampling.py:233-237).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2110_14514_b200 as P
from paper_2110_14514_b200 import _lib
from paper_2110_14514_b200.synthetic import gen_slice
from oracle import ogcp_oracle as O

DIMS = (1_000_000, 1_000_000, 1_000)
NNZ = 100_000_000
Q = 1 << 24
KEY = (31, 3, 0, 17)   # (t, PHASE_FACTOR_GRAD, epoch, it) of rng_at(seed, ...), solvers.py:345


@pytest.fixture(scope="module")
def c4():
    X, factors, mix, total = gen_slice(DIMS, NNZ, 32, "poisson", seed=42)
    subs0 = X.subs0
    lin = subs0 @ O.strides_of(DIMS)
    assert lin.size == NNZ and bool(np.all(np.diff(lin) > 0))  # stored in ascending linear order
    yield X, lin
    del X
    torch.cuda.empty_cache()


def numpy_draw(lin_sorted, p, q, seed, key):
    """sampling.py:108-153 on the keyed numpy stream, membership by binary search (tensor.py:163-169)."""
    gen = O.keyed_rng(seed, *key)
    ords = gen.integers(0, lin_sorted.size, size=p)
    hi = np.asarray(DIMS, dtype=np.int64)
    st = O.strides_of(DIMS)
    kept, need = [], q
    while need > 0:
        cand = gen.integers(0, hi, size=(need, len(DIMS)), dtype=np.int64)
        cl = cand @ st
        pos = np.minimum(np.searchsorted(lin_sorted, cl), lin_sorted.size - 1)
        miss = lin_sorted[pos] != cl
        kept.append(cand[miss])
        need -= int(miss.sum())
    return ords, np.concatenate(kept)


def test_c4_draw_bit_exact(c4):
    X, lin = c4
    s = P.draw_samples(X, NNZ, Q, P.rng_at(7, *KEY))
    ords, zeros = numpy_draw(lin, NNZ, Q, 7, KEY)
    got = s.ord_dev.cpu().numpy()
    assert got.shape == (NNZ,)
    assert np.array_equal(got.astype(np.int64), ords)
    assert np.array_equal(s.zero_subs0, zeros)


@pytest.mark.parametrize("buckets,sort_zeros", [(0, False), (4, False), (4, True)])
def test_c4_merged_counts_equal_bincount(c4, buckets, sort_zeros):
    X, lin = c4
    ords, zeros = numpy_draw(lin, NNZ, Q, 7, KEY)
    counts = np.bincount(ords, minlength=NNZ)
    del ords
    _lib.set_buckets(buckets)  # 0: plain ordinal order; 4: the bench's row-bucketed walk
    _lib.set_sort_zeros(sort_zeros)
    try:
        o, c, z = _lib.debug_solve_draw(X, 7, KEY, None, Q, ldr=32)
    finally:
        _lib.set_buckets(1)
        _lib.set_sort_zeros(False)
    order = np.argsort(o, kind="stable")
    o, c = o[order], c[order]
    nzr = np.flatnonzero(counts)
    assert np.array_equal(o, nzr), "merged ordinals differ from the distinct drawn ordinals"
    assert np.array_equal(c, counts[nzr]), "multiplicities differ from np.bincount"
    assert int(c.sum()) == NNZ
    if sort_zeros:
        # OGCP_OPT_SORT_ZEROS: bucketed solves walk the zero rows sorted (stably) by (row bucket of mode 1, mode-0 row):
        # the same rows as the reference's draw, in the walk order (sampler.cu k_zero_sort_keys)
        key = (zeros[:, 1] * buckets // DIMS[1]) * DIMS[0] + zeros[:, 0]
        zeros = zeros[np.argsort(key, kind="stable")]
    assert np.array_equal(z, zeros)


@pytest.mark.parametrize("world", [4, 8])
def test_c4_word_sharded_draw_partitions_bincount(c4, world):
    """The multi-GPU draw sharded by RNG word range (OGCP_OPT_SHARD_DRAWS), at the bench
    scale: each of `world` simulated ranks generates its 1/world of the words, the tile
    maps / zero-row records are all-gathered and the nibble counters reduce-scattered
    (exact device-side stand-ins on this GPU).  Rank r's merged set holds exactly the
    np.bincount entries of its own ordinal chunk, and the ranks' zero rows, in rank
    order, are the reference's accepted zero rows in draw order."""
    X, lin = c4
    ords, zeros = numpy_draw(lin, NNZ, Q, 7, KEY)
    counts = np.bincount(ords, minlength=NNZ)
    del ords
    cw = (-(-NNZ // 8) + world - 1) // world
    zparts = []
    _lib.set_buckets(4)
    try:
        for r in range(world):
            _lib.set_shard_sim(r, world)
            o, c, z = _lib.debug_solve_draw(X, 7, KEY, None, Q, ldr=32)
            lo, hi = min(8 * cw * r, NNZ), min(8 * cw * (r + 1), NNZ)
            order = np.argsort(o, kind="stable")
            o, c = o[order], c[order]
            nzr = lo + np.flatnonzero(counts[lo:hi])
            assert np.array_equal(o, nzr), r
            assert np.array_equal(c, counts[nzr]), r
            zparts.append(z)
    finally:
        _lib.set_shard_sim(0, 1)
        _lib.set_buckets(1)
    z = np.concatenate(zparts)
    assert np.array_equal(z, zeros)
    # the rows are split roughly evenly (word ranges of equal length)
    sizes = np.array([len(p_) for p_ in zparts])
    assert sizes.min() > 0.8 * Q / world and sizes.max() < 1.2 * Q / world


def test_c4_factor_gradient_tma_walk_matches_generic(c4):
    """The bench-scale K3 walk: one factor iteration at rate ~0 (u = (1 - b1) g) on the c4
    slice (p = all, q = 2^24, R = 32, row-bucketed merged set) with the TMA-fed
    warp-specialised walk (csrc/walk_tma.cuh) and with the generic sample kernels gives
    the same factor gradients (fp32 reduction order only), and the weight gradient of the
    same draw matches too."""
    from paper_2110_14514_b200.solvers import solve_factors_device, solve_weights_device
    X, _ = c4
    R = 32
    rng = np.random.default_rng(3)
    init = [rng.uniform(0.5, 1.5, (d, R)) / np.sqrt(d) for d in DIMS]
    w = np.full(R, 2.0)
    cfg = P.SolverConfig(max_epochs_factors=1, iters_factors=1, rate_factors=1e-30,
                         samples=P.SamplerConfig(None, Q, 1 << 20, 1 << 20, seed=9))
    loss = P.make_loss("poisson")

    def u_of(impl):
        _lib.set_walk_impl(impl)
        try:
            model = P.DeviceModel.from_numpy(init)
            adam = cfg.make_adam(cfg.rate_factors, loss)
            adam.init_device(model.dims, model.rank)
            solve_factors_device(X, model, w, None, [], cfg, loss, adam, 0, 1)
            out = [t[:, :R].double().cpu().numpy() for t in adam._buf["u"]]
            del model, adam
            return out
        finally:
            _lib.set_walk_impl("tma")

    a, b = u_of("tma"), u_of("generic")
    for k in range(3):
        assert np.linalg.norm(a[k] - b[k]) <= 1e-5 * np.linalg.norm(b[k]), k
