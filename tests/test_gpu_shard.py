"""The multi-GPU shard partition, checked in one process: a context put in
shard-simulation mode (OGCP_OPT_SHARD_SIM, no communicator) runs exactly the
share of rank r of a world-N solve.  For merged (count-form) gradient draws --
with and without the row-bucketed layout, replicated or sharded by RNG word
range (OGCP_OPT_SHARD_DRAWS: the simulation then runs every rank's part in lock
step with exact device-side stand-ins for the all-gathers / reduce-scatter) --
the ranks' nonzero shares (their own ordinal ranges) and zero-row shares must
partition the single-GPU set exactly; for plain draws the contiguous split must
too."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2110_14514_b200 as P
from paper_2110_14514_b200 import _lib


@pytest.fixture(scope="module")
def slice_1e5():
    rng = np.random.default_rng(21)
    dims = (300, 200, 40)
    lin = rng.choice(int(np.prod(dims)), size=100_000, replace=False)
    subs0 = np.array(np.unravel_index(np.sort(lin), dims)).T
    vals = rng.integers(1, 4, size=lin.size).astype(float)
    return P.SparseTensor.from_zero_based(dims, subs0, vals)


def _draw(X, p, q, world=1, rank=0):
    _lib.set_shard_sim(rank, world)
    try:
        return _lib.debug_solve_draw(X, 5, (7, 3, 0, 1), p, q, ldr=8)
    finally:
        _lib.set_shard_sim(0, 1)


def owner_range(eta, r, world):
    """shard_owner_range: chunks of whole nibble words (8 ordinals) per rank."""
    cw = (-(-eta // 8) + world - 1) // world
    return min(8 * cw * r, eta), min(8 * cw * (r + 1), eta)


@pytest.mark.parametrize("shard_draws", [0, 1])
@pytest.mark.parametrize("buckets", [1, 4])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_merged_draw_shards_partition(slice_1e5, buckets, world, shard_draws):
    X = slice_1e5
    _lib.set_buckets(buckets)
    _lib.set_shard_draws(shard_draws)
    try:
        o, c, z = _draw(X, None, 4000)  # p = all: merged form
        assert c.sum() == X.nnz and len(z) == 4000
        parts = [_draw(X, None, 4000, world, r) for r in range(world)]
    finally:
        _lib.set_buckets(1)
        _lib.set_shard_draws(1)
    po = np.concatenate([q[0] for q in parts])
    pc = np.concatenate([q[1] for q in parts])
    a, b = np.argsort(o, kind="stable"), np.argsort(po, kind="stable")
    np.testing.assert_array_equal(po[b], o[a])
    np.testing.assert_array_equal(pc[b], c[a])
    for r, (ro, _, _) in enumerate(parts):  # each rank holds its own ordinal range
        lo, hi = owner_range(X.nnz, r, world)
        assert ro.size == 0 or (ro.min() >= lo and ro.max() < hi)
    np.testing.assert_array_equal(np.concatenate([q[2] for q in parts]), z)


def test_plain_draw_shards_partition(slice_1e5):
    X = slice_1e5
    o, c, z = _draw(X, 3000, 2000)  # p << eta: per-draw form, contiguous split of [nonzeros | zeros]
    parts = [_draw(X, 3000, 2000, 3, r) for r in range(3)]
    np.testing.assert_array_equal(np.concatenate([q[0] for q in parts]), o)
    np.testing.assert_array_equal(np.concatenate([q[2] for q in parts]), z)


@pytest.mark.parametrize("shard_draws", [0, 1])
@pytest.mark.parametrize("R", [6, 20])
def test_sharded_gradients_sum_to_single_gpu(slice_1e5, R, shard_draws):
    """Shard-simulated factor solves of one iteration with rate ~0: every rank's
    K3 output is its partial gradient, so the per-rank first Adam moments
    (u = (1-b1) g) must sum to the single-GPU one (R = 20: the lean 3-way walks)."""
    X = slice_1e5
    rng = np.random.default_rng(2)
    init = [rng.uniform(0.2, 1.0, (d, R)) for d in X.dims]
    w = np.full(R, 1.1)
    cfg = P.SolverConfig(max_epochs_factors=1, iters_factors=1, rate_factors=1e-30,
                         samples=P.SamplerConfig(None, 3000, 5000, 5000, seed=4))
    loss = P.make_loss("poisson")

    def u_of(world, rank):
        _lib.set_shard_sim(rank, world)
        _lib.set_shard_draws(shard_draws)
        try:
            model = P.DeviceModel.from_numpy(init)
            adam = cfg.make_adam(cfg.rate_factors, loss)
            adam.init_device(model.dims, model.rank)
            from paper_2110_14514_b200.solvers import solve_factors_device
            solve_factors_device(X, model, w, None, [], cfg, loss, adam, 0, 1)
            return [t[:, :R].double().cpu().numpy() for t in adam._buf["u"]]
        finally:
            _lib.set_shard_sim(0, 1)
            _lib.set_shard_draws(1)

    full = u_of(1, 0)
    for world in (2, 4):
        parts = [u_of(world, r) for r in range(world)]
        for k in range(3):
            tot = sum(p_[k] for p_ in parts)
            assert np.linalg.norm(tot - full[k]) <= 1e-5 * np.linalg.norm(full[k])


def test_nccl_entry_points_one_rank():
    """The run-time loaded NCCL (libnccl.so.2) and every collective signature the
    multi-GPU solves use, exercised on a one-rank communicator."""
    import ctypes as C
    bad = C.c_int32(-1)
    _lib.check(_lib.lib().ogcp_comm_selftest(_lib.ctx(), C.byref(bad)))
    assert bad.value == 0


def test_row_sharded_update_partitions_rows():
    """Models past the small-model size run K5 owner-computes across ranks: a
    shard-simulated rank r of a world-N factor solve updates exactly its
    contiguous row block [I r/N, I (r+1)/N) of every mode (factors and Adam
    moments) and leaves every other row untouched; with N = 1 all rows move.
    The blocks partition the rows, so after the owners' broadcasts every rank
    holds one full, identical update."""
    rng = np.random.default_rng(5)
    dims = (5000, 300, 20)  # mode 0 past kSmallRows (4096): the per-mode K5 path
    lin = rng.choice(int(np.prod(dims)), size=60_000, replace=False)
    subs0 = np.array(np.unravel_index(np.sort(lin), dims)).T
    X = P.SparseTensor.from_zero_based(dims, subs0, rng.integers(1, 4, size=lin.size).astype(float))
    R = 6
    init = [rng.uniform(0.2, 1.0, (d, R)) for d in dims]
    w = np.full(R, 1.1)
    cfg = P.SolverConfig(max_epochs_factors=1, iters_factors=2, rate_factors=1e-2,
                         samples=P.SamplerConfig(None, 20000, 5000, 5000, seed=4))
    loss = P.make_loss("poisson")
    from paper_2110_14514_b200.solvers import solve_factors_device

    def run(world, rank):
        _lib.set_shard_sim(rank, world)
        try:
            model = P.DeviceModel.from_numpy(init)
            adam = cfg.make_adam(cfg.rate_factors, loss)
            adam.init_device(model.dims, model.rank)
            _, tr = solve_factors_device(X, model, w, None, [], cfg, loss, adam, 0, 1)
            A = [t[:, :R].double().cpu().numpy() for t in model.tensors]
            u = [t[:, :R].double().cpu().numpy() for t in adam._buf["u"]]
            return A, u, tr.rejections
        finally:
            _lib.set_shard_sim(0, 1)

    A1, u1, rej = run(1, 0)
    assert rej == 0
    for k in range(3):
        assert np.mean(np.any(A1[k] != init[k], axis=1)) > 0.99 and np.mean(np.any(u1[k] != 0, axis=1)) > 0.99
    world = 3
    accepted = 0
    for r in range(world):
        # rank r's objective share can reject the epoch, which restores the entry state
        A, u, rej = run(world, r)
        accepted += rej == 0
        for k, d in enumerate(dims):
            lo, hi = d * r // world, d * (r + 1) // world
            own = np.zeros(d, bool)
            own[lo:hi] = True
            np.testing.assert_array_equal(A[k][~own], init[k][~own].astype(np.float32))
            assert not np.any(u[k][~own])
            if rej:
                np.testing.assert_array_equal(A[k], init[k].astype(np.float32))
                continue
            # owned rows move unless rank r's sample share never touched them
            assert np.mean(np.any(A[k][own] != init[k][own].astype(np.float32), axis=1)) > 0.9
            assert np.mean(np.any(u[k][own] != 0, axis=1)) > 0.9
    assert accepted >= 1


@pytest.mark.parametrize("impl", ["tma", "tma-all", "tma-a2", "lean"])
@pytest.mark.parametrize("R", [12, 20])
@pytest.mark.parametrize("buckets", [1, 4])
def test_walk_kernels_gradient_match_generic(slice_1e5, impl, R, buckets):
    """One factor iteration with rate ~0 (u = (1-b1) g): the TMA-fed / register-pipelined
    3-way walk kernels and the generic sample kernels give the same factor gradients
    (fp32 reduction order only)."""
    X = slice_1e5
    rng = np.random.default_rng(5)
    init = [rng.uniform(0.2, 1.0, (d, R)) for d in X.dims]
    w = np.full(R, 0.9)
    cfg = P.SolverConfig(max_epochs_factors=1, iters_factors=1, rate_factors=1e-30,
                         samples=P.SamplerConfig(None, 7000, 5000, 5000, seed=9))
    loss = P.make_loss("poisson")

    def u_of(which):
        _lib.set_walk_impl(which)
        _lib.set_buckets(buckets)
        try:
            model = P.DeviceModel.from_numpy(init)
            adam = cfg.make_adam(cfg.rate_factors, loss)
            adam.init_device(model.dims, model.rank)
            from paper_2110_14514_b200.solvers import solve_factors_device
            solve_factors_device(X, model, w, None, [], cfg, loss, adam, 0, 1)
            return [t[:, :R].double().cpu().numpy() for t in adam._buf["u"]]
        finally:
            _lib.set_walk_impl("tma")
            _lib.set_buckets(1)

    a, b = u_of(impl), u_of("generic")
    for k in range(3):
        assert np.linalg.norm(a[k] - b[k]) <= 1e-6 * np.linalg.norm(b[k])
