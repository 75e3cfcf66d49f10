"""GPU coverage beyond the golden cases: every mode count / rank layout the kernels
specialise (D = 1..6, ldr = 4..256), error paths with the reference's messages,
checkpoint resume, empty slices, and the statistical laws of the GPU sampler."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2110_14514_b200 as P
from oracle import ogcp_oracle as O


def rel_err(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def _slice(seed, dims, nnz, kind="poisson"):
    rng = np.random.default_rng(seed)
    lin = rng.choice(int(np.prod(dims)), size=nnz, replace=False)
    subs0 = np.array(np.unravel_index(lin, dims)).T.reshape(-1, len(dims))
    vals = rng.integers(1, 4, size=lin.size).astype(float) if kind == "poisson" else rng.standard_normal(nnz)
    return subs0, vals


@pytest.mark.parametrize("dims,R", [((97,), 3), ((12, 9, 8, 7), 4), ((6, 5, 4, 6, 5), 3), ((5, 4, 3, 4, 3, 2), 2),
                                     ((60, 50, 20), 1), ((60, 50, 20), 40), ((40, 30, 10), 100),
                                     ((30, 20, 10), 200)])
def test_gradient_tensor_modes_and_ranks(dims, R):
    """factor_gradients with history/reg + weight gradient against the oracle for every
    specialised (mode count, padded rank) layout."""
    rng = np.random.default_rng(len(dims) * 100 + R)
    nnz = min(400, int(np.prod(dims)) // 2)
    subs0, vals = _slice(R, dims, nnz, "gaussian")
    A = [rng.uniform(-1, 1, (d, R)) for d in dims]
    Aold = [a + 0.05 * rng.uniform(-1, 1, a.shape) for a in A]
    s = rng.uniform(0.5, 1.5, R)
    window = [(1, rng.uniform(0.1, 1.0, R)), (2, rng.uniform(0.1, 1.0, R))]
    Y = P.SparseTensor.from_zero_based(dims, subs0, vals, allow_zero_values=True)
    G = P.factor_gradients(Y, A, s, old_factors=Aold, window=window, hist_weight=1.5, hist_decay=0.9, t=3,
                           reg_factors=0.2) if len(dims) > 1 else None
    if G is not None:
        want = O.assemble_factor_grads(subs0, vals, dims, A, s, Aold, window, 1.5, 0.9, 3, 0.2)
        for g, w in zip(G, want):
            assert rel_err(g, w) < 2e-5
    gw = P.weight_gradient_mttkrp(Y, A)
    assert rel_err(gw, O.weight_grad(subs0, vals, A)) < 2e-5
    for k in range(len(dims)):
        assert rel_err(P.sampled_mttkrp(Y, A, k), O.mttkrp(subs0, vals, dims, A, k)) < 2e-5


@pytest.mark.parametrize("R", [2, 20, 48, 130])
def test_factor_solve_vs_oracle_ranks(R):
    """solve_factors (history + regularisation, fused K5 incl. the wide-rank variant)."""
    dims = (40, 30, 12)
    subs0, vals = _slice(R + 1, dims, 900)
    rng = np.random.default_rng(R)
    A = [rng.uniform(0.2, 1.0, (d, R)) for d in dims]
    Aold = [a * (1 + 0.02 * rng.uniform(-1, 1, a.shape)) for a in A]
    s = rng.uniform(0.5, 1.5, R)
    window = [(1, rng.uniform(0.1, 1.0, R)), (3, rng.uniform(0.1, 1.0, R))]
    cfg = P.SolverConfig(max_epochs_factors=2, iters_factors=5, rate_factors=1e-2, hist_weight=2.0, hist_decay=0.95,
                         reg_factors=0.05, samples=P.SamplerConfig(500, 600, 1500, 1500, seed=4))
    loss = P.make_loss("poisson")
    adam = cfg.make_adam(cfg.rate_factors, loss)
    adam.init([a.copy() for a in A])
    X = P.SparseTensor.from_zero_based(dims, subs0, vals)
    res = P.solve_factors(X, A, s, Aold, window, cfg, loss, adam, 0, t=4)
    ocfg = O.Cfg(kappa_f=2, tau_f=5, rate_f=1e-2, hist_weight=2.0, hist_decay=0.95, reg_factors=0.05, p=500, q=600,
                 p_obj=1500, q_obj=1500, seed=4)
    oadam = O.AdamOracle(1e-2, lower=0.0)
    oadam.init([a.copy() for a in A])
    fo, it, tr, _, _ = O.factor_solve(O.Slice(dims, subs0, vals), A, s, Aold, window, ocfg, "poisson", oadam, 0, 4)
    assert res.iteration == it
    np.testing.assert_allclose(res.trace.objective, tr, rtol=1e-4)
    for a, b in zip(res.factors, fo):
        assert rel_err(a, b) < 1e-4


@pytest.mark.parametrize("R", [3, 20, 32])
def test_factor_solve_vs_oracle_per_mode_k5(R):
    """solve_factors with history + regularisation on a model past the small-model
    size (a 5000-row mode): the per-mode K5 launches (shared-memory staged history
    apply for R >= 4, shuffles below) against the oracle."""
    dims = (5000, 30, 12)
    subs0, vals = _slice(R + 7, dims, 3000)
    rng = np.random.default_rng(R + 1)
    A = [rng.uniform(0.2, 1.0, (d, R)) for d in dims]
    Aold = [a * (1 + 0.02 * rng.uniform(-1, 1, a.shape)) for a in A]
    s = rng.uniform(0.5, 1.5, R)
    window = [(1, rng.uniform(0.1, 1.0, R)), (2, rng.uniform(0.1, 1.0, R))]
    cfg = P.SolverConfig(max_epochs_factors=2, iters_factors=4, rate_factors=1e-2, hist_weight=2.0, hist_decay=0.9,
                         reg_factors=0.05, samples=P.SamplerConfig(1500, 1500, 3000, 3000, seed=6))
    loss = P.make_loss("poisson")
    adam = cfg.make_adam(cfg.rate_factors, loss)
    adam.init([a.copy() for a in A])
    X = P.SparseTensor.from_zero_based(dims, subs0, vals)
    res = P.solve_factors(X, A, s, Aold, window, cfg, loss, adam, 0, t=3)
    ocfg = O.Cfg(kappa_f=2, tau_f=4, rate_f=1e-2, hist_weight=2.0, hist_decay=0.9, reg_factors=0.05, p=1500, q=1500,
                 p_obj=3000, q_obj=3000, seed=6)
    oadam = O.AdamOracle(1e-2, lower=0.0)
    oadam.init([a.copy() for a in A])
    fo, it, tr, _, _ = O.factor_solve(O.Slice(dims, subs0, vals), A, s, Aold, window, ocfg, "poisson", oadam, 0, 3)
    assert res.iteration == it
    np.testing.assert_allclose(res.trace.objective, tr, rtol=1e-4)
    for a, b in zip(res.factors, fo):
        assert rel_err(a, b) < 1e-4


def test_errors_carry_reference_messages():
    dims = (20, 15, 10)
    subs0, vals = _slice(9, dims, 300)
    R = 3
    init = [np.full((d, R), 0.5) for d in dims]
    # divergence: a huge temporal rate, as test_cli.py:167-173 forces it (--rate-w 1e200)
    cfg = P.SolverConfig(max_epochs_weights=2, max_epochs_factors=1, iters_weights=3, iters_factors=3,
                         rate_weights=1e200, rate_decay=0.9, samples=P.SamplerConfig(200, 200, 400, 400, seed=1))
    loss = P.make_loss("gaussian")
    st = P.fresh_state(dims, R, loss, cfg, factors=init)
    X = P.SparseTensor.from_zero_based(dims, subs0, vals)
    with pytest.raises(P.DivergenceError, match=r"^slice 1: temporal weight solve"):
        P.process_slice(st, X, loss, cfg, exact_loss=False)
    # data error: bernoulli loss on count data (losses.py:54)
    cfg2 = P.SolverConfig(max_epochs_weights=1, max_epochs_factors=1, iters_weights=2, iters_factors=2,
                          samples=P.SamplerConfig(50, 50, 100, 100, seed=1))
    st2 = P.fresh_state(dims, R, P.make_loss("bernoulli"), cfg2, factors=init)
    with pytest.raises(P.DataError, match=r"^slice 1: bernoulli loss requires x in \{0, 1\}"):
        P.process_slice(st2, X, P.make_loss("bernoulli"), cfg2)
    # sampling error: zero draws on a full tensor (sampling.py:122-123)
    full = np.indices((3, 4)).reshape(2, -1).T
    Xf = P.SparseTensor.from_zero_based((3, 4), full, np.ones(12))
    with pytest.raises(P.SamplingError, match="tensor has no zeros"):
        P.draw_samples(Xf, 2, 3, P.rng_at(0, 1))
    # duplicates / bounds at construction (tensor.py:91-114)
    with pytest.raises(P.DataError, match="duplicate coordinate"):
        P.SparseTensor((3, 3), [[1, 1], [2, 2], [1, 1]], [1.0, 2.0, 3.0])
    with pytest.raises(P.DataError, match="out of bounds"):
        P.SparseTensor((3, 3), [[1, 4]], [1.0])
    with pytest.raises(P.DataError, match="exactly 0 are disallowed"):
        P.SparseTensor((3, 3), [[1, 2]], [0.0])


def test_empty_slice_and_zero_only_draws():
    dims = (10, 8, 6)
    X = P.SparseTensor.from_zero_based(dims, np.empty((0, 3), np.int64), np.empty(0))
    s = P.draw_samples(X, 0, 50, P.rng_at(0, 1))
    ref = O.draw(O.Slice(dims, np.empty((0, 3)), np.empty(0)), 0, 50, O.keyed_rng(0, 1))
    np.testing.assert_array_equal(s.zero_subs0, ref.zero_subs0)
    cfg = P.SolverConfig(max_epochs_weights=1, max_epochs_factors=1, iters_weights=3, iters_factors=3,
                         samples=P.SamplerConfig(None, 40, None, 80, seed=2))
    loss = P.make_loss("poisson")
    st = P.fresh_state(dims, 2, loss, cfg, factors=[np.full((d, 2), 0.3) for d in dims])
    m = P.process_slice(st, X, loss, cfg, exact_loss=True)
    assert np.isfinite(m.local_loss_exact)


def test_checkpoint_resume_matches_uninterrupted(tmp_path):
    dims = (25, 20, 6, 4)
    subs0, vals = _slice(11, dims, 900)
    cfg = P.SolverConfig(max_epochs_weights=1, max_epochs_factors=1, iters_weights=10, iters_factors=10,
                         rate_weights=0.05, rate_factors=1e-2, hist_weight=1.0, warm_start_weights=True,
                         samples=P.SamplerConfig(None, 300, None, 600, seed=3))
    loss = P.make_loss("poisson")
    Xs = [P.SparseTensor.from_zero_based(dims[:-1], subs0[subs0[:, -1] == t, :-1], vals[subs0[:, -1] == t])
          for t in range(dims[-1])]
    init = [np.full((d, 3), 0.4) for d in dims[:-1]]

    def fresh():
        st = P.fresh_state(dims[:-1], 3, loss, cfg, factors=init)
        st.window = P.HistoryWindow(capacity=2)
        st.weights_log.append(np.ones(3))
        st.window.observe(1, np.ones(3), P.rng_at(3, 1, 5))
        st.t = 1
        return st

    a = fresh()
    for X in Xs:
        P.process_slice(a, X, loss, cfg, exact_loss=False)
    b = fresh()
    for X in Xs[:2]:
        P.process_slice(b, X, loss, cfg, exact_loss=False)
    path = os.path.join(tmp_path, "ck.npz")
    P.save_checkpoint(b, path)
    c = P.load_checkpoint(path, loss, cfg)
    for X in Xs[2:]:
        P.process_slice(c, X, loss, cfg, exact_loss=False)
    assert c.t == a.t and c.iteration == a.iteration
    assert c.window.step_ids() == a.window.step_ids()
    for x, y in zip(c.factors, a.factors):
        assert rel_err(x, y) < 1e-4


def test_gpu_zero_draws_uniform_chi2():
    """test_sampling.py:57-72 pattern on the GPU sampler: zero cells are uniform."""
    from scipy import stats
    rng = np.random.default_rng(2)
    dims = (10, 10)
    lin = rng.choice(100, size=20, replace=False)
    subs0 = np.array(np.unravel_index(lin, dims)).T
    X = P.SparseTensor.from_zero_based(dims, subs0, np.ones(20))
    z = P.draw_samples(X, 2000, 100_000, P.rng_at(0, 7)).zero_subs0
    cells = z[:, 0] * 10 + z[:, 1]
    counts = np.bincount(cells, minlength=100)
    assert counts[lin].sum() == 0
    zero_cells = np.setdiff1d(np.arange(100), lin)
    assert stats.chisquare(counts[zero_cells]).pvalue > 1e-3


def test_gpu_objective_unbiased():
    """test_acceptance.py:104-144 pattern: the GPU objective estimate is unbiased."""
    rng = np.random.default_rng(6)
    dims = (4, 4, 3)
    lin = rng.choice(48, size=12, replace=False)
    subs0 = np.array(np.unravel_index(lin, dims)).T
    vals = rng.integers(1, 4, size=12).astype(float)
    w = rng.uniform(0.2, 1.0, 2)
    A = [rng.uniform(0.1, 1.0, (d, 2)) for d in dims]
    X = P.SparseTensor.from_zero_based(dims, subs0, vals)
    dense_x = np.zeros(dims)
    dense_x[tuple(subs0.T)] = vals
    exact = float(np.sum(O.loss_f("poisson", dense_x.ravel(), np.einsum("ir,jr,kr,r->ijk", *A, w).ravel())))
    reps = 600
    v = np.array([P.estimate_objective(X, A, w, P.make_loss("poisson"), P.draw_samples(X, 6, 10, P.rng_at(77, r)))
                  for r in range(reps)])
    assert abs(v.mean() - exact) < 4 * v.std(ddof=1) / np.sqrt(reps)


def test_large_slice_prefiltered_zero_draws_bit_exact():
    """Slices with >= 2^20 nonzeros probe zero candidates through the membership
    prefilter (one-hash bitmap) before the hash table: rejections (2.4% density)
    and accepted zeros stay bit-exact with the reference draw."""
    dims = (1000, 1000, 50)
    rng = np.random.default_rng(17)
    lin = np.sort(rng.choice(int(np.prod(dims)), size=1_200_000, replace=False))
    subs0 = np.array(np.unravel_index(lin, dims)).T
    vals = np.ones(lin.size)
    X = P.SparseTensor.from_zero_based(dims, subs0, vals)
    s = P.draw_samples(X, 5000, 200_000, P.rng_at(3, 9))
    ref = O.draw(O.Slice(dims, subs0, vals), 5000, 200_000, O.keyed_rng(3, 9))
    np.testing.assert_array_equal(s.nz_ordinals, ref.ordinals)
    np.testing.assert_array_equal(s.zero_subs0, ref.zero_subs0)


@pytest.mark.parametrize("R", [64, 130])
def test_weight_solve_vs_oracle_large_ranks(R):
    """solve_weights at ranks whose temporal row no longer fits a 64-double host mirror."""
    dims = (40, 30, 12)
    subs0, vals = _slice(R + 5, dims, 900)
    rng = np.random.default_rng(R + 1)
    A = [rng.uniform(0.2, 1.0, (d, R)) / 3 for d in dims]
    cfg = P.SolverConfig(max_epochs_weights=2, iters_weights=5, rate_weights=0.05, reg_weights=0.1,
                         samples=P.SamplerConfig(500, 600, 1500, 1500, seed=4))
    X = P.SparseTensor.from_zero_based(dims, subs0, vals)
    res = P.solve_weights(X, A, P.make_loss("poisson"), cfg, t=3)
    ocfg = O.Cfg(kappa_w=2, tau_w=5, rate_w=0.05, reg_weights=0.1, p=500, q=600, p_obj=1500, q_obj=1500, seed=4)
    s, tr, _, _ = O.temporal_solve(O.Slice(dims, subs0, vals), A, "poisson", ocfg, 3)
    assert rel_err(res.weights, s) < 1e-4
    np.testing.assert_allclose(res.trace.objective, tr, rtol=1e-4)


@pytest.mark.parametrize("umma", [True, False])
@pytest.mark.parametrize("R", [40, 64, 100, 128])
def test_tensor_core_grams_vs_oracle(R, umma):
    """ldr 64 / 128 Grams run on tensor cores -- tcgen05.mma kind::tf32 with TMEM
    accumulators (csrc/gram_umma.cuh) or the mma.sync kernel -- with the split-TF32
    3-product scheme: fp32-level accuracy, checked norm-wise like the gradients
    (entries of a Hadamard of Grams of random signs cancel, so elementwise relative
    error is meaningless near 0).  Mode sizes 3000 / 257 / 40 cover full chunks, a
    ragged tail chunk and a single partial chunk."""
    from paper_2110_14514_b200 import _lib
    rng = np.random.default_rng(R)
    dims = (3000, 257, 40)
    A = [rng.uniform(-1, 1, (d, R)) for d in dims]
    B = [a + 0.1 * rng.uniform(-1, 1, a.shape) for a in A]
    _lib.set_umma_gram(umma)
    try:
        for mode in (None, 1):
            g, want = P.gram(A, mode), O.hadamard_gram(A, mode)
            assert rel_err(g, want) < 1e-5
            np.testing.assert_allclose(np.diag(g), np.diag(want), rtol=1e-5)
            assert rel_err(P.gram(A, mode, other_factors=B), O.hadamard_gram(A, mode, B)) < 1e-5
    finally:
        _lib.set_umma_gram(True)



@pytest.mark.parametrize("umma", [True, False])
@pytest.mark.parametrize("R", [20, 32])
def test_ldr32_grams_vs_oracle(R, umma):
    """ldr 32 (the c4 rank): the tcgen05 Gram with its decoupled raw-tile ring
    (k_gram_umma32) and the mma.sync kernel against fp64 numpy.  Mode 0 past the
    small-model size (5000 rows) so the Grams take the large-model path; 257 and
    40 rows cover a ragged tail chunk and a single partial chunk."""
    from paper_2110_14514_b200 import _lib
    rng = np.random.default_rng(R)
    dims = (5000, 257, 40)
    A = [rng.uniform(-1, 1, (d, R)) for d in dims]
    B = [a + 0.1 * rng.uniform(-1, 1, a.shape) for a in A]
    _lib.set_umma_gram(umma)
    try:
        for mode in (None, 1):
            g, want = P.gram(A, mode), O.hadamard_gram(A, mode)
            assert rel_err(g, want) < 1e-5
            np.testing.assert_allclose(np.diag(g), np.diag(want), rtol=1e-5)
            assert rel_err(P.gram(A, mode, other_factors=B), O.hadamard_gram(A, mode, B)) < 1e-5
    finally:
        _lib.set_umma_gram(True)


def test_tcgen05_gram_at_c5_scale():
    """The tcgen05 / TMEM Gram at the c5 shape (100K rows, ldr 128: 3125 32-row chunks over
    148 CTAs) against the mma.sync kernel and fp64 numpy (norm-wise 1e-5)."""
    from paper_2110_14514_b200 import _lib
    rng = np.random.default_rng(128)
    A = rng.uniform(-1, 1, (100_000, 128))
    B = A + 0.05 * rng.uniform(-1, 1, A.shape)
    want_p, want_c = A.T @ A, B.T @ A
    out = {}
    for umma in (True, False):
        _lib.set_umma_gram(umma)
        try:
            out[umma] = (P.gram([A], None), P.gram([A], None, other_factors=[B]))
        finally:
            _lib.set_umma_gram(True)
    for umma in (True, False):
        assert rel_err(out[umma][0], want_p) < 1e-5
        assert rel_err(out[umma][1], want_c) < 1e-5
