"""GPU parity of the Gaussian special cases (dense-Gaussian gradient mode,
least-squares temporal solve, exact residual), congruence and the stream feed
against golden vectors from the reference (tests/golden/gaussian.npz).
Direct quantities within 1e-5 relative (fp32 factors, fp64 accumulation);
stream / static fits within 1e-3 (BASELINE.json north_star)."""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2110_14514_b200 as P
from oracle import ogcp_oracle as O

DIRECT_RTOL = 1e-5
FIT_RTOL = 1e-3


def rel_err(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def fx(golden_dir):
    g = np.load(os.path.join(golden_dir, "gaussian.npz"), allow_pickle=False)
    dims = tuple(int(d) for d in g["dims"])
    X = P.SparseTensor.from_zero_based(dims, g["subs0"], g["vals"])
    init = [g[f"init{k}"] for k in range(len(dims) - 1)]
    return g, X, init


def test_direct_terms_vs_reference(fx):
    g, X, init = fx
    X1, w0 = X.slice_view(1), g["warm_weights"][0]
    assert P.gaussian_sum_sq_residual(X1, init, w0) == pytest.approx(float(g["resid"]), rel=DIRECT_RTOL)
    assert rel_err(P.solve_weights_least_squares(X1, init, 0.0), g["ls_mu0"]) < DIRECT_RTOL
    assert rel_err(P.solve_weights_least_squares(X1, init, 0.3), g["ls_mu"]) < DIRECT_RTOL
    from paper_2110_14514_b200.solvers import dense_gaussian_weight_gradient
    assert rel_err(dense_gaussian_weight_gradient(X1, init, w0, 0.2), g["dense_wgrad"]) < DIRECT_RTOL
    grads = P.dense_gaussian_factor_gradients(X1, init, w0, reg_factors=0.1)
    for k, gk in enumerate(grads):
        assert rel_err(gk, g[f"dense_fgrad{k}"]) < DIRECT_RTOL
    assert rel_err(P.dense_gaussian_mttkrp_gradient(X1, init, w0, 1),
                   g["dense_fgrad1"] - 0.1 * init[1]) < DIRECT_RTOL


def test_dense_gradients_with_history_vs_oracle(fx):
    g, X, init = fx
    X1 = X.slice_view(2)
    rng = np.random.default_rng(3)
    cur = [a + 0.05 * rng.standard_normal(a.shape) for a in init]
    window = [(1, g["warm_weights"][0]), (2, g["warm_weights"][1])]
    s = np.array([0.7, 1.1, 0.9])
    got = P.dense_gaussian_factor_gradients(X1, cur, s, old_factors=init, window=window, hist_weight=2.0,
                                            hist_decay=0.8, t=3, reg_factors=0.05)
    OX = O.Slice(X1.dims, X1.subs0, X1.vals)
    want = O.dense_factor_grads(OX, cur, s, init, window, 2.0, 0.8, 3, 0.05)
    for a, b in zip(got, want):
        assert rel_err(a, b) < DIRECT_RTOL


@pytest.mark.parametrize("name", ["dense", "ls"])
def test_gaussian_streams_vs_reference(fx, name):
    g, X, init = fx
    kw = json.loads(str(g[f"{name}_cfg"]))
    p = 100 if name == "dense" else 150
    cfg = P.SolverConfig(**kw, samples=P.SamplerConfig(p, 0, 200 if name == "dense" else 200, 0, seed=4))
    loss = P.make_loss("gaussian")
    st = P.fresh_state(X.dims[:-1], 3, loss, cfg, factors=init)
    st.window = P.HistoryWindow(capacity=2)
    for h in (1, 2):
        st.weights_log.append(g["warm_weights"][h - 1])
        st.window.observe(h, g["warm_weights"][h - 1], P.rng_at(cfg.samples.seed, h, 5))
    st.t = 2
    rows = P.run_stream(st, [X.slice_view(t) for t in range(3, X.dims[-1] + 1)], loss, cfg)
    np.testing.assert_allclose([r.local_loss_exact for r in rows], g[f"{name}_local_exact"], rtol=FIT_RTOL)
    assert rel_err(np.vstack(st.weights_log), g[f"{name}_weights_log"]) < FIT_RTOL
    for k, a in enumerate(st.factors):
        assert rel_err(a, g[f"{name}_final{k}"]) < FIT_RTOL
    assert st.iteration == int(g[f"{name}_iteration"])
    for (_, w, f), wr, fr in zip(st.trace_log, json.loads(str(g[f"{name}_wtrace"])),
                                 json.loads(str(g[f"{name}_ftrace"]))):
        np.testing.assert_allclose(w, wr, rtol=FIT_RTOL)
        np.testing.assert_allclose(f, fr, rtol=FIT_RTOL)
    if name == "ls":
        assert all(r.epochs_weights == 0 for r in rows)


def test_dense_static_restarts_vs_reference(fx):
    g, X, init = fx
    cfg = P.SolverConfig(gradient_mode="dense-gaussian", max_epochs_factors=3, iters_factors=10, rate_factors=2e-2,
                         reg_factors=0.01, reg_weights=0.02, samples=P.SamplerConfig(100, 0, 200, 0, seed=4))
    res = P.solve_static(X, 3, P.make_loss("gaussian"), cfg, restarts=2, seed_key=3)
    assert rel_err(res.model.weights, g["static_weights"]) < FIT_RTOL
    for k, a in enumerate(res.model.factors):
        assert rel_err(a, g[f"static_A{k}"]) < FIT_RTOL
    np.testing.assert_allclose(res.trace.objective, g["static_trace"], rtol=FIT_RTOL)


def test_congruence_vs_reference(fx):
    g, _, _ = fx
    for i, want in enumerate(g["cong_scores"]):
        M1 = P.KTensor(g[f"cong{i}_w1"], [g[f"cong{i}_f1_{k}"] for k in range(3)])
        M2 = P.KTensor(g[f"cong{i}_w2"], [g[f"cong{i}_f2_{k}"] for k in range(3)])
        assert P.congruence_score(M1, M2) == pytest.approx(float(want), rel=DIRECT_RTOL, abs=1e-6)
    M = P.KTensor(g["cong0_w1"], [g[f"cong0_f1_{k}"] for k in range(3)])
    assert P.congruence_score(M, M) == pytest.approx(1.0, abs=1e-6)


def test_feed_and_errors(fx):
    g, X, init = fx
    sl = list(P.stream_slices(X))
    assert len(sl) == X.dims[-1]
    for t, s in enumerate(sl, start=1):
        ref = X.slice_view(t)
        assert s.nnz == ref.nnz and s.dims == ref.dims
    B = P.leading_block(X, 2)
    assert B.dims == X.dims[:-1] + (2,) and B.nnz == int((X.subs0[:, -1] < 2).sum())
    with pytest.raises(P.DataError):
        P.leading_block(X, 0)
    with pytest.raises(P.DataError):  # dense-gaussian needs the gaussian loss
        P.solve_weights(X.slice_view(1), init, P.make_loss("poisson"),
                        P.SolverConfig(gradient_mode="dense-gaussian"))
    st = P.fresh_state(X.dims[:-1], 3, P.make_loss("poisson"), P.SolverConfig(temporal_solver="least-squares"),
                       factors=init)
    with pytest.raises(P.DataError, match="least-squares temporal solve requires gaussian loss"):
        P.process_slice(st, X.slice_view(1), P.make_loss("poisson"), P.SolverConfig(temporal_solver="least-squares"))
    with pytest.raises(P.DataError, match="singular"):
        P.solve_weights_least_squares(X.slice_view(1), [np.zeros_like(a) for a in init], 0.0)
