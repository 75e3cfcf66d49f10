"""GPU parity of the static fit and warm start (solvers.py:371-493,
streaming.py:113-151) against golden vectors from the reference and the pinned
oracle.  Tolerances as in test_gpu_parity: the fit within 1e-3 relative (fp32
factors over hundreds of Adam steps), epoch/rejection counts exact."""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2110_14514_b200 as P
from paper_2110_14514_b200 import _lib
from oracle import ogcp_oracle as O

FIT_RTOL = 1e-3


def rel_err(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def case(golden_dir, name):
    g = np.load(os.path.join(golden_dir, "static.npz"), allow_pickle=False)
    c = lambda k: g[f"{name}_{k}"]
    kw = json.loads(str(c("cfg")))
    sm = json.loads(str(c("samples")))
    cfg = P.SolverConfig(**kw, samples=P.SamplerConfig(sm["p"], sm["q"], sm["p_obj"], sm["q_obj"], seed=sm["seed"]))
    dims = tuple(int(d) for d in c("dims"))
    X = P.SparseTensor.from_zero_based(dims, c("subs0"), c("vals"))
    return c, P.make_loss(str(c("kind"))), int(c("R")), cfg, X


@pytest.mark.parametrize("name", ["gauss", "pois", "bern"])
def test_solve_static_vs_reference(golden_dir, name):
    c, loss, R, cfg, X = case(golden_dir, name)
    res = P.solve_static(X, R, loss, cfg, seed_key=4)
    assert rel_err(res.model.weights, c("static_weights")) < FIT_RTOL
    for k, a in enumerate(res.model.factors):
        assert rel_err(a, c(f"static_A{k}")) < FIT_RTOL
    np.testing.assert_allclose(res.trace.objective, c("static_trace"), rtol=FIT_RTOL)
    assert (res.trace.epochs, res.trace.rejections) == (int(c("static_epochs")), int(c("static_rejections")))


@pytest.mark.parametrize("name", ["gauss", "pois", "bern"])
def test_warm_start_vs_reference(golden_dir, name):
    c, loss, R, cfg, X = case(golden_dir, name)
    st = P.warm_start(X, R, loss, cfg, int(c("capacity")), restarts=int(c("restarts")))
    for k, a in enumerate(st.factors):
        assert rel_err(a, c(f"warm_A{k}")) < FIT_RTOL
    assert rel_err(np.vstack(st.weights_log), c("warm_weights_log")) < FIT_RTOL
    assert st.window.step_ids() == c("warm_window_ids").tolist()
    assert st.t == int(c("warm_t"))


@pytest.mark.parametrize("merge", [True, False])
def test_dense_static_vs_oracle(merge):
    """p = all nonzeros of a 1e5-nnz block: the merged-draw and per-draw forms
    of the static fit both follow the oracle."""
    rng = np.random.default_rng(5)
    dims = (200, 150, 60, 4)
    lin = rng.choice(int(np.prod(dims)), size=100_000, replace=False)
    subs0 = np.array(np.unravel_index(np.sort(lin), dims)).T
    vals = rng.integers(1, 4, size=lin.size).astype(float)
    R = 5
    _lib.set_merge_draws(merge)
    try:
        X = P.SparseTensor.from_zero_based(dims, subs0, vals)
        cfg = P.SolverConfig(max_epochs_factors=2, iters_factors=3, rate_factors=1e-2, reg_factors=0.01,
                             samples=P.SamplerConfig(None, 5000, 20000, 20000, seed=9))
        loss = P.make_loss("poisson")
        res = P.solve_static(X, R, loss, cfg, seed_key=1)
    finally:
        _lib.set_merge_draws(True)
    ocfg = O.Cfg(kappa_f=2, tau_f=3, rate_f=1e-2, reg_factors=0.01, p=None, q=5000, p_obj=20000, q_obj=20000, seed=9)
    w, fs, trace, epochs, rej = O.static_solve(O.Slice(dims, subs0, vals), R, "poisson", ocfg, seed_key=1)
    assert rel_err(res.model.weights, w) < FIT_RTOL
    for a, b in zip(res.model.factors, fs):
        assert rel_err(a, b) < FIT_RTOL
    np.testing.assert_allclose(res.trace.objective, trace, rtol=FIT_RTOL)
    assert (res.trace.epochs, res.trace.rejections) == (epochs, rej)


def test_static_errors():
    X = P.SparseTensor.from_zero_based((3, 4), np.array([[0, 1], [2, 3]]), np.array([1.0, 2.0]))
    with pytest.raises(P.DataError):
        P.warm_start(P.SparseTensor.from_zero_based((5,), np.array([[1]]), np.array([1.0])), 2,
                     P.make_loss("gaussian"), P.SolverConfig(), 0)
    with pytest.raises(P.DataError):
        P.solve_static(X, 2, P.make_loss("gaussian"), P.SolverConfig(), init=P.KTensor(np.ones(2), [np.ones((3, 2)),
                       np.ones((4, 2))]), restarts=2)
    with pytest.raises(P.DivergenceError):
        P.solve_static(X, 2, P.make_loss("gaussian"),
                       P.SolverConfig(rate_factors=1e200, rate_decay=0.9, max_epochs_factors=2, iters_factors=5,
                                      samples=P.SamplerConfig(4, 4, 4, 4, seed=1)))
