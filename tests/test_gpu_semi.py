"""GPU tests of the semi-stratified extension (parity against the restated oracle,
which tests/test_oracle_semi.py pins by Monte-Carlo unbiasedness)."""

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2110_14514_b200 as P
from paper_2110_14514_b200 import _lib
from paper_2110_14514_b200.tensor import DeviceModel
from oracle import ogcp_oracle as O


def _slice(seed, dims, nnz):
    rng = np.random.default_rng(seed)
    lin = rng.choice(int(np.prod(dims)), size=nnz, replace=False)
    subs0 = np.array(np.unravel_index(lin, dims)).T
    vals = rng.integers(1, 4, size=lin.size).astype(float)
    return subs0, vals


@pytest.mark.parametrize("dims,nnz,p,q", [((50, 40, 30), 3000, 5000, 7000), ((1, 60, 9), 200, 300, 400),
                                           ((4, 4), 16, 10, 50)])
def test_semi_draws_bit_exact(dims, nnz, p, q):
    subs0, vals = _slice(1, dims, nnz)
    X = P.SparseTensor.from_zero_based(dims, subs0, vals)
    s = P.draw_samples(X, p, q, P.rng_at(5, 3, 1), semi_stratified=True)
    ref = O.draw_semi(O.Slice(dims, subs0, vals), p, q, O.keyed_rng(5, 3, 1))
    np.testing.assert_array_equal(s.nz_ordinals, ref.ordinals)
    np.testing.assert_array_equal(s.zero_subs0, ref.zero_subs0)


@pytest.mark.parametrize("kind", ["poisson", "bernoulli", "gaussian"])
def test_semi_gradient_vs_oracle(kind):
    dims = (40, 30, 20)
    subs0, vals = _slice(2, dims, 2000)
    if kind == "bernoulli":
        vals = np.ones_like(vals)
    rng = np.random.default_rng(3)
    R = 5
    A = [rng.uniform(0.2, 1.0, (d, R)) for d in dims]
    w = rng.uniform(0.5, 1.5, R)
    X = P.SparseTensor.from_zero_based(dims, subs0, vals)
    s = P.draw_samples(X, 3000, 4000, P.rng_at(8, 1), semi_stratified=True)
    model = DeviceModel.from_numpy(A)
    grads = DeviceModel.zeros_like(model)
    gw = torch.zeros(R, dtype=torch.float64, device="cuda")
    wa, wp = _lib.f64arr(w)
    gp = grads.ptrs()
    _lib.check(_lib.lib().ogcp_sampled_gradient_ex(
        _lib.ctx(), X._handle, C.c_void_p(s.ord_dev.data_ptr()), s.p, C.c_void_p(s.zero_dev.data_ptr()), s.q,
        C.byref(model.c()), wp, C.byref(P.make_loss(kind)._c()), 1, C.cast(gp, C.POINTER(C.c_void_p)),
        C.c_void_p(gw.data_ptr())))
    os_ = O.draw_semi(O.Slice(dims, subs0, vals), 3000, 4000, O.keyed_rng(8, 1))
    ys, yv = O.semi_y(O.Slice(dims, subs0, vals), A, w, kind, os_)
    for k, g in enumerate(grads.to_numpy()):
        want = O.mttkrp(ys, yv, dims, A, k) * w
        assert np.linalg.norm(g - want) <= 1e-5 * np.linalg.norm(want)
    want = O.weight_grad(ys, yv, A)
    assert np.linalg.norm(gw.cpu().numpy() - want) <= 1e-5 * np.linalg.norm(want)


def test_semi_stratified_stream_runs():
    """A c3-like (Bernoulli, semi-stratified) solve makes progress on the sampled objective."""
    dims = (300, 200, 50)
    subs0, vals = _slice(4, dims, 20000)
    vals = np.ones_like(vals)
    rng = np.random.default_rng(5)
    R = 4
    init = [rng.uniform(0.05, 0.3, (d, R)) for d in dims]
    cfg = P.SolverConfig(max_epochs_weights=2, max_epochs_factors=2, iters_weights=20, iters_factors=20,
                         rate_weights=0.05, rate_factors=1e-2,
                         samples=P.SamplerConfig(4000, 4000, 8000, 8000, seed=1, semi_stratified=True))
    loss = P.make_loss("bernoulli")
    st = P.fresh_state(dims, R, loss, cfg, factors=init)
    X = P.SparseTensor.from_zero_based(dims, subs0, vals)
    m = P.process_slice(st, X, loss, cfg, exact_loss=True)
    assert np.isfinite(m.local_loss_exact)
    _, wtr, ftr = st.trace_log[-1]
    assert all(b <= a for a, b in zip(wtr, wtr[1:])) and all(b <= a for a, b in zip(ftr, ftr[1:]))


@pytest.mark.parametrize("p,buckets", [(6000, 1), (None, 1), (None, 4)])
def test_semi_stream_step_vs_oracle(p, buckets):
    """A full semi-stratified slice step (weight + factor solves, history) against the
    oracle restatement: per-draw and merged (count-form) draws, with and without the
    row-bucketed walk."""
    dims = (300, 200, 40)
    subs0, vals = _slice(6, dims, 100_000)
    rng = np.random.default_rng(7)
    R = 5
    init = [rng.uniform(0.2, 1.0, (d, R)) for d in dims]
    _lib.set_buckets(buckets)
    try:
        cfg = P.SolverConfig(max_epochs_weights=1, max_epochs_factors=1, iters_weights=4, iters_factors=4,
                             rate_weights=0.05, rate_factors=1e-2, hist_weight=1.0, warm_start_weights=True,
                             samples=P.SamplerConfig(p, 5000, 20000, 20000, seed=3, semi_stratified=True))
        loss = P.make_loss("poisson")
        st = P.fresh_state(dims, R, loss, cfg, factors=init)
        st.window = P.HistoryWindow(capacity=2)
        for h in (1, 2):
            s_h = np.full(R, 1.0 + 0.1 * h)
            st.weights_log.append(s_h)
            st.window.observe(h, s_h, P.rng_at(3, h, 5))
        st.t = 2
        X = P.SparseTensor.from_zero_based(dims, subs0, vals)
        m = P.process_slice(st, X, loss, cfg, exact_loss=True)
    finally:
        _lib.set_buckets(1)
    ocfg = O.Cfg(kappa_w=1, kappa_f=1, tau_w=4, tau_f=4, rate_w=0.05, rate_f=1e-2, hist_weight=1.0,
                 warm_weights=True, p=p, q=5000, p_obj=20000, q_obj=20000, seed=3, semi=True)
    ost = O.new_stream(init, "poisson", ocfg, capacity=2)
    for h in (1, 2):
        s_h = np.full(R, 1.0 + 0.1 * h)
        ost.weights_log.append(s_h)
        O.window_observe(ost, h, s_h, 3)
    ost.t = 2
    Xo = O.Slice(dims, subs0, vals)
    s_t = O.slice_step(ost, Xo, "poisson", ocfg)
    want = O.exact_local_loss(Xo, ost.factors, s_t, "poisson")
    assert m.local_loss_exact == pytest.approx(want, rel=1e-4)
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
    for a, b in zip(st.factors, ost.factors):
        assert rel(a, b) < 1e-4
    assert rel(st.weights_log[-1], s_t) < 1e-4
    for (_, w, f), (_, ow, of) in zip(st.trace_log[-1:], ost.traces[-1:]):
        np.testing.assert_allclose(w, ow, rtol=1e-4)
        np.testing.assert_allclose(f, of, rtol=1e-4)
