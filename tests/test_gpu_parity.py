"""GPU parity: the CUDA engine against golden vectors from the reference and the
pinned CPU oracle, through the C ABI.  Tolerances: sampled indices bit-exact;
fp32 gradients/objectives within 1e-5 relative (norm-wise per mode); stream fit
within 1e-3 (BASELINE.json north_star)."""

import ctypes as C
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2110_14514_b200 as P
from paper_2110_14514_b200 import _lib
from paper_2110_14514_b200.tensor import DeviceModel
from oracle import ogcp_oracle as O

GRAD_RTOL = 1e-5


def load(golden_dir, name):
    return np.load(os.path.join(golden_dir, name), allow_pickle=False)


def rel_err(a, b):
    den = max(np.linalg.norm(b), 1e-300)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / den


def test_draws_bit_exact_vs_reference(golden_dir):
    g = load(golden_dir, "draws.npz")
    for ci in range(int(g["ncases"])):
        c = lambda k: g[f"c{ci}_{k}"]
        dims = tuple(int(d) for d in c("dims"))
        X = P.SparseTensor.from_zero_based(dims, c("subs0"), c("vals"))
        mr = int(c("max_rejects"))
        err = str(c("error"))
        if err:
            with pytest.raises(P.SamplingError) as ei:
                P.draw_samples(X, int(c("p")), int(c("q")), P.rng_at(int(c("seed")), *c("key").tolist()),
                               None if mr < 0 else mr)
            assert err.endswith(str(ei.value)), (ci, err, str(ei.value))
            continue
        s = P.draw_samples(X, int(c("p")), int(c("q")), P.rng_at(int(c("seed")), *c("key").tolist()),
                           None if mr < 0 else mr)
        np.testing.assert_array_equal(s.nz_ordinals, c("ordinals"), err_msg=f"case {ci}")
        np.testing.assert_array_equal(s.zero_subs0, c("zero_subs0"), err_msg=f"case {ci}")


@pytest.mark.parametrize("dims,nnz,p,q,seed,key", [
    ((1000, 997, 64), 200_000, 300_001, 200_000, 3, (7, 3, 1, 9)),
    ((100_000, 100_000, 1000), 1_000_000, 1_000_000, 1_000_000, 7, (5, 3, 0, 2)),
    ((4096, 4096), 3_000_000, 50_000, 1_000_000, 1, (2, 4)),     # 18% dense: many rejection rounds
    ((65536, 300, 7, 3), 500_000, 77_777, 333_333, 9, (1, 1, 1, 1)),
])
def test_draws_bit_exact_large(dims, nnz, p, q, seed, key):
    rng = np.random.default_rng(5)
    cells = int(np.prod(dims, dtype=object))
    lin = np.unique(rng.integers(0, cells, size=int(nnz * 1.05)))[:nnz]
    rng.shuffle(lin)
    subs0 = np.array(np.unravel_index(lin, dims)).T
    vals = rng.integers(1, 5, size=lin.size).astype(float)
    X = P.SparseTensor.from_zero_based(dims, subs0, vals)
    s = P.draw_samples(X, p, q, P.rng_at(seed, *key))
    ref = O.draw(O.Slice(dims, subs0, vals), p, q, O.keyed_rng(seed, *key))
    np.testing.assert_array_equal(s.nz_ordinals, ref.ordinals)
    np.testing.assert_array_equal(s.zero_subs0, ref.zero_subs0)


def _fused(X, factors, weights, kind, s, want_grads=True):
    model = DeviceModel.from_numpy(factors)
    grads = DeviceModel.zeros_like(model)
    gw = torch.zeros(model.rank, dtype=torch.float64, device="cuda")
    w, wp = _lib.f64arr(weights)
    gp = grads.ptrs()
    _lib.check(_lib.lib().ogcp_sampled_gradient(
        _lib.ctx(), X._handle, C.c_void_p(s.ord_dev.data_ptr() if s.p else None), s.p,
        C.c_void_p(s.zero_dev.data_ptr() if s.q else None), s.q, C.byref(model.c()), wp,
        C.byref(P.make_loss(kind)._c()), C.cast(gp, C.POINTER(C.c_void_p)), C.c_void_p(gw.data_ptr())))
    return grads.to_numpy(), gw.cpu().numpy()


def test_fused_sampled_gradient_vs_reference(golden_dir):
    g = load(golden_dir, "grads.npz")
    for ci in range(int(g["ncases"])):
        c = lambda k: g[f"c{ci}_{k}"]
        dims = tuple(int(d) for d in c("dims"))
        kind = str(c("kind"))
        X = P.SparseTensor.from_zero_based(dims, c("subs0"), c("vals"))
        A = [c(f"A{k}") for k in range(len(dims))]
        s = c("weights")
        t = 5
        smp = P.draw_samples(X, int(c("p")), int(c("q")), P.rng_at(13, t, 3, 0, ci))
        grads, gw = _fused(X, A, s, kind, smp)
        ys, yv = c("Y_subs0"), c("Y_vals")
        for k in range(len(dims)):
            want = O.mttkrp(ys, yv, dims, A, k) * s[None, :]
            assert rel_err(grads[k], want) < GRAD_RTOL, (ci, k, rel_err(grads[k], want))
        assert rel_err(gw, c("gw")) < GRAD_RTOL, (ci, rel_err(gw, c("gw")))


def test_factor_gradients_with_history_vs_reference(golden_dir):
    g = load(golden_dir, "grads.npz")
    for ci in range(int(g["ncases"])):
        c = lambda k: g[f"c{ci}_{k}"]
        dims = tuple(int(d) for d in c("dims"))
        A = [c(f"A{k}") for k in range(len(dims))]
        Aold = [c(f"Aold{k}") for k in range(len(dims))]
        window = list(zip(c("window_ids").tolist(), list(c("window_s"))))
        Y = P.SparseTensor.from_zero_based(dims, c("Y_subs0"), c("Y_vals"), allow_zero_values=True)
        G = P.factor_gradients(Y, A, c("weights"), old_factors=Aold, window=window, hist_weight=2.0, hist_decay=0.9,
                               t=5, reg_factors=0.3)
        for k in range(len(dims)):
            assert rel_err(G[k], c(f"G{k}")) < GRAD_RTOL, (ci, k, rel_err(G[k], c(f"G{k}")))
        gw = P.weight_gradient_mttkrp(Y, A)
        assert rel_err(gw, c("gw")) < GRAD_RTOL


def test_objective_vs_reference(golden_dir):
    g = load(golden_dir, "grads.npz")
    for ci in range(int(g["ncases"])):
        c = lambda k: g[f"c{ci}_{k}"]
        dims = tuple(int(d) for d in c("dims"))
        kind = str(c("kind"))
        X = P.SparseTensor.from_zero_based(dims, c("subs0"), c("vals"))
        A = [c(f"A{k}") for k in range(len(dims))]
        Aold = [c(f"Aold{k}") for k in range(len(dims))]
        window = list(zip(c("window_ids").tolist(), list(c("window_s"))))
        smp = P.draw_samples(X, int(c("p")), int(c("q")), P.rng_at(13, 5, 4))
        f = P.estimate_objective(X, A, c("weights"), P.make_loss(kind), smp, old_factors=Aold, window=window,
                                 hist_weight=2.0, hist_decay=0.9, t=5, reg_factors=0.3, reg_weights=0.2)
        assert f == pytest.approx(float(c("fobj")), rel=GRAD_RTOL), ci


def test_gram_identities():
    rng = np.random.default_rng(3)
    A = [rng.uniform(-1, 1, (d, 6)) for d in (50, 40, 7)]
    B = [rng.uniform(-1, 1, (d, 6)) for d in (50, 40, 7)]
    for mode in (None, 0, 2):
        np.testing.assert_allclose(P.gram(A, mode), O.hadamard_gram(A, mode), rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(P.gram(A, mode, other_factors=B), O.hadamard_gram(A, mode, B), rtol=1e-5,
                                   atol=1e-6)
    # known answer: all-ones 2x2, 3 modes, skip none -> 2*2*2... (kernels test KAT gram=12 analogue)
    ones = [np.ones((2, 1)), np.ones((3, 1)), np.ones((2, 1))]
    assert P.gram(ones)[0, 0] == pytest.approx(12.0)


def test_adam_matches_reference(golden_dir):
    g = load(golden_dir, "adam.npz")
    ad = P.Adam(0.1, lower_bound=0.0)
    a = np.array([1.0, 0.05, 2.0])
    ad.init(a)
    a = ad.update(a, True)
    seq = []
    for i in range(1, 6):
        a = ad.step(a, np.array([1.0, 2.0, -0.5]) * i, i)
        seq.append(a.copy())
    a = ad.update(a, False)
    seq.append(a.copy())
    np.testing.assert_allclose(np.vstack(seq), g["seq"], rtol=1e-6, atol=1e-7)
    assert ad.rate == pytest.approx(float(g["rate"]))


def run_engine_stream(g, name):
    c = lambda k: g[f"{name}_{k}"]
    kind = str(c("kind"))
    dims = tuple(int(d) for d in c("dims"))
    kw = json.loads(str(c("cfg")))
    sm = json.loads(str(c("samples")))
    cfg = P.SolverConfig(**kw, samples=P.SamplerConfig(sm["p"], sm["q"], sm["p_obj"], sm["q_obj"], seed=sm["seed"]))
    loss = P.make_loss(kind)
    st = P.fresh_state(dims[:-1], int(c("R")), loss, cfg, factors=[c(f"init{k}") for k in range(len(dims) - 1)])
    st.window = P.HistoryWindow(capacity=int(c("H")))
    for h, s_h in enumerate(c("warm_weights"), start=1):
        st.weights_log.append(s_h)
        st.window.observe(h, s_h, P.rng_at(cfg.samples.seed, h, 5))
    st.t = int(c("n_warm"))
    full_s, full_v = c("subs0"), c("vals")
    rows = []
    for t in range(st.t + 1, st.t + int(c("n_stream")) + 1):
        mask = full_s[:, -1] == t - 1
        X = P.SparseTensor.from_zero_based(dims[:-1], full_s[mask, :-1], full_v[mask])
        rows.append(P.process_slice(st, X, loss, cfg, exact_loss=True))
    return st, rows


@pytest.mark.parametrize("name", ["gauss", "pois", "bern"])
def test_stream_fit_vs_reference(golden_dir, name):
    g = load(golden_dir, "streams.npz")
    c = lambda k: g[f"{name}_{k}"]
    st, rows = run_engine_stream(g, name)
    loc_x = np.array([r.local_loss_exact for r in rows])
    loc_s = np.array([r.local_loss_sampled for r in rows])
    np.testing.assert_allclose(loc_x, c("local_exact"), rtol=1e-3)
    np.testing.assert_allclose(loc_s, c("local_sampled"), rtol=1e-3)
    for k, a in enumerate(st.factors):
        assert rel_err(a, c(f"final{k}")) < 1e-3
    assert rel_err(np.vstack(st.weights_log), c("weights_log")) < 1e-3
    assert st.iteration == int(c("iteration"))
    assert st.window.step_ids() == c("window_ids").tolist()


@pytest.mark.parametrize("merge,buckets,R,impl", [(True, 1, 6, "tma"), (False, 1, 6, "tma"), (True, 4, 6, "tma"),
                                                  (True, 32, 6, "tma"), (True, 4, 12, "tma"), (True, 1, 20, "tma"),
                                                  (True, 4, 20, "tma"), (True, 32, 20, "tma"), (True, 4, 20, "lean"),
                                                  (True, 4, 20, "generic"), (True, 1, 12, "lean"),
                                                  (True, 4, 20, "tma-all"), (True, 1, 12, "tma-all"),
                                                  (True, 4, 20, "tma-a2")])
def test_dense_draw_solve_vs_oracle(merge, buckets, R, impl):
    """p = all nonzeros on a 1e5-nnz slice: the merged (count) form -- walked in
    ordinal order or in the slice's row-bucket order, by the TMA-fed or the
    register-pipelined 3-way walk kernels (ldr 16 / 32, csrc/walk_tma.cuh,
    csrc/walk3.cuh) or the generic ones -- and the per-draw
    form of the solve all match the oracle's slice step."""
    rng = np.random.default_rng(21)
    dims = (300, 200, 40)
    lin = rng.choice(int(np.prod(dims)), size=100_000, replace=False)
    subs0 = np.array(np.unravel_index(np.sort(lin), dims)).T
    vals = rng.integers(1, 4, size=lin.size).astype(float)
    init = [rng.uniform(0.2, 1.0, (d, R)) for d in dims]
    _lib.set_merge_draws(merge)
    _lib.set_buckets(buckets)
    _lib.set_walk_impl(impl)
    try:
        X = P.SparseTensor.from_zero_based(dims, subs0, vals)
        cfg = P.SolverConfig(max_epochs_weights=1, max_epochs_factors=1, iters_weights=4, iters_factors=4,
                             rate_weights=0.05, rate_factors=1e-2, hist_weight=1.0, warm_start_weights=True,
                             samples=P.SamplerConfig(None, 5000, 20000, 20000, seed=3))
        loss = P.make_loss("poisson")
        st = P.fresh_state(dims, R, loss, cfg, factors=init)
        st.window = P.HistoryWindow(capacity=2)
        for h in (1, 2):
            s_h = np.full(R, 1.0 + 0.1 * h)
            st.weights_log.append(s_h)
            st.window.observe(h, s_h, P.rng_at(3, h, 5))
        st.t = 2
        m = P.process_slice(st, X, loss, cfg, exact_loss=True)
    finally:
        _lib.set_merge_draws(True)
        _lib.set_buckets(1)
        _lib.set_walk_impl("tma")
    ocfg = O.Cfg(kappa_w=1, kappa_f=1, tau_w=4, tau_f=4, rate_w=0.05, rate_f=1e-2, hist_weight=1.0,
                 warm_weights=True, p=None, q=5000, p_obj=20000, q_obj=20000, seed=3)
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
    for a, b in zip(st.factors, ost.factors):
        assert rel_err(a, b) < 1e-4
    assert rel_err(st.weights_log[-1], s_t) < 1e-4


def test_gradient_tensor_layout_bit_exact(golden_dir):
    """Row A6: merged Y (np.unique + bincount, sampling.py:233-239) and the per-mode
    row-segment layouts are bit-exact; values within fp32-factor tolerance."""
    g = load(golden_dir, "grads.npz")
    for ci in range(int(g["ncases"])):
        c = lambda k: g[f"c{ci}_{k}"]
        dims = tuple(int(d) for d in c("dims"))
        X = P.SparseTensor.from_zero_based(dims, c("subs0"), c("vals"))
        A = [c(f"A{k}") for k in range(len(dims))]
        Y = P.sampled_gradient_tensor(X, A, c("weights"), P.make_loss(str(c("kind"))), int(c("p")), int(c("q")),
                                      P.rng_at(13, 5, 3, 0, ci))
        np.testing.assert_array_equal(Y.subs0, c("Y_subs0"))
        assert rel_err(Y.vals, c("Y_vals")) < GRAD_RTOL
        for k in range(len(dims)):
            perm, offs = P.segment_layout(Y, k)
            np.testing.assert_array_equal(perm, np.argsort(c("Y_subs0")[:, k], kind="stable"))
            want = np.concatenate([[0], np.cumsum(np.bincount(c("Y_subs0")[:, k], minlength=dims[k]))])
            np.testing.assert_array_equal(offs, want)


def test_gradient_tensor_large_merge_vs_oracle():
    rng = np.random.default_rng(12)
    dims = (2000, 1500, 30)
    lin = rng.choice(int(np.prod(dims)), size=300_000, replace=False)
    subs0 = np.array(np.unravel_index(lin, dims)).T
    vals = rng.integers(1, 5, size=lin.size).astype(float)
    R = 5
    A = [rng.uniform(0.1, 1.0, (d, R)) for d in dims]
    w = rng.uniform(0.5, 1.5, R)
    X = P.SparseTensor.from_zero_based(dims, subs0, vals)
    Y = P.sampled_gradient_tensor(X, A, w, P.make_loss("poisson"), 600_000, 200_000, P.rng_at(2, 9, 3, 1, 4))
    _, ys, yv = O.sampled_y(O.Slice(dims, subs0, vals), A, w, "poisson", 600_000, 200_000, O.keyed_rng(2, 9, 3, 1, 4))
    np.testing.assert_array_equal(Y.subs0, ys)
    assert rel_err(Y.vals, yv) < GRAD_RTOL


@pytest.mark.parametrize("kind", ["gaussian", "poisson", "bernoulli"])
def test_global_loss_vs_oracle(kind):
    """global_loss (metrics.py:73-92): the average over the stream's slices of the exact
    local loss of [[s_t; final factors]] -- every cell, zeros included, over ||X_t||^2 --
    against the oracle's exact_local_loss (metrics.py:50-57) slice by slice."""
    rng = np.random.default_rng(11)
    dims, R, T = (14, 9, 6), 4, 3
    factors = [rng.uniform(0.2, 1.0, (d, R)) for d in dims]
    weights_log = [rng.uniform(0.5, 1.5, R) for _ in range(T)]
    slices, want = [], []
    for t in range(T):
        lin = rng.choice(int(np.prod(dims)), size=150, replace=False)
        subs0 = np.array(np.unravel_index(np.sort(lin), dims)).T
        vals = (np.ones(lin.size) if kind == "bernoulli" else
                rng.integers(1, 5, size=lin.size).astype(float) if kind == "poisson" else rng.normal(size=lin.size))
        slices.append(P.SparseTensor.from_zero_based(dims, subs0, vals))
        want.append(O.exact_local_loss(O.Slice(dims, subs0, vals), factors, weights_log[t], kind))
    got = P.global_loss(slices, factors, weights_log, P.make_loss(kind))
    assert got == pytest.approx(float(np.mean(want)), rel=1e-5)
    with pytest.raises(P.DataError):
        P.global_loss(slices, factors, weights_log[:1], P.make_loss(kind))
