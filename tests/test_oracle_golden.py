"""Pin the CPU oracle against golden vectors produced by the reference itself."""

import json
import os

import numpy as np
import pytest

from oracle import ogcp_oracle as O


def load(golden_dir, name):
    return np.load(os.path.join(golden_dir, name), allow_pickle=False)


def test_draws_match_reference(golden_dir):
    g = load(golden_dir, "draws.npz")
    for ci in range(int(g["ncases"])):
        c = lambda k: g[f"c{ci}_{k}"]
        X = O.Slice(tuple(int(d) for d in c("dims")), c("subs0"), c("vals"))
        mr = int(c("max_rejects"))
        err = str(c("error"))
        try:
            s = O.draw(X, int(c("p")), int(c("q")), O.keyed_rng(int(c("seed")), *c("key").tolist()),
                       None if mr < 0 else mr)
        except O.OracleError as exc:
            assert err.endswith(str(exc)), (ci, err, exc)
            continue
        assert err == "", ci
        np.testing.assert_array_equal(s.ordinals, c("ordinals"))
        np.testing.assert_array_equal(s.zero_subs0, c("zero_subs0"))


def test_gradients_objective_match_reference(golden_dir):
    g = load(golden_dir, "grads.npz")
    for ci in range(int(g["ncases"])):
        c = lambda k: g[f"c{ci}_{k}"]
        dims = tuple(int(d) for d in c("dims"))
        kind = str(c("kind"))
        X = O.Slice(dims, c("subs0"), c("vals"))
        A = [c(f"A{k}") for k in range(len(dims))]
        Aold = [c(f"Aold{k}") for k in range(len(dims))]
        s = c("weights")
        window = list(zip(c("window_ids").tolist(), list(c("window_s"))))
        t = 5
        _, ys, yv = O.sampled_y(X, A, s, kind, int(c("p")), int(c("q")), O.keyed_rng(13, t, 3, 0, ci))
        np.testing.assert_array_equal(ys, c("Y_subs0"))
        np.testing.assert_allclose(yv, c("Y_vals"), rtol=1e-12, atol=0)
        G = O.assemble_factor_grads(ys, yv, dims, A, s, Aold, window, 2.0, 0.9, t, 0.3)
        for k in range(len(dims)):
            np.testing.assert_allclose(G[k], c(f"G{k}"), rtol=1e-10, atol=1e-10 * np.abs(G[k]).max())
        np.testing.assert_allclose(O.weight_grad(ys, yv, A), c("gw"), rtol=1e-10)
        d = O.draw(X, int(c("p")), int(c("q")), O.keyed_rng(13, t, 4))
        f = O.objective(X, A, s, kind, d, old_factors=Aold, window=window, hist_weight=2.0, hist_decay=0.9,
                        t=t, reg_factors=0.3, reg_weights=0.2)
        assert f == pytest.approx(float(c("fobj")), rel=1e-12)


def test_adam_matches_reference(golden_dir):
    g = load(golden_dir, "adam.npz")
    ad = O.AdamOracle(0.1, lower=0.0)
    a = [np.array([1.0, 0.05, 2.0])]
    ad.init(a)
    a = ad.epoch_end(a, True)
    seq = []
    for i in range(1, 6):
        a = ad.step(a, [np.array([1.0, 2.0, -0.5]) * i], i)
        seq.append(a[0].copy())
    a = ad.epoch_end(a, False)
    seq.append(a[0].copy())
    np.testing.assert_array_equal(np.vstack(seq), g["seq"])
    assert ad.rate == float(g["rate"])


def run_oracle_stream(g, name):
    c = lambda k: g[f"{name}_{k}"]
    kind = str(c("kind"))
    dims = tuple(int(d) for d in c("dims"))
    kw = json.loads(str(c("cfg")))
    sm = json.loads(str(c("samples")))
    cfg = O.Cfg(kappa_w=kw["max_epochs_weights"], kappa_f=kw["max_epochs_factors"], tau_w=kw["iters_weights"],
                tau_f=kw["iters_factors"], rate_w=kw["rate_weights"], rate_f=kw["rate_factors"],
                hist_weight=kw.get("hist_weight", 0.0), hist_decay=kw.get("hist_decay", 1.0),
                warm_weights=kw.get("warm_start_weights", False), reg_factors=kw.get("reg_factors", 0.0),
                reg_weights=kw.get("reg_weights", 0.0), p=sm["p"], q=sm["q"], p_obj=sm["p_obj"],
                q_obj=sm["q_obj"], seed=sm["seed"])
    R = int(c("R"))
    st = O.new_stream([c(f"init{k}") for k in range(len(dims) - 1)], kind, cfg, capacity=int(c("H")))
    for h, s_h in enumerate(c("warm_weights"), start=1):
        st.weights_log.append(s_h)
        O.window_observe(st, h, s_h, cfg.seed)
    st.t = int(c("n_warm"))
    full = O.Slice(dims, c("subs0"), c("vals"))
    loc_s, loc_x = [], []
    for t in range(st.t + 1, st.t + int(c("n_stream")) + 1):
        mask = full.subs0[:, -1] == t - 1
        X = O.Slice(dims[:-1], full.subs0[mask, :-1], full.vals[mask])
        s_t = O.slice_step(st, X, kind, cfg)
        loc_s.append(O.sampled_local_loss(X, st.factors, s_t, kind, cfg, t))
        loc_x.append(O.exact_local_loss(X, st.factors, s_t, kind))
    return st, cfg, np.array(loc_s), np.array(loc_x)


@pytest.mark.parametrize("name", ["gauss", "pois", "bern"])
def test_stream_matches_reference(golden_dir, name):
    g = load(golden_dir, "streams.npz")
    c = lambda k: g[f"{name}_{k}"]
    st, cfg, loc_s, loc_x = run_oracle_stream(g, name)
    for k, a in enumerate(st.factors):
        np.testing.assert_allclose(a, c(f"final{k}"), rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(np.vstack(st.weights_log), c("weights_log"), rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(loc_s, c("local_sampled"), rtol=1e-9)
    np.testing.assert_allclose(loc_x, c("local_exact"), rtol=1e-9)
    assert st.iteration == int(c("iteration"))
    assert [h for h, _ in st.window] == c("window_ids").tolist()
    assert st.adam.rate == pytest.approx(float(c("adam_rate")))
    ftr = json.loads(str(c("ftrace")))
    for (_, _, f), ref in zip(st.traces, ftr):
        np.testing.assert_allclose(f, ref, rtol=1e-9)


def static_case(g, name):
    c = lambda k: g[f"{name}_{k}"]
    kw = json.loads(str(c("cfg")))
    sm = json.loads(str(c("samples")))
    cfg = O.Cfg(kappa_f=kw["max_epochs_factors"], tau_f=kw["iters_factors"], rate_f=kw["rate_factors"],
                reg_factors=kw.get("reg_factors", 0.0), reg_weights=kw.get("reg_weights", 0.0),
                rate_decay=kw.get("rate_decay", 0.1), p=sm["p"], q=sm["q"], p_obj=sm["p_obj"],
                q_obj=sm["q_obj"], seed=sm["seed"])
    X = O.Slice(tuple(int(d) for d in c("dims")), c("subs0"), c("vals"))
    return c, str(c("kind")), int(c("R")), cfg, X


@pytest.mark.parametrize("name", ["gauss", "pois", "bern"])
def test_static_and_warm_start_match_reference(golden_dir, name):
    g = load(golden_dir, "static.npz")
    c, kind, R, cfg, X = static_case(g, name)
    w, fs, trace, epochs, rej = O.static_solve(X, R, kind, cfg, seed_key=4)
    np.testing.assert_allclose(w, c("static_weights"), rtol=1e-9, atol=1e-12)
    for k, a in enumerate(fs):
        np.testing.assert_allclose(a, c(f"static_A{k}"), rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(trace, c("static_trace"), rtol=1e-9)
    assert (epochs, rej) == (int(c("static_epochs")), int(c("static_rejections")))
    st = O.warm_start(X, R, kind, cfg, int(c("capacity")), restarts=int(c("restarts")))
    for k, a in enumerate(st.factors):
        np.testing.assert_allclose(a, c(f"warm_A{k}"), rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(np.vstack(st.weights_log), c("warm_weights_log"), rtol=1e-9, atol=1e-12)
    assert [h for h, _ in st.window] == c("warm_window_ids").tolist()
    assert st.t == int(c("warm_t"))


def gaussian_fixture(golden_dir):
    g = load(golden_dir, "gaussian.npz")
    dims = tuple(int(d) for d in g["dims"])
    full = O.Slice(dims, g["subs0"], g["vals"])
    init = [g[f"init{k}"] for k in range(len(dims) - 1)]

    def slice_at(t):
        mask = full.subs0[:, -1] == t - 1
        return O.Slice(dims[:-1], full.subs0[mask, :-1], full.vals[mask])
    return g, dims, full, init, slice_at


def gaussian_cfg(kw, seed=0):
    return O.Cfg(kappa_w=kw.get("max_epochs_weights", 20), kappa_f=kw["max_epochs_factors"],
                 tau_w=kw.get("iters_weights", 100), tau_f=kw["iters_factors"],
                 rate_w=kw.get("rate_weights", 0.1), rate_f=kw["rate_factors"],
                 hist_weight=kw.get("hist_weight", 0.0), hist_decay=kw.get("hist_decay", 1.0),
                 reg_factors=kw.get("reg_factors", 0.0), reg_weights=kw.get("reg_weights", 0.0),
                 p=100 if kw.get("gradient_mode") else 150, q=0, p_obj=200, q_obj=0, seed=4,
                 dense=kw.get("gradient_mode") == "dense-gaussian",
                 least_squares=kw.get("temporal_solver") == "least-squares")


def test_gaussian_direct_match_reference(golden_dir):
    g, dims, full, init, slice_at = gaussian_fixture(golden_dir)
    X1, w0 = slice_at(1), g["warm_weights"][0]
    assert O.gaussian_residual(X1, init, w0) == pytest.approx(float(g["resid"]), rel=1e-12)
    np.testing.assert_allclose(O.least_squares_weights(X1, init, 0.0), g["ls_mu0"], rtol=1e-10)
    np.testing.assert_allclose(O.least_squares_weights(X1, init, 0.3), g["ls_mu"], rtol=1e-10)
    np.testing.assert_allclose(O.dense_weight_grad(X1, init, w0, 0.2), g["dense_wgrad"], rtol=1e-10)
    for k, gk in enumerate(O.dense_factor_grads(X1, init, w0, None, (), 0.0, 1.0, 0, 0.1)):
        np.testing.assert_allclose(gk, g[f"dense_fgrad{k}"], rtol=1e-10, atol=1e-12)
    for i, want in enumerate(g["cong_scores"]):
        got = O.congruence(g[f"cong{i}_w1"], [g[f"cong{i}_f1_{k}"] for k in range(3)],
                           g[f"cong{i}_w2"], [g[f"cong{i}_f2_{k}"] for k in range(3)])
        assert got == pytest.approx(float(want), rel=1e-12, abs=1e-14)


@pytest.mark.parametrize("name", ["dense", "ls"])
def test_gaussian_streams_match_reference(golden_dir, name):
    g, dims, full, init, slice_at = gaussian_fixture(golden_dir)
    cfg = gaussian_cfg(json.loads(str(g[f"{name}_cfg"])))
    st = O.new_stream(init, "gaussian", cfg, capacity=2)
    for h in (1, 2):
        st.weights_log.append(g["warm_weights"][h - 1])
        O.window_observe(st, h, g["warm_weights"][h - 1], cfg.seed)
    st.t = 2
    loc = []
    for t in range(3, dims[-1] + 1):
        s_t = O.slice_step(st, slice_at(t), "gaussian", cfg)
        loc.append(O.exact_local_loss(slice_at(t), st.factors, s_t, "gaussian"))
    np.testing.assert_allclose(np.vstack(st.weights_log), g[f"{name}_weights_log"], rtol=1e-8, atol=1e-12)
    for k, a in enumerate(st.factors):
        np.testing.assert_allclose(a, g[f"{name}_final{k}"], rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(loc, g[f"{name}_local_exact"], rtol=1e-8)
    assert st.iteration == int(g[f"{name}_iteration"])
    for (_, w, f), wr, fr in zip(st.traces, json.loads(str(g[f"{name}_wtrace"])),
                                 json.loads(str(g[f"{name}_ftrace"]))):
        np.testing.assert_allclose(w, wr, rtol=1e-8)
        np.testing.assert_allclose(f, fr, rtol=1e-8)


def test_gaussian_static_restarts_match_reference(golden_dir):
    g, dims, full, init, slice_at = gaussian_fixture(golden_dir)
    cfg = O.Cfg(kappa_f=3, tau_f=10, rate_f=2e-2, reg_factors=0.01, reg_weights=0.02, p=100, q=0, p_obj=200,
                q_obj=0, seed=4, dense=True)
    w, fs, trace, *_ = O.static_fit(full, 3, "gaussian", cfg, restarts=2, seed_key=3)
    np.testing.assert_allclose(w, g["static_weights"], rtol=1e-8)
    for k, a in enumerate(fs):
        np.testing.assert_allclose(a, g[f"static_A{k}"], rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(trace, g["static_trace"], rtol=1e-8)
