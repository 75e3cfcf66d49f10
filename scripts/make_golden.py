"""Generate golden vectors from the REFERENCE implementation (build container only).

Runs the reference package ``ogcp`` 0.1.0 from /root/reference/pkg/src and writes
small fixtures under tests/golden/ that pin both the CPU oracle (oracle/) and the
CUDA engine.  /root/reference does not exist on the GPU box; the fixtures travel
instead.  Re-run with:  python scripts/make_golden.py
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")


def random_sparse(ogcp, rng, dims, nnz, kind):
    cells = int(np.prod(dims))
    lin = rng.choice(cells, size=nnz, replace=False)
    subs0 = np.array(np.unravel_index(lin, dims)).T.reshape(-1, len(dims))
    if kind == "poisson":
        vals = rng.integers(1, 6, nnz).astype(float)
    elif kind == "bernoulli":
        vals = np.ones(nnz)
    else:
        vals = rng.standard_normal(nnz)
        vals[vals == 0] = 1.0
    return ogcp.SparseTensor.from_zero_based(dims, subs0, vals)


def main():
    sys.path.insert(0, REF)
    import ogcp
    from ogcp import sampling, solvers, streaming, metrics

    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(20211027)

    # ---------------------------------------------------------------- draws
    draw_cases = [
        # dims, nnz, seed, key, p, q, max_rejects
        ((10, 10), 20, 0, (3,), 10, 16, None),
        ((6, 7, 5), 40, 7, (4, 3, 0, 1), 300, 200, None),
        ((1, 9, 4), 10, 1, (2, 1), 50, 50, None),          # unit dim consumes no words
        ((13, 11, 3, 2), 60, 11, (9, 3, 2, 7), 77, 91, None),
        ((32, 77, 24), 900, 7, (5, 3, 0, 17), 900, 1000, None),
        ((40, 1, 1), 1, 5, (1, 1), 33, 12, None),          # eta == 1 consumes no words
        ((5, 5), 0, 3, (1, 2), 0, 8, None),                # empty slice
        ((4, 4), 15, 0, (6,), 5, 40, None),                # dense: many rejections
        ((3, 3), 8, 2, (1,), 0, 5, 3),                     # exhausted budget -> SamplingError
        ((1000, 997, 64), 5000, 99, (12, 3, 4, 99), 4096, 4096, None),
    ]
    draws = {}
    for ci, (dims, nnz, seed, key, p, q, mr) in enumerate(draw_cases):
        X = random_sparse(ogcp, rng, dims, nnz, "gaussian")
        rec = dict(dims=np.array(dims), subs0=X.subs0.copy(), vals=X.vals.copy(),
                   seed=np.array(seed), key=np.array(key), p=np.array(p), q=np.array(q),
                   max_rejects=np.array(-1 if mr is None else mr))
        try:
            s = sampling.draw_samples(X, p, q, sampling.rng_at(seed, *key), mr)
            rec.update(ordinals=s.nz_ordinals.copy(), zero_subs0=s.zero_subs0.copy(), error=np.array(""))
        except ogcp.OgcpError as exc:
            rec.update(ordinals=np.empty(0, np.int64), zero_subs0=np.empty((0, len(dims)), np.int64),
                       error=np.array(f"{type(exc).__name__}: {exc}"))
        for k, v in rec.items():
            draws[f"c{ci}_{k}"] = v
    draws["ncases"] = np.array(len(draw_cases))
    np.savez_compressed(os.path.join(OUT, "draws.npz"), **draws)

    # ------------------------------------------- gradients / objective per loss
    grads = {}
    gcases = [("gaussian", (7, 6, 5), 60, 4, 200, 150), ("poisson", (9, 8, 7), 80, 5, 300, 400),
              ("bernoulli", (12, 10, 6), 90, 3, 250, 300), ("poisson", (20, 15), 70, 6, 150, 120)]
    for ci, (kind, dims, nnz, R, p, q) in enumerate(gcases):
        X = random_sparse(ogcp, rng, dims, nnz, kind)
        lo = 0.1 if kind != "gaussian" else -1.0
        factors = [rng.uniform(lo, 1.0, (d, R)) for d in dims]
        old = [a + 0.05 * rng.uniform(-1, 1, a.shape) for a in factors]
        if kind != "gaussian":
            old = [np.abs(a) for a in old]
        weights = rng.uniform(0.2, 1.5, R)
        window = [(h, rng.uniform(0.1, 1.0, R)) for h in (1, 3, 4)]
        loss = ogcp.make_loss(kind)
        t = 5
        Y = sampling.sampled_gradient_tensor(X, factors, weights, loss, p, q, sampling.rng_at(13, t, 3, 0, ci))
        G = solvers.factor_gradients(Y, factors, weights, old_factors=old, window=window, hist_weight=2.0,
                                     hist_decay=0.9, t=t, reg_factors=0.3)
        gw = ogcp.weight_gradient_mttkrp(Y, factors)
        objs = sampling.draw_samples(X, p, q, sampling.rng_at(13, t, 4))
        fobj = sampling.estimate_objective(X, factors, weights, loss, objs, old_factors=old, window=window,
                                           hist_weight=2.0, hist_decay=0.9, t=t, reg_factors=0.3,
                                           reg_weights=0.2)
        rec = dict(kind=np.array(kind), dims=np.array(dims), subs0=X.subs0, vals=X.vals, weights=weights,
                   R=np.array(R), p=np.array(p), q=np.array(q), Y_subs0=Y.subs0, Y_vals=Y.vals, gw=gw,
                   fobj=np.array(fobj), window_ids=np.array([h for h, _ in window]),
                   window_s=np.vstack([s for _, s in window]))
        for k in range(len(dims)):
            rec[f"A{k}"] = factors[k]
            rec[f"Aold{k}"] = old[k]
            rec[f"G{k}"] = G[k]
        for k, v in rec.items():
            grads[f"c{ci}_{k}"] = v
    grads["ncases"] = np.array(len(gcases))
    np.savez_compressed(os.path.join(OUT, "grads.npz"), **grads)

    # ----------------------------------------------------------- Adam KATs
    adam = ogcp.Adam(0.1, lower_bound=0.0)
    a = np.array([1.0, 0.05, 2.0])
    adam.init(a)
    a = adam.update(a, True)
    seq = []
    for i in range(1, 6):
        a = adam.step(a, np.array([1.0, 2.0, -0.5]) * i, i)
        seq.append(a.copy())
    a = adam.update(a, False)
    seq.append(a.copy())
    np.savez_compressed(os.path.join(OUT, "adam.npz"), seq=np.vstack(seq), rate=np.array(adam.rate))

    # -------------------------------------------------------------- streams
    streams = {}
    scases = [
        # name, kind, dims(with time), R, density, cfg kwargs, H, n_warm, n_stream
        ("gauss", "gaussian", (6, 5, 4, 6), 3, None,
         dict(max_epochs_weights=3, max_epochs_factors=2, iters_weights=20, iters_factors=20,
              rate_weights=0.5, rate_factors=1e-2, hist_weight=1.0, hist_decay=0.95,
              samples=sampling.SamplerConfig(200, 0, 300, 0, seed=3)), 3, 2, 4),
        ("pois", "poisson", (8, 9, 5, 7), 3, 0.2,
         dict(max_epochs_weights=2, max_epochs_factors=2, iters_weights=15, iters_factors=15,
              rate_weights=0.1, rate_factors=1e-2, hist_weight=10.0, warm_start_weights=True,
              reg_factors=0.01, reg_weights=0.02,
              samples=sampling.SamplerConfig(None, 60, None, 200, seed=7)), 2, 2, 5),
        ("bern", "bernoulli", (7, 6, 8, 6), 2, 0.15,
         dict(max_epochs_weights=2, max_epochs_factors=2, iters_weights=10, iters_factors=10,
              rate_weights=0.1, rate_factors=1e-2, hist_weight=5.0, hist_decay=0.8,
              samples=sampling.SamplerConfig(30, 40, 60, 80, seed=5)), 2, 2, 4),
    ]
    for name, kind, dims, R, dens, kw, H, n_warm, n_stream in scases:
        if kind == "gaussian":
            X, _ = ogcp.gen_gaussian(ogcp.SyntheticSpec("gaussian", dims=dims, rank=R, noise=0.1, seed=42))
        else:
            X, _ = ogcp.gen_poisson(ogcp.SyntheticSpec("poisson", dims=dims, rank=R, density=dens, seed=42))
            if kind == "bernoulli":
                X = ogcp.SparseTensor.from_zero_based(X.dims, X.subs0, np.ones(X.nnz))
        loss = ogcp.make_loss(kind)
        cfg = solvers.SolverConfig(**kw)
        init = [rng.uniform(0.2, 1.0, (d, R)) for d in dims[:-1]]
        state = streaming.fresh_state(dims[:-1], R, loss, cfg, factors=init)
        state.window = streaming.HistoryWindow(capacity=H)
        # pretend-warm: fixed weights for the first n_warm steps
        for h in range(1, n_warm + 1):
            s_h = rng.uniform(0.5, 1.5, R)
            state.weights_log.append(s_h)
            state.window.observe(h, s_h, sampling.rng_at(cfg.samples.seed, h, sampling.PHASE_WINDOW))
        state.t = n_warm
        rec = dict(kind=np.array(kind), dims=np.array(dims), subs0=X.subs0, vals=X.vals, R=np.array(R),
                   H=np.array(H), n_warm=np.array(n_warm), n_stream=np.array(n_stream),
                   cfg=np.array(json.dumps({k: v for k, v in kw.items() if k != "samples"})),
                   samples=np.array(json.dumps(dict(p=kw["samples"].grad_nonzeros, q=kw["samples"].grad_zeros,
                                                    p_obj=kw["samples"].obj_nonzeros,
                                                    q_obj=kw["samples"].obj_zeros, seed=kw["samples"].seed))),
                   warm_weights=np.vstack(state.weights_log))
        for k, a in enumerate(init):
            rec[f"init{k}"] = a
        loc_s, loc_x, wtr, ftr = [], [], [], []
        for t in range(n_warm + 1, n_warm + n_stream + 1):
            m = streaming.process_slice(state, X.slice_view(t), loss, cfg, exact_loss=True)
            loc_s.append(m.local_loss_sampled)
            loc_x.append(m.local_loss_exact)
            wtr.append(state.trace_log[-1][1])
            ftr.append(state.trace_log[-1][2])
        for k, a in enumerate(state.factors):
            rec[f"final{k}"] = a
        rec.update(weights_log=np.vstack(state.weights_log), local_sampled=np.array(loc_s),
                   local_exact=np.array(loc_x), iteration=np.array(state.iteration),
                   window_ids=np.array(state.window.step_ids()),
                   wtrace=np.array(json.dumps(wtr)), ftrace=np.array(json.dumps(ftr)),
                   adam_rate=np.array(state.adam_factors.rate))
        for k, v in rec.items():
            streams[f"{name}_{k}"] = v
    streams["names"] = np.array(json.dumps([c[0] for c in scases]))
    np.savez_compressed(os.path.join(OUT, "streams.npz"), **streams)
    make_static()
    make_gaussian()
    print("golden fixtures written to", os.path.abspath(OUT))


def make_static():
    """solve_static / warm_start fixtures (solvers.py:371-493, streaming.py:113-151)."""
    sys.path.insert(0, REF)
    import ogcp
    from ogcp import sampling, solvers, streaming

    static = {}
    cases = [
        # name, kind, dims (last = time), R, density, cfg kwargs, restarts, capacity
        ("gauss", "gaussian", (6, 5, 4, 3), 3, None,
         dict(max_epochs_factors=3, iters_factors=20, rate_factors=1e-2, reg_factors=0.01, reg_weights=0.02,
              samples=sampling.SamplerConfig(200, 0, 300, 0, seed=3)), 1, 2),
        ("pois", "poisson", (8, 9, 5, 4), 3, 0.2,
         dict(max_epochs_factors=2, iters_factors=15, rate_factors=1e-2,
              samples=sampling.SamplerConfig(None, 60, None, 200, seed=7)), 2, 3),
        ("bern", "bernoulli", (7, 6, 8, 3), 2, 0.15,
         dict(max_epochs_factors=3, iters_factors=10, rate_factors=5e-2, rate_decay=0.5,
              samples=sampling.SamplerConfig(30, 40, 60, 80, seed=5)), 1, 2),
    ]
    for name, kind, dims, R, dens, kw, restarts, cap in cases:
        if kind == "gaussian":
            X, _ = ogcp.gen_gaussian(ogcp.SyntheticSpec("gaussian", dims=dims, rank=R, noise=0.1, seed=11))
        else:
            X, _ = ogcp.gen_poisson(ogcp.SyntheticSpec("poisson", dims=dims, rank=R, density=dens, seed=11))
            if kind == "bernoulli":
                X = ogcp.SparseTensor.from_zero_based(X.dims, X.subs0, np.ones(X.nnz))
        loss = ogcp.make_loss(kind)
        cfg = solvers.SolverConfig(**kw)
        res = solvers.solve_static(X, R, loss, cfg, seed_key=4)
        state = streaming.warm_start(X, R, loss, cfg, cap, restarts=restarts)
        rec = dict(kind=np.array(kind), dims=np.array(dims), subs0=X.subs0, vals=X.vals, R=np.array(R),
                   restarts=np.array(restarts), capacity=np.array(cap),
                   cfg=np.array(json.dumps({k: v for k, v in kw.items() if k != "samples"})),
                   samples=np.array(json.dumps(dict(p=kw["samples"].grad_nonzeros, q=kw["samples"].grad_zeros,
                                                    p_obj=kw["samples"].obj_nonzeros,
                                                    q_obj=kw["samples"].obj_zeros, seed=kw["samples"].seed))),
                   static_weights=res.model.weights, static_trace=np.array(res.trace.objective),
                   static_epochs=np.array(res.trace.epochs), static_rejections=np.array(res.trace.rejections),
                   warm_weights_log=np.vstack(state.weights_log), warm_window_ids=np.array(state.window.step_ids()),
                   warm_t=np.array(state.t))
        for k, a in enumerate(res.model.factors):
            rec[f"static_A{k}"] = a
        for k, a in enumerate(state.factors):
            rec[f"warm_A{k}"] = a
        for k, v in rec.items():
            static[f"{name}_{k}"] = v
    static["names"] = np.array(json.dumps([c[0] for c in cases]))
    np.savez_compressed(os.path.join(OUT, "static.npz"), **static)


def make_gaussian():
    """Gaussian special cases (kernels.py:117-146, solvers.py:145-185, 271-288) and
    congruence (metrics.py:95-148)."""
    sys.path.insert(0, REF)
    import ogcp
    from ogcp import kernels, metrics, sampling, solvers, streaming

    rng = np.random.default_rng(77)
    out = {}
    X, _ = ogcp.gen_gaussian(ogcp.SyntheticSpec("gaussian", dims=(7, 6, 5, 6), rank=3, noise=0.1, seed=13))
    out.update(subs0=X.subs0, vals=X.vals, dims=np.array(X.dims))
    R = 3
    init = [rng.uniform(0.2, 1.0, (d, R)) for d in X.dims[:-1]]
    for k, a in enumerate(init):
        out[f"init{k}"] = a
    warm = rng.uniform(0.5, 1.5, (2, R))
    out["warm_weights"] = warm
    # direct calls on slice 1
    X1 = X.slice_view(1)
    out["resid"] = np.array(kernels.gaussian_sum_sq_residual(X1, init, warm[0]))
    out["ls_mu0"] = solvers.solve_weights_least_squares(X1, init, 0.0)
    out["ls_mu"] = solvers.solve_weights_least_squares(X1, init, 0.3)
    out["dense_wgrad"] = solvers._dense_gaussian_weight_gradient(X1, init, warm[0], 0.2)
    for k, g in enumerate(solvers.dense_gaussian_factor_gradients(X1, init, warm[0], reg_factors=0.1)):
        out[f"dense_fgrad{k}"] = g
    cases = {
        "dense": dict(gradient_mode="dense-gaussian", max_epochs_weights=3, max_epochs_factors=2, iters_weights=20,
                      iters_factors=20, rate_weights=0.2, rate_factors=1e-2, hist_weight=1.0, hist_decay=0.9,
                      reg_factors=0.01, reg_weights=0.05, samples=sampling.SamplerConfig(100, 0, 200, 0, seed=4)),
        "ls": dict(temporal_solver="least-squares", max_epochs_factors=2, iters_factors=15, rate_factors=1e-2,
                   hist_weight=2.0, reg_weights=0.1, samples=sampling.SamplerConfig(150, 0, 200, 0, seed=4)),
    }
    loss = ogcp.make_loss("gaussian")
    for name, kw in cases.items():
        cfg = solvers.SolverConfig(**kw)
        state = streaming.fresh_state(X.dims[:-1], R, loss, cfg, factors=init)
        state.window = streaming.HistoryWindow(capacity=2)
        for h in (1, 2):
            state.weights_log.append(warm[h - 1])
            state.window.observe(h, warm[h - 1], sampling.rng_at(cfg.samples.seed, h, sampling.PHASE_WINDOW))
        state.t = 2
        loc = []
        for t in range(3, X.dims[-1] + 1):
            m = streaming.process_slice(state, X.slice_view(t), loss, cfg, exact_loss=True)
            loc.append(m.local_loss_exact)
        out[f"{name}_cfg"] = np.array(json.dumps({k: v for k, v in kw.items() if k != "samples"}))
        out[f"{name}_weights_log"] = np.vstack(state.weights_log)
        out[f"{name}_local_exact"] = np.array(loc)
        out[f"{name}_iteration"] = np.array(state.iteration)
        out[f"{name}_ftrace"] = np.array(json.dumps([tr[2] for tr in state.trace_log]))
        out[f"{name}_wtrace"] = np.array(json.dumps([tr[1] for tr in state.trace_log]))
        for k, a in enumerate(state.factors):
            out[f"{name}_final{k}"] = a
    # static, dense-gaussian, two restarts
    cfg = solvers.SolverConfig(gradient_mode="dense-gaussian", max_epochs_factors=3, iters_factors=10,
                               rate_factors=2e-2, reg_factors=0.01, reg_weights=0.02,
                               samples=sampling.SamplerConfig(100, 0, 200, 0, seed=4))
    st = solvers.solve_static(X, R, loss, cfg, restarts=2, seed_key=3)
    out["static_weights"] = st.model.weights
    for k, a in enumerate(st.model.factors):
        out[f"static_A{k}"] = a
    out["static_trace"] = np.array(st.trace.objective)
    # congruence pairs
    pairs = []
    for i in range(4):
        R1, R2 = (3, 3) if i < 2 else (3, 4 + i - 2)
        dims = (5, 4, 6)
        w1 = rng.uniform(0.5, 2.0, R1)
        f1 = [rng.standard_normal((d, R1)) for d in dims]
        if i == 1:
            w2 = w1[::-1] * 1.3
            f2 = [a[:, ::-1] * (-1.0 if k == 0 else 1.0) for k, a in enumerate(f1)]
            w2 = w2 * -1.0
        else:
            w2 = rng.uniform(-1.0, 2.0, R2)
            f2 = [rng.standard_normal((d, R2)) for d in dims]
            if i == 3:
                f2[1][:, 0] = 0.0
        sc = metrics.congruence_score(ogcp.KTensor(w1, f1), ogcp.KTensor(w2, f2))
        out[f"cong{i}_w1"], out[f"cong{i}_w2"] = w1, np.array(w2)
        for k in range(3):
            out[f"cong{i}_f1_{k}"], out[f"cong{i}_f2_{k}"] = f1[k], np.array(f2[k])
        pairs.append(sc)
    out["cong_scores"] = np.array(pairs)
    np.savez_compressed(os.path.join(OUT, "gaussian.npz"), **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["static"]:
        make_static()
    elif sys.argv[1:] == ["gaussian"]:
        make_gaussian()
    else:
        main()
