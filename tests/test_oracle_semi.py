"""Pins the semi-stratified restatement (an extension; no reference golden vectors exist)
by Monte-Carlo unbiasedness against exact dense sums, the pattern of the reference's
test_acceptance.py:104-144 and test_sampling.py:133-150."""

import numpy as np

from oracle import ogcp_oracle as O


def _dense_setup(seed=6):
    rng = np.random.default_rng(seed)
    dims = (4, 5, 3)
    lin = rng.choice(int(np.prod(dims)), size=14, replace=False)
    subs0 = np.array(np.unravel_index(lin, dims)).T
    vals = rng.integers(1, 4, size=lin.size).astype(float)
    X = O.Slice(dims, subs0, vals)
    R = 2
    A = [rng.uniform(0.2, 1.0, (d, R)) for d in dims]
    w = rng.uniform(0.3, 1.0, R)
    dense_x = np.zeros(dims)
    dense_x[tuple(subs0.T)] = vals
    dense_m = np.einsum("ir,jr,kr,r->ijk", *A, w)
    return X, A, w, dense_x, dense_m


def test_semi_objective_unbiased():
    X, A, w, dx, dm = _dense_setup()
    exact = float(np.sum(O.loss_f("poisson", dx.ravel(), dm.ravel())))
    reps = 3000
    vals = np.array([O.semi_objective_data(X, A, w, "poisson", O.draw_semi(X, 5, 9, O.keyed_rng(11, r)))
                     for r in range(reps)])
    se = vals.std(ddof=1) / np.sqrt(reps)
    assert abs(vals.mean() - exact) < 4 * se


def test_semi_gradient_tensor_unbiased():
    X, A, w, dx, dm = _dense_setup(7)
    exact = O.loss_df("gaussian", dx, dm)
    reps = 3000
    acc = np.zeros(X.dims)
    sq = np.zeros(X.dims)
    for r in range(reps):
        subs, y = O.semi_y(X, A, w, "gaussian", O.draw_semi(X, 6, 10, O.keyed_rng(5, r)))
        d = np.zeros(X.dims)
        np.add.at(d, tuple(subs.T), y)
        acc += d
        sq += d * d
    mean = acc / reps
    se = np.sqrt(np.maximum(sq / reps - mean ** 2, 0) / reps)
    assert (np.abs(mean - exact) <= 4 * se + 1e-12).all()


def test_semi_draw_stream_layout():
    X, *_ = _dense_setup()
    s = O.draw_semi(X, 7, 5, O.keyed_rng(3, 1, 2))
    g = O.keyed_rng(3, 1, 2)
    np.testing.assert_array_equal(s.ordinals, g.integers(0, X.eta, size=7))
    np.testing.assert_array_equal(s.zero_subs0, g.integers(0, np.asarray(X.dims), size=(5, 3)))
