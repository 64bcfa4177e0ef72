"""The Eigen-free decoder solve (csrc/host/decoders.cpp, C ABI
neng_solve_decoders) — SURVEY §8(f)3.  The reference's solve_decoders
(frontend.cpp:56-76) needs Eigen, which is absent, so it cannot be built
here: parity is anchored on the reference's own known-answer tests for it
(test_frontend.cpp:114-172, replayed below) and on an independent numpy
solve of the same normal equations."""
import math

import numpy as np
import pytest

from paper_1805_11144_b200 import networks, passes
from paper_1805_11144_b200.ir import BuildError
from paper_1805_11144_b200.rng import Rng


def test_identity_system_returns_identity():  # test_frontend.cpp:114-121
    a = np.eye(3)
    d = passes.solve_decoders(a, a, 0.0)
    assert np.allclose(d, np.eye(3), rtol=0, atol=1e-14)


def test_zero_targets_give_exactly_zero():  # test_frontend.cpp:123-130
    rng = Rng(5)
    a = np.array([rng.uniform(0.0, 100.0) for _ in range(40 * 6)]).reshape(40, 6)
    d = passes.solve_decoders(a, np.zeros((40, 2)))
    assert np.all(d == 0.0)


def test_unregularized_singular_system_rejected():  # test_frontend.cpp:132-137
    a = np.array([[1.0, 0.0], [2.0, 0.0]])  # second activity identically zero
    y = np.array([1.0, 2.0])
    with pytest.raises(BuildError, match="singular"):
        passes.solve_decoders(a, y, 0.0)
    passes.solve_decoders(a, y, 0.1)


def test_stronger_regularization_shrinks_decoders():  # test_frontend.cpp:139-153
    rng = Rng(11)
    m, n = 50, 8
    a = np.array([rng.uniform(0.0, 200.0) for _ in range(m * n)]).reshape(m, n)
    y = np.array([rng.uniform(-1.0, 1.0) for _ in range(m)])
    norms = [np.linalg.norm(passes.solve_decoders(a, y, reg)) for reg in (0.01, 0.1, 1.0)]
    assert norms[1] <= norms[0] and norms[2] <= norms[1]


def _lif_rate(j, tau_rc=0.02, tau_ref=0.002):
    out = np.zeros_like(j)
    on = j > 1.0
    out[on] = 1.0 / (tau_ref + tau_rc * np.log1p(1.0 / (j[on] - 1.0)))
    return out


def test_hundred_lif_neurons_decode_identity():  # test_frontend.cpp:155-172
    # sample_ensemble_parameters(100, 1, {}, 99) (frontend.cpp:78-118): unit encoders from
    # Rng(99) normals, then U(200, 400) max rates, then U(-1, 1) intercepts
    n, m = 100, 201
    rng = Rng(99)
    enc = np.array([math.copysign(1.0, rng.gaussian()) for _ in range(n)])
    max_rates = np.array([rng.uniform(200.0, 400.0) for _ in range(n)])
    intercepts = np.array([rng.uniform(-1.0, 1.0) for _ in range(n)])
    gain, bias = networks.gain_bias_lif(max_rates, intercepts)
    x = -1.0 + 2.0 * np.arange(m) / (m - 1)
    acts = _lif_rate(gain[None, :] * enc[None, :] * x[:, None] + bias[None, :])
    d = passes.solve_decoders(acts, x)
    rmse = math.sqrt(np.mean((acts @ d[:, 0] - x) ** 2))
    assert rmse < 0.05, rmse


@pytest.mark.parametrize("m,n,d,reg", [(30, 7, 1, 0.1), (200, 50, 3, 0.01), (64, 64, 2, 0.5)])
def test_matches_an_independent_normal_equation_solve(m, n, d, reg):
    rng = np.random.default_rng(m * n)
    a = rng.uniform(0.0, 300.0, size=(m, n))
    y = rng.normal(size=(m, d))
    sigma = reg * np.abs(a).max()
    want = np.linalg.solve(a.T @ a + m * sigma * sigma * np.eye(n), a.T @ y)
    got = passes.solve_decoders(a, y, reg)
    assert np.allclose(got, want, rtol=1e-9, atol=1e-12 * np.abs(want).max())


def test_bad_systems_rejected():
    with pytest.raises(BuildError, match="non-negative"):
        passes.solve_decoders(np.ones((3, 2)), np.ones(3), -1.0)
    with pytest.raises(ValueError):
        passes.solve_decoders(np.ones((3, 2)), np.ones(4))


def test_least_squares_product_decoders_decode_the_product():
    # config 1's product ensembles (decoders="ls"): 2-D ensembles of 100 LIF decoding x0 * x1
    nb = networks.NetBuilder(7)
    e = nb.ensemble(100, 2)
    D = nb.solve_decoders(e, lambda p: p[:, :1] * p[:, 1:2], 1, eval_points_per_dim=100, radius=1.5)
    assert D.shape == (1, 100)
    E = np.asarray(nb.m.signals[e.enc].initial).reshape(100, 2)
    bias = next(np.asarray(op.value) for op in nb.m.operators if op.operands[0].signal == e.j and op.value is not None)
    pts = np.random.default_rng(3).uniform(-1.0, 1.0, size=(400, 2))
    est = _lif_rate(pts @ E.T + bias[None, :]) @ D[0]
    err = np.sqrt(np.mean((est - pts[:, 0] * pts[:, 1]) ** 2))
    rand = _lif_rate(pts @ E.T + bias[None, :]) @ np.random.default_rng(1).normal(0.0, 0.1, 100)
    err_rand = np.sqrt(np.mean((rand - pts[:, 0] * pts[:, 1]) ** 2))
    assert err < 0.2 and err < 0.1 * err_rand, (err, err_rand)
