"""GPU: the density callers (FactorGaussian, reference density.hpp:24-260) on
the B200 operator, against a dense fp64 restatement of the same formulas
(the kernel matrix built explicitly as in oracle.hpp's dense reference)."""
import numpy as np
import pytest

import paper_2605_24584_b200 as L
from paper_2605_24584_b200.density import FactorGaussian

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    return torch


def _model(torch, phased, seed=0, n=3000, kl=40, C=2, t=0.7):
    rng = np.random.default_rng(seed)
    a, b = rng.uniform(-10, 10, n), rng.uniform(-10, 10, kl)
    phi, psi = (rng.uniform(0, 6.28, n), rng.uniform(0, 6.28, kl)) if phased else (None, None)
    mean = rng.uniform(-1, 1, n)
    d = rng.uniform(0.5, 1.5, n)
    W = [rng.uniform(-1, 1, n) for _ in range(C)]
    Ls = [np.tril(rng.uniform(-0.3, 0.3, (kl, kl))) + np.eye(kl) for _ in range(C)]
    T = lambda v: None if v is None else torch.tensor(v, dtype=torch.float64, device="cuda")  # noqa: E731
    op = L.DeviceOperator(T(a), T(b), t, T(phi), T(psi))
    fg = FactorGaussian(mean, d, W, op, Ls)
    A = np.exp(-np.abs(a[:, None] - b[None, :]) / t)
    if phased:
        A = A * np.cos(phi[:, None] - psi[None, :])
    F = sum(W[c][:, None] * (A @ Ls[c].T) for c in range(C))
    return fg, dict(A=A, F=F, mean=mean, d=d, W=W, Ls=Ls, n=n, kl=kl)


@pytest.mark.parametrize("phased", [False, True])
def test_factor_gaussian_against_dense(torch, phased):
    fg, D = _model(torch, phased)
    F, mean, d, n, kl = D["F"], D["mean"], D["d"], D["n"], D["kl"]
    rng = np.random.default_rng(5)
    Z = rng.normal(size=(3, kl))
    R = rng.normal(size=(3, n))
    got = fg.apply_F(torch.tensor(Z, device="cuda")).cpu().numpy()
    assert np.allclose(got, Z @ F.T, rtol=1e-11, atol=1e-11 * np.abs(Z @ F.T).max())
    got = fg.apply_Ft(torch.tensor(R, device="cuda")).cpu().numpy()
    assert np.allclose(got, R @ F, rtol=1e-11, atol=1e-11 * np.abs(R @ F).max())
    M = np.eye(kl) + F.T @ (F / (d * d)[:, None])
    assert np.allclose(fg.capacitance().cpu().numpy(), M, rtol=1e-10, atol=1e-10 * np.abs(M).max())
    x = mean + F @ rng.normal(size=kl) + d * rng.normal(size=n)
    Sigma = np.diag(d * d) + F @ F.T
    sign, logdet = np.linalg.slogdet(Sigma)
    r = x - mean
    want = -0.5 * (r @ np.linalg.solve(Sigma, r) + logdet + n * np.log(2 * np.pi))
    assert abs(fg.log_likelihood(x) - want) <= 1e-9 * abs(want)
    z, xh = fg.map_reconstruct(x)
    zw = np.linalg.solve(M, F.T @ (r / (d * d)))
    assert np.allclose(z.cpu().numpy(), zw, rtol=1e-9, atol=1e-9 * np.abs(zw).max())
    assert np.allclose(xh.cpu().numpy(), mean + F @ zw, rtol=1e-9, atol=1e-9)
    B, Fb = fg.build_blocks()
    assert np.allclose(Fb.cpu().numpy(), F, rtol=1e-11, atol=1e-11 * np.abs(F).max())
    for c in range(len(B)):
        want_b = D["A"] @ D["Ls"][c].T
        assert np.allclose(B[c].cpu().numpy(), want_b, rtol=1e-11, atol=1e-11 * np.abs(want_b).max())
    S = fg.sample(4000, 3).cpu().numpy()
    assert S.shape == (4000, n)
    # first two moments of the draws (statistical, generous bounds)
    emp = (S - mean).mean(0)
    assert np.abs(emp).mean() < 0.1
    var = ((S - mean) ** 2).mean(0)
    assert np.allclose(var.mean(), np.diag(Sigma).mean(), rtol=0.05)


def test_factor_gaussian_validation_order(torch):
    fg, D = _model(torch, False, n=500, kl=8, C=1)
    op = fg.op
    with pytest.raises(L.EmptyInput):
        FactorGaussian([], [], [[]], op, [np.eye(8)])
    with pytest.raises(L.DimensionMismatch):
        FactorGaussian(np.zeros(499), np.ones(499), [np.ones(499)], op, [np.eye(8)])
    with pytest.raises(L.DimensionMismatch):
        FactorGaussian(np.zeros(500), np.ones(500), [np.ones(500)], op, [])
    with pytest.raises(L.NonFinite):
        FactorGaussian(np.zeros(500), -np.ones(500), [np.ones(500)], op, [np.eye(8)])
    with pytest.raises(L.DimensionMismatch):
        FactorGaussian(np.zeros(500), np.ones(500), [np.ones(500)], op, [np.eye(7)])
    with pytest.raises(L.DimensionMismatch):
        fg.apply_F(torch.zeros(7, device="cuda", dtype=torch.float64))
    with pytest.raises(L.EmptyInput):
        fg.sample(0, 1)
