"""Pins of the oracle's stage 1: SLM (Eq 1-2) and the per-view
likelihoods P(S|V) (Eq 5-9).

Each test compares the oracle with something other than itself: a worked
example printed by the specification, a textbook/library routine
(scipy.stats.norm.logpdf), a special case, or an invariant."""
import math

import numpy as np
import pytest
from scipy.special import expit
from scipy.stats import norm

import oracle

LN_U = -3.0 * math.log(256.0)  # uniform foreground density (1/256)^3


def _px(I, mu, sigma, floor=1.0, p_occ=0.5):
    I = np.asarray(I, np.uint8).reshape(-1, 3)
    mu = np.asarray(mu, np.float32).reshape(-1, 3)
    sigma = np.asarray(sigma, np.float32).reshape(-1, 3)
    return oracle.slm_image(I, mu, sigma, floor, p_occ)


def test_spec_worked_example_sigma5(golden):
    """sigma=5, I=mu -> SLM ~= 1.17e-4."""
    g = golden("slm_worked_examples.json")["sigma5_at_mean"]
    slm, _, _ = _px([100, 100, 100], [100, 100, 100], [5, 5, 5])
    assert slm[0] == pytest.approx(g["slm"], rel=g["rel_tol"])
    # and the two densities it is built from: SLM = u/(u+g)
    assert slm[0] == pytest.approx(g["u"] / (g["u"] + g["g"]), rel=g["rel_tol"])


def test_appendix_constants_at_mean(golden):
    """d and t(p_O=1/2) at I = mu for several sigma."""
    gd = golden("slm_worked_examples.json")
    tol = gd["abs_tol_appendix"]
    for s, d_ref in gd["d_at_mean"].items():
        s = float(s)
        slm, l1, l0 = _px([128] * 3, [128] * 3, [s] * 3)
        d = math.log(1.0 / slm[0] - 1.0)  # SLM = 1/(1+e^d)
        assert d == pytest.approx(d_ref, abs=tol)
        assert l1[0] - l0[0] == pytest.approx(gd["t_half_at_mean"][str(int(s))], abs=tol)


def test_library_routine_scipy_logpdf():
    """SLM = expit(-(sum_ch norm.logpdf(I; mu, sigma) - ln u)) on random inputs."""
    rng = np.random.default_rng(7)
    n = 20000
    I = rng.integers(0, 256, size=(n, 3)).astype(np.uint8)
    mu = rng.uniform(0, 255, size=(n, 3)).astype(np.float32)
    # bias some pixels to sit near their mean so SLM spans (0, 1)
    near = rng.random(n) < 0.5
    mu[near] = np.clip(I[near] + rng.normal(0, 6, size=(near.sum(), 3)), 0, 255).astype(np.float32)
    sigma = rng.uniform(1.0, 40.0, size=(n, 3)).astype(np.float32)
    slm, l1, l0 = _px(I, mu, sigma)
    d = norm.logpdf(I.astype(np.float64), mu.astype(np.float64), sigma.astype(np.float64)).sum(1) - LN_U
    ref = expit(-d)
    np.testing.assert_allclose(slm, ref, rtol=1e-11, atol=1e-300)
    # p_O = 1/2: t = ln(2 SLM) (the Eq 5-9 collapse, P(S|V=0) = 1/2)
    np.testing.assert_allclose(l1 - l0, np.log(2.0 * ref), rtol=1e-10, atol=1e-12)
    assert (slm >= 0).all() and (slm <= 1).all()


def test_p_occ_limits_match_likelihood_ratio():
    """p_O -> 0: t = ln SLM - ln(1-SLM) = -d (pure Gaussian-vs-uniform ratio);
    p_O -> 1: t -> 0 (every branch is SLM, the view says nothing)."""
    rng = np.random.default_rng(3)
    n = 2000
    I = rng.integers(0, 256, size=(n, 3)).astype(np.uint8)
    mu = np.clip(I + rng.normal(0, 8, size=(n, 3)), 0, 255).astype(np.float32)
    sigma = rng.uniform(2, 8, size=(n, 3)).astype(np.float32)
    d = norm.logpdf(I.astype(float), mu.astype(float), sigma.astype(float)).sum(1) - LN_U
    _, l1, l0 = _px(I, mu, sigma, p_occ=1e-15)
    ok = d > -10.0  # where (1-SLM) ~ e^d dominates p_O = 1e-15 in Eq 6-7
    assert ok.sum() > 500
    np.testing.assert_allclose((l1 - l0)[ok], -d[ok], rtol=1e-9, atol=1e-9)
    # p_O = 1 - e: |t| ~ e (1 - SLM) / SLM, and SLM >= ~1e-5 here (sigma >= 2)
    _, l1, l0 = _px(I, mu, sigma, p_occ=1.0 - 1e-14)
    assert np.abs(l1 - l0).max() < 1e-8


def test_ten_sigma_deviation_is_foreground():
    """I deviates >= 10 sigma on every channel -> SLM >= 1 - 1e-6."""
    slm, _, _ = _px([200, 10, 180], [140, 70, 120], [6, 6, 6])
    assert slm[0] >= 1 - 1e-6
    slm, _, _ = _px([255, 0, 255], [0, 255, 0], [1, 1, 1])
    assert slm[0] == 1.0


def test_g_equals_u_gives_half(golden):
    """g = u -> SLM = 1/2.  With sigma = 1 on all channels,
    |I - mu| = 3.0417886 makes sum ln N = ln u (d = 0)."""
    dev = golden("slm_worked_examples.json")["d_zero_deviation_sigma1"]
    slm, l1, l0 = _px([100] * 3, [100 - dev] * 3, [1, 1, 1])
    # mu is float32: |dmu| <= ulp(97)/2 = 3.8e-6 -> |d| <= 3*3.04*3.8e-6 = 3.5e-5
    assert slm[0] == pytest.approx(0.5, abs=1e-5)
    assert l1[0] - l0[0] == pytest.approx(0.0, abs=2e-5)
    # exact double version of the same case (sigma = 1 so float rounding only in mu)
    _, l1x, l0x = _px([100] * 3, [100 - 3.0] * 3, [1, 1, 1])
    assert l1x[0] - l0x[0] < 0 < l1[0] - l0[0] + 2e-5  # still below at |I-mu| = 3


def test_monotone_in_deviation():
    """increasing |I - mu| on one channel never decreases SLM."""
    mu = np.float32(120.25)
    I = np.arange(121, 256).astype(np.uint8)
    n = I.shape[0]
    img = np.stack([I, np.full(n, 90, np.uint8), np.full(n, 90, np.uint8)], 1)
    m = np.stack([np.full(n, mu), np.full(n, 91.5), np.full(n, 88.0)], 1).astype(np.float32)
    slm, _, _ = _px(img, m, np.full((n, 3), 3.5, np.float32))
    assert (np.diff(slm) >= 0).all()
    assert slm[0] < 0.01 and slm[-1] == pytest.approx(1.0)


def test_sigma_floor():
    """R#6: sigma' = max(sigma, sigma_floor) per channel."""
    a = _px([10, 20, 30], [11, 19.5, 30], [0.2, 0.7, 1.0])
    b = _px([10, 20, 30], [11, 19.5, 30], [1.0, 1.0, 1.0])
    for x, y in zip(a, b):
        assert x[0] == y[0]
    c = _px([10, 20, 30], [11, 19.5, 30], [0.2, 0.7, 1.0], floor=2.0)
    d = _px([10, 20, 30], [11, 19.5, 30], [2.0, 2.0, 2.0])
    assert c[0][0] == d[0][0]


def test_view_likelihood_spec_examples():
    """(0.8, occupied) -> 0.8; (0.8, empty, p_O=1/2) -> 0.5;
    (s, empty, p_O=1/2) -> 0.5 for every s."""
    l1, l0 = oracle.view_likelihood(0.8, 0.5)
    assert math.exp(l1) == pytest.approx(0.8, abs=1e-15)
    assert math.exp(l0) == pytest.approx(0.5, abs=1e-15)
    for s in np.linspace(0.0, 1.0, 11):
        _, l0 = oracle.view_likelihood(s, 0.5)
        assert math.exp(l0) == pytest.approx(0.5, abs=1e-15)
    # Eq 6-7 at general p_O: P(S|V=0) = (1-p_O)(1-s) + p_O s
    l1, l0 = oracle.view_likelihood(0.8, 0.3)
    assert math.exp(l0) == pytest.approx(0.7 * 0.2 + 0.3 * 0.8, abs=1e-15)
    assert math.exp(l1) == pytest.approx(0.8, abs=1e-15)


def test_term_bounds():
    """t in [-ln(p_O + (1-p_O) e^{d_max}), -ln p_O] with d_max = 3 ln(256) -
    1.5 ln(2 pi) - 3 ln(sigma_floor) (all-channel exact match at the floor)."""
    rng = np.random.default_rng(11)
    n = 50000
    I = rng.integers(0, 256, size=(n, 3)).astype(np.uint8)
    mu = np.clip(I + rng.normal(0, 3, size=(n, 3)), 0, 255).astype(np.float32)
    sigma = rng.uniform(0.5, 10, size=(n, 3)).astype(np.float32)
    for p in (0.5, 0.3, 0.8):
        _, l1, l0 = _px(I, mu, sigma, p_occ=p)
        t = l1 - l0
        dmax = -LN_U - 1.5 * math.log(2 * math.pi)
        lo = -math.log(p + (1 - p) * math.exp(dmax))
        assert t.max() <= -math.log(p) + 1e-12
        assert t.min() >= lo - 1e-12
