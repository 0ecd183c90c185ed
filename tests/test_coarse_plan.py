"""Host-side coarse-code plan (psfs_coarse_plan), no GPU.

The plan must give codes c + bias in [0, 255] for every term t the method can
produce, t in [-ln p_O - softplus(dm_max), -ln p_O] (Eq 5-9 with d <= d_max at
I = mu, sigma' = sigma_floor), widened by the FP32 error bound,
with the smallest such quantum 2^sh; and the bracket width wc = 2^sh - 1 +
ceil(2 eps 2^20)."""
import math

import pytest

from paper_1311_6811_b200 import psfs


def _t_range(po, sigma_floor):
    dmax = 24 * math.log(2) - 1.5 * math.log(2 * math.pi) - 3 * math.log(sigma_floor)
    x = dmax + math.log((1 - po) / po)
    # -ln p_O - ln(1 + e^x): the most negative term (I = mu at the floor)
    return -math.log(po) - (x + math.log1p(math.exp(-x)) if x > 0 else math.log1p(math.exp(x))), -math.log(po)


@pytest.mark.parametrize("po,sf", [(0.5, 1.0), (0.3, 1.0), (0.9, 2.0), (0.01, 0.5), (0.999, 0.25),
                                   (0.001, 1.0)])
def test_plan_codes_cover_every_term(po, sf):
    p = psfs.coarse_plan(dict(occlusion_prior=po, sigma_floor=sf), 8)
    assert p["ok"]
    lo, hi = _t_range(po, sf)
    s = 2.0 ** (20 - p["sh"])
    eps = p["eps"]
    assert eps >= 2.0 ** -10
    # code of the smallest and largest possible FP32 t (within eps of the exact one)
    c_lo = math.floor((lo - 2 * eps) * s) + p["bias"]
    c_hi = math.floor(hi * s) + p["bias"]
    assert 0 <= c_lo and c_hi <= 255
    # t = 0 (out of view) codes to the bias exactly when t - eps < 0 <= t ... the pad
    # stores the bias itself, i.e. c = 0, whose bracket [0, wc] contains q = 0
    assert p["wc"] == 2 ** p["sh"] - 1 + math.ceil(2 * eps * 2 ** 20)
    # minimal quantum: one step finer would not fit a byte
    s2 = 2.0 * s
    assert math.floor(hi * s2) - math.floor((lo - 2 * eps) * s2) + 2 > 255 or p["sh"] == 8


def test_plan_default_is_sixteen():
    """p_O = 1/2, sigma_floor = 1: t in [-13.1856, ln 2] -> 1/16 quantum (sh = 16)."""
    p = psfs.coarse_plan(None, 8)
    assert p["ok"] and p["sh"] == 16
    lo, hi = _t_range(0.5, 1.0)
    assert abs(lo + 13.185570) < 1e-5 and abs(hi - math.log(2)) < 1e-12


@pytest.mark.parametrize("params", [dict(sigma_floor=0.1), dict(occlusion_prior=1e-4),
                                    dict(occlusion_prior=1 - 1e-4)])
def test_plan_rejects_unbounded_params(params):
    """Outside the admitted range the FP32 error bound is not claimed: exact path."""
    assert not psfs.coarse_plan(params, 8)["ok"]


@pytest.mark.parametrize("params", [dict(), dict(occlusion_prior=0.3, voxel_prior=0.2, threshold=0.7),
                                    dict(occlusion_prior=0.05, threshold=0.3), dict(sigma_floor=0.5),
                                    dict(voxel_prior=0.9, threshold=0.2)])
@pytest.mark.parametrize("ncam", [1, 4, 8, 16, 32])
def test_thresholds_decide_exactly_where_the_bracket_allows(params, ncam):
    """Brute force over every code sum U = sum(c + bias) of ncam cameras: the exact
    S lies in [2^sh sum c, 2^sh sum c + ncam wc] (each camera's bracket; an
    out-of-view camera's exact 0 is in its c = 0 bracket).  U >= K1 must imply S >
    T_q for every S in that range, U < K0 must imply S <= T_q, and every U in
    [K0, K1) must leave both outcomes possible (nothing decided that needs no fix-up
    is sent to it, nothing undecided is decided)."""
    p = psfs.coarse_plan(params, ncam)
    assert p["ok"]
    q, wc, bias, Tq, K0, K1 = 1 << p["sh"], p["wc"], p["bias"], p["Tq"], p["K0"], p["K1"]
    # T_q from the definition: floor((logit tau - logit p_V) 2^20)
    tau, pv = params.get("threshold", 0.5), params.get("voxel_prior", 0.5)
    assert Tq == math.floor((math.log(tau / (1 - tau)) - math.log(pv / (1 - pv))) * 2 ** 20)
    assert 0 <= K0 <= K1 <= 32767
    for U in range(0, 255 * ncam + 1):
        sc = U - ncam * bias
        lo, hi = q * sc, q * sc + ncam * wc
        if U >= K1:
            assert lo > Tq, (U, lo, Tq)
        elif U < K0:
            assert hi <= Tq, (U, hi, Tq)
        else:
            assert lo <= Tq < hi, (U, lo, hi, Tq)
