"""An independent NumPy float64 re-derivation of the oracle's O1-O8 on C1
(SURVEY.md 8(c) "Independent re-derivation": agreement to 1e-9 in L and exact
bits).  Written from the paper, not from oracle/psfs_oracle.c:

* O1-O3 (Eq 1-2; Eq 5-9): d = ln N(I | mu, sigma') - ln U
  with U = 256^-3 and sigma' = max(sigma, floor), vectorised over pixels;
  t = ln P(S|V=1) - ln P(S|V=0) = -logaddexp(ln p_O, ln(1 - p_O) + d);
* O4-O5: the voxel centre origin + spacing (idx + 1/2) projected in float64
  straight from P (no pre-composed float matrix), nearest pixel floor(x/w + 1/2),
  in view iff w > 0 and inside the image (R#10-R#13);
* O6-O8 (Eq 3-4): L = logit p_V + sum of in-view t, bit =
  posterior > tau, x-fastest words LSB first (R#19).

The oracle's projection is the pinned FP32 chain, so voxel-cameras whose exact
position lies within 1e-3 px of a pixel edge (where FP32 rounding may pick the
neighbour) are excluded -- the only place the two definitions may differ."""
import math

import numpy as np
import pytest

import oracle
from synth.scene import make_frames, make_scene


def _terms(frame, mu, sigma, floor, p_occ):
    I = frame.astype(np.float64)
    s = np.maximum(sigma.astype(np.float64), floor)
    m = mu.astype(np.float64)
    ln_g = np.sum(-0.5 * ((I - m) / s) ** 2 - np.log(s) - 0.5 * math.log(2 * math.pi), axis=-1)
    d = ln_g + 3 * math.log(256.0)
    return -np.logaddexp(math.log(p_occ), math.log1p(-p_occ) + d)


def _numpy_reconstruct(scene, frames, floor=1.0, p_occ=0.5, p_vox=0.5, tau=0.5, margin=1e-3):
    g = scene.grid
    k, j, i = np.meshgrid(np.arange(g.zlen), np.arange(g.ylen), np.arange(g.xlen), indexing="ij")
    X = g.origin[0] + g.spacing * (i.ravel() + 0.5)
    Y = g.origin[1] + g.spacing * (j.ravel() + 0.5)
    Z = g.origin[2] + g.spacing * (k.ravel() + 0.5)
    L = np.full(g.nvox, math.log(p_vox) - math.log1p(-p_vox))
    ambiguous = np.zeros(g.nvox, bool)
    for c, cam in enumerate(scene.cameras):
        t = _terms(frames[c], scene.mu[c], scene.sigma[c], floor, p_occ)
        P = scene.P[c]
        x = P[0, 0] * X + P[0, 1] * Y + P[0, 2] * Z + P[0, 3]
        y = P[1, 0] * X + P[1, 1] * Y + P[1, 2] * Z + P[1, 3]
        w = P[2, 0] * X + P[2, 1] * Y + P[2, 2] * Z + P[2, 3]
        with np.errstate(divide="ignore", invalid="ignore"):
            u = x / w + 0.5
            v = y / w + 0.5
        inview = (w > 0) & (u >= 0) & (u < cam.width) & (v >= 0) & (v < cam.height)
        near_edge = (np.abs(u - np.round(u)) < margin) | (np.abs(v - np.round(v)) < margin)
        ambiguous |= near_edge & (w > 0)
        px = np.where(inview, np.floor(u), 0).astype(np.int64)
        py = np.where(inview, np.floor(v), 0).astype(np.int64)
        L += np.where(inview, t[py, px], 0.0)
    post = 1.0 / (1.0 + np.exp(-L))
    occ = post > tau
    bits = np.packbits(occ, bitorder="little").view(np.uint8)
    words = np.zeros((g.nvox + 31) // 32, np.uint32)
    words.view(np.uint8)[: bits.size] = bits
    return L, post, words, ambiguous


@pytest.mark.parametrize("params", [dict(), dict(p_occ=0.3, p_vox=0.2, tau=0.7, floor=1.5)])
@pytest.mark.parametrize("body", ["skeleton", "ellipsoid"])
def test_numpy_rederivation_matches_oracle_on_c1(params, body):
    s = make_scene("C1", body=body)
    fr = make_frames(s, 0)
    L, post, words, amb = _numpy_reconstruct(s, fr, **params)
    orc = oracle.scene_reconstruct(s, fr, sigma_floor=params.get("floor", 1.0),
                                   p_occ=params.get("p_occ", 0.5), p_vox=params.get("p_vox", 0.5),
                                   tau=params.get("tau", 0.5))
    keep = ~amb
    assert keep.mean() > 0.95  # the exclusion is a thin set
    assert np.abs(L[keep] - orc["L"][keep]).max() <= 1e-9
    bn = np.unpackbits(words.view(np.uint8), bitorder="little")[: s.grid.nvox].astype(bool)
    bo = np.unpackbits(orc["bits"].view(np.uint8), bitorder="little")[: s.grid.nvox].astype(bool)
    assert np.array_equal(bn[keep], bo[keep])
    assert bo.sum() > 0
