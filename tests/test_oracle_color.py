"""Pins of the oracle's voxel colour (NEXT-4; P:222, P:229, P:273-275;
S:223-231), against what the paper / SPEC and closed forms fix:

* S:228  every qualifying view samples (100, 50, 25) -> (100, 50, 25);
* S:229  a voxel behind every camera -> colour unset;
* S:230  two qualifying views (100,0,0) and (200,0,0) -> (150,0,0);
* the SLM gate at the closed-form SLM of an exact-background pixel
  with sigma = 5: SLM = 1/(1 + (5 sqrt(2 pi))^-3 / 256^-3) = 1.17330e-4;
* which cameras take part = the in-view set of the exact double projection
  (an independent implementation), away from image borders.
"""
import math

import numpy as np
import pytest

import oracle
from synth.scene import Grid, look_at_camera, make_scene

SLM_SIGMA5 = 1.0 / (1.0 + (1.0 / (5.0 * math.sqrt(2.0 * math.pi))) ** 3 * 256.0 ** 3)


def _rig(cams, grid):
    P = np.stack([c.P for c in cams]).astype(np.float64)
    W = np.array([c.width for c in cams], np.int32)
    H = np.array([c.height for c in cams], np.int32)
    return P, W, H


def _const_images(W, H, colours, mu_value=200.0, sigma_value=2.0):
    frames = [np.broadcast_to(np.asarray(col, np.uint8), (h, w, 3)).copy()
              for w, h, col in zip(W, H, colours)]
    mu = [np.full((h, w, 3), mu_value, np.float32) for w, h in zip(W, H)]
    sg = [np.full((h, w, 3), sigma_value, np.float32) for w, h in zip(W, H)]
    return frames, mu, sg


def _exact_inview(P, W, H, grid, vox):
    """In-view flags from the exact double projection (oracle_project_exact), and
    whether the exact sub-pixel position is at least 1e-3 px from every border."""
    out, safe = [], []
    for v in vox:
        i, j, k = v % grid.xlen, (v // grid.xlen) % grid.ylen, v // (grid.xlen * grid.ylen)
        row, srow = [], []
        for c in range(len(W)):
            X = np.asarray(grid.origin) + grid.spacing * (np.array([i, j, k]) + 0.5)
            x, y, w = P[c] @ np.append(X, 1.0)
            r, _, _ = oracle.project_exact(P[c], grid.origin, grid.spacing, W[c], H[c], i, j, k)
            row.append(bool(r))
            if w > 0:
                u, vv = x / w + 0.5, y / w + 0.5
                d = min(abs(u), abs(u - W[c]), abs(vv), abs(vv - H[c]))
                srow.append(d > 1e-3)
            else:
                srow.append(True)
        out.append(row)
        safe.append(all(srow))
    return np.array(out), np.array(safe)


def test_every_view_same_colour():
    s = make_scene("C1")
    P, W, H = s.P, s.widths, s.heights
    frames, mu, sg = _const_images(W, H, [(100, 50, 25)] * len(W))
    rng = np.random.default_rng(3)
    vox = rng.integers(0, s.grid.nvox, 400)
    rgb, cnt, _ = oracle.color(P, W, H, s.grid, frames, mu, sg, vox)
    seen = cnt > 0
    assert seen.sum() > 300
    assert np.array_equal(rgb[seen], np.tile([100.0, 50.0, 25.0], (seen.sum(), 1)))
    assert (rgb[~seen] == 0).all()
    inview, safe = _exact_inview(P, W, H, s.grid, vox)
    assert np.array_equal(cnt[safe], inview[safe].sum(axis=1))


def test_voxel_behind_every_camera_is_unset():
    g = Grid((-100.0, -100.0, 900.0), 50.0, 4, 4, 4)
    cam = look_at_camera((0.0, -4000.0, 1000.0), (0.0, -8000.0, 1000.0), 64, 48)  # looks away
    P, W, H = _rig([cam], g)
    frames, mu, sg = _const_images(W, H, [(100, 50, 25)])
    rgb, cnt, margin = oracle.color(P, W, H, g, frames, mu, sg, np.arange(g.nvox))
    assert (cnt == 0).all() and (rgb == 0).all() and np.isinf(margin).all()


def test_two_views_average():
    s = make_scene("C1")
    cams = [s.cameras[0], s.cameras[2]]  # opposite cameras of the ring
    P, W, H = _rig(cams, s.grid)
    frames, mu, sg = _const_images(W, H, [(100, 0, 0), (200, 0, 0)])
    g = s.grid
    centre = (g.xlen // 2) + g.xlen * ((g.ylen // 2) + g.ylen * (g.zlen // 2))
    rgb, cnt, _ = oracle.color(P, W, H, g, frames, mu, sg, [centre])
    assert cnt[0] == 2
    assert np.array_equal(rgb[0], [150.0, 0.0, 0.0])


def test_camera_dependent_colours_mean_over_inview_set():
    s = make_scene("C1")
    P, W, H = s.P, s.widths, s.heights
    cols = [(10, 20, 30), (40, 80, 120), (200, 100, 0), (7, 7, 7)]
    frames, mu, sg = _const_images(W, H, cols)
    rng = np.random.default_rng(5)
    vox = rng.integers(0, s.grid.nvox, 300)
    rgb, cnt, _ = oracle.color(P, W, H, s.grid, frames, mu, sg, vox)
    inview, safe = _exact_inview(P, W, H, s.grid, vox)
    C = np.asarray(cols, np.float64)
    for n in np.nonzero(safe & (inview.sum(axis=1) > 0))[0]:
        want = C[inview[n]].mean(axis=0)
        assert np.allclose(rgb[n], want, rtol=0, atol=1e-12)


@pytest.mark.parametrize("gate,qualifies", [(1.17e-4, True), (1.18e-4, False), (0.5, False)])
def test_slm_gate_at_closed_form_slm(gate, qualifies):
    """Exact background (I = mu, integer) with sigma = 5 gives SLM = 1.17330e-4
    at every pixel: the gate lets every in-view camera through below
    that value and none above it."""
    assert abs(SLM_SIGMA5 - 1.17330e-4) < 1e-9
    s = make_scene("C1")
    P, W, H = s.P, s.widths, s.heights
    frames, mu, sg = _const_images(W, H, [(90, 120, 150)] * len(W), sigma_value=5.0)
    mu = [np.broadcast_to(np.asarray((90, 120, 150), np.float32), m.shape).copy() for m in mu]
    vox = np.arange(0, s.grid.nvox, 97)
    rgb, cnt, margin = oracle.color(P, W, H, s.grid, frames, mu, sg, vox, slm_gate=gate)
    inview, safe = _exact_inview(P, W, H, s.grid, vox)
    if qualifies:
        assert np.array_equal(cnt[safe], inview[safe].sum(axis=1))
        assert (rgb[cnt > 0] == [90.0, 120.0, 150.0]).all()
    else:
        assert (cnt == 0).all()
    seen = inview.any(axis=1) & safe
    assert np.allclose(margin[seen], abs(SLM_SIGMA5 - gate), rtol=1e-9, atol=0)
