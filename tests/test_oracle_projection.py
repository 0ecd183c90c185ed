"""Pins of the oracle's voxel -> pixel projection ("the pixel ... is the
projection of voxel V_i"; readings R#10-R#13 in DESIGN.md): worked examples of
SPEC.md:46-47 and :346, scale invariance, the ring camera's
principal point, and brute force against the exact
double-precision nearest pixel."""
import numpy as np
import pytest

import oracle
from synth.scene import Grid, cube_grid, look_at_camera, ring_rig

IDENTITY = np.array([[1.0, 0, 0, 0], [0, 1.0, 0, 0], [0, 0, 1.0, 0]])


def _grid_at(point, spacing=1.0):
    """1x1x1 grid whose single voxel centre is `point`."""
    o = np.asarray(point, float) - 0.5 * spacing
    return Grid(tuple(o), spacing, 1, 1, 1)


def _pixel_of(P, point, W=64, H=64, spacing=1.0):
    g = _grid_at(point, spacing)
    A = oracle.precompose(P[None], g.origin, g.spacing)[0]
    return oracle.project_pinned(A, W, H, [[0, 0, 0]])[0]


def test_identity_camera_examples(golden):
    """P = [I|0]: (0,0,2) -> (0,0); (2,4,2) -> (1,2)."""
    for ex in golden("projection_examples.json")["identity_camera"]:
        inview, px, py = _pixel_of(IDENTITY, ex["point"])
        assert inview == 1
        assert (px, py) == tuple(ex["pixel"])


def test_round_half_up_example(golden):
    """projected (10.2, 20.7) -> pixel (10, 21)."""
    ex = golden("projection_examples.json")["round_half_up"]
    u, v = ex["uv"]
    inview, px, py = _pixel_of(IDENTITY, [2 * u, 2 * v, 2.0])
    assert inview == 1 and (px, py) == tuple(ex["pixel"])
    # exact ties round up: (0.5, 1.5) -> (1, 2); (-0.5,...) -> 0 is in view
    inview, px, py = _pixel_of(IDENTITY, [1.0, 3.0, 2.0])
    assert (inview, px, py) == (1, 1, 2)
    inview, px, py = _pixel_of(IDENTITY, [-1.0, 0.0, 2.0])
    assert (inview, px, py) == (1, 0, 0)
    inview, _, _ = _pixel_of(IDENTITY, [-1.25, 0.0, 2.0])  # u = -0.625 -> pixel -1: out
    assert inview == 0


def test_behind_camera_and_outside_image_are_out_of_view():
    """R#12: w <= 0 or pixel outside [0,W)x[0,H) -> out of view."""
    assert _pixel_of(IDENTITY, [0.0, 0.0, -2.0])[0] == 0
    assert _pixel_of(IDENTITY, [0.0, 0.0, 0.0])[0] == 0     # w = 0
    assert _pixel_of(IDENTITY, [127.0, 0.0, 2.0], W=64)[0] == 0   # u = 63.5 -> pixel 64
    inview, px, _ = _pixel_of(IDENTITY, [126.9, 0.0, 2.0], W=64)
    assert inview == 1 and px == 63
    assert _pixel_of(IDENTITY, [0.0, 200.0, 2.0], H=64)[0] == 0


def test_image_border_exact():
    # u + 1/2 == W exactly -> pixel W -> out of view; just below -> W-1
    assert _pixel_of(IDENTITY, [2 * 63.5, 0.0, 2.0], W=64)[0] == 0
    r = _pixel_of(IDENTITY, [2 * 63.49, 0.0, 2.0], W=64)
    assert r[0] == 1 and r[1] == 63


def test_power_of_two_scale_is_bit_invariant():
    """P -> lambda P leaves pixels unchanged; for lambda = 2^e every
    pinned float operation scales exactly, so the result is bit-identical."""
    cams = ring_rig([(4, 1000.0, 0.0)], 64, 48)
    g = cube_grid(16)
    ijk = np.stack(np.meshgrid(np.arange(16), np.arange(16), np.arange(16), indexing="ij"),
                   -1).reshape(-1, 3)
    for cam in cams:
        A1 = oracle.precompose(cam.P[None], g.origin, g.spacing)[0]
        A2 = oracle.precompose((8.0 * cam.P)[None], g.origin, g.spacing)[0]
        assert (oracle.project_pinned(A1, 64, 48, ijk) == oracle.project_pinned(A2, 64, 48, ijk)).all()


def test_general_scale_invariance_exact_projection():
    rng = np.random.default_rng(5)
    cam = look_at_camera((3000.0, -2500.0, 1400.0), (0, 0, 1000), 320, 240)
    g = cube_grid(8)
    for lam in (0.37, 3.1, 1e3):
        for _ in range(50):
            i, j, k = rng.integers(0, 8, 3)
            assert oracle.project_exact(cam.P, g.origin, g.spacing, 320, 240, i, j, k) == \
                oracle.project_exact(lam * cam.P, g.origin, g.spacing, 320, 240, i, j, k)


def test_ring_camera_principal_point():
    """the look-at point projects to the principal point
    ((W-1)/2, (H-1)/2).  For even W, H that is an exact pixel-edge tie, so the
    pinned pixel may land on either side (W/2 - 1 or W/2)."""
    for W, H in ((64, 48), (640, 480), (1920, 1080)):
        for cam in ring_rig([(8, 1000.0, 0.0), (8, 1600.0, 22.5)], W, H):
            X = np.array([0.0, 0.0, 1000.0, 1.0])
            x = cam.P @ X
            assert x[0] / x[2] == pytest.approx((W - 1) / 2, abs=1e-6)
            assert x[1] / x[2] == pytest.approx((H - 1) / 2, abs=1e-6)
            r = _pixel_of(cam.P, [0.0, 0.0, 1000.0], W, H)
            assert r[0] == 1 and r[1] in (W // 2 - 1, W // 2) and r[2] in (H // 2 - 1, H // 2)


@pytest.mark.parametrize("cfg", [("C1", 32, [(4, 1000.0, 0.0)], 64, 48),
                                 ("C2-ish", 64, [(8, 1000.0, 0.0)], 640, 480),
                                 ("tilted", 32, [(8, 600.0, 0.0), (8, 1600.0, 22.5)], 192, 108)])
def test_pinned_matches_exact_nearest_pixel(cfg):
    """Brute force: on every voxel x camera the pinned FP32 projection equals the
    exact double nearest pixel floor(x/w + 1/2), except a small number of
    near-boundary flips (pixel-edge ties within FP32 rounding), which we bound."""
    name, n, rings, W, H = cfg
    cams = ring_rig(rings, W, H)
    g = cube_grid(n)
    P = np.stack([c.P for c in cams])
    Ws = np.full(len(cams), W, np.int32)
    Hs = np.full(len(cams), H, np.int32)
    flips = oracle.projection_flips(P, Ws, Hs, g, nthreads=4)
    total = g.nvox * len(cams)
    assert flips <= 0.01 * total, (flips, total)
    # and the pinned projection really is "nearest pixel": for sampled voxels,
    # |(x/w) - px| <= 1/2 + 1e-3 in double
    A = oracle.precompose(P, g.origin, g.spacing)
    rng = np.random.default_rng(1)
    ijk = rng.integers(0, n, size=(2000, 3))
    for c in range(len(cams)):
        res = oracle.project_pinned(A[c], W, H, ijk)
        Xw = np.asarray(g.origin) + g.spacing * (ijk + 0.5)
        x = np.concatenate([Xw, np.ones((len(ijk), 1))], 1) @ P[c].T
        u, v = x[:, 0] / x[:, 2], x[:, 1] / x[:, 2]
        m = res[:, 0] == 1
        assert np.abs(u[m] - res[m, 1]).max() <= 0.5 + 1e-3
        assert np.abs(v[m] - res[m, 2]).max() <= 0.5 + 1e-3
        # out-of-view ones really are outside (up to the same slack)
        out = ~m
        outside = (x[:, 2] <= 0) | (u < -0.5 + 1e-3) | (u >= W - 0.5 - 1e-3) | \
            (v < -0.5 + 1e-3) | (v >= H - 0.5 - 1e-3)
        assert outside[out].all()
