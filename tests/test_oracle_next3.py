"""Pins of the oracle's NEXT-3 boundary variants:
grayscale input (U = 256^-1, R#25) and bilinear SLM sampling
(clamped at image borders, R#26).

Pinned by values derived by hand (tests/golden/next3_examples.json), a library
re-derivation (scipy.stats.norm.logpdf), the RGB special case (nch = 3 equals
oracle_pixel bit for bit), closed forms for linear SLM images (bilinear
interpolation reproduces a linear field exactly), the reduction to the
nearest-pixel fusion for constant images and at pixel centres, and the
classical-SFS limit on a grayscale scene by brute force."""
import math

import numpy as np
import pytest

import oracle
from synth.scene import Grid, make_frames, make_scene

IDENTITY = np.array([[1.0, 0, 0, 0], [0, 1.0, 0, 0], [0, 0, 1.0, 0]])


# ------------------------------------------------------------------ grayscale

@pytest.mark.parametrize("key", ["gray_I_eq_mu_sigma5", "gray_I_eq_mu_sigma2"])
def test_gray_worked_examples(golden, key):
    g = golden("next3_examples.json")
    ex = g[key]
    slm, l1, l0 = oracle.pixel_nch([ex["I"]], [ex["mu"]], [ex["sigma"]])
    assert slm == pytest.approx(ex["slm"], abs=g["abs_tol"])
    assert l1 - l0 == pytest.approx(ex["t_half"], abs=g["abs_tol"])
    # RGB at the same pixel is a different number (U = 256^-3): the channel count matters
    slm3, _, _ = oracle.pixel_nch([ex["I"]] * 3, [ex["mu"]] * 3, [ex["sigma"]] * 3)
    assert abs(slm3 - slm) > 1e-3


def test_gray_crossing(golden):
    """g = u at I = mu when sigma = 256/sqrt(2 pi): SLM = 1/2 (up to sigma's
    float rounding)."""
    ex = golden("next3_examples.json")["gray_crossing_sigma"]
    slm, l1, l0 = oracle.pixel_nch([128], [128.0], [ex["sigma"]])
    assert slm == pytest.approx(0.5, abs=1e-6)
    assert l1 - l0 == pytest.approx(0.0, abs=1e-5)


def test_gray_scipy_rederivation():
    """d = ln N(I; mu, sigma') + ln 256 (scipy), SLM = 1/(1 + e^d),
    t = -logaddexp(ln p_O, ln(1 - p_O) + d), random pixels, general p_O."""
    from scipy.stats import norm
    rng = np.random.default_rng(31)
    n = 2000
    I = rng.integers(0, 256, size=(n, 1)).astype(np.uint8)
    mu = rng.uniform(0, 255, size=(n, 1)).astype(np.float32)
    sg = rng.uniform(0.3, 40.0, size=(n, 1)).astype(np.float32)
    for floor, po in ((1.0, 0.5), (2.0, 0.3), (0.5, 0.9)):
        slm, l1, l0 = oracle.slm_image(I, mu, sg, floor, po)
        s = np.maximum(sg[:, 0].astype(np.float64), floor)
        d = norm.logpdf(I[:, 0].astype(np.float64), mu[:, 0].astype(np.float64), s) + math.log(256.0)
        np.testing.assert_allclose(slm, 1.0 / (1.0 + np.exp(d)), rtol=1e-12, atol=1e-15)
        t = -np.logaddexp(math.log(po), math.log1p(-po) + d)
        np.testing.assert_allclose(l1 - l0, t, rtol=0, atol=1e-11)


def test_nch3_is_oracle_pixel_bit_for_bit():
    rng = np.random.default_rng(5)
    n = 500
    I = rng.integers(0, 256, size=(n, 3)).astype(np.uint8)
    mu = rng.uniform(0, 255, size=(n, 3)).astype(np.float32)
    sg = rng.uniform(0.3, 40.0, size=(n, 3)).astype(np.float32)
    a = oracle.slm_image(I, mu, sg, 1.0, 0.4)
    for p in range(0, n, 7):
        b = oracle.pixel_nch(I[p], mu[p], sg[p], 1.0, 0.4)
        assert (a[0][p], a[1][p], a[2][p]) == b


def test_gray_monotone_and_bounded():
    mu = np.full((256, 1), 120.0, np.float32)
    sg = np.full((256, 1), 6.0, np.float32)
    I = np.arange(256, dtype=np.uint8).reshape(256, 1)
    slm, l1, l0 = oracle.slm_image(I, mu, sg)
    dev = np.abs(np.arange(256) - 120.0)
    order = np.argsort(dev, kind="stable")
    assert (np.diff(slm[order]) >= -1e-15).all()
    assert (slm >= 0).all() and (slm <= 1).all()


def test_gray_train_background():
    """S:105-106 on one channel: identical frames -> sigma = floor; 90/110 -> 100, 10."""
    a = [np.full((4, 5, 1), 100, np.uint8)] * 10
    m, s = oracle.train_background(a)
    assert (m == 100).all() and (s == 1.0).all()
    b = [np.full((4, 5, 1), 90 if f % 2 else 110, np.uint8) for f in range(10)]
    m, s = oracle.train_background(b)
    assert (m == 100).all() and (s == 10).all()


def test_gray_sfs_limit_brute_force():
    """PAPER.md:59-65 on a grayscale C1 scene: noise-free frames, background
    I = mu with sigma = 2 (t_bg = -3.259, golden), foreground 80 grey levels from
    mu (t_fg = ln 2): with <= 4 cameras a single background view outweighs the
    rest (3 ln 2 < 3.259), so PSFS occupancy is the visual hull, and
    L = n_fg ln 2 + n_bg t_bg."""
    from tests.test_oracle_fusion import _visual_hull_and_counts
    s = make_scene("C1", body="skeleton", integer_mu=True, const_sigma=2.0, channels=1)
    labels = []
    frames = make_frames(s, 0, mode="clean", labels_out=labels)
    sils = [lab >= 0 for lab in labels]
    r = oracle.scene_reconstruct(s, frames)
    occ = np.unpackbits(r["bits"].view(np.uint8), bitorder="little")[: s.grid.nvox].astype(bool)
    vh, nv, nfg = _visual_hull_and_counts(s, sils, return_fg=True)
    assert vh.sum() > 50
    assert (occ == vh).all()
    u = 1.0 / 256
    g = 1.0 / (2.0 * math.sqrt(2 * math.pi))
    t_bg = math.log(2 * u / (u + g))
    ref = nfg * math.log(2.0) + (nv - nfg) * t_bg
    np.testing.assert_allclose(r["L"], ref, atol=1e-10, rtol=0)


# ------------------------------------------------------------------ bilinear

def _one_cam_fuse(slm_yx, origin, p_occ=0.5, p_vox=0.5):
    S = np.asarray(slm_yx, np.float64)
    H, W = S.shape
    g = Grid(tuple(origin), 1.0, 1, 1, 1)
    r = oracle.fuse_bilinear_slm(IDENTITY[None], np.array([W], np.int32), np.array([H], np.int32),
                                 g, [S], p_occ=p_occ, p_vox=p_vox)
    return r


@pytest.mark.parametrize("pri", ["half_priors", "general_priors"])
def test_bilinear_worked_example(golden, pri):
    gd = golden("next3_examples.json")
    ex = gd["bilinear_2x2"]
    # the pinned projection really lands on (x, y) + 1/2
    A = oracle.precompose(IDENTITY[None], ex["grid_origin"], ex["spacing"])[0]
    inview, u, v = oracle.project_pinned_uv(A, ex["W"], ex["H"], 0, 0, 0)
    assert inview and u - 0.5 == ex["x"] and v - 0.5 == ex["y"]
    assert oracle.bilinear(np.array(ex["slm_image_yx"]), ex["x"], ex["y"]) == pytest.approx(
        ex["slm_sample"], abs=gd["abs_tol"])
    e = ex[pri]
    r = _one_cam_fuse(ex["slm_image_yx"], ex["grid_origin"], e["p_occ"], e["p_vox"])
    assert r["L"][0] == pytest.approx(e["L"], abs=gd["abs_tol"])
    assert r["post"][0] == pytest.approx(e["posterior"], abs=gd["abs_tol"])
    assert int(r["bits"][0] & 1) == int(e["posterior"] > 0.5)


@pytest.mark.parametrize("key", ["left_x_lt_0", "right_x_in_1_1p5", "bottom_y_in_1_1p5"])
def test_bilinear_clamped_borders(golden, key):
    gd = golden("next3_examples.json")
    ex = gd["bilinear_clamp"][key]
    S = gd["bilinear_2x2"]["slm_image_yx"]
    r = _one_cam_fuse(S, ex["grid_origin"])
    assert r["L"][0] == pytest.approx(math.log(2 * ex["slm_sample"]), abs=1e-7)


def test_bilinear_reproduces_linear_fields():
    """SLM(x, y) = a + b x + c y over a realistic C1 rig: at every in-view voxel
    whose continuous projection lies inside the pixel-centre hull, the bilinear
    sample is a + b x + c y with (x, y) the EXACT double projection x/w, y/w of
    the voxel centre (P directly, not the oracle), up to the float rounding of
    (u, v) (<= 1e-5 px).  A wrong 1/2 shift, swapped weights or axes, or a
    wrong neighbour fails by >= 1e-3."""
    s = make_scene("C1")
    g = s.grid
    A = oracle.precompose(s.P, g.origin, g.spacing)
    rng = np.random.default_rng(8)
    for c, cam in enumerate(s.cameras):
        W, H = cam.width, cam.height
        a, b, cc = 0.3, 0.5 / W, 0.15 / H
        yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
        S = a + b * xx + cc * yy
        P = s.P[c]
        checked = 0
        for _ in range(400):
            i, j, k = rng.integers(0, g.xlen), rng.integers(0, g.ylen), rng.integers(0, g.zlen)
            inview, u, v = oracle.project_pinned_uv(A[c], W, H, i, j, k)
            if not inview:
                continue
            X = np.array([g.origin[0] + g.spacing * (i + 0.5), g.origin[1] + g.spacing * (j + 0.5),
                          g.origin[2] + g.spacing * (k + 0.5), 1.0])
            h = P @ X
            x, y = h[0] / h[2], h[1] / h[2]
            if not (0.01 < x < W - 1.01 and 0.01 < y < H - 1.01):
                continue
            got = oracle.bilinear(S, u - 0.5, v - 0.5)
            assert got == pytest.approx(a + b * x + cc * y, abs=1e-7)
            checked += 1
        assert checked > 100


def test_bilinear_constant_images_equal_nearest():
    """Constant SLM per camera: every bilinear sample equals the nearest pixel's,
    so oracle_fuse_bilinear equals oracle_fuse (both from the same SLMs)."""
    s = make_scene("C1")
    g = s.grid
    vals = [0.2, 0.7, 0.9, 0.45]
    slm = [np.full((cam.height, cam.width), v) for cam, v in zip(s.cameras, vals)]
    l1 = [np.full(x.shape, oracle.view_likelihood(v, 0.4)[0]) for x, v in zip(slm, vals)]
    l0 = [np.full(x.shape, oracle.view_likelihood(v, 0.4)[1]) for x, v in zip(slm, vals)]
    a = oracle.fuse_bilinear_slm(s.P, s.widths, s.heights, g, slm, p_occ=0.4, p_vox=0.3)
    b = oracle.fuse_views(s.P, s.widths, s.heights, g, l1, l0, p_occ=0.4, p_vox=0.3)
    np.testing.assert_allclose(a["L"], b["L"], atol=1e-12, rtol=0)
    assert np.array_equal(a["bits"], b["bits"])


def test_bilinear_at_pixel_centres_equals_nearest():
    """P = [I|0] with voxel centres projecting exactly onto pixel centres
    (x/w, y/w integers): fx = fy = 0, the sample is that pixel's SLM, so the
    bilinear and nearest fusions agree on random SLM images."""
    rng = np.random.default_rng(12)
    X, Y = 6, 5
    g = Grid((-0.5, -0.5, 0.5), 1.0, X, Y, 1)  # voxel (i, j) -> centre (i, j, 1) -> pixel (i, j)
    slms = [rng.uniform(0.01, 0.99, size=(Y, X)) for _ in range(3)]
    l1 = [np.vectorize(lambda v: oracle.view_likelihood(v, 0.5)[0])(s_) for s_ in slms]
    l0 = [np.vectorize(lambda v: oracle.view_likelihood(v, 0.5)[1])(s_) for s_ in slms]
    P = np.stack([IDENTITY] * 3)
    W = np.full(3, X, np.int32)
    H = np.full(3, Y, np.int32)
    a = oracle.fuse_bilinear_slm(P, W, H, g, slms)
    b = oracle.fuse_views(P, W, H, g, l1, l0)
    np.testing.assert_allclose(a["L"], b["L"], atol=1e-12, rtol=0)


def test_bilinear_invariants():
    """Camera-order invariance; unseen voxels keep the prior; posterior in [0,1]."""
    s = make_scene("C1")
    fr = make_frames(s, 0)
    a = oracle.scene_reconstruct(s, fr, sampling="bilinear", want_slm=True)
    assert (a["post"] >= 0).all() and (a["post"] <= 1).all()
    perm = [2, 0, 3, 1]
    P = s.P[perm]
    b = oracle.reconstruct(P, s.widths[perm], s.heights[perm], s.grid, fr[perm], s.mu[perm],
                           s.sigma[perm], sampling="bilinear")
    np.testing.assert_allclose(a["L"], b["L"], atol=1e-12, rtol=0)
    g = Grid((-6000.0, -6000.0, -3000.0), 12000.0 / 16, 16, 16, 16)
    s2 = make_scene("C1", grid=g)
    c = oracle.scene_reconstruct(s2, make_frames(s2, 0), sampling="bilinear", p_vox=0.3)
    n = oracle.scene_reconstruct(s2, make_frames(s2, 0), p_vox=0.3)
    unseen = np.abs(n["L"] - math.log(0.3 / 0.7)) < 1e-15
    assert unseen.sum() > 100
    np.testing.assert_allclose(c["L"][unseen], math.log(0.3 / 0.7), atol=1e-15)
    # bilinear and nearest differ (the variant is not a no-op), but not by much
    assert np.abs(a["L"] - oracle.scene_reconstruct(s, fr)["L"]).max() > 1e-3
