"""Pins of the oracle's stage 2: occupancy posterior (Eq 3-4)
with the occlusion latent (Eq 5-9) and thresholding.

Pinned against closed forms, invariants
(BASELINE.json north_star: posterior in [0,1], camera-order
invariance, an unseen voxel keeps its prior, all-background images give an
empty hull), and brute force on tiny grids (the classical-SFS limit,
PAPER.md:59-61, and visual-hull fidelity)."""
import math

import numpy as np
import pytest

import oracle
from synth.scene import (Grid, body_parts, cube_grid, make_frames, make_scene,
                         render_silhouette)

IDENTITY = np.array([[1.0, 0, 0, 0], [0, 1.0, 0, 0], [0, 0, 1.0, 0]])


def handset_fuse(slm_images, p_occ=0.5, p_vox=0.5, tau=0.5):
    """n identical cameras P=[I|0] looking at a 1-voxel-thick X x Y grid whose
    voxel (i, j) projects to pixel (i, j) of every view; view c's SLM image is
    given by hand.  Returns the oracle's L / posterior / bits."""
    slm_images = [np.asarray(s, np.float64) for s in slm_images]
    Y, X = slm_images[0].shape
    g = Grid((-0.5, -0.5, 0.5), 1.0, X, Y, 1)
    l1s, l0s = [], []
    for s in slm_images:
        flat = s.reshape(-1)
        pairs = np.array([oracle.view_likelihood(v, p_occ) for v in flat])
        l1s.append(pairs[:, 0].reshape(Y, X))
        l0s.append(pairs[:, 1].reshape(Y, X))
    n = len(slm_images)
    P = np.stack([IDENTITY] * n)
    W = np.full(n, X, np.int32)
    H = np.full(n, Y, np.int32)
    return oracle.fuse_views(P, W, H, g, l1s, l0s, p_occ=p_occ, p_vox=p_vox, tau=tau)


def _one_voxel(slms, **kw):
    r = handset_fuse([np.array([[s]]) for s in slms], **kw)
    return r["post"][0], r["L"][0], int(r["bits"][0] & 1)


@pytest.mark.parametrize("key", ["four_views_slm_one", "all_half", "any_zero",
                                 "n8_half_priors", "n8_general_priors"])
def test_worked_examples(golden, key):
    g = golden("fusion_worked_examples.json")
    ex = g[key]
    post, L, bit = _one_voxel(ex["slm"], p_occ=ex["p_occ"], p_vox=ex["p_vox"])
    assert post == pytest.approx(ex["posterior"], abs=g["abs_tol"])
    if "L" in ex:
        assert L == pytest.approx(ex["L"], abs=g["abs_tol"])
    assert bit == int(ex["posterior"] > 0.5)


def test_closed_form_1e4_voxels_8_views():
    """SPEC.md:563 (acceptance #1): priors 1/2 -> posterior = prod SLM /
    (prod SLM + 2^-n) within 1e-12 on 10^4 random voxels x 8 random SLMs."""
    rng = np.random.default_rng(2024)
    slms = [rng.uniform(0.0, 1.0, size=(100, 100)) for _ in range(8)]
    r = handset_fuse(slms)
    prod = np.prod(np.stack(slms), axis=0).reshape(-1)
    ref = prod / (prod + 2.0 ** -8)
    np.testing.assert_allclose(r["post"], ref, rtol=0, atol=1e-12)
    assert (r["post"] >= 0).all() and (r["post"] <= 1).all()
    bits = np.unpackbits(r["bits"].view(np.uint8), bitorder="little")[:10000]
    assert (bits == (ref > 0.5)).all() or np.abs(ref[bits != (ref > 0.5)] - 0.5).max() < 1e-12


def test_camera_permutation_invariance():
    """fusion is invariant to camera order (double: <= 1e-12)."""
    rng = np.random.default_rng(9)
    slms = [rng.uniform(0.01, 0.99, size=(20, 30)) for _ in range(6)]
    a = handset_fuse(slms, p_occ=0.3, p_vox=0.4)
    perm = rng.permutation(6)
    b = handset_fuse([slms[i] for i in perm], p_occ=0.3, p_vox=0.4)
    np.testing.assert_allclose(a["L"], b["L"], atol=1e-12, rtol=0)


def test_monotone_in_slm():
    """raising any sampled SLM never lowers the posterior."""
    rng = np.random.default_rng(4)
    base = [rng.uniform(0.05, 0.95, size=(10, 10)) for _ in range(5)]
    for p_occ in (0.5, 0.2, 0.9):
        a = handset_fuse(base, p_occ=p_occ)
        up = [b.copy() for b in base]
        up[2] = np.minimum(up[2] + 0.04, 1.0)
        b = handset_fuse(up, p_occ=p_occ)
        assert (b["post"] >= a["post"] - 1e-15).all()


def test_unseen_voxel_keeps_prior():
    """BJ:5: a voxel seen by no camera keeps its prior (L = logit p_V exactly)."""
    for p_vox in (0.5, 0.2, 0.7):
        # a seen voxel moves off the prior; a 3x3 grid behind every camera (w = -1)
        # is seen by none and keeps it
        r = handset_fuse([np.array([[0.9]]), np.array([[0.8]])], p_vox=p_vox)
        assert r["post"][0] > p_vox
        g = Grid((-0.5, -0.5, -1.5), 1.0, 3, 3, 1)  # behind: w = -1
        P = np.stack([IDENTITY] * 3)
        l1 = [np.zeros((3, 3))] * 3
        l0 = [np.zeros((3, 3)) - 1.0] * 3
        rr = oracle.fuse_views(P, np.full(3, 3, np.int32), np.full(3, 3, np.int32), g, l1, l0,
                               p_vox=p_vox)
        np.testing.assert_allclose(rr["L"], math.log(p_vox) - math.log(1 - p_vox), atol=1e-14)
        np.testing.assert_allclose(rr["post"], p_vox, atol=1e-15)


def test_all_background_frames_give_empty_hull():
    """BJ:5 / SURVEY §8(c): I = round(mu) everywhere and sigma in [2, 8]:
    d >= K - 3 (0.5/2)^2/2 > 0 so every in-view term is negative -> empty."""
    s = make_scene("C1")
    frames = make_frames(s, 0, mode="background")
    r = oracle.scene_reconstruct(s, frames)
    assert r["bits"].sum() == 0
    assert r["L"].max() <= 0.0


def _visual_hull_and_counts(scene, sils, return_fg=False):
    """Brute-force visual hull with the oracle's (pinned) projection: voxel is in
    the hull iff n_v >= 1 and every camera that sees it sees silhouette."""
    g = scene.grid
    A = oracle.precompose(scene.P, g.origin, g.spacing)
    ii, jj, kk = np.meshgrid(np.arange(g.xlen), np.arange(g.ylen), np.arange(g.zlen),
                             indexing="ij")
    ijk = np.stack([ii.ravel(), jj.ravel(), kk.ravel()], 1)
    lin = ijk[:, 0] + g.xlen * (ijk[:, 1] + g.ylen * ijk[:, 2])
    nv = np.zeros(g.nvox, np.int32)
    nfg = np.zeros(g.nvox, np.int32)
    allfg = np.ones(g.nvox, bool)
    for c, cam in enumerate(scene.cameras):
        res = oracle.project_pinned(A[c], cam.width, cam.height, ijk)
        seen = res[:, 0] == 1
        fg = np.zeros(len(ijk), bool)
        fg[seen] = sils[c][res[seen, 2], res[seen, 1]]
        nv[lin[seen]] += 1
        nfg[lin[seen & fg]] += 1
        allfg[lin[seen & ~fg]] = False
    if return_fg:
        return (nv >= 1) & allfg, nv, nfg
    return (nv >= 1) & allfg, nv


def test_sfs_limit_brute_force():
    """with noise-free frames, background I = mu (sigma = 5) and
    foreground >= 16 sigma from mu, t_fg = ln 2 and t_bg = -8.357; for voxels
    seen by n_v <= 13 cameras PSFS occupancy equals the classical visual hull
    (every seeing camera's pixel is silhouette foreground)."""
    s = make_scene("C1", body="skeleton", integer_mu=True, const_sigma=5.0)
    labels = []
    frames = make_frames(s, 0, mode="clean", labels_out=labels)
    sils = [lab >= 0 for lab in labels]
    r = oracle.scene_reconstruct(s, frames)
    occ = np.unpackbits(r["bits"].view(np.uint8), bitorder="little")[: s.grid.nvox].astype(bool)
    vh, nv, nfg = _visual_hull_and_counts(s, sils, return_fg=True)
    assert nv.max() <= 13
    assert vh.sum() > 50
    assert (occ == vh).all()
    # and the log-odds are the closed form n_fg ln 2 + n_bg t_bg, where at I = mu
    # and sigma = 5: d_bg = 3 ln 256 - 1.5 ln 2 pi - 3 ln 5, t_bg = ln 2 - softplus(d_bg)
    # (Eq 5-9 at p_O = 1/2), and t_fg = ln 2 - softplus(d_fg) = ln 2 (d_fg ~ -375)
    d_bg = 3 * math.log(256.0) - 1.5 * math.log(2 * math.pi) - 3 * math.log(5.0)
    t_bg = math.log(2.0) - (d_bg + math.log1p(math.exp(-d_bg)))
    ref = nfg * math.log(2.0) + (nv - nfg) * t_bg
    np.testing.assert_allclose(r["L"], ref, atol=1e-10, rtol=0)


def test_sphere_fidelity_iou():
    """SPEC.md:565 (acceptance #3): noisy ellipsoid, 8-camera ring: occupancy IoU
    vs the rasterised visual hull >= 0.85, and the hull-containment ordering
    (SPEC.md:500): mean posterior inside the true body > outside every cone."""
    g = cube_grid(48)
    s = make_scene("C2", body="ellipsoid", grid=g, W=200, H=150)
    labels = []
    frames = make_frames(s, 0, labels_out=labels)
    sils = [lab >= 0 for lab in labels]
    r = oracle.scene_reconstruct(s, frames, nthreads=4)
    occ = np.unpackbits(r["bits"].view(np.uint8), bitorder="little")[: g.nvox].astype(bool)
    vh, nv = _visual_hull_and_counts(s, sils)
    iou = (occ & vh).sum() / max((occ | vh).sum(), 1)
    assert iou >= 0.85, iou
    assert r["post"][vh].mean() > r["post"][~vh & (nv > 0)].mean()


def test_sampled_mode_equals_full_mode():
    """oracle_fuse_sample (terms on demand) == oracle_fuse (term images)."""
    s = make_scene("C1")
    fr = make_frames(s, 0)
    full = oracle.scene_reconstruct(s, fr)
    rng = np.random.default_rng(0)
    vox = rng.integers(0, s.grid.nvox, 500)
    L, post = oracle.fuse_sample(s.P, s.widths, s.heights, s.grid, fr, s.mu, s.sigma, vox)
    np.testing.assert_array_equal(L, full["L"][vox])


def test_slab_outputs_are_slices_of_full():
    """k0/k1 slab evaluation returns exactly the slab of the full grid (used by
    the z-slab multi-GPU partition tests)."""
    s = make_scene("C1")
    fr = make_frames(s, 0)
    full = oracle.scene_reconstruct(s, fr)
    plane = s.grid.xlen * s.grid.ylen
    part = oracle.scene_reconstruct(s, fr, k0=8, k1=20)
    np.testing.assert_array_equal(part["L"], full["L"][8 * plane: 20 * plane])
    np.testing.assert_array_equal(part["bits"], full["bits"][8 * plane // 32: 20 * plane // 32])
