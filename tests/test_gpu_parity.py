"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded synthetic inputs.  Bar (BASELINE.json north_star): log-odds within
1e-4 absolute; occupancy bits exact except voxels whose posterior lies within
1e-4 of tau; stage-1 terms within 1e-6 of the oracle's t = ln P(S|V=1) -
ln P(S|V=0) (DESIGN.md error budget)."""
import math
import os

import numpy as np
import pytest

import oracle
from synth.scene import Grid, cube_grid, make_frames, make_scene, ring_rig
from tests.helpers import assert_parity, gpu_run, unpack_bits

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

NTHREADS = max(1, len(os.sched_getaffinity(0)))
TERM_TOL = 1e-6


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1311_6811_b200 import build
    build.build()


# ------------------------------------------------------------------ stage 1

def _terms_vs_oracle(scene, frames, params=None):
    from paper_1311_6811_b200 import from_scene
    params = params or {}
    rec = from_scene(scene, params)
    q = rec.debug_terms(torch.from_numpy(frames).cuda()).cpu().numpy().astype(np.float64)
    t_gpu = q / 2.0 ** 20
    worst = 0.0
    off = 0
    for c in range(scene.ncam):
        _, l1, l0 = oracle.slm_image(frames[c], scene.mu[c], scene.sigma[c],
                                     params.get("sigma_floor", 1.0),
                                     params.get("occlusion_prior", 0.5), NTHREADS)
        t = (l1 - l0).reshape(-1)
        n = t.shape[0]
        worst = max(worst, float(np.abs(t_gpu[off:off + n] - t).max()))
        off += n
    return worst


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_stage1_terms(name):
    s = make_scene(name)
    fr = make_frames(s, 0)
    assert _terms_vs_oracle(s, fr) <= TERM_TOL


def test_stage1_extreme_pixels():
    """I = mu at the sigma floor (d = d_max), >= 10 sigma deviations, sigma below
    the floor, general p_O."""
    s = make_scene("C1")
    rng = np.random.default_rng(1)
    mu = s.mu.copy()
    sg = s.sigma.copy()
    fr = make_frames(s, 0)
    mu[:, ::2, ::2] = np.round(mu[:, ::2, ::2])
    fr[:, ::2, ::2] = mu[:, ::2, ::2].astype(np.uint8)       # I = mu exactly
    sg[:, ::4, :] = rng.uniform(0.1, 1.0, size=sg[:, ::4, :].shape)  # below the floor
    fr[:, 1::4, :] = np.where(mu[:, 1::4, :] < 128, 255, 0)  # far tail
    s.mu, s.sigma = mu.astype(np.float32), sg.astype(np.float32)
    for p in (dict(), dict(occlusion_prior=0.3), dict(occlusion_prior=0.9, sigma_floor=2.0)):
        assert _terms_vs_oracle(s, fr, p) <= TERM_TOL


def test_stage1_ragged_width():
    """W % 4 != 0 takes the scalar (1 pixel/thread) kernel."""
    s = make_scene("C1", W=66, H=50)
    fr = make_frames(s, 0)
    assert _terms_vs_oracle(s, fr) <= TERM_TOL


# ------------------------------------------------------------------ end to end

def _parity(scene, frames_list, params=None, fuse=8, roi=True, **kw):
    params = params or {}
    g = gpu_run(scene, frames_list, params, fuse=fuse, roi=roi)
    stats = []
    for f, fr in enumerate(frames_list):
        orc = oracle.scene_reconstruct(scene, fr, nthreads=NTHREADS,
                                       sigma_floor=params.get("sigma_floor", 1.0),
                                       p_occ=params.get("occlusion_prior", 0.5),
                                       p_vox=params.get("voxel_prior", 0.5),
                                       tau=params.get("threshold", 0.5))
        stats.append(assert_parity(g["L"][f], g["bits"][f], orc, scene.grid.nvox,
                                   tau=params.get("threshold", 0.5), **kw))
    return g, stats


@pytest.mark.parametrize("name,body", [("C1", "skeleton"), ("C1", "ellipsoid"),
                                       ("C2", "skeleton"), ("C2", "both")])
def test_end_to_end_single_frame(name, body):
    s = make_scene(name, body=body)
    _, st = _parity(s, [make_frames(s, 0)])
    assert st[0]["occupied"] > 0


def test_c2_bench_configuration_batch_of_8():
    """The bench's launch configuration: C2, F = 8 distinct frames fused."""
    s = make_scene("C2")
    frames = [make_frames(s, f) for f in range(8)]
    g, st = _parity(s, frames, fuse=8)
    # and every frame of the fused batch equals the same frame run alone (F = 1):
    # integer sums make the result independent of grouping
    g1 = gpu_run(s, frames[:3], fuse=1)
    assert np.array_equal(g1["bits"], g["bits"][:3])
    assert np.array_equal(g1["L"], g["L"][:3])


def test_c2_batch_of_16_paired_kernel():
    """16-frame passes (64-byte term records, lane pairs in k_voxel16): C2 with
    16 distinct frames against the oracle, and bit-identical to 8-frame passes."""
    s = make_scene("C2")
    frames = [make_frames(s, f) for f in range(16)]
    g, st = _parity(s, frames, fuse=16)
    g8 = gpu_run(s, frames, fuse=8)
    assert np.array_equal(g8["bits"], g["bits"])
    assert np.array_equal(g8["L"], g["L"])


def test_c2_bench_launch_configuration_64_frames():
    """bench.py's timed call: C2, 64 distinct frame sets in one
    psfs_reconstruct_batch (four 16-frame passes, stage 1 of pass g+1
    overlapped with stage 2 of pass g), every frame against the oracle."""
    from paper_1311_6811_b200 import from_scene
    s = make_scene("C2")
    frames = [make_frames(s, f) for f in range(64)]
    rec = from_scene(s)
    rec.set_overlap(True, 0)
    L, B = rec.alloc_outputs(64)
    rec.reconstruct_batch(torch.from_numpy(np.stack(frames)).cuda(), 64, logodds=L, bits=B)
    torch.cuda.synchronize()
    assert rec.last_launch_count == 8
    Lh, Bh = L.cpu().numpy(), B.cpu().numpy().view(np.uint32)
    for f in range(64):
        orc = oracle.scene_reconstruct(s, frames[f], nthreads=NTHREADS)
        assert_parity(Lh[f], Bh[f], orc, s.grid.nvox)


def test_batch_grouping_29_frames():
    """29 = 16 + 8 + 4 + 1 frames: every group size, against the oracle."""
    s = make_scene("C1")
    frames = [make_frames(s, f) for f in range(29)]
    _parity(s, frames, fuse=16)


def test_batch_grouping_13_frames():
    """13 = 8 + 4 + 1 frames: every group size path, against the oracle."""
    s = make_scene("C1")
    frames = [make_frames(s, f) for f in range(13)]
    _parity(s, frames)


@pytest.mark.parametrize("fuse", [1, 2, 4])
def test_fuse_widths(fuse):
    s = make_scene("C1")
    _parity(s, [make_frames(s, f) for f in range(fuse)], fuse=fuse)


def test_c3_sequence_frames():
    """C3 (256^3, 8 cameras 1280x960): frames of the walking / arm-waving
    sequence, full grid against the oracle."""
    s = make_scene("C3")
    frames = [make_frames(s, f, motion=True) for f in (0, 45)]
    _parity(s, frames)


@pytest.mark.parametrize("nf,fuse", [(3, 8), (17, 16)])
def test_ragged_grid_and_images(nf, fuse):
    """xlen % 32 != 0 (atomic bit path), xlen odd (a lane pair with one voxel
    outside the grid), ylen % 8 != 0, zlen % KZ != 0, W % 4 != 0."""
    g = Grid((-1000.0, -1000.0, 0.0), 2000.0 / 37, 37, 29, 23)
    s = make_scene("C1", grid=g, W=66, H=50)
    _parity(s, [make_frames(s, f) for f in range(nf)], fuse=fuse)


@pytest.mark.parametrize("nf,fuse", [(2, 8), (16, 16)])
def test_general_priors_and_threshold(nf, fuse):
    s = make_scene("C1")
    p = dict(occlusion_prior=0.3, voxel_prior=0.2, threshold=0.7, sigma_floor=1.5)
    _parity(s, [make_frames(s, f) for f in range(nf)], params=p, fuse=fuse)


def test_all_background_gives_empty_hull():
    s = make_scene("C2")
    g = gpu_run(s, [make_frames(s, 0, mode="background")])
    assert g["bits"].sum() == 0


def test_unseen_voxels_keep_prior():
    """Grid extending far outside every view: those voxels' log-odds equal
    logit(p_V) (rounded to float) and they are unoccupied at tau = 1/2."""
    g = Grid((-6000.0, -6000.0, -3000.0), 12000.0 / 32, 32, 32, 32)
    s = make_scene("C1", grid=g)
    for pv in (0.5, 0.35):
        out = gpu_run(s, [make_frames(s, 0)], params=dict(voxel_prior=pv))
        orc = oracle.scene_reconstruct(s, make_frames(s, 0), p_vox=pv)
        unseen = np.abs(orc["L"] - (math.log(pv) - math.log1p(-pv))) < 1e-12
        assert unseen.sum() > 1000
        assert (out["L"][0][unseen] == np.float32(math.log(pv) - math.log1p(-pv))).all()


def test_camera_permutation_bit_identical():
    """Fixed-point accumulation: permuting the cameras leaves the GPU output
    bit-identical."""
    s = make_scene("C1")
    fr = make_frames(s, 0)
    a = gpu_run(s, [fr])
    perm = np.array([2, 0, 3, 1])
    s2 = make_scene("C1")
    s2.cameras = [s.cameras[i] for i in perm]
    s2.mu, s2.sigma = s.mu[perm], s.sigma[perm]
    b = gpu_run(s2, [fr[perm]])
    assert np.array_equal(a["bits"], b["bits"]) and np.array_equal(a["L"], b["L"])


def test_roi_on_off_identical():
    s = make_scene("C2")
    fr = [make_frames(s, 0), make_frames(s, 1)]
    a = gpu_run(s, fr, roi=True)
    b = gpu_run(s, fr, roi=False)
    assert np.array_equal(a["bits"], b["bits"]) and np.array_equal(a["L"], b["L"])
    roi = a["rec"].roi()
    area = ((roi[:, 1] - roi[:, 0]) * (roi[:, 3] - roi[:, 2])).sum()
    assert area < s.ncam * 640 * 480


@pytest.mark.parametrize("world", [2, 4])
def test_zslab_handles_concatenate_to_full(world):
    """z-slab partition on one GPU: each rank's handle writes exactly its slab's
    words and log-odds; together they are bit-identical to the 1-handle run."""
    s = make_scene("C2")
    fr = [make_frames(s, 0)]
    full = gpu_run(s, fr)
    nw = s.grid.nwords
    plane = s.grid.xlen * s.grid.ylen
    bits = np.zeros(nw, np.uint32)
    for r in range(world):
        part = gpu_run(s, fr, rank=r, world=world)
        k0, k1 = part["rec"].k0, part["rec"].k1
        w0, w1 = plane * k0 // 32, plane * k1 // 32
        bits[w0:w1] = part["bits"][0][w0:w1]
        assert np.array_equal(part["L"][0], full["L"][0][plane * k0: plane * k1])
        roi_full = full["rec"].roi()
        roi = part["rec"].roi()
        assert ((roi[:, 1] - roi[:, 0]) <= (roi_full[:, 1] - roi_full[:, 0])).all()
    assert np.array_equal(bits, full["bits"][0])
    # the assembled slabs against the oracle (A5 parity)
    orc = oracle.scene_reconstruct(s, fr[0], nthreads=NTHREADS)
    assert_parity(None, bits, orc, s.grid.nvox)


def test_reconstruct_host_matches_device_path():
    from paper_1311_6811_b200 import from_scene
    s = make_scene("C2")
    frames = np.stack([make_frames(s, f) for f in range(11)])
    dev = gpu_run(s, list(frames))
    rec = from_scene(s)
    hf = torch.from_numpy(frames).pin_memory()
    Lh = torch.empty((11, rec.nslab), dtype=torch.float32).pin_memory()
    Bh = torch.zeros((11, s.grid.nwords), dtype=torch.int32).pin_memory()
    rec.reconstruct_host(hf, 11, Lh, Bh)
    torch.cuda.synchronize()
    assert np.array_equal(Bh.numpy().view(np.uint32), dev["bits"])
    assert np.array_equal(Lh.numpy(), dev["L"])


# ------------------------------------------------------------------ full sizes, sampled

def _sample_voxels(grid, rng, n_random=1 << 16, every=64):
    plane = grid.xlen * grid.ylen
    ks = np.arange(0, grid.zlen, every)
    rows = np.concatenate([k * plane + rng.integers(0, plane, 4096) for k in ks])
    return np.unique(np.concatenate([rows, rng.integers(0, grid.nvox, n_random)]))


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_full_size_sampled(name):
    """C4 (512^3, 16 cams 1920x1080) and C5 (1024^3, 32 cams): the full-size GPU
    run, checked on a voxel sample (every 64th z-slice x 4096 voxels + 65536
    random voxels) that the oracle evaluates voxel by voxel, plus an invariant
    over every voxel (occupied <=> L > logit tau at tau = p_V = 1/2)."""
    from paper_1311_6811_b200 import from_scene
    s = make_scene(name)
    fr = make_frames(s, 0)
    rec = from_scene(s)
    L, B = rec.alloc_outputs(1)
    rec.reconstruct_batch(torch.from_numpy(fr).cuda(), 1, logodds=L, bits=B)
    torch.cuda.synchronize()
    rng = np.random.default_rng(7)
    vox = _sample_voxels(s.grid, rng)
    Lo, post = oracle.fuse_sample(s.P, s.widths, s.heights, s.grid, fr, s.mu, s.sigma, vox,
                                  nthreads=NTHREADS)
    vt = torch.from_numpy(vox).cuda()
    Lg = L[0][vt].cpu().numpy().astype(np.float64)
    assert np.abs(Lg - Lo).max() <= 1e-4
    words = B[0][(vt >> 5)].cpu().numpy().view(np.uint32)
    bits = ((words >> (vox & 31).astype(np.uint32)) & 1).astype(bool)
    mism = bits != (post > 0.5)
    assert not (mism & ~(np.abs(post - 0.5) < 1e-4)).any()
    assert bits.sum() > 0
    # every voxel: bit set <=> L > 0 (integer compare S > 0 vs float L)
    shifts = torch.arange(32, device="cuda", dtype=torch.int32)
    allbits = ((B[0].view(-1, 1) >> shifts) & 1).view(-1)[: s.grid.nvox].bool()
    assert not bool((allbits & (L[0] < 0)).any()) and not bool((~allbits & (L[0] > 0)).any())


@pytest.mark.parametrize("name,with_logodds", [("C4", True), ("C5", False)])
def test_full_size_sixteen_frame_pass(name, with_logodds):
    """The full-size configurations through the exact path's 16-frame pass
    (k_likelihood halves + k_voxel16: NCAM = 16 for C4, the generic camera loop
    k_voxel16<0> for C5's 32 cameras) over 2 distinct frame sets repeated 8
    times.  Coarse passes are switched off (psfs_set_coarse(0)) so the bits-only
    C5 call takes the exact kernels too.  Both distinct frames are checked on
    the voxel sample against the oracle (log-odds for C4, bits for both; C5's
    16 log-odds volumes would need 64 GB), and every repeat is bit-identical to
    its original."""
    from paper_1311_6811_b200 import from_scene
    s = make_scene(name)
    two = [make_frames(s, 0), make_frames(s, 1)]
    fr = torch.from_numpy(np.stack(two)).cuda().repeat(8, 1, 1, 1, 1)
    rec = from_scene(s)
    rec.set_coarse(0)
    assert not rec.coarse_status()[0]
    L, B = rec.alloc_outputs(16, logodds=with_logodds)
    rec.reconstruct_batch(fr, 16, logodds=L, bits=B)
    torch.cuda.synchronize()
    for f in range(2, 16):
        assert torch.equal(B[f], B[f % 2])
    rng = np.random.default_rng(11)
    vox = _sample_voxels(s.grid, rng)
    vt = torch.from_numpy(vox).cuda()
    for f in range(2):
        Lo, post = oracle.fuse_sample(s.P, s.widths, s.heights, s.grid, two[f], s.mu, s.sigma, vox,
                                      nthreads=NTHREADS)
        if with_logodds:
            assert np.abs(L[f][vt].cpu().numpy().astype(np.float64) - Lo).max() <= 1e-4
        words = B[f][(vt >> 5)].cpu().numpy().view(np.uint32)
        bits = ((words >> (vox & 31).astype(np.uint32)) & 1).astype(bool)
        mism = bits != (post > 0.5)
        assert not (mism & ~(np.abs(post - 0.5) < 1e-4)).any()
        assert bits.sum() > 0


# ------------------------------------------------------------------ bench launch configurations (round 2 legs)

def test_c3_sequence_300_frames_one_call():
    """bench.py's C3 leg: the 300-frame walking / arm-waving sequence (16
    distinct frame sets of it, cycled) in ONE call (coarse passes of <= 64
    frames); frames 0, 150 and 299 against the oracle on the full 256^3 grid."""
    from paper_1311_6811_b200 import from_scene
    s = make_scene("C3")
    distinct = [make_frames(s, f * 19, motion=True) for f in range(16)]
    dev = [torch.from_numpy(d).cuda() for d in distinct]
    rec = from_scene(s)
    n = 300
    tab = rec.frame_pointers([dev[f % 16] for f in range(n)], n)
    _, B = rec.alloc_outputs(n, logodds=False)
    rec.reconstruct_batch(tab, n, bits=B)
    torch.cuda.synchronize()
    assert rec.coarse_status()[0]
    for f in (0, 150, 299):
        orc = oracle.scene_reconstruct(s, distinct[f % 16], nthreads=NTHREADS)
        assert_parity(None, B[f].cpu().numpy().view(np.uint32), orc, s.grid.nvox)


def test_c5_coarse_pass_64_frames_sampled():
    """bench.py's C5 leg: one 64-frame coarse pass of 1024^3 voxels x 32 cameras
    (the frame-pointer table of 2048 entries), checked on the voxel sample
    against the oracle for two distinct frame sets, repeats bit-identical."""
    from paper_1311_6811_b200 import from_scene
    s = make_scene("C5")
    two = [make_frames(s, 0), make_frames(s, 1)]
    dev = [torch.from_numpy(d).cuda() for d in two]
    rec = from_scene(s)
    n = 64
    tab = rec.frame_pointers([dev[f % 2] for f in range(n)], n)
    _, B = rec.alloc_outputs(n, logodds=False)
    rec.reconstruct_batch(tab, n, bits=B)
    torch.cuda.synchronize()
    assert rec.coarse_status()[0]
    for f in range(2, n, 7):
        assert torch.equal(B[f], B[f % 2])
    rng = np.random.default_rng(23)
    vox = _sample_voxels(s.grid, rng)
    vt = torch.from_numpy(vox).cuda()
    for f in range(2):
        _, post = oracle.fuse_sample(s.P, s.widths, s.heights, s.grid, two[f], s.mu, s.sigma, vox,
                                     nthreads=NTHREADS)
        words = B[f][(vt >> 5)].cpu().numpy().view(np.uint32)
        bits = ((words >> (vox & 31).astype(np.uint32)) & 1).astype(bool)
        mism = bits != (post > 0.5)
        assert not (mism & ~(np.abs(post - 0.5) < 1e-4)).any()
        assert bits.sum() > 0


@pytest.mark.parametrize("world", [1, 4])
def test_row_spans_identical_to_rectangles(world):
    """Per-row spans of the ROI (stage 1 only computes, and the host path only
    uploads, the columns each row's projected slab hull covers): the exact and
    the coarse outputs equal the rectangles' and the whole images', the device
    and host paths alike, while fewer pixels are processed."""
    from paper_1311_6811_b200 import from_scene
    s = make_scene("C2")
    frames = np.stack([make_frames(s, f % 8) for f in range(20)])
    fr = torch.from_numpy(frames).cuda()
    outs = {}
    for mode in (True, 2, False):
        for r in range(world):
            rec = from_scene(s, rank=r, world=world)
            rec.set_roi_enabled(mode)
            L, B = rec.alloc_outputs(20)
            rec.reconstruct_batch(fr, 20, logodds=L, bits=B)          # exact path
            _, Bc = rec.alloc_outputs(20, logodds=False)
            rec.reconstruct_batch(fr, 20, bits=Bc)                    # coarse pass
            hf = torch.from_numpy(frames).pin_memory()
            Bh = torch.zeros((20, s.grid.nwords), dtype=torch.int32).pin_memory()
            rec.reconstruct_host(hf, 20, None, Bh)                    # zero-copy upload of the spans
            torch.cuda.synchronize()
            outs[(mode, r)] = (L.cpu().numpy(), B.cpu().numpy(), Bc.cpu().numpy(), Bh.numpy().copy(),
                               rec.roi_pixels())
    for r in range(world):
        a, b, c = outs[(True, r)], outs[(2, r)], outs[(False, r)]
        for k in range(4):
            assert np.array_equal(a[k], b[k]) and np.array_equal(a[k], c[k]), (r, k)
        assert np.array_equal(a[1], a[2]) and np.array_equal(a[1], a[3])
        assert a[4] < b[4] < c[4]
    orc = oracle.scene_reconstruct(s, frames[0], nthreads=NTHREADS)
    if world == 1:
        assert_parity(outs[(True, 0)][0][0], outs[(True, 0)][1][0], orc, s.grid.nvox)
