"""GPU tests of the coarse passes (bits-only calls).

* the bracket: for every pixel, the coarse code c (k_likelihood_c8, FP32)
  brackets the exact Q11.20 term q of k_likelihood: c 2^sh <= q <= c 2^sh + wc
  (adversarial pixels included: I = mu at the sigma floor, far tails, sigma below
  the floor, general p_O);
* the bitmask: coarse passes give exactly the exact path's bits (which the
  parity tests pin to the oracle) -- 1..64 frames, partial passes, overlap on and
  off, z-slab handles, the host-buffer path, and the test mode in which every
  voxel-frame goes through the exact fix-up;
* against the oracle directly (bits within the BASELINE.json ambiguity band)."""
import os

import numpy as np
import pytest

import oracle
from synth.scene import Grid, make_frames, make_scene
from tests.helpers import assert_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

NTHREADS = max(1, len(os.sched_getaffinity(0)))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1311_6811_b200 import build
    build.build()


def _rec(scene, params=None, mode=1, **kw):
    from paper_1311_6811_b200 import from_scene
    rec = from_scene(scene, params or {}, **kw)
    rec.set_coarse(mode, 64, 1)  # coarse passes for every bits-only call
    return rec


def _bits(rec, frames, nf):
    _, B = rec.alloc_outputs(nf, logodds=False)
    rec.reconstruct_batch(frames, nf, bits=B)
    torch.cuda.synchronize()
    return B


# ------------------------------------------------------------------ the bracket

def _adversarial_scene():
    s = make_scene("C1")
    rng = np.random.default_rng(5)
    mu, sg = s.mu.copy(), s.sigma.copy()
    fr = make_frames(s, 0)
    mu[:, ::2, ::2] = np.round(mu[:, ::2, ::2])
    fr[:, ::2, ::2] = mu[:, ::2, ::2].astype(np.uint8)             # I = mu exactly
    sg[:, ::4, :] = rng.uniform(0.1, 1.0, size=sg[:, ::4, :].shape)  # below the floor
    fr[:, 1::4, :] = np.where(mu[:, 1::4, :] < 128, 255, 0)        # far tail
    fr[:, 2::4, 1::2] = np.clip(mu[:, 2::4, 1::2] + rng.integers(-12, 13, fr[:, 2::4, 1::2].shape),
                                0, 255).astype(np.uint8)          # |I - mu| of a few sigma
    s.mu, s.sigma = mu.astype(np.float32), sg.astype(np.float32)
    return s, fr


@pytest.mark.parametrize("params", [dict(), dict(occlusion_prior=0.3), dict(occlusion_prior=0.02),
                                    dict(occlusion_prior=0.97, sigma_floor=2.0),
                                    dict(sigma_floor=0.25)])
@pytest.mark.parametrize("which", ["C2", "adversarial"])
def test_codes_bracket_exact_terms(params, which):
    from paper_1311_6811_b200 import psfs
    if which == "C2":
        s = make_scene("C2")
        fr = make_frames(s, 3)
    else:
        s, fr = _adversarial_scene()
    rec = _rec(s, params)
    plan = psfs.coarse_plan(params, s.ncam)
    f = torch.from_numpy(fr).cuda()
    q = rec.debug_terms(f).cpu().numpy().astype(np.int64)
    c = rec.debug_codes(f).cpu().numpy().astype(np.int64) - plan["bias"]
    lo = c << plan["sh"]
    assert (q >= lo).all(), int((lo - q).max())
    assert (q <= lo + plan["wc"]).all(), int((q - lo - plan["wc"]).max())
    assert 0 < c.min() + plan["bias"] and c.max() + plan["bias"] < 255  # no clamping


# ------------------------------------------------------------------ bits == exact path

@pytest.mark.parametrize("nf", [1, 5, 32, 37, 64])
@pytest.mark.parametrize("overlap", [True, False])
def test_c2_bits_identical_to_exact_path(nf, overlap):
    s = make_scene("C2")
    frames = torch.from_numpy(np.stack([make_frames(s, f % 24) for f in range(nf)])).cuda()
    a = _rec(s, mode=1)
    a.set_overlap(overlap, 0)
    assert a.coarse_status()[0]
    Ba = _bits(a, frames, nf)
    assert a.last_launch_count == 3 * ((nf + 63) // 64)  # k_likelihood_c8p, k_voxel_c8(w), k_fixup_c8
    b = _rec(s, mode=0)
    Bb = _bits(b, frames, nf)
    assert torch.equal(Ba, Bb)
    assert int(Ba.ne(0).sum()) > 0
    if nf < 16:  # the default policy: calls below 16 frames take the exact path
        a.set_coarse(1)
        assert torch.equal(_bits(a, frames, nf), Bb)
        groups = len([g for g in (16, 8, 4, 2, 1) if nf & g])
        # + one k_fill_pads per record-size change on a term buffer (serial: one buffer)
        assert a.last_launch_count == 2 * groups + (0 if overlap else groups - 1)


@pytest.mark.parametrize("params", [dict(), dict(occlusion_prior=0.3, voxel_prior=0.2, threshold=0.7),
                                    dict(occlusion_prior=0.05, threshold=0.3)])
@pytest.mark.parametrize("capacity", [0, 1000])
@pytest.mark.parametrize("nf", [11, 40])
def test_fixup_everywhere_equals_exact_path(params, capacity, nf):
    """Test mode 2 sends every voxel-frame through the exact fix-up: listed and
    summed by k_fixup_c8 (capacity 2^20), or, past a 1000-entry list, summed in
    place by k_voxel_c8 (coarse_exact_sum).  The result must still be the exact
    path's bitmask."""
    s = make_scene("C1")
    frames = torch.from_numpy(np.stack([make_frames(s, f % 13) for f in range(nf)])).cuda()
    a = _rec(s, params, mode=2)
    a.set_coarse(2, 64, 1, capacity)
    a.coarse_status(reset=True)
    Ba = _bits(a, frames, nf)
    _, nfix = a.coarse_status(reset=True)
    assert nfix == nf * s.grid.nvox
    b = _rec(s, params, mode=0)
    assert torch.equal(Ba, _bits(b, frames, nf))


@pytest.mark.parametrize("max_frames", [1, 7, 8, 9, 32, 33, 40, 64])
def test_pass_sizes(max_frames):
    """Narrow (<= 32 frames, k_voxel_c8) and wide (33..64, k_voxel_c8w) passes,
    partial quarters, balanced splits of 70 frames."""
    s = make_scene("C1")
    nf = 70
    frames = torch.from_numpy(np.stack([make_frames(s, f) for f in range(nf)])).cuda()
    a = _rec(s)
    a.set_coarse(1, max_frames, 1)
    b = _rec(s, mode=0)
    assert torch.equal(_bits(a, frames, nf), _bits(b, frames, nf))


def test_fixups_are_rare_on_c2():
    s = make_scene("C2")
    nf = 32
    frames = torch.from_numpy(np.stack([make_frames(s, f) for f in range(nf)])).cuda()
    a = _rec(s)
    a.coarse_status(reset=True)
    _bits(a, frames, nf)
    _, nfix = a.coarse_status(reset=True)
    assert nfix < 1e-3 * nf * s.grid.nvox


@pytest.mark.parametrize("world", [2, 4])
def test_zslab_handles(world):
    s = make_scene("C2")
    nf = 9
    frames = torch.from_numpy(np.stack([make_frames(s, f) for f in range(nf)])).cuda()
    full = _bits(_rec(s, mode=0), frames, nf)
    plane = s.grid.xlen * s.grid.ylen
    out = torch.zeros_like(full)
    for r in range(world):
        rec = _rec(s, rank=r, world=world)
        assert rec.coarse_status()[0]
        B = _bits(rec, frames, nf)
        w0, w1 = plane * rec.k0 // 32, plane * rec.k1 // 32
        out[:, w0:w1] = B[:, w0:w1]
    assert torch.equal(out, full)
    # the assembled slabs against the oracle, every frame
    Bh = out.cpu().numpy().view(np.uint32)
    for f in range(nf):
        orc = oracle.scene_reconstruct(s, make_frames(s, f), nthreads=NTHREADS)
        assert_parity(None, Bh[f], orc, s.grid.nvox)


@pytest.mark.parametrize("dims,coarse", [((37, 29, 23), False), ((64, 29, 23), True),
                                         ((32, 8, 5), True)])
def test_ragged_grids(dims, coarse):
    """xlen % 32 != 0: coarse passes do not apply (bits-only calls stay exact);
    ylen % 8 != 0 and zlen % kz != 0 with xlen % 32 == 0 take coarse passes."""
    g = Grid((-1000.0, -1000.0, 0.0), 2000.0 / dims[0], *dims)
    s = make_scene("C1", grid=g, W=66, H=50)
    nf = 35
    frames = torch.from_numpy(np.stack([make_frames(s, f % 7) for f in range(nf)])).cuda()
    a = _rec(s)
    assert a.coarse_status()[0] == coarse
    b = _rec(s, mode=0)
    assert torch.equal(_bits(a, frames, nf), _bits(b, frames, nf))


@pytest.mark.parametrize("upload", [1, 0])
@pytest.mark.parametrize("pinned", [True, False])
def test_host_path_coarse(upload, pinned):
    """psfs_reconstruct_host, coarse passes: zero-copy upload kernel (mapped pinned
    frames) or DMA 2-D copies (mode 0, or pageable frames: the kernel path must
    refuse them), bits identical to the device path."""
    s = make_scene("C2")
    nf = 80
    frames = np.stack([make_frames(s, f % 16) for f in range(nf)])
    a = _rec(s)
    a.set_host_upload(upload)
    hf = torch.from_numpy(frames)
    if pinned:
        hf = hf.pin_memory()
    Bh = torch.zeros((nf, s.grid.nwords), dtype=torch.int32).pin_memory()
    a.reconstruct_host(hf, nf, None, Bh)
    torch.cuda.synchronize()
    passes = (nf + 63) // 64  # 3 kernels per pass (+ 1 upload kernel each on the zero-copy path)
    assert a.last_launch_count in (3 * passes, 4 * passes)
    kernel_used = a.last_launch_count == 4 * passes
    assert kernel_used == (upload == 1 and pinned)
    b = _rec(s, mode=0)
    assert torch.equal(Bh.cuda(), _bits(b, torch.from_numpy(frames).cuda(), nf))


# ------------------------------------------------------------------ against the oracle

@pytest.mark.parametrize("name,params", [("C1", dict()), ("C2", dict()),
                                         ("C1", dict(occlusion_prior=0.3, voxel_prior=0.2,
                                                     threshold=0.7))])
def test_coarse_bits_vs_oracle(name, params):
    s = make_scene(name)
    nf = 3
    frames = [make_frames(s, f) for f in range(nf)]
    a = _rec(s, params)
    B = _bits(a, torch.from_numpy(np.stack(frames)).cuda(), nf).cpu().numpy().view(np.uint32)
    for f in range(nf):
        orc = oracle.scene_reconstruct(s, frames[f], nthreads=NTHREADS,
                                       p_occ=params.get("occlusion_prior", 0.5),
                                       p_vox=params.get("voxel_prior", 0.5),
                                       tau=params.get("threshold", 0.5))
        st = assert_parity(None, B[f], orc, s.grid.nvox, tau=params.get("threshold", 0.5))
        assert st["occupied"] > 0


@pytest.mark.parametrize("name,nf", [("C4", 40)])
def test_full_size_wide_pass_vs_oracle(name, nf):
    """C4 (512^3, 16 cameras at 1920x1080) in one wide coarse pass (k_voxel_c8w with
    NCAM = 16): 2 distinct frame sets repeated; both checked against the oracle on a
    voxel sample (every 64th slice x 4096 voxels + 65536 random voxels), every
    repeat bit-identical to its original, and the whole bitmask equal to the exact
    int32 path's."""
    s = make_scene(name)
    two = [make_frames(s, 0), make_frames(s, 1)]
    fr = torch.from_numpy(np.stack(two)).cuda().repeat(nf // 2, 1, 1, 1, 1)
    a = _rec(s)
    a.coarse_status(reset=True)
    Ba = _bits(a, fr, nf)
    assert a.last_launch_count == 3
    _, nfix = a.coarse_status(reset=True)
    for f in range(2, nf):
        assert torch.equal(Ba[f], Ba[f % 2])
    rng = np.random.default_rng(13)
    plane = s.grid.xlen * s.grid.ylen
    vox = np.unique(np.concatenate([np.concatenate([k * plane + rng.integers(0, plane, 4096)
                                                    for k in range(0, s.grid.zlen, 64)]),
                                    rng.integers(0, s.grid.nvox, 1 << 16)]))
    vt = torch.from_numpy(vox).cuda()
    for f in range(2):
        _, post = oracle.fuse_sample(s.P, s.widths, s.heights, s.grid, two[f], s.mu, s.sigma, vox,
                                     nthreads=NTHREADS)
        words = Ba[f][(vt >> 5)].cpu().numpy().view(np.uint32)
        bits = ((words >> (vox & 31).astype(np.uint32)) & 1).astype(bool)
        assert not ((bits != (post > 0.5)) & ~(np.abs(post - 0.5) < 1e-4)).any()
        assert bits.sum() > 0
    b = _rec(s, mode=0)
    Bb = _bits(b, fr[:2].contiguous(), 2)
    assert torch.equal(Ba[:2], Bb)
    assert 0 < nfix < 1e-3 * nf * s.grid.nvox


# ------------------------------------------------------------------ frame addressing

@pytest.mark.parametrize("coarse_mode", [1, 0])
def test_strided_and_table_frame_pointers_agree(coarse_mode):
    """Stage 1 computes per-frame image addresses by arithmetic when the call's
    frame pointers are uniformly strided (one [frame][camera] tensor), and loads
    them from the pointer table otherwise (separately allocated images).  Both
    must give the same bitmask -- coarse passes (k_likelihood_c8p) and the exact
    path (k_likelihood_x4p) -- and the oracle's bits."""
    s = make_scene("C1")
    nf = 24
    frames = np.stack([make_frames(s, f % 7) for f in range(nf)])
    strided = torch.from_numpy(frames).cuda()
    table = [[torch.from_numpy(frames[f, c].copy()).cuda() for c in range(s.ncam)] for f in range(nf)]
    rec = _rec(s, mode=coarse_mode)
    Ba = _bits(rec, strided, nf)
    Bb = _bits(rec, table, nf)
    assert torch.equal(Ba, Bb)
    o = oracle.scene_reconstruct(s, frames[5], nthreads=NTHREADS)
    assert_parity(None, Ba[5].cpu().numpy().view(np.uint32), o, s.grid.nvox)
