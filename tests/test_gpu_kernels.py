"""GPU checks of kernel building blocks that parity tests cannot isolate."""
import numpy as np
import pytest

import oracle
from synth.scene import Grid, look_at_camera, make_frames, make_scene, ring_rig
from tests.helpers import assert_parity, gpu_run

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1311_6811_b200 import build
    build.build()


def test_fast_reciprocal_is_ieee_rn_over_planner_range():
    """The planner enables the MUFU+Newton reciprocal only when every in-front w
    lies in [2^-60, 2^60]; over every float of that range it must equal
    __frcp_rn (IEEE RN(1/w)) bit for bit."""
    from paper_1311_6811_b200.psfs import debug_rcp_check
    assert debug_rcp_check(2.0 ** -60, 2.0 ** 60) == 0


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_planner_enables_fast_reciprocal_for_ring_rigs(name):
    from paper_1311_6811_b200 import Reconstructor
    s = make_scene(name) if name in ("C1", "C2") else None
    from synth.scene import CONFIGS, cube_grid
    cfg = CONFIGS[name]
    cams = ring_rig(cfg["rings"], cfg["W"], cfg["H"])
    rec = Reconstructor(cube_grid(cfg["n"]))
    rec.set_cameras(np.stack([c.P for c in cams]), [c.width for c in cams],
                    [c.height for c in cams])
    assert rec.fast_rcp


def test_camera_inside_grid_uses_exact_reciprocal_and_matches_oracle():
    """A camera whose principal plane cuts the grid (w changes sign inside it):
    the planner must fall back to __frcp_rn; parity with the oracle holds,
    including voxels behind that camera."""
    s = make_scene("C1")
    inner = look_at_camera((0.0, -300.0, 1000.0), (0.0, 3000.0, 1000.0), 64, 48)
    s.cameras = s.cameras[:3] + [inner]
    g = gpu_run(s, [make_frames(s, 0)])
    assert not g["rec"].fast_rcp
    orc = oracle.scene_reconstruct(s, make_frames(s, 0))
    assert_parity(g["L"][0], g["bits"][0], orc, s.grid.nvox)


@pytest.mark.parametrize("path", [0, 2, 3, 4, 5, 6])
def test_stage1_paths_bit_identical(path):
    """The three stage-1 kernels (TMA ring with cp.async.bulk + mbarrier, used
    when frames are 16-byte aligned and W % 16 == 0; pipelined persistent; one
    pixel per thread) give bit-identical terms and outputs."""
    from paper_1311_6811_b200 import from_scene
    s = make_scene("C2")
    frames = np.stack([make_frames(s, f) for f in range(8)])
    rec = from_scene(s)
    ref = from_scene(s)
    ref.set_stage1_path(1)
    rec.set_stage1_path(path)
    n = frames.size
    aligned = torch.from_numpy(frames).cuda()
    raw = torch.empty(n + 4, dtype=torch.uint8, device="cuda")
    raw[4:].copy_(aligned.view(-1))
    shifted = raw[4:].view(frames.shape)            # 4-byte misaligned -> generic kernel
    assert shifted.data_ptr() % 16 == 4
    La, Ba = rec.alloc_outputs(8)
    Lb, Bb = rec.alloc_outputs(8)
    Lc, Bc = rec.alloc_outputs(8)
    ref.reconstruct_batch(aligned, 8, logodds=La, bits=Ba)      # TMA ring
    ref.reconstruct_batch(shifted, 8, logodds=Lb, bits=Bb)      # misaligned: path 0
    rec.reconstruct_batch(aligned, 8, logodds=Lc, bits=Bc)
    torch.cuda.synchronize()
    assert torch.equal(Ba, Bb) and torch.equal(La, Lb)
    assert torch.equal(Ba, Bc) and torch.equal(La, Lc)
    for r in (rec, ref):
        assert torch.equal(r.debug_terms(aligned[0]), ref.debug_terms(shifted[0]))


@pytest.mark.parametrize("path,ty,kz", [(0, 1, 1), (4, 1, 4), (0, 1, 16), (0, 4, 1), (4, 4, 3), (5, 1, 4),
                                        (6, 1, 4), (6, 4, 3)])
def test_sixteen_frame_passes_bit_identical(path, ty, kz):
    """16-frame passes (stage 1 as two 8-frame halves, warp-row or one-pixel
    loads; k_voxel16 with lane pairs) equal 8-frame passes bit for bit, for
    several z-depths of the stage-2 tile."""
    from paper_1311_6811_b200 import from_scene
    s = make_scene("C2")
    frames = np.stack([make_frames(s, f) for f in range(16)])
    fr = torch.from_numpy(frames).cuda()
    a = from_scene(s)
    a.set_max_fuse(8)
    b = from_scene(s)
    b.set_max_fuse(16)
    b.set_stage1_path(path)
    b.set_voxel_tile(ty, kz)
    La, Ba = a.alloc_outputs(16)
    Lb, Bb = b.alloc_outputs(16)
    a.reconstruct_batch(fr, 16, logodds=La, bits=Ba)
    b.reconstruct_batch(fr, 16, logodds=Lb, bits=Bb)
    torch.cuda.synchronize()
    assert b.last_launch_count == 2  # one stage-1 and one stage-2 launch
    assert torch.equal(Ba, Bb) and torch.equal(La, Lb)


@pytest.mark.parametrize("ty,kz", [(1, 1), (4, 2), (1, 16)])
def test_voxel_tile_shapes_bit_identical(ty, kz):
    from tests.helpers import gpu_run
    from paper_1311_6811_b200 import from_scene
    s = make_scene("C2")
    frames = np.stack([make_frames(s, f) for f in range(8)])
    a = from_scene(s)
    b = from_scene(s)
    b.set_voxel_tile(ty, kz)
    fr = torch.from_numpy(frames).cuda()
    La, Ba = a.alloc_outputs(8)
    Lb, Bb = b.alloc_outputs(8)
    a.reconstruct_batch(fr, 8, logodds=La, bits=Ba)
    b.reconstruct_batch(fr, 8, logodds=Lb, bits=Bb)
    torch.cuda.synchronize()
    assert torch.equal(Ba, Bb) and torch.equal(La, Lb)


@pytest.mark.parametrize("fuse", [8, 16])
def test_overlapped_batches_bit_identical(fuse):
    """Stage 1 of group g+1 on the auxiliary stream beside stage 2 of group g
    (two term buffers) gives the same bits / log-odds as the serial schedule,
    including mixed group sizes (21 = 8 + 8 + 4 + 1 or 16 + 4 + 1)."""
    from paper_1311_6811_b200 import from_scene
    s = make_scene("C2")
    frames = np.stack([make_frames(s, f % 16) for f in range(21)])
    fr = torch.from_numpy(frames).cuda()
    a = from_scene(s)
    a.set_overlap(False)
    a.set_max_fuse(8)  # the serial reference always runs 8-frame passes
    b = from_scene(s)
    b.set_overlap(True, 2)
    b.set_max_fuse(fuse)
    La, Ba = a.alloc_outputs(21)
    Lb, Bb = b.alloc_outputs(21)
    a.reconstruct_batch(fr, 21, logodds=La, bits=Ba)
    for _ in range(2):  # twice: the second call reuses both term buffers
        b.reconstruct_batch(fr, 21, logodds=Lb, bits=Bb)
    torch.cuda.synchronize()
    assert torch.equal(Ba, Bb) and torch.equal(La, Lb)


@pytest.mark.parametrize("params,nf", [(dict(), 8), (dict(), 16),
                                       (dict(occlusion_prior=0.3, voxel_prior=0.2, threshold=0.7), 16)])
def test_carve_bits_identical(params, nf):
    """psfs_set_carve: the bits-only early exit leaves the bitmask unchanged
    (C2 skeleton frames and C1 with general priors; 8- and 16-frame passes),
    and is ignored when log-odds are requested."""
    from paper_1311_6811_b200 import from_scene
    name = "C2" if not params else "C1"
    s = make_scene(name)
    frames = np.stack([make_frames(s, f) for f in range(nf)])
    fr = torch.from_numpy(frames).cuda()
    a = from_scene(s, params)
    b = from_scene(s, params)
    b.set_carve(True)
    _, Ba = a.alloc_outputs(nf, logodds=False)
    _, Bb = b.alloc_outputs(nf, logodds=False)
    a.reconstruct_batch(fr, nf, bits=Ba)
    b.reconstruct_batch(fr, nf, bits=Bb)
    Lc, Bc = b.alloc_outputs(nf)
    b.reconstruct_batch(fr, nf, logodds=Lc, bits=Bc)
    La, Bd = a.alloc_outputs(nf)
    a.reconstruct_batch(fr, nf, logodds=La, bits=Bd)
    torch.cuda.synchronize()
    assert torch.equal(Ba, Bb)
    assert torch.equal(Bc, Bd) and torch.equal(Lc, La)
