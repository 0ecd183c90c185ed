"""GPU parity of the merged filtering + thresholding (NEXT-1,
psfs_smooth_threshold) against the oracle: smoothed posterior within 1e-5,
bits exact except where the oracle's smoothed value is within 1e-4 of tau."""
import math

import numpy as np
import pytest

import oracle
from synth.scene import Grid, make_frames, make_scene
from tests.helpers import unpack_bits

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1311_6811_b200 import build
    build.build()


def _gpu_smooth(rec, L):
    Lt = torch.from_numpy(np.ascontiguousarray(L, np.float32)).cuda()
    sm = torch.empty_like(Lt)
    bits = torch.zeros((Lt.numel() + 31) // 32, dtype=torch.int32, device="cuda")
    rec.smooth_threshold(Lt, smoothed=sm, bits=bits)
    torch.cuda.synchronize()
    return sm.cpu().numpy().astype(np.float64), bits.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("name,grid", [("C1", None), ("C2", None),
                                       ("C1", Grid((-1000.0, -1000.0, 0.0), 2000.0 / 37, 37, 29, 23))])
def test_smooth_from_reconstruction(name, grid):
    from paper_1311_6811_b200 import from_scene
    s = make_scene(name, grid=grid)
    fr = make_frames(s, 0)
    rec = from_scene(s)
    L, B = rec.alloc_outputs(1)
    rec.reconstruct(torch.from_numpy(fr).cuda(), logodds=L, bits=B)
    torch.cuda.synchronize()
    sm_g, bits_g = _gpu_smooth(rec, L[0].cpu().numpy())
    orc = oracle.scene_reconstruct(s, fr)
    sm_o, bits_o = oracle.smooth_threshold(orc["post"], s.grid, 0.5)
    assert np.abs(sm_g - sm_o).max() <= 1e-5
    n = s.grid.nvox
    mism = unpack_bits(bits_g, n) != unpack_bits(bits_o, n)
    assert not (mism & ~(np.abs(sm_o - 0.5) < 1e-4)).any()
    assert unpack_bits(bits_o, n).sum() > 0


def test_smooth_handset_all_ones():
    from paper_1311_6811_b200 import Reconstructor
    g = Grid((0.0, 0.0, 0.0), 1.0, 32, 8, 6)
    rec = Reconstructor(g)
    sm, bits = _gpu_smooth(rec, np.full(g.nvox, 40.0))
    sm = sm.reshape(6, 8, 32)
    assert sm[0, 0, 0] == pytest.approx(8 / 27, abs=1e-6)
    assert sm[3, 3, 3] == pytest.approx(1.0, abs=1e-6)
    occ = unpack_bits(bits, g.nvox).reshape(6, 8, 32)
    assert occ[0, 0, 0] == 0 and occ[0, 3, 3] == 1 and occ.sum() == (sm > 0.5).sum()


# ------------------------------------------------------------------ merged with reconstruction

def _oracle_smooth(s, fr):
    orc = oracle.scene_reconstruct(s, fr)
    return oracle.smooth_threshold(orc["post"], s.grid, 0.5)


def _check_smooth(s, sm_g, bits_g, sm_o, bits_o, word0=0):
    n = sm_o.size
    assert np.abs(sm_g.astype(np.float64) - sm_o).max() <= 1e-5
    mism = unpack_bits(np.asarray(bits_g)[word0:], n) != unpack_bits(bits_o, n)
    assert not (mism & ~(np.abs(sm_o - 0.5) < 1e-4)).any()


@pytest.mark.parametrize("name,grid,nf", [("C1", None, 3), ("C2", None, 2), ("C1", None, 17),
                                          ("C1", Grid((-1000.0, -1000.0, 0.0), 2000.0 / 37, 37, 29, 23), 2)])
def test_reconstruct_smoothed_from_sums(name, grid, nf):
    """psfs_reconstruct_smoothed (exact int32 sums -> k_box_sums, no float volume
    in between) against the oracle's box filter of its own posterior, frame by
    frame, and equal to the two-call form (psfs_reconstruct_sums +
    psfs_smooth_sums)."""
    from paper_1311_6811_b200 import from_scene
    s = make_scene(name, grid=grid)
    frames = [make_frames(s, f % 7) for f in range(nf)]
    fr = torch.from_numpy(np.stack(frames)).cuda()
    rec = from_scene(s)
    sm = torch.empty((nf, s.grid.nvox), dtype=torch.float32, device="cuda")
    bits = torch.zeros((nf, s.grid.nwords), dtype=torch.int32, device="cuda")
    rec.reconstruct_smoothed(fr, nf, smoothed=sm, bits=bits)
    sums = torch.empty((nf, s.grid.nvox), dtype=torch.int32, device="cuda")
    rec.reconstruct_sums(fr, nf, sums)
    sm2 = torch.empty_like(sm)
    bits2 = torch.zeros_like(bits)
    rec.smooth_sums(nf, sums, smoothed=sm2, bits=bits2)
    torch.cuda.synchronize()
    assert torch.equal(sm, sm2) and torch.equal(bits, bits2)
    smh, bh = sm.cpu().numpy(), bits.cpu().numpy().view(np.uint32)
    for f in {0, nf - 1}:
        sm_o, bits_o = _oracle_smooth(s, frames[f])
        _check_smooth(s, smh[f], bh[f], sm_o, bits_o)


def test_sums_are_the_log_odds():
    """The sums output is the exact path's S: L = S 2^-20 + logit p_V rounded
    once to float equals psfs_reconstruct's log-odds bit for bit."""
    from paper_1311_6811_b200 import from_scene
    s = make_scene("C1")
    fr = torch.from_numpy(np.stack([make_frames(s, f) for f in range(5)])).cuda()
    rec = from_scene(s, dict(voxel_prior=0.3))
    L, _ = rec.alloc_outputs(5)
    rec.reconstruct_batch(fr, 5, logodds=L)
    sums = torch.empty((5, s.grid.nvox), dtype=torch.int32, device="cuda")
    rec.reconstruct_sums(fr, 5, sums)
    torch.cuda.synchronize()
    Lh = (sums.cpu().numpy().astype(np.float64) / 2 ** 20 + (math.log(0.3) - math.log1p(-0.3))).astype(np.float32)
    assert np.array_equal(Lh, L.cpu().numpy())


@pytest.mark.parametrize("world", [2, 4])
def test_smooth_sums_zslab_handles(world):
    """NEXT-1 on z-slabs (one process): every rank's sums, one-slice halos taken
    from the neighbours' boundary slices, psfs_smooth_sums per rank; the slabs
    together equal the world-1 result bit for bit and meet the oracle."""
    from paper_1311_6811_b200 import PsfsError, from_scene
    s = make_scene("C2")
    frames = [make_frames(s, 0), make_frames(s, 3)]
    fr = torch.from_numpy(np.stack(frames)).cuda()
    nf, g = 2, s.grid
    plane = g.xlen * g.ylen
    full = from_scene(s)
    smf = torch.empty((nf, g.nvox), dtype=torch.float32, device="cuda")
    bf = torch.zeros((nf, g.nwords), dtype=torch.int32, device="cuda")
    full.reconstruct_smoothed(fr, nf, smoothed=smf, bits=bf)
    recs = [from_scene(s, rank=r, world=world) for r in range(world)]
    sums = []
    for r, rec in enumerate(recs):
        t = torch.empty((nf, rec.nslab), dtype=torch.int32, device="cuda")
        rec.reconstruct_sums(fr, nf, t)
        sums.append(t)
    bits = torch.zeros((nf, g.nwords), dtype=torch.int32, device="cuda")
    sm_all = torch.empty((nf, g.nvox), dtype=torch.float32, device="cuda")
    for r, rec in enumerate(recs):
        lo = sums[r - 1][:, -plane:].contiguous() if r > 0 else None
        hi = sums[r + 1][:, :plane].contiguous() if r < world - 1 else None
        if r > 0:
            with pytest.raises(PsfsError):
                rec.smooth_sums(nf, sums[r], None, hi, bits=bits)  # the lower halo is required
        sm = torch.empty((nf, rec.nslab), dtype=torch.float32, device="cuda")
        rec.smooth_sums(nf, sums[r], lo, hi, smoothed=sm, bits=bits)
        sm_all[:, plane * rec.k0: plane * rec.k1] = sm
    torch.cuda.synchronize()
    assert torch.equal(sm_all, smf) and torch.equal(bits, bf)
    smh, bh = sm_all.cpu().numpy(), bits.cpu().numpy().view(np.uint32)
    for f in range(nf):
        sm_o, bits_o = _oracle_smooth(s, frames[f])
        _check_smooth(s, smh[f], bh[f], sm_o, bits_o)
