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
