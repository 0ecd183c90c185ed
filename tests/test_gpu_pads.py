"""GPU parity of the out-of-view pad records when one handle's passes change
record size (the pad column / row of the padded term and code
images are the neutral value only for the record size last written).

The grid extends far outside every view, so many voxel-camera pairs read the
pad (t = 0, R#12).  One handle runs a sequence of calls whose
passes use different record sizes -- exact path: 16-frame then 1-frame calls,
7 overlapped frames (4 + 2 + 1 across two term buffers); coarse passes: 20
frames (32-byte records), 40 frames (64-byte), 65 frames (33 + 32, both sizes
across two code buffers), then 20 again -- and every frame is checked against
the oracle."""
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


def _scene():
    # 32^3 voxels over a 12 m cube around the 2 m capture volume: most voxels
    # project outside some (or every) view
    g = Grid((-6000.0, -6000.0, -3000.0), 12000.0 / 32, 32, 32, 32)
    return make_scene("C1", grid=g)


def _oracle_cache(s, n):
    frames = [make_frames(s, f % 8) for f in range(n)]
    orcs = [oracle.scene_reconstruct(s, frames[f], nthreads=NTHREADS) for f in range(8)]
    return frames, orcs


def test_pad_scene_reads_pads():
    """The scene really sends voxels out of view (the test below is not vacuous),
    and some of them are in view of other cameras."""
    s = _scene()
    fr = make_frames(s, 0)
    orc = oracle.scene_reconstruct(s, fr, nthreads=NTHREADS)
    unseen = np.abs(orc["L"]) < 1e-12
    assert unseen.sum() > 1000 and (~unseen).sum() > 1000


def test_exact_path_record_size_changes():
    from paper_1311_6811_b200 import from_scene
    s = _scene()
    frames, orcs = _oracle_cache(s, 16)
    rec = from_scene(s)
    rec.set_overlap(True, 0)
    for n in (16, 1, 7, 2, 16, 3):
        fr = torch.from_numpy(np.stack(frames[:n])).cuda()
        L, B = rec.alloc_outputs(n)
        rec.reconstruct_batch(fr, n, logodds=L, bits=B)
        torch.cuda.synchronize()
        Lh, Bh = L.cpu().numpy(), B.cpu().numpy().view(np.uint32)
        for f in range(n):
            assert_parity(Lh[f], Bh[f], orcs[f % 8], s.grid.nvox)


@pytest.mark.parametrize("overlap", [True, False])
def test_coarse_record_size_changes(overlap):
    from paper_1311_6811_b200 import from_scene
    s = _scene()
    frames, orcs = _oracle_cache(s, 65)
    rec = from_scene(s)
    rec.set_overlap(overlap, 0)
    for n in (20, 40, 65, 20, 1, 33):
        fr = torch.from_numpy(np.stack(frames[:n])).cuda()
        _, B = rec.alloc_outputs(n, logodds=False)
        rec.reconstruct_batch(fr, n, bits=B)
        torch.cuda.synchronize()
        if n >= 16:
            assert rec.coarse_status()[0], f"{n} frames did not take the coarse passes"
        Bh = B.cpu().numpy().view(np.uint32)
        for f in range(n):
            assert_parity(None, Bh[f], orcs[f % 8], s.grid.nvox)


def test_exact_then_coarse_then_exact():
    """The two buffer kinds are separate; alternating kinds on one handle keeps
    both correct."""
    from paper_1311_6811_b200 import from_scene
    s = _scene()
    frames, orcs = _oracle_cache(s, 40)
    rec = from_scene(s)
    for n, lo in ((16, True), (40, False), (1, True), (17, False), (4, True)):
        fr = torch.from_numpy(np.stack(frames[:n])).cuda()
        L, B = rec.alloc_outputs(n, logodds=lo)
        rec.reconstruct_batch(fr, n, logodds=L, bits=B)
        torch.cuda.synchronize()
        Lh = L.cpu().numpy() if lo else None
        Bh = B.cpu().numpy().view(np.uint32)
        for f in range(n):
            assert_parity(None if Lh is None else Lh[f], Bh[f], orcs[f % 8], s.grid.nvox)
