"""GPU parity of the surface extraction (NEXT-2, psfs_surface) against the
oracle: bit-exact index lists (integer work), on random volumes of ragged
shapes, on a real reconstruction, per z-slab, and with a short output buffer."""
import numpy as np
import pytest

import oracle
from synth.scene import Grid, make_frames, make_scene
from tests.test_oracle_surface import _bits_of

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1311_6811_b200 import build
    build.build()


def _gpu_surface(grid, words, rank=0, world=1, capacity=None):
    from paper_1311_6811_b200 import Reconstructor
    r = Reconstructor(grid, rank=rank, world=world)
    b = torch.from_numpy(np.asarray(words).view(np.int32).copy()).cuda()
    cap = (grid.xlen * grid.ylen * grid.zlen) if capacity is None else capacity
    idx = torch.full((max(cap, 1),), -1, dtype=torch.int64, device="cuda")
    sb = torch.zeros_like(b)
    cnt, _, _ = r.surface(b, surface_bits=sb, indices=idx)
    torch.cuda.synchronize()
    return int(cnt.item()), idx.cpu().numpy(), sb.cpu().numpy().view(np.uint32), r


@pytest.mark.parametrize("shape,p", [((32, 32, 32), 0.6), ((23, 29, 37), 0.7), ((9, 17, 64), 0.9),
                                     ((5, 3, 33), 0.5), ((40, 40, 96), 0.97)])
def test_random_volumes(shape, p):
    rng = np.random.default_rng(sum(shape))
    occ = rng.random(shape) < p
    z, y, x = shape
    g = Grid((0.0, 0.0, 0.0), 1.0, x, y, z)
    words = _bits_of(occ)
    ref = oracle.surface(words, g)
    n, idx, sb, _ = _gpu_surface(g, words)
    assert n == len(ref)
    np.testing.assert_array_equal(idx[:n], ref)
    surf = np.zeros(occ.size, bool)
    surf[ref] = True
    np.testing.assert_array_equal(sb, _bits_of(surf.reshape(shape)))


def test_surface_of_reconstruction_and_slabs():
    s = make_scene("C2")
    from tests.helpers import gpu_run
    out = gpu_run(s, [make_frames(s, 0)], logodds=False)
    words = out["bits"][0]
    ref = oracle.surface(words, s.grid)
    assert len(ref) > 1000
    n, idx, _, _ = _gpu_surface(s.grid, words)
    np.testing.assert_array_equal(idx[:n], ref)
    parts = []
    for r in range(4):
        n, idx, _, rec = _gpu_surface(s.grid, words, rank=r, world=4)
        parts.append(idx[:n])
        plane = s.grid.xlen * s.grid.ylen
        assert ((idx[:n] >= rec.k0 * plane) & (idx[:n] < rec.k1 * plane)).all()
    np.testing.assert_array_equal(np.concatenate(parts), ref)


def test_short_output_buffer_keeps_exact_count():
    rng = np.random.default_rng(0)
    occ = rng.random((16, 16, 32)) < 0.5
    g = Grid((0.0, 0.0, 0.0), 1.0, 32, 16, 16)
    words = _bits_of(occ)
    ref = oracle.surface(words, g)
    n, idx, _, _ = _gpu_surface(g, words, capacity=100)
    assert n == len(ref)
    np.testing.assert_array_equal(idx[:100], ref[:100])
