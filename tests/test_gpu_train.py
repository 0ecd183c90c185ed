"""GPU parity of the background training (NEXT-3, psfs_train_background) against
the oracle (oracle.train_background): mean and sigma agree to float rounding;
the SPEC's examples hold exactly; an installed model gives the
same reconstruction as uploading the same values with psfs_set_background."""
import numpy as np
import pytest

import oracle
from synth.scene import make_frames, make_scene

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1311_6811_b200 import build
    build.build()


def _rec(scene="C1"):
    from paper_1311_6811_b200 import from_scene
    s = make_scene(scene)
    return s, from_scene(s)


@pytest.mark.parametrize("n,misaligned", [(1, False), (7, False), (8, True), (33, False),
                                         (33, True)])
def test_mean_sigma_parity(n, misaligned):
    """misaligned: frames at an odd address (the byte-load kernel variant)."""
    s, rec = _rec()
    rng = np.random.default_rng(n)
    H, W = int(s.heights[1]), int(s.widths[1])
    base = rng.integers(0, 256, (1, H, W, 3))
    fr = np.clip(base + rng.integers(-40, 41, (n, H, W, 3)), 0, 255).astype(np.uint8)
    t = torch.from_numpy(fr).cuda()
    if misaligned:
        raw = torch.empty(t.numel() + 1, dtype=torch.uint8, device="cuda")
        raw[1:].copy_(t.view(-1))
        t = raw[1:].view(t.shape)
        assert t.data_ptr() % 4 == 1
    m, sg = rec.train_background(1, t, install=False)
    torch.cuda.synchronize()
    mo, so = oracle.train_background(list(fr), sigma_floor=1.0)
    assert np.allclose(m.cpu().numpy(), mo, rtol=1e-6, atol=0)
    assert np.allclose(sg.cpu().numpy(), so, rtol=1e-6, atol=0)


def test_spec_examples():
    """S:105 identical frames -> sigma = floor; S:106 alternating 90/110 -> 100, 10."""
    s, rec = _rec()
    H, W = int(s.heights[0]), int(s.widths[0])
    same = torch.full((10, H, W, 3), 100, dtype=torch.uint8, device="cuda")
    m, sg = rec.train_background(0, same, install=False)
    alt = torch.stack([torch.full((H, W, 3), 90 if f % 2 == 0 else 110, dtype=torch.uint8,
                                  device="cuda") for f in range(8)])
    m2, sg2 = rec.train_background(0, alt, install=False)
    torch.cuda.synchronize()
    assert (m == 100).all() and (sg == 1.0).all() and (m2 == 100).all() and (sg2 == 10).all()


def test_installed_model_equals_uploaded_model():
    """Train every camera on background-only frames, install on the device, and
    reconstruct a noisy frame: bit-identical to a handle whose backgrounds were
    set from the same float values through psfs_set_background."""
    from paper_1311_6811_b200 import Reconstructor
    s = make_scene("C1")
    a = Reconstructor(s.grid)
    b = Reconstructor(s.grid)
    for r in (a, b):
        r.set_cameras(s.P, s.widths, s.heights)
    bg = np.stack([make_frames(s, f, mode="background") for f in range(12)])  # [n, ncam, H, W, 3]
    for c in range(s.ncam):
        m, sg = a.train_background(c, torch.from_numpy(np.ascontiguousarray(bg[:, c])).cuda())
        torch.cuda.synchronize()
        b.set_background(c, m.cpu().numpy(), sg.cpu().numpy())
    fr = torch.from_numpy(make_frames(s, 0)).cuda()
    La, Ba = a.alloc_outputs(1)
    Lb, Bb = b.alloc_outputs(1)
    a.reconstruct(fr, logodds=La, bits=Ba)
    b.reconstruct(fr, logodds=Lb, bits=Bb)
    torch.cuda.synchronize()
    assert torch.equal(La, Lb) and torch.equal(Ba, Bb)
    assert int(Ba.ne(0).sum()) > 0
