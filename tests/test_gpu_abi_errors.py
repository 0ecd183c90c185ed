"""Error behaviour of the C ABI (include/psfs.h) on a GPU: every documented
status code is returned for the documented misuse, nothing aborts."""
import numpy as np
import pytest

from synth.scene import make_frames, make_scene

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1311_6811_b200 import build
    build.build()


def _rec(scene):
    from paper_1311_6811_b200 import Reconstructor
    return Reconstructor(scene.grid)


def test_error_codes():
    from paper_1311_6811_b200.psfs import PsfsError
    s = make_scene("C1")
    fr = torch.from_numpy(make_frames(s, 0)).cuda()
    r = _rec(s)
    # ESTATE: background before cameras, reconstruct before cameras
    with pytest.raises(PsfsError) as e:
        r.set_background(0, s.mu[0], s.sigma[0])
    assert e.value.code == 5
    # EDEGENERATE: singular 3x3 block; W <= 0
    P = s.P.copy()
    P[1, :, 2] = 0.0
    P[1, :, 1] = 0.0
    with pytest.raises(PsfsError) as e:
        r.set_cameras(P, s.widths, s.heights)
    assert e.value.code == 2
    with pytest.raises(PsfsError) as e:
        r.set_cameras(s.P, [64, 64, 0, 64], s.heights)
    assert e.value.code == 2
    # EINVAL: non-finite matrix
    P = s.P.copy()
    P[0, 0, 0] = np.nan
    with pytest.raises(PsfsError) as e:
        r.set_cameras(P, s.widths, s.heights)
    assert e.value.code == 1
    # ELIMIT: more than 64 cameras
    with pytest.raises(PsfsError) as e:
        r.set_cameras(np.repeat(s.P[:1], 65, 0), [64] * 65, [48] * 65)
    assert e.value.code == 8
    r.set_cameras(s.P, s.widths, s.heights)
    # EDIM: background size differs from the camera
    with pytest.raises(PsfsError) as e:
        r.set_background(0, s.mu[0][:, :32], s.sigma[0][:, :32])
    assert e.value.code == 3
    # ECOUNT: reconstruct while some camera has no background
    L, B = r.alloc_outputs(1)
    with pytest.raises(PsfsError) as e:
        r.reconstruct(fr, logodds=L, bits=B)
    assert e.value.code == 4
    for c in range(s.ncam):
        r.set_background(c, s.mu[c], s.sigma[c])
    # EINVAL: both outputs NULL; non-finite background
    with pytest.raises(PsfsError) as e:
        r.reconstruct(fr)
    assert e.value.code == 1
    bad = s.sigma[0].copy()
    bad[0, 0, 0] = np.inf
    with pytest.raises(PsfsError) as e:
        r.set_background(0, s.mu[0], bad)
    assert e.value.code == 1
    # and the handle still works after every error
    r.reconstruct(fr, logodds=L, bits=B)
    torch.cuda.synchronize()
    assert torch.isfinite(L).all()


def test_fixed_point_headroom_rejected():
    """ncam * max|t| * 2^20 must fit int32: a tiny sigma floor makes d_max huge."""
    from paper_1311_6811_b200 import Reconstructor
    from paper_1311_6811_b200.psfs import PsfsError
    s = make_scene("C1")
    r = Reconstructor(s.grid, params=dict(sigma_floor=1e-100))
    with pytest.raises(PsfsError) as e:
        r.set_cameras(s.P, s.widths, s.heights)
    assert e.value.code == 1


def test_create_rejects_bad_slab():
    from paper_1311_6811_b200 import Reconstructor
    from paper_1311_6811_b200.psfs import PsfsError
    s = make_scene("C1")
    with pytest.raises(PsfsError):
        Reconstructor(s.grid, world=3, rank=0)   # 32 slices not divisible by 3
