"""The seeded input generator (synth/) -- determinism and geometry checks.
It holds none of the method's arithmetic; these tests pin the scene recipe."""
import math

import numpy as np
import pytest

from synth.scene import (ellipsoid_part, look_at_camera, make_frames, make_scene, render_labels,
                         ring_rig)


def test_same_seed_same_bytes():
    a = make_scene("C1")
    b = make_scene("C1")
    assert np.array_equal(a.mu, b.mu) and np.array_equal(a.sigma, b.sigma)
    assert np.array_equal(make_frames(a, 3), make_frames(b, 3))
    assert not np.array_equal(make_frames(a, 3), make_frames(a, 4))


def test_ring_azimuths():
    """n = 4 -> cameras at azimuths 0, 90, 180, 270 degrees."""
    cams = ring_rig([(4, 1000.0, 0.0)], 64, 48, radius=3000.0)
    az = [math.degrees(math.atan2(c.center[1], c.center[0])) % 360 for c in cams]
    assert az == pytest.approx([0, 90, 180, 270], abs=1e-9)


def test_projected_sphere_area():
    """a sphere of radius r at distance d images to a disk of
    radius f r / sqrt(d^2 - r^2); rasterised area within 2%."""
    W, H = 640, 480
    cam = look_at_camera((4000.0, 0.0, 1000.0), (0, 0, 1000.0), W, H)
    r, d = 300.0, 4000.0
    lab = render_labels(cam, [ellipsoid_part((0, 0, 1000.0), (r, r, r))])
    f = cam.K[0, 0]
    rad = f * r / math.sqrt(d * d - r * r)
    assert (lab >= 0).sum() == pytest.approx(math.pi * rad * rad, rel=0.02)


def test_background_ranges():
    s = make_scene("C1")
    assert s.mu.min() >= 20 and s.mu.max() <= 235
    assert s.sigma.min() >= 2 and s.sigma.max() <= 8
    assert s.mu.dtype == np.float32 and s.sigma.dtype == np.float32
