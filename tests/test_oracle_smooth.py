"""Pins of the oracle's merged probability filtering + thresholding (NEXT-1;
P:111): S:211 (all-ones grid: corner 8/27 ->
unoccupied, interior 1), S:212 (single voxel: max 1/27 -> empty), all-zero
grid, edge / face counts of the zero-padded box, constant and linear fields
(a box average reproduces them in the interior), and permutation of axes."""
import numpy as np
import pytest

import oracle
from synth.scene import Grid


def _g(z, y, x):
    return Grid((0.0, 0.0, 0.0), 1.0, x, y, z)


def test_all_ones():
    z, y, x = 6, 7, 8
    sm, bits = oracle.smooth_threshold(np.ones(z * y * x), _g(z, y, x))
    sm = sm.reshape(z, y, x)
    assert sm[0, 0, 0] == pytest.approx(8 / 27, abs=1e-15)      # corner
    assert sm[0, 0, 3] == pytest.approx(12 / 27, abs=1e-15)     # edge
    assert sm[0, 3, 3] == pytest.approx(18 / 27, abs=1e-15)     # face
    assert sm[3, 3, 3] == pytest.approx(1.0, abs=1e-15)         # interior
    occ = np.unpackbits(bits.view(np.uint8), bitorder="little")[: z * y * x].reshape(z, y, x)
    assert occ[0, 0, 0] == 0 and occ[0, 0, 3] == 0 and occ[0, 3, 3] == 1 and occ[3, 3, 3] == 1


def test_single_voxel_and_zero():
    p = np.zeros(9 * 9 * 9)
    p[4 + 9 * (4 + 9 * 4)] = 1.0
    sm, bits = oracle.smooth_threshold(p, _g(9, 9, 9))
    assert sm.max() == pytest.approx(1 / 27, abs=1e-15)
    assert (sm > 0).sum() == 27 and bits.sum() == 0
    sm, bits = oracle.smooth_threshold(np.zeros(8 * 8 * 8), _g(8, 8, 8))
    assert sm.max() == 0 and bits.sum() == 0


def test_constant_and_linear_fields_in_the_interior():
    z, y, x = 7, 8, 9
    kk, jj, ii = np.meshgrid(np.arange(z), np.arange(y), np.arange(x), indexing="ij")
    for field in (np.full((z, y, x), 0.37), 0.01 * ii + 0.02 * jj + 0.03 * kk):
        sm, _ = oracle.smooth_threshold(field.reshape(-1), _g(z, y, x))
        sm = sm.reshape(z, y, x)
        np.testing.assert_allclose(sm[1:-1, 1:-1, 1:-1], field[1:-1, 1:-1, 1:-1], atol=1e-14)


def test_threshold_is_strict_and_axes_symmetric():
    rng = np.random.default_rng(5)
    p = rng.random((5, 6, 7))
    sm, bits = oracle.smooth_threshold(p.reshape(-1), _g(5, 6, 7), tau=0.5)
    occ = np.unpackbits(bits.view(np.uint8), bitorder="little")[: p.size].astype(bool)
    assert (occ == (sm > 0.5)).all()
    # transposing the volume transposes the result (the box is symmetric)
    pt = np.ascontiguousarray(p.transpose(2, 1, 0))
    smt, _ = oracle.smooth_threshold(pt.reshape(-1), _g(7, 6, 5))
    np.testing.assert_allclose(smt.reshape(7, 6, 5), sm.reshape(5, 6, 7).transpose(2, 1, 0), atol=1e-15)
