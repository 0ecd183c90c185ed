"""Pins of the oracle's surface extraction (NEXT-2):
closed-form counts for solid blocks (n^3 - (n-2)^3), S:220 (3^3 block -> 26),
S:221 (single voxel -> 1), S:222 (5^3 block -> 98), structures whose every
occupied voxel is surface (checkerboard, 1-voxel planes), the volume boundary
rule, and slab evaluation."""
import numpy as np
import pytest

import oracle
from synth.scene import Grid


def _bits_of(occ):
    """occ: bool [z, y, x] -> uint32 words, bit v = i + X (j + Y k), LSB first."""
    flat = np.ascontiguousarray(occ.reshape(-1)).astype(np.uint8)
    pad = (-flat.size) % 32
    flat = np.concatenate([flat, np.zeros(pad, np.uint8)])
    return np.packbits(flat, bitorder="little").view(np.uint32)


def _grid(shape):
    z, y, x = shape
    return Grid((0.0, 0.0, 0.0), 1.0, x, y, z)


@pytest.mark.parametrize("n,expect", [(1, 1), (2, 8), (3, 26), (4, 56), (5, 98), (7, 218)])
def test_solid_blocks(n, expect):
    occ = np.zeros((12, 11, 13), bool)
    occ[3:3 + n, 2:2 + n, 4:4 + n] = True
    s = oracle.surface(_bits_of(occ), _grid(occ.shape))
    assert len(s) == expect == n ** 3 - max(n - 2, 0) ** 3
    assert (np.diff(s) > 0).all()


def test_full_volume_boundary_counts_as_outside():
    """a completely occupied volume keeps exactly its boundary layer."""
    occ = np.ones((6, 7, 8), bool)
    assert len(oracle.surface(_bits_of(occ), _grid(occ.shape))) == 6 * 7 * 8 - 4 * 5 * 6


def test_checkerboard_and_planes_are_all_surface():
    z, y, x = np.meshgrid(np.arange(9), np.arange(10), np.arange(11), indexing="ij")
    occ = ((x + y + z) % 2 == 0)
    s = oracle.surface(_bits_of(occ), _grid(occ.shape))
    assert len(s) == occ.sum()
    plane = np.zeros((9, 10, 11), bool)
    plane[4] = True
    assert len(oracle.surface(_bits_of(plane), _grid(plane.shape))) == 110


def test_hollow_shell_removes_only_interior():
    occ = np.zeros((10, 10, 10), bool)
    occ[1:9, 1:9, 1:9] = True         # 8^3 solid
    n_inner = 6 ** 3
    s = oracle.surface(_bits_of(occ), _grid(occ.shape))
    assert len(s) == 8 ** 3 - n_inner
    # the surface of the surface (a closed shell of thickness 1) is itself
    shell = np.zeros(1000, bool)
    shell[s] = True
    assert len(oracle.surface(_bits_of(shell.reshape(10, 10, 10)), _grid((10, 10, 10)))) == len(s)


def test_slab_is_slice_of_full():
    rng = np.random.default_rng(3)
    occ = rng.random((16, 9, 32)) < 0.7
    g = _grid(occ.shape)
    full = oracle.surface(_bits_of(occ), g)
    plane = 9 * 32
    part = oracle.surface(_bits_of(occ), g, 4, 12)
    np.testing.assert_array_equal(part, full[(full >= 4 * plane) & (full < 12 * plane)])
