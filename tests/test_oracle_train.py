"""Pins of the oracle's background training (NEXT-3): the SPEC's
worked examples and numpy's mean / population std (ddof = 0) on random
frames (a library routine for the special case without the floor)."""
import numpy as np
import pytest

import oracle


def test_identical_frames_give_floor_sigma():
    """10 identical frames of value 100 -> mean 100, sigma = sigma_floor."""
    fr = [np.full((5, 7, 3), 100, np.uint8)] * 10
    m, s = oracle.train_background(fr, sigma_floor=1.0)
    assert (m == 100.0).all() and (s == 1.0).all()
    m, s = oracle.train_background(fr, sigma_floor=2.5)
    assert (s == 2.5).all()


def test_alternating_frames_population_sigma():
    """frames alternating 90 / 110 -> mean 100, sigma 10 (population)."""
    fr = [np.full((4, 6, 3), 90 if f % 2 == 0 else 110, np.uint8) for f in range(8)]
    m, s = oracle.train_background(fr)
    assert (m == 100.0).all() and (s == 10.0).all()


def test_errors():
    """EmptyInput; frames of differing sizes -> DimensionMismatch."""
    with pytest.raises(ValueError, match="EmptyInput"):
        oracle.train_background([])
    with pytest.raises(ValueError, match="DimensionMismatch"):
        oracle.train_background([np.zeros((4, 4, 3), np.uint8), np.zeros((4, 5, 3), np.uint8)])


@pytest.mark.parametrize("n", [1, 2, 7, 33])
def test_matches_numpy_mean_std(n):
    rng = np.random.default_rng(n)
    base = rng.integers(0, 256, (1, 9, 11, 3))
    fr = np.clip(base + rng.integers(-30, 31, (n, 9, 11, 3)), 0, 255).astype(np.uint8)
    m, s = oracle.train_background(list(fr), sigma_floor=1e-300)
    assert np.allclose(m, fr.astype(np.float64).mean(axis=0), rtol=0, atol=1e-12)
    assert np.allclose(s, np.maximum(fr.astype(np.float64).std(axis=0, ddof=0), 1e-300),
                       rtol=1e-12, atol=1e-12)
    m1, s1 = oracle.train_background(list(fr), sigma_floor=4.0)
    assert np.array_equal(m1, m) and np.array_equal(s1, np.maximum(s, 4.0))
