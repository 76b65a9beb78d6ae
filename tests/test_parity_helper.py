"""CPU checks of the GPU tests' comparison (tests/_parity.py, R17) and of the input
recipe's wide-angle option: the element-wise term catches a single outlier the norm bound would
pass, complex inputs compare as (re, im) pairs, and synth.theta(half_range) keeps its range."""
import numpy as np

import synth
from _parity import ELEM_FACTOR, rel


def test_norm_error_alone():
    rng = np.random.default_rng(0)
    b = rng.standard_normal(10000)
    a = b * (1 + 1e-7)
    assert rel(a, b) < 2e-7


def test_single_outlier_is_caught():
    rng = np.random.default_rng(1)
    b = rng.standard_normal(523776)
    a = b.copy()
    a[12345] *= 1.07  # one angle off by 7%: the norm error is ~1e-4, the element error ~7e-2
    nb = np.linalg.norm(b)
    assert np.linalg.norm(a - b) / nb < 2e-4
    assert rel(a, b) > 1e-3


def test_elem_factor_and_zero_reference():
    b = np.zeros(8)
    b[0] = 1.0
    a = b.copy()
    a[3] = 4e-5 * ELEM_FACTOR * np.sqrt(1 / 8)  # relative to rms(b) = sqrt(1/8)
    assert abs(rel(a, b) - max(np.linalg.norm(a - b), 4e-5)) < 1e-9


def test_complex_pairs():
    b = np.array([1 + 1j, 2 - 1j, 0.5j])
    a = b + np.array([0, 1e-6j, 0])
    assert 0 < rel(a, b) < 1e-5


def test_nonfinite_fails():
    assert rel(np.array([np.nan, 1.0]), np.array([1.0, 1.0])) == float("inf")


def test_theta_half_range():
    th = synth.theta(100000, seed=3, half_range=8 * np.pi)
    assert th.dtype == np.float32
    assert th.min() >= -8 * np.pi - 1e-3 and th.max() <= 8 * np.pi + 1e-3
    assert th.max() > 7 * np.pi and th.min() < -7 * np.pi
    assert np.array_equal(synth.theta(1000, seed=3), synth.theta(1000, seed=3, half_range=np.pi))
