"""Input-generator checks (workload/): calibration, determinism, monotone cap."""
import numpy as np

from workload.lengths import LengthModel, sample_lengths
from workload.prompts import make_prompts


def test_length_calibration_paper_shape():
    """~80% within 3K tokens and a few % at the limit (0.848 / 0.031 at 8k)."""
    L = sample_lengths(LengthModel(cap=8192), 0, 100000)
    assert 0.83 <= (L <= 3000).mean() <= 0.87
    assert 0.025 <= (L == 8192).mean() <= 0.037
    L4 = sample_lengths(LengthModel(cap=4096), 0, 100000)
    assert 0.06 <= (L4 == 4096).mean() <= 0.085


def test_length_trivial_cases_and_range():
    assert (sample_lengths(LengthModel(tail=1.0, cap=4096), 1, 100) == 4096).all()
    L = sample_lengths(LengthModel(median=100, sigma=0.0, tail=0.0, cap=500), 1, 100)
    assert (L == 100).all()
    L = sample_lengths(LengthModel(median=12, sigma=0.6, tail=0.1, floor=1, cap=64), 2, 5000)
    assert L.min() >= 1 and L.max() <= 64


def test_length_determinism_and_monotone_cap():
    a = sample_lengths(LengthModel(cap=8192), 3, 1000)
    b = sample_lengths(LengthModel(cap=8192), 3, 1000)
    np.testing.assert_array_equal(a, b)
    c = sample_lengths(LengthModel(cap=16384), 3, 1000)
    assert (c >= a).all()
    # offsets address the same stream
    np.testing.assert_array_equal(sample_lengths(LengthModel(cap=8192), 3, 10, offset=500), a[500:510])


def test_prompts():
    off, toks = make_prompts(1, 16, 512, 4, 16)
    lens = np.diff(off)
    assert off[0] == 0 and lens.min() >= 4 and lens.max() <= 16
    assert toks.min() >= 1 and toks.max() < 512
    off2, toks2 = make_prompts(1, 16, 512, 4, 16)
    np.testing.assert_array_equal(toks, toks2)
    off, toks = make_prompts(1, 3, 128256, 256)
    assert (np.diff(off) == 256).all()
