"""Host-side behaviour of the reference's spectrum / selection helpers
(ct/spectral.py:27-66,187-208, ct/kvcore.py:70-105) and the drop-in model
names (ct/toymodel.py:31-55).  The device transforms are in test_gpu_parity."""

import numpy as np
import pytest

from paper_2605_24022_b200.errors import InvalidParam, ShapeError
from paper_2605_24022_b200.kvcore import ComplexSpectrum
from paper_2605_24022_b200.model import ModelConfig, ToyModelConfig
from paper_2605_24022_b200.spectral import cutoff_index, highpass, jaccard_overlap, lowpass


def _spec(n=10, h=2, d=4, seed=0):
    x = np.random.default_rng(seed).standard_normal((n, h, d))
    return ComplexSpectrum.from_complex(np.fft.rfft(x, axis=0), origin_len=n)


def test_complex_spectrum_validates_shape():
    s = _spec()
    assert s.n_freqs == 6 and s.re.dtype == np.float64
    assert not s.re.flags.writeable
    with pytest.raises(ShapeError):
        ComplexSpectrum(np.zeros((5, 2, 4)), np.zeros((5, 2, 4)), origin_len=10)
    with pytest.raises(ShapeError):
        ComplexSpectrum(np.zeros((6, 2, 4)), np.zeros((6, 2, 3)), origin_len=10)


@pytest.mark.parametrize("alpha", [0.0, 0.3, 0.5, 1.0])
def test_lowpass_highpass_partition_the_bins(alpha):
    s = _spec(n=11)
    c = cutoff_index(alpha, s.n_freqs)
    lo, hi = lowpass(s, alpha), highpass(s, alpha)
    assert np.all(lo.to_complex()[c:] == 0) and np.array_equal(lo.to_complex()[:c], s.to_complex()[:c])
    assert np.all(hi.to_complex()[:c] == 0) and np.array_equal(hi.to_complex()[c:], s.to_complex()[c:])
    assert np.array_equal(lo.to_complex() + hi.to_complex(), s.to_complex())


def test_band_filters_reject_bad_alpha():
    for a in (-0.1, 1.1, float("nan")):
        with pytest.raises(InvalidParam):
            lowpass(_spec(), a)
        with pytest.raises(InvalidParam):
            highpass(_spec(), a)


def test_jaccard_known_answers():
    assert jaccard_overlap([], []) == 1.0
    assert jaccard_overlap([1, 2, 3], [2, 3, 4]) == 0.5
    assert jaccard_overlap([5, 5, 1], [1]) == 0.5
    assert jaccard_overlap(np.arange(10), np.arange(10)) == 1.0
    assert jaccard_overlap([1], []) == 0.0


def test_toy_model_config_is_the_reference_config():
    c = ToyModelConfig()
    assert ToyModelConfig is ModelConfig
    assert (c.seed, c.n_layers, c.n_heads, c.head_dim, c.vocab_size, c.mlp, c.rope_base) == \
        (0, 4, 2, 8, 256, False, 10000.0)
    assert c.hidden_dim == 16
    with pytest.raises(ShapeError):
        ToyModelConfig(head_dim=7)
