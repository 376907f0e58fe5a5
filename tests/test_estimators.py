"""sklearn wrappers (ct/estimators.py) — the reference's own test cases
(pkg/tests/test_estimators.py) against this package: parameter handling and
the calibrator on CPU, the ranker's device scorer against the oracle on GPU."""

import numpy as np
import pytest
from sklearn.base import clone

from oracle import cachetune_oracle as O
from paper_2605_24022_b200.errors import InvalidParam
from paper_2605_24022_b200.estimators import FrequencyTokenRanker, RatioCalibrator
from paper_2605_24022_b200.pipesim import RequestSpec
from paper_2605_24022_b200.scheduler import HardwareProfile, ttft_model


def test_ranker_get_set_params_and_clone():
    est = FrequencyTokenRanker(alpha=0.3)
    assert est.get_params() == {"alpha": 0.3}
    est.set_params(alpha=0.7)
    assert est.alpha == 0.7
    assert clone(est).get_params() == {"alpha": 0.7}


def test_ranker_requires_fit():
    with pytest.raises(InvalidParam):
        FrequencyTokenRanker().transform(r=0.1)
    with pytest.raises(InvalidParam):
        FrequencyTokenRanker().complement(0.1)


def test_calibrator_fits_r_star():
    p = HardwareProfile(t_c=2e-6, t_i=3e-6, t_o=0.0)
    est = RatioCalibrator(evaluator=lambda s, r: ttft_model(r, s.n_tokens, s.n_layers, p),
                          profile=p)
    est.fit([RequestSpec(chunk_tokens=(64, 64), n_layers=4)] * 5)
    assert abs(est.r_star_ - 0.6) < est.epsilon
    assert est.predict() == est.r_star_
    assert est.r0_ == pytest.approx(0.6)
    assert len(est.trace_) == est.eval_count_


def test_calibrator_clone_keeps_params():
    est = RatioCalibrator(epsilon=0.02, r_min=0.2)
    cloned = clone(est)
    assert cloned.epsilon == 0.02 and cloned.r_min == 0.2
    with pytest.raises(InvalidParam):
        RatioCalibrator().fit([1, 2])
    with pytest.raises(InvalidParam):
        RatioCalibrator().predict()


@pytest.mark.gpu
def test_ranker_matches_oracle_on_device():
    import torch
    import paper_2605_24022_b200 as ct
    rng = np.random.default_rng(5)
    layers = [(rng.standard_normal((18, 2, 4)).astype(np.float32),
               rng.standard_normal((18, 2, 4)).astype(np.float32)) for _ in range(2)]
    chunk = ct.KvChunk("c", tuple(ct.SeqTensor(k) for k, _ in layers),
                       tuple(ct.SeqTensor(v) for _, v in layers))
    est = FrequencyTokenRanker(alpha=0.5).fit(chunk)
    scores, _, agg = O.rank_chunk([k for k, _ in layers], [v for _, v in layers], 0.5)
    assert np.array_equal(est.aggregate_order_, agg)
    np.testing.assert_allclose(est.scores_, scores, rtol=1e-11)
    assert np.array_equal(est.transform(r=0.2), O.indices_for_ratio(agg, 0.2))
    got = set(est.transform(r=0.3).tolist()) | set(est.complement(0.3).tolist())
    assert got == set(range(18))
    # (keys, values) array pair, and an HBM-resident DeviceChunk scored in place
    k, v = layers[0]
    est2 = FrequencyTokenRanker().fit((k, v))
    assert est2.n_tokens_ == 18 and est2.scores_.shape == (1, 18)
    dc = ct.DeviceChunk("d", torch.from_numpy(np.stack([k for k, _ in layers])).cuda(),
                        torch.from_numpy(np.stack([v for _, v in layers])).cuda())
    assert np.array_equal(FrequencyTokenRanker().fit(dc).aggregate_order_, agg)
    np.testing.assert_allclose(est.score_tokens(k, v), O.low_freq_scores(k, v, 0.5), rtol=1e-11)
