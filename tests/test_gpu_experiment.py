"""Attention-recovery experiment on the device path
against the reference's own per-seed deviations (tests/golden/experiment_cases.npz,
made by running ct/toymodel.py:382-419) and the ordering the reference's
acceptance criterion 8 asserts (pkg/tests/test_acceptance.py:187-201)."""

import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ex():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_24022_b200 import experiments
    return experiments


@pytest.fixture(scope="module")
def committed(ex):
    g = golden("experiment_cases")
    seeds = [int(s) for s in g["seeds"]]
    per = {s: dict(ex.run_selection_experiment(seeds, r=0.15, strategy=s))
           for s in ex.STRATEGIES}
    return g, seeds, per


def test_per_seed_deviation_matches_reference(committed):
    g, seeds, per = committed
    for strategy, res in per.items():
        got = np.array([res[s] for s in seeds])
        want = g[f"dev_{strategy}"]
        # fp32 device forward vs the reference's float64 numpy forward
        np.testing.assert_allclose(got, want, rtol=2e-4, atol=2e-7, err_msg=strategy)


def test_criterion_08_attention_recovery_ordering(committed):
    _, seeds, per = committed
    means = {k: float(np.mean(list(v.values()))) for k, v in per.items()}
    assert means["lowfreq"] < means["none"]
    assert means["lowfreq"] <= means["random"]
    assert means["full"] <= 1e-5
    assert all(means["none"] >= m for m in means.values())
    wins = sum(per["lowfreq"][s] < per["none"][s] for s in seeds)
    assert wins >= 0.8 * len(seeds)


def test_small_and_mlp_variants(ex):
    g = golden("experiment_cases")
    for strategy in ("lowfreq", "none"):
        res = ex.run_selection_experiment([0, 1, 2], 0.25, strategy, chunk_tokens=(24, 24),
                                          suffix_len=6)
        np.testing.assert_allclose([d for _, d in res], g[f"small_{strategy}"], rtol=2e-4,
                                   atol=2e-7)
    res = ex.run_selection_experiment([3, 4], r=0.3, strategy="lowfreq", mlp=True)
    np.testing.assert_allclose([d for _, d in res], g["mlp_lowfreq"], rtol=2e-4, atol=2e-7)


def test_strategies_share_budget(ex):
    import paper_2605_24022_b200 as ct
    from paper_2605_24022_b200.model import GpuModel, ModelConfig
    m = GpuModel.reference_init(ModelConfig(seed=0))
    rng = np.random.default_rng(0)
    chunk = ct.encode_chunk_isolated(m, rng.integers(0, 256, size=30))
    for strategy in ("lowfreq", "highfreq", "random"):
        rk = ex.strategy_ranking(chunk, strategy, rng=np.random.default_rng(0))
        assert rk.n_tokens == 30
        assert np.array_equal(np.sort(rk.aggregate_order), np.arange(30))
    with pytest.raises(ct.InvalidPlan):
        ex.strategy_ranking(chunk, "random")
    with pytest.raises(ct.InvalidPlan):
        ex.run_selection_experiment([0], strategy="bogus")


def test_spectrum_report_matches_reference(ex):
    import paper_2605_24022_b200 as ct
    g = golden("spectrum_cases")
    for i in range(int(g["count"])):
        chunk = ct.KvChunk("s", tuple(ct.SeqTensor(k) for k in g[f"s{i}_keys"]),
                           tuple(ct.SeqTensor(v) for v in g[f"s{i}_vals"]))
        rep = ex.spectrum_report(chunk, int(g[f"s{i}_bands"]))
        np.testing.assert_allclose(rep["key"], g[f"s{i}_key"], rtol=1e-10, atol=1e-14)
        np.testing.assert_allclose(rep["value"], g[f"s{i}_value"], rtol=1e-10, atol=1e-14)


def test_suffix_only_record_equals_full_record(ex):
    """record_attention=<history> (device suffix rows, TC main pass) gives the
    same deviation as the full host record on the toy model."""
    import paper_2605_24022_b200 as ct
    from paper_2605_24022_b200.model import GpuModel, ModelConfig
    m = GpuModel.reference_init(ModelConfig(seed=3))
    rng = np.random.default_rng([3, 1])
    toks = [rng.integers(0, 256, size=n) for n in (64, 64)]
    suffix = rng.integers(0, 256, size=8)
    full_a = ct.full_prefill(m, np.concatenate(toks + [suffix]), record_attention=True)
    full_b = ct.full_prefill(m, np.concatenate(toks + [suffix]), record_attention=128)
    chunks = [ct.encode_chunk_isolated(m, t) for t in toks]
    ranks = [ct.rank_chunk(c) for c in chunks]
    sel_a = ct.selective_prefill(m, chunks, ranks, suffix, 0.2, record_attention=True)
    sel_b = ct.selective_prefill(m, chunks, ranks, suffix, 0.2, record_attention=128)
    da = ct.attention_deviation(full_a.attention.suffix_view(128), sel_a.attention.suffix_view(128))
    db = ct.attention_deviation(full_b.attention.suffix_view(128), sel_b.attention.suffix_view(128))
    assert abs(da - db) <= 1e-6 * da


def test_attention_recovery_llama_geometry_bf16(ex):
    """§8(f) row 4 at a BASELINE geometry (Llama-3-8B layer shapes, 4 layers,
    4 x 1024-token chunks, bf16, tensor-core selective pass): recomputing the
    low-frequency tokens recovers more of the full-recompute suffix attention
    than recomputing nothing, at r=0.15."""
    import paper_2605_24022_b200 as ct
    cfg = ct.ModelConfig.llama3_8b(n_layers=4, vocab_size=4096, seed=21)
    m = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
    rng = np.random.default_rng(21)
    toks = [rng.integers(0, 4096, size=1024) for _ in range(4)]
    suffix = rng.integers(0, 4096, size=32)
    dev = ex.attention_recovery_at_scale(m, toks, suffix, 0.15)
    assert set(dev) == {"lowfreq", "highfreq", "random", "none"}
    assert dev["lowfreq"] < dev["none"]
    full = ex.attention_recovery_at_scale(m, toks, suffix, 0.15, strategies=("full",))
    assert full["full"] < 0.05 * dev["none"]
