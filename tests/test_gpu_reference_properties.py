"""Property checks of the reference's own unit tests, run against this
implementation's drop-in API.

Sources:
- scoring and selection: pkg/tests/test_spectral.py;
- rotary embedding: pkg/tests/test_rope.py;
- toy-model prefill: pkg/tests/test_toymodel.py:24-140;
- chunk pool: pkg/tests/test_cachepool.py:127-210.

The checks are restated, not copied.  They use the same properties and
tolerances, and run through the GPU scorer (FFT energy kernel, device
orders), the GPU RoPE kernel and the GPU prefill engine in fp32 mode."""

import numpy as np
import pytest
import torch

import paper_2605_24022_b200 as ct
from paper_2605_24022_b200.errors import InvalidParam, InvalidPlan, ShapeError

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def seq(rng, n, h=2, d=4):
    return ct.SeqTensor(rng.standard_normal((n, h, d)).astype(np.float32))


def chunk_of(rng, n, layers=3, h=2, d=4, chunk_id="c"):
    return ct.KvChunk(chunk_id, tuple(seq(rng, n, h, d) for _ in range(layers)),
                      tuple(seq(rng, n, h, d) for _ in range(layers)))


def one_lane(values):
    """[N, 1, 2] tensor whose two lanes both carry `values`."""
    v = np.asarray(values, np.float32)
    return ct.SeqTensor(np.stack([v, v], axis=-1)[:, None, :])


def row_norms(a):
    a = np.asarray(a, np.float64)
    return np.sqrt((a.reshape(a.shape[0], -1) ** 2).sum(axis=1))


def dft_lowpass(x, alpha):
    """O(N^2) low-pass reconstruction of every lane of x [N, ...] (f64):
    keep rfft bins k < floor(alpha (N//2 + 1)) and their mirrors."""
    n = x.shape[0]
    t = np.arange(n)
    w = np.exp(-2j * np.pi * np.outer(t, t) / n)          # forward DFT matrix
    spec = w @ x.reshape(n, -1)
    c = int(np.floor(alpha * (n // 2 + 1)))
    k = np.minimum(t, n - t)
    spec[k >= c] = 0.0
    return (np.conj(w) @ spec / n).real.reshape(x.shape)


# --------------------------------------------------------------- spectrum

def test_spectrum_of_constant_and_alternating_lanes():
    dc = ct.rfft_seq(one_lane([1.0] * 4)).to_complex()[:, 0, 0]
    assert abs(dc[0] - 4.0) < 1e-12 and np.all(np.abs(dc[1:]) < 1e-12)
    ny = ct.rfft_seq(one_lane([1.0, -1.0, 1.0, -1.0])).to_complex()[:, 0, 0]
    assert np.all(np.abs(ny[:2]) < 1e-12) and abs(ny[2] - 4.0) < 1e-12


def test_lowpass_identity_null_cutoff_idempotence(rng):
    s = ct.rfft_seq(seq(rng, 10))
    full = s.to_complex()
    assert np.array_equal(ct.lowpass(s, 1.0).to_complex(), full)
    assert not np.any(ct.lowpass(s, 0.0).to_complex())
    half = ct.lowpass(s, 0.5).to_complex()   # 6 bins, cutoff 3
    assert np.array_equal(half[:3], full[:3]) and not np.any(half[3:])
    once = ct.lowpass(ct.rfft_seq(seq(rng, 12)), 0.4)
    assert np.array_equal(ct.lowpass(once, 0.4).to_complex(), once.to_complex())
    with pytest.raises(InvalidParam):
        ct.lowpass(s, 1.5)


def test_inverse_transform_cases(rng):
    t = seq(rng, 16, 2, 4)
    assert np.max(np.abs(ct.irfft_seq(ct.rfft_seq(t), 16).data - t.data)) < 1e-6
    ramp = one_lane([1.0, 2.0, 3.0, 4.0])
    assert not np.any(ct.irfft_seq(ct.lowpass(ct.rfft_seq(ramp), 0.0), 4).data)
    flat = ct.irfft_seq(ct.rfft_seq(one_lane([1.0] * 4)), 4).data
    assert np.max(np.abs(flat - 1.0)) < 1e-7
    with pytest.raises(ShapeError):
        ct.irfft_seq(ct.rfft_seq(seq(rng, 8)), 9)


def test_parseval(rng):
    t = seq(rng, 17, 2, 4)                   # odd length: no Nyquist bin
    spec = ct.rfft_seq(t).to_complex()
    w = np.full(spec.shape[0], 2.0)
    w[0] = 1.0
    lhs = float((w[:, None, None] * np.abs(spec) ** 2).sum())
    rhs = 17 * float((t.data.astype(np.float64) ** 2).sum())
    assert abs(lhs - rhs) / rhs < 1e-6


# ----------------------------------------------------------------- scores

def test_scores_at_full_band_are_the_raw_row_norms(rng):
    k, v = seq(rng, 9), seq(rng, 9)
    got = ct.low_freq_scores(k, v, 1.0)
    assert np.allclose(got, 0.5 * row_norms(k.data) + 0.5 * row_norms(v.data), atol=1e-6)


def test_scores_with_equal_keys_and_values(rng):
    t = seq(rng, 8)
    want = row_norms(ct.irfft_seq(ct.lowpass(ct.rfft_seq(t), 0.5), 8).data)
    assert np.allclose(ct.low_freq_scores(t, t, 0.5), want, atol=1e-5)


@pytest.mark.parametrize("n", [12, 7, 64])
def test_scores_against_a_quadratic_dft(rng, n):
    k, v = seq(rng, n, 2, 4), seq(rng, n, 2, 4)
    want = (0.5 * row_norms(dft_lowpass(k.data.astype(np.float64), 0.5))
            + 0.5 * row_norms(dft_lowpass(v.data.astype(np.float64), 0.5)))
    assert np.max(np.abs(ct.low_freq_scores(k, v, 0.5) - want)) < 1e-6


def test_scores_reject_mismatched_shapes(rng):
    with pytest.raises(ShapeError):
        ct.low_freq_scores(seq(rng, 8), seq(rng, 9), 0.5)


# -------------------------------------------------------- ranking, ratios

def test_one_layer_aggregate_is_the_layer_order(rng):
    r = ct.rank_chunk(chunk_of(rng, 10, layers=1), 0.5)
    assert np.array_equal(r.aggregate_order, r.per_layer_order[0])


def test_boosted_token_ranks_first(rng):
    base = chunk_of(rng, 12, layers=3)
    boost = np.where(np.arange(12) == 3, 10.0, 1.0).astype(np.float32)[:, None, None]
    c = ct.KvChunk("boost", tuple(ct.SeqTensor(k.data * boost) for k in base.keys_raw),
                   tuple(ct.SeqTensor(v.data * boost) for v in base.values))
    for k, v in zip(c.keys_raw, c.values):
        assert int(np.argmax(ct.low_freq_scores(k, v, 0.5))) == 3
    assert ct.rank_chunk(c, 0.5).aggregate_order[0] == 3


def test_identical_tokens_keep_index_order(rng):
    a = rng.standard_normal((6, 2, 4)).astype(np.float32)
    a[4] = a[1]
    t = ct.SeqTensor(a)
    order = list(ct.rank_chunk(ct.KvChunk("tie", (t,), (t,)), 0.5).aggregate_order)
    assert order.index(1) < order.index(4)


def test_ratio_boundaries_and_counts(rng):
    r9 = ct.rank_chunk(chunk_of(rng, 9), 0.5)
    assert ct.indices_for_ratio(r9, 0.0).size == 0
    assert np.array_equal(ct.indices_for_ratio(r9, 1.0), np.arange(9))
    with pytest.raises(InvalidParam):
        ct.indices_for_ratio(r9, -0.1)
    assert ct.selection_count(0.15, 20) == 3
    assert ct.indices_for_ratio(ct.rank_chunk(chunk_of(rng, 20), 0.5), 0.15).size == 3
    # decimal ratios whose binary product lands just above the integer
    assert (ct.selection_count(0.1, 1000), ct.selection_count(0.05, 1000),
            ct.selection_count(0.3, 10)) == (100, 50, 3)


def test_selections_nest_and_complement(rng):
    for _ in range(50):
        n = int(rng.integers(4, 40))
        rk = ct.rank_chunk(chunk_of(rng, n), 0.5)
        lo, hi = np.sort(rng.uniform(0, 1, size=2))
        small = set(ct.indices_for_ratio(rk, lo).tolist())
        assert small <= set(ct.indices_for_ratio(rk, hi).tolist())
        assert set(ct.complement_for_ratio(rk, lo).tolist()) == set(range(n)) - small


def test_orders_survive_positive_scaling(rng):
    c = chunk_of(rng, 24, layers=2)
    base = ct.rank_chunk(c, 0.5)
    for s in (0.01, 3.0, 1000.0):
        sc = ct.KvChunk("s", tuple(ct.SeqTensor(k.data * s) for k in c.keys_raw),
                        tuple(ct.SeqTensor(v.data * s) for v in c.values))
        other = ct.rank_chunk(sc, 0.5)
        assert np.array_equal(other.aggregate_order, base.aggregate_order)
        assert np.array_equal(other.per_layer_order, base.per_layer_order)


# ------------------------------------------------------------------- RoPE

def test_rope_parameter_validation():
    for bad in (dict(head_dim=3), dict(head_dim=4, base=1.0),
                dict(head_dim=4, pairing="interleaved-ish")):
        with pytest.raises(InvalidParam):
            ct.RopeParams(**bad)


def test_rope_identity_unit_angle_and_inverse(rng):
    t = seq(rng, 5, 2, 8)
    assert np.array_equal(ct.rope_apply(t, [0] * 5, ct.RopeParams(head_dim=8)).data, t.data)
    one = ct.rope_apply(ct.SeqTensor(np.array([[[1.0, 0.0]]], np.float32)), [1],
                        ct.RopeParams(head_dim=2)).data[0, 0]
    assert abs(one[0] - np.cos(1.0)) < 1e-7 and abs(one[1] - np.sin(1.0)) < 1e-7
    x = seq(rng, 7, 2, 8)
    pos = rng.integers(0, 500, size=7)
    p = ct.RopeParams(head_dim=8)
    back = ct.rope_apply(ct.rope_apply(x, pos, p), -pos, p)
    assert np.max(np.abs(back.data - x.data)) < 1e-6


def test_rope_preserves_norms_pairings_and_scaling(rng):
    t = seq(rng, 9, 2, 8)
    out = ct.rope_apply(t, rng.integers(0, 2048, size=9), ct.RopeParams(head_dim=8))
    assert np.max(np.abs(row_norms(out.data) - row_norms(t.data))) < 1e-6
    u = seq(rng, 4, 1, 8)
    adj = ct.rope_apply(u, [3] * 4, ct.RopeParams(head_dim=8, pairing="adjacent")).data
    spl = ct.rope_apply(u, [3] * 4, ct.RopeParams(head_dim=8, pairing="split")).data
    assert not np.allclose(adj, spl)
    assert np.allclose(row_norms(spl), row_norms(u.data), atol=1e-6)
    w = seq(rng, 3, 1, 4)
    assert np.allclose(ct.rope_apply(w, [2, 4, 6], ct.RopeParams(head_dim=4)).data,
                       ct.rope_apply(w, [1, 2, 3], ct.RopeParams(head_dim=4, scaling=2.0)).data,
                       atol=1e-7)
    with pytest.raises(ShapeError):
        ct.rope_apply(seq(rng, 4, 1, 4), [0, 1], ct.RopeParams(head_dim=4))


# ------------------------------------------------------------ toy prefill

@pytest.fixture(scope="module")
def toy():
    return ct.ToyModel(ct.ToyModelConfig(seed=0))


def toks(model, n, seed=5):
    return np.random.default_rng(seed).integers(0, model.config.vocab_size, size=n)


def mats(rec):
    return [np.asarray(m.cpu().numpy() if isinstance(m, torch.Tensor) else m) for m in rec.matrices]


def test_attention_record_shape_normalisation_causality(toy):
    for m in mats(ct.full_prefill(toy, [42], record_attention=True).attention):
        assert m.shape[1:] == (1, 1) and np.allclose(m, 1.0)
    for m in mats(ct.full_prefill(toy, toks(toy, 33), record_attention=True).attention):
        assert np.max(np.abs(m.sum(axis=-1) - 1.0)) < 1e-5
        assert not np.any(np.triu(m, k=1))


def test_full_prefill_is_deterministic_and_validates(toy):
    t = toks(toy, 20)
    a, b = ct.full_prefill(toy, t), ct.full_prefill(toy, t)
    assert torch.equal(a.logits, b.logits)
    assert all(torch.equal(ka, kb) for (ka, _), (kb, _) in zip(a.kv, b.kv))
    with pytest.raises(ShapeError):
        ct.full_prefill(toy, [toy.config.vocab_size + 5])


def _roped(chunk, layer, positions, model):
    return ct.rope_apply(chunk.keys[layer].float().cpu().numpy(), positions,
                         model.config.rope_params).data


def test_isolated_chunk_equals_prefix_context_only_at_layer_one(toy):
    prompt = toks(toy, 48, seed=9)
    full = ct.full_prefill(toy, prompt)
    piece = ct.encode_chunk_isolated(toy, prompt[19:35])
    want = full.kv[0][0][19:35].float().cpu().numpy()
    assert np.max(np.abs(_roped(piece, 0, np.arange(19, 35), toy) - want)) < 1e-6
    # a chunk after other context differs from the full prefill beyond layer 1
    prompt = toks(toy, 40, seed=11)
    full = ct.full_prefill(toy, prompt)
    late = ct.encode_chunk_isolated(toy, prompt[24:])
    diffs = [np.max(np.abs(_roped(late, l, np.arange(24, 40), toy)
                           - full.kv[l][0][24:].float().cpu().numpy()))
             for l in range(1, toy.config.n_layers)]
    assert max(diffs) > 1e-4


def test_single_token_chunk_matches_every_layer(toy):
    t = toks(toy, 1, seed=3)
    piece, full = ct.encode_chunk_isolated(toy, t), ct.full_prefill(toy, t)
    for l in range(toy.config.n_layers):
        assert np.max(np.abs(_roped(piece, l, [0], toy)
                             - full.kv[l][0].float().cpu().numpy())) < 1e-6
        assert np.max(np.abs(piece.values[l].float().cpu().numpy()
                             - full.kv[l][1].float().cpu().numpy())) < 1e-6


def test_selective_prefill_at_r1_and_r0(toy):
    parts = [toks(toy, 24, seed=s) for s in (1, 2)]
    suffix = toks(toy, 6, seed=4)
    chunks = [ct.encode_chunk_isolated(toy, t, chunk_id=f"c{i}") for i, t in enumerate(parts)]
    ranks = [ct.rank_chunk(c) for c in chunks]
    sel = ct.selective_prefill(toy, chunks, ranks, suffix, 1.0, record_attention=True)
    full = ct.full_prefill(toy, np.concatenate(parts + [suffix]), record_attention=True)
    assert (sel.logits.double() - full.logits.double()).abs().max().item() < 1e-5
    assert ct.attention_deviation(full.attention.suffix_view(48),
                                  sel.attention.suffix_view(48)) < 1e-5
    # r = 0, no suffix: pure reuse, the cache is the rotated chunk itself
    body = toks(toy, 20, seed=8)
    piece = ct.encode_chunk_isolated(toy, body)
    out = ct.selective_prefill(toy, [piece], [ct.rank_chunk(piece)], [], 0.0)
    assert tuple(out.logits.shape) == (0, toy.config.vocab_size)
    for l, (k, v) in enumerate(out.kv):
        assert np.array_equal(k.float().cpu().numpy(), _roped(piece, l, np.arange(20), toy))
        assert torch.equal(v.float(), piece.values[l].float())
    # r = 0 with a suffix: layer 1 already equals the full prefill
    sfx = toks(toy, 5, seed=12)
    out = ct.selective_prefill(toy, [piece], [ct.rank_chunk(piece)], sfx, 0.0)
    full = ct.full_prefill(toy, np.concatenate([body, sfx]))
    assert (out.kv[0][0].double() - full.kv[0][0].double()).abs().max().item() < 1e-6


def test_selective_prefill_rejects_a_foreign_ranking(toy):
    piece = ct.encode_chunk_isolated(toy, toks(toy, 10))
    other = ct.encode_chunk_isolated(toy, toks(toy, 12, seed=2))
    with pytest.raises(InvalidPlan):
        ct.selective_prefill(toy, [piece], [ct.rank_chunk(other)], [], 0.5)


# ------------------------------------------------- chunk pool (CachePool)
# pkg/tests/test_cachepool.py:127-210, restated: plans and sparse fetches of
# the registry, with the fetched rows landing in HBM

@pytest.fixture
def pool16(rng):
    from paper_2605_24022_b200.pipesim import TierConfig
    c = chunk_of(rng, 16, layers=3, chunk_id="c0")
    rk = ct.rank_chunk(c, 0.5)
    p = ct.CachePool()
    p.put_chunk(c, rk, TierConfig("cpu-mem", read_bw=20e9, write_bw=20e9))
    return p, c, rk


def test_pool_plans_at_the_ratio_extremes(pool16):
    from paper_2605_24022_b200.cachepool import token_row_bytes
    p, c, _ = pool16
    keep_all = p.plan_sparse_fetch("c0", 0, 0.0)
    assert len(keep_all.keep_indices) == 16
    assert keep_all.expected_bytes == 16 * token_row_bytes(2, 4) * 2
    none = p.plan_sparse_fetch("c0", 1, 1.0)
    assert len(none.keep_indices) == 0 and none.expected_bytes == 0
    k, v, keep = p.fetch_sparse(none)
    assert k is None and v is None and keep.size == 0
    k, v, keep = p.fetch_sparse(p.plan_sparse_fetch("c0", 2, 0.0))
    assert np.array_equal(keep, np.arange(16))
    assert np.array_equal(k.cpu().numpy(), c.keys_raw[2].data)
    assert np.array_equal(v.cpu().numpy(), c.values[2].data)


def test_pool_paper_ratio_and_monotone_bytes(rng, pool16):
    from paper_2605_24022_b200.pipesim import TierConfig
    p, _, _ = pool16
    sizes = [p.plan_sparse_fetch("c0", 0, r).expected_bytes for r in np.linspace(0, 1, 11)]
    assert all(a >= b for a, b in zip(sizes, sizes[1:]))
    q = ct.CachePool()
    c20 = chunk_of(rng, 20, layers=2, chunk_id="p")
    q.put_chunk(c20, ct.rank_chunk(c20, 0.5), TierConfig("cpu-mem", read_bw=20e9, write_bw=20e9))
    plan = q.plan_sparse_fetch("p", 0, 0.15)     # 20 tokens, r = 0.15: 17 kept
    assert len(plan.keep_indices) == 17 and plan.expected_bytes == 17 * 2 * 4 * 4 * 2


def test_pool_fetch_plus_recompute_rows_rebuild_the_layer(pool16):
    p, c, rk = pool16
    k, _, keep = p.fetch_sparse(p.plan_sparse_fetch("c0", 1, 0.3))
    rec = ct.indices_for_ratio(rk, 0.3)
    layer = c.keys_raw[1].data
    out = ct.tensor_scatter_tokens(ct.SeqTensor(np.zeros_like(layer)),
                                   ct.SeqTensor(k.cpu().numpy()), keep)
    out = ct.tensor_scatter_tokens(out, ct.SeqTensor(layer[rec]), rec)
    assert np.array_equal(np.asarray(out.data), layer)


def test_pool_byte_ranges_disjoint_and_coalesced(pool16):
    from paper_2605_24022_b200.cachepool import token_row_bytes
    p, _, _ = pool16
    plan = p.plan_sparse_fetch("c0", 0, 0.2)
    spans = sorted(plan.byte_ranges)
    assert sum(n for _, n in spans) == plan.expected_bytes
    row = token_row_bytes(2, 4)
    for (o1, n1), (o2, _) in zip(spans, spans[1:]):
        assert o1 + n1 <= o2                          # disjoint
        assert o2 != o1 + n1 or n1 % row != 0          # adjacent rows merged
