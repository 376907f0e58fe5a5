"""Parity at BASELINE config-2 size (32 layers, Llama-3-8B geometry, 16 x 2048
chunks + 64 suffix, r = 0.15) through properties that do not need the float64
oracle to run the whole request:

* the scorer on one full chunk (32 layers x [2048, 8, 128]) vs the oracle:
  per-layer and aggregate orders bit-exact;
* the device selection plan vs the reference's integer rules
  (ct/spectral.py:162-184, ct/toymodel.py:246-267) on the same orders;
* blended cache rows: reused K = RoPE(pool K, global position) within one bf16
  rounding, reused V bit-exact, at three layers;
* HBM pool == pinned pool == CUDA-graph replay == a second step, bit for bit;
* r = 1 selective prefill == full-recompute prefill, bit for bit (same kernels,
  same shapes, every token recomputed)."""

import numpy as np
import pytest
import torch

from oracle import cachetune_oracle as O

pytestmark = pytest.mark.gpu

C, N, S, R = 16, 2048, 64, 0.15


@pytest.fixture(scope="module")
def big():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2605_24022_b200 as ct
    cfg = ct.ModelConfig.llama3_8b(n_layers=32, seed=11)
    m = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
    rng = np.random.default_rng(11)
    toks = [rng.integers(0, cfg.vocab_size, size=N) for _ in range(C)]
    chunks = [ct.encode_chunk_isolated(m, t, chunk_id=f"c{j}") for j, t in enumerate(toks)]
    ranks = ct.rank_chunks(chunks)
    suffix = torch.as_tensor(rng.integers(0, cfg.vocab_size, size=S).astype(np.int32),
                             device="cuda")
    return ct, m, toks, chunks, ranks, suffix


def test_fullsize_scorer_chunk_vs_oracle(big):
    ct, m, toks, chunks, ranks, suffix = big
    c0 = chunks[0]
    keys = [c0.keys[l].float().cpu().numpy() for l in range(c0.n_layers)]
    vals = [c0.values[l].float().cpu().numpy() for l in range(c0.n_layers)]
    scores, orders, agg = O.rank_chunk(keys, vals, 0.5)
    assert np.array_equal(ranks[0].aggregate_order, agg)
    assert np.array_equal(ranks[0].per_layer_order, orders)
    np.testing.assert_allclose(ranks[0].per_layer_scores, scores, rtol=1e-11)


def test_fullsize_selection_and_blend(big):
    ct, m, toks, chunks, ranks, suffix = big
    from paper_2605_24022_b200.pipeline import SelectivePrefillEngine
    from paper_2605_24022_b200.pool import KvPool
    from paper_2605_24022_b200.rope import rope_table
    eng = SelectivePrefillEngine(m, KvPool(chunks, ranks, "hbm"), R, S)
    eng.step(suffix)
    torch.cuda.synchronize()
    k = O.selection_count(R, N)
    rec = np.concatenate([O.indices_for_ratio(rk.aggregate_order, R) + j * N
                          for j, rk in enumerate(ranks)])
    keep = np.concatenate([O.complement_for_ratio(rk.aggregate_order, R) + j * N
                           for j, rk in enumerate(ranks)])
    assert eng.k == k
    assert np.array_equal(eng.positions[:C * k].cpu().numpy(), rec)
    assert np.array_equal(eng.positions[C * k:].cpu().numpy(), np.arange(C * N, C * N + S))
    assert np.array_equal(eng.keep.cpu().numpy(), keep)
    # reused rows of three layers: K rotated at its global position, V copied
    cfg = m.config
    table = rope_table(cfg.rope_params, eng.n_ctx, "f32", m.device)
    g = torch.Generator().manual_seed(0)
    sample = torch.as_tensor(keep)[torch.randperm(keep.size, generator=g)[:1024]].cuda()
    for l in (0, 17, 31):
        ch, tok = sample // N, sample % N
        kraw = torch.stack([chunks[int(c)].keys[l][int(t)] for c, t in zip(ch, tok)]).float()
        vraw = torch.stack([chunks[int(c)].values[l][int(t)] for c, t in zip(ch, tok)])
        cs = table[sample.long()]
        cos, sin = cs[..., 0][:, None, :], cs[..., 1][:, None, :]
        a, b = kraw[..., 0::2], kraw[..., 1::2]
        want = torch.empty_like(kraw)
        want[..., 0::2] = a * cos - b * sin
        want[..., 1::2] = a * sin + b * cos
        got = eng.cache[l, 0][sample.long()].float()
        tol = want.abs() * 2.0 ** -8 + (a.abs() + b.abs()).repeat_interleave(2, -1) * 2.0 ** -20
        assert bool(((got - want).abs() <= tol).all()), l
        assert torch.equal(eng.cache[l, 1][sample.long()], vraw), l


def test_fullsize_pools_graph_and_repeat_bit_identical(big):
    ct, m, toks, chunks, ranks, suffix = big
    from paper_2605_24022_b200.pipeline import SelectivePrefillEngine
    from paper_2605_24022_b200.pool import KvPool
    hbm = SelectivePrefillEngine(m, KvPool(chunks, ranks, "hbm"), R, S)
    a = hbm.step(suffix).clone()
    b = hbm.step(suffix).clone()
    assert torch.equal(a, b)
    hbm.capture(suffix)
    assert torch.equal(hbm.replay().clone(), a)
    del hbm
    pin = SelectivePrefillEngine(m, KvPool(chunks, ranks, "pinned"), R, S)
    assert torch.equal(pin.step(suffix), a)


def test_fullsize_r1_equals_full_prefill(big):
    ct, m, toks, chunks, ranks, suffix = big
    from paper_2605_24022_b200.pipeline import FullPrefillEngine, SelectivePrefillEngine
    from paper_2605_24022_b200.pool import KvPool
    sel = SelectivePrefillEngine(m, KvPool(chunks, ranks, "hbm"), 1.0, S)
    got = sel.step(suffix).clone()
    del sel
    torch.cuda.empty_cache()
    full = FullPrefillEngine(m, C * N + S)
    tokens = torch.cat([torch.as_tensor(np.concatenate(toks).astype(np.int32), device="cuda"),
                        suffix])
    want = full.step(tokens)
    assert torch.equal(got, want)


def test_fullsize_oracle_attention_and_blend(big):
    """Float64 oracle at full config-2 context (32,832 tokens) on layers 0, 15
    and 31: the whole blended cache of each layer vs O.fuse_layer, attention
    of 64 sampled query rows (incl. the first-token row) x 8 q heads vs the
    oracle attention over that cache.  bf16 mode: <= 2e-2 normwise."""
    from fullsize_oracle import check_request
    from paper_2605_24022_b200.pipeline import SelectivePrefillEngine
    from paper_2605_24022_b200.pool import KvPool
    ct, m, toks, chunks, ranks, suffix = big
    eng = SelectivePrefillEngine(m, KvPool(chunks, ranks, "hbm"), R, S)
    errs = check_request(eng, chunks, suffix, (0, 15, 31))
    print("cfg2 oracle errors", errs)
    # reused K rows are one bf16 rounding of the float64 rotation
    assert all(e["blend_k_reused"] <= 2.0 ** -8 for e in errs.values()), errs
