"""Pin the CPU oracle (oracle/cachetune_oracle.py) against fixtures produced by
the live reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import golden
from oracle import cachetune_oracle as O


def test_spectral_cases_bit_exact():
    g = golden("spectral_cases")
    for i in range(int(g["count"])):
        keys, vals, alpha = g[f"c{i}_keys"], g[f"c{i}_vals"], float(g[f"c{i}_alpha"])
        scores, orders, agg = O.rank_chunk(list(keys), list(vals), alpha)
        assert np.array_equal(agg, g[f"c{i}_agg"]), i
        assert np.array_equal(orders, g[f"c{i}_orders"]), i
        # same numpy pocketfft arithmetic -> identical float64 scores
        np.testing.assert_allclose(scores, g[f"c{i}_scores"], rtol=1e-12, atol=1e-300)
        for r, tag in ((0.15, "sel15"), (0.05, "sel05"), (0.5, "sel50")):
            assert np.array_equal(O.indices_for_ratio(agg, r), g[f"c{i}_{tag}"]), (i, r)


def test_highband_cases_bit_exact():
    """Oracle high band vs the reference's highfreq strategy ranking."""
    g = golden("highband_cases")
    for i in range(int(g["count"])):
        keys, vals, alpha = g[f"c{i}_keys"], g[f"c{i}_vals"], float(g[f"c{i}_alpha"])
        scores = np.stack([O.high_freq_scores(k, v, alpha) for k, v in zip(keys, vals)])
        np.testing.assert_allclose(scores, g[f"c{i}_scores"], rtol=1e-12, atol=1e-300)
        assert np.array_equal(np.stack([O.descending_order(s) for s in scores]),
                              g[f"c{i}_orders"]), i
        assert np.array_equal(O.descending_order(scores.mean(axis=0)), g[f"c{i}_agg"]), i


def test_big_chunk_regenerated_inputs_and_orders():
    g = golden("big_chunks")
    l, n, h, d = g["geometry"]
    s = int(g["seeds"][0])
    rng = np.random.default_rng(s)
    keys = [rng.standard_normal((n, h, d)).astype(np.float32) for _ in range(l)]
    vals = [rng.standard_normal((n, h, d)).astype(np.float32) for _ in range(l)]
    chk = sum(float(np.sum(k.astype(np.float64))) for k in keys + vals)
    assert chk == float(g[f"s{s}_checksum"]), "numpy RNG stream drifted"
    scores, orders, agg = O.rank_chunk(keys, vals, 0.5)
    assert np.array_equal(agg, g[f"s{s}_agg"])
    assert np.array_equal(orders, g[f"s{s}_orders"])


def test_selection_count_known_answers():
    # tests/test_spectral.py:170-181 worked examples
    assert O.selection_count(0.15, 20) == 3
    assert O.selection_count(0.1, 1000) == 100
    assert O.selection_count(0.15, 2048) == 308
    assert O.selection_count(0.0, 7) == 0
    assert O.selection_count(1.0, 7) == 7
    with pytest.raises(ValueError):
        O.selection_count(1.5, 3)


def test_rope_cases():
    g = golden("rope_cases")
    for i in range(int(g["count"])):
        d, base, scaling, pairing = g[f"r{i}_params"]
        rope = O.Rope(int(d), float(base), float(scaling),
                      "adjacent" if int(pairing) == 0 else "split")
        y = O.rope_apply(g[f"r{i}_x"], g[f"r{i}_pos"], rope)
        assert np.array_equal(y, g[f"r{i}_y"]), i


def test_fuse_cases():
    g = golden("fuse_cases")
    for i in range(int(g["count"])):
        f = lambda k: g[f"f{i}_{k}"]
        keep, rec = f("keep"), f("rec")
        d = f("kr").shape[2] if keep.size else f("kn").shape[2]
        K, V = O.fuse_layer(f("kr") if keep.size else None, f("vr") if keep.size else None,
                            keep, f("kn") if rec.size else None,
                            f("vn") if rec.size else None, rec, keep, O.Rope(d),
                            keep.size + rec.size)
        assert np.array_equal(K, f("K")) and np.array_equal(V, f("V"))


@pytest.mark.parametrize("tag,mlp", [("cfg1", False), ("cfg1mlp", True)])
def test_toy_cfg1_selective_prefill(tag, mlp):
    g = golden("toy_cfg1")
    model = O.Model(O.ModelConfig(seed=0, n_layers=2, mlp=mlp))
    chunks, aggs = [], []
    for j in range(4):
        keys, vals = g[f"{tag}_chunk{j}_keys"], g[f"{tag}_chunk{j}_vals"]
        src = g[f"{tag}_tokens"][j]
        # the oracle's isolated encoding reproduces the reference's chunk KV
        kr, vs = O.encode_chunk_isolated(model, src)
        assert max(O.normwise_rel(a, b) for a, b in zip(kr, keys)) < 1e-6
        assert max(O.normwise_rel(a, b) for a, b in zip(vs, vals)) < 1e-6
        _, _, agg = O.rank_chunk(list(keys), list(vals))
        assert np.array_equal(agg, g[f"{tag}_chunk{j}_agg"])
        chunks.append((list(keys), list(vals), src))
        aggs.append(agg)
    out = O.selective_prefill(model, chunks, aggs, g[f"{tag}_suffix"], 0.15)
    assert np.array_equal(out["query_positions"], g[f"{tag}_qpos"])
    assert O.normwise_rel(out["logits"], g[f"{tag}_logits"]) < 1e-12
    for l in range(2):
        assert np.array_equal(out["kv"][l][0], g[f"{tag}_kv{l}_k"]) or \
            O.normwise_rel(out["kv"][l][0], g[f"{tag}_kv{l}_k"]) < 1e-6
        assert O.normwise_rel(out["kv"][l][1], g[f"{tag}_kv{l}_v"]) < 1e-6
        hist = 2048
        rows = np.flatnonzero(out["query_positions"] >= hist)[-4:]
        got = out["attention"][l][:, rows, :hist]
        assert O.normwise_rel(got, g[f"{tag}_attn{l}_suffix"]) < 1e-10
