"""Importance-ordered pool: sparse plan/fetch byte accounting and bit-exact rows
against the reference's plans (tests/golden/pool_cases.npz), plus the serving
engine's HBM vs pinned-host paths agreeing bit for bit."""

import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ct():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_24022_b200 as ct
    return ct


@pytest.mark.parametrize("location", ["hbm", "pinned"])
def test_pool_plans_match_reference_accounting(ct, location):
    from paper_2605_24022_b200.pool import KvPool
    g = golden("pool_cases")
    for i in range(int(g["count"])):
        layers, n, h, d, layer = (int(x) for x in g[f"p{i}_geom"])
        r = float(g[f"p{i}_r"])
        keys, vals = g[f"p{i}_keys"], g[f"p{i}_vals"]
        chunk = ct.KvChunk(f"p{i}", tuple(ct.SeqTensor(k) for k in keys),
                           tuple(ct.SeqTensor(v) for v in vals), source_tokens=np.arange(n))
        rk = ct.rank_chunk(chunk)
        dc = ct.DeviceChunk.from_host(chunk)
        pool = KvPool([dc], [rk], location)
        plan = pool.plan_sparse_fetch(f"p{i}", layer, r)
        # same keep set and byte count as the reference's CTKV plan
        assert np.array_equal(plan.keep_indices, g[f"p{i}_keep"])
        assert plan.expected_bytes == int(g[f"p{i}_expected"])
        # one contiguous range instead of the reference's coalesced runs
        assert len(plan.byte_ranges) == (1 if plan.keep_count else 0)
        before = pool.io_stats["bytes_read"]
        K, V, keep = pool.fetch_sparse(plan)
        if plan.keep_count:
            assert pool.io_stats["bytes_read"] - before == plan.expected_bytes
            assert np.array_equal(K.cpu().numpy(), keys[layer][keep])
            assert np.array_equal(V.cpu().numpy(), vals[layer][keep])


def test_engine_hbm_and_pinned_pools_agree(ct):
    from paper_2605_24022_b200.pipeline import SelectivePrefillEngine
    from paper_2605_24022_b200.pool import KvPool
    cfg = ct.ModelConfig.llama3_8b(n_layers=2, vocab_size=1024, seed=5)
    m = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
    rng = np.random.default_rng(5)
    chunks = [ct.encode_chunk_isolated(m, rng.integers(0, 1024, size=512), chunk_id=f"c{j}")
              for j in range(3)]
    ranks = ct.rank_chunks(chunks)
    suffix = torch.as_tensor(rng.integers(0, 1024, size=16).astype(np.int32), device="cuda")
    outs = []
    for loc in ("hbm", "pinned"):
        eng = SelectivePrefillEngine(m, KvPool(chunks, ranks, loc), 0.15, 16)
        outs.append(eng.step(suffix).float().cpu())
        caches = eng.cache.float().cpu()
        outs.append(caches)
    assert torch.equal(outs[0], outs[2])
    assert torch.equal(outs[1], outs[3])
    # and the drop-in selective_prefill on the same inputs gives the same logits
    ref = ct.selective_prefill(m, chunks, ranks, suffix.cpu().numpy(), 0.15, logits_rows="last",
                               record_attention=False)  # records force the SIMT path
    assert torch.equal(ref.logits.float().cpu(), outs[0])


@pytest.mark.parametrize("location", ["hbm", "pinned"])
def test_corpus_pool_requests_match_dedicated_pools(ct, location):
    """Config-5 style serving: one importance-ordered corpus pool, each request
    binds a different subset of its chunks (in its own order).  Logits and the
    blended cache equal those of an engine over a pool built from exactly the
    request's chunks, bit for bit, and rebinding between requests is clean."""
    from paper_2605_24022_b200.pipeline import SelectivePrefillEngine
    from paper_2605_24022_b200.pool import KvPool
    cfg = ct.ModelConfig.llama3_8b(n_layers=2, vocab_size=1024, seed=6)
    m = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
    rng = np.random.default_rng(6)
    chunks = [ct.encode_chunk_isolated(m, rng.integers(0, 1024, size=512), chunk_id=f"d{j}")
              for j in range(5)]
    ranks = ct.rank_chunks(chunks)
    corpus = KvPool(chunks, ranks, location)
    eng = SelectivePrefillEngine(m, corpus, 0.15, 16, n_chunks=3)
    suffix = torch.as_tensor(rng.integers(0, 1024, size=16).astype(np.int32), device="cuda")
    for req in ([4, 1, 2], ["d0", "d3", "d1"], [4, 1, 2]):
        eng.bind(req)
        got = eng.step(suffix).float().cpu()
        got_cache = eng.cache.float().cpu()
        idx = [corpus.chunk_index(c) for c in req]
        own = SelectivePrefillEngine(m, KvPool([chunks[i] for i in idx], [ranks[i] for i in idx],
                                               location), 0.15, 16)
        assert torch.equal(got, own.step(suffix).float().cpu())
        assert torch.equal(got_cache, own.cache.float().cpu())
    with pytest.raises(ValueError):
        eng.bind([0, 1])


def test_real_three_stream_timeline_audited(ct):
    """CUDA-event timeline of a pinned-pool request in the simulator's schema
    (ct/pipesim.py:93-105), checked with validate_timeline (ct/pipesim.py:257-279):
    per-stream order, fusion after its transfer and recompute, and real overlap
    of the PCIe transfer with the per-layer compute."""
    from paper_2605_24022_b200 import pipesim
    from paper_2605_24022_b200.pipeline import SelectivePrefillEngine
    from paper_2605_24022_b200.pool import KvPool
    cfg = ct.ModelConfig.llama3_8b(n_layers=4, vocab_size=1024, seed=6)
    m = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
    rng = np.random.default_rng(6)
    chunks = [ct.encode_chunk_isolated(m, rng.integers(0, 1024, size=2048), chunk_id=f"c{j}")
              for j in range(4)]
    ranks = ct.rank_chunks(chunks)
    eng = SelectivePrefillEngine(m, KvPool(chunks, ranks, "pinned"), 0.15, 64)
    eng.step()
    eng.record_timeline = True
    eng.step()
    torch.cuda.synchronize()
    tl = eng.timeline()
    plan = pipesim.synthetic_plan([2048] * 4, 4, 0.15, 8, 128)
    assert pipesim.validate_timeline(tl, plan) == []
    csv = pipesim.timeline_to_csv(tl)
    assert len(csv.splitlines()) == 1 + 3 * 4
    busy = sum(e.end_s - e.start_s for e in tl.events)
    assert busy > tl.ttft_s  # streams overlapped


def test_offline_prepare_pool_and_ctkv_export(ct, tmp_path):
    """GPU offline stage: encode + rank + importance-ordered pool, CTKV export
    readable by the reference format parser, rankings identical to rank_chunk."""
    from paper_2605_24022_b200 import ctkv
    from paper_2605_24022_b200.offline import prepare_pool
    from oracle import cachetune_oracle as O
    om = O.Model(O.ModelConfig(seed=2, n_layers=2))
    rng = np.random.default_rng(9)
    toks = [rng.integers(0, 256, size=256) for _ in range(3)]
    timings = {}
    pool = prepare_pool(om, toks, location="pinned", ctkv_dir=tmp_path, timings=timings)
    assert {"encode_ms", "rank_ms", "pool_ms"} <= set(timings)
    assert timings["permute_launches"] == 1  # the batch layout: one pool_permute launch
    for i in range(3):
        chunk, rk = ctkv.read_ctkv((tmp_path / f"chunk{i}.ctkv").read_bytes(), f"chunk{i}")
        assert np.array_equal(rk.aggregate_order, pool.agg[i].cpu().numpy())
        again = ct.rank_chunk(chunk)
        assert np.array_equal(again.aggregate_order, rk.aggregate_order)
        # the exported chunk KV is the oracle's isolated encoding (fp32 mode)
        kr, vs = O.encode_chunk_isolated(om, toks[i])
        assert O.normwise_rel(chunk.keys_raw[1].data, kr[1]) < 1e-5


@pytest.mark.parametrize("file_backed", [False, True])
def test_cachepool_fetch_sparse_bit_exact_into_hbm(ct, tmp_path, file_backed):
    """CachePool.fetch_sparse (ct/cachepool.py:437-481): exactly the planned
    byte ranges (the reference's, pinned in tests/test_cachepool.py) staged in
    pinned memory and moved to HBM in one copy; rows bit-identical to the
    chunk's K/V at the keep indices, bytes read == expected_bytes; the
    registry converts to the engine's importance-ordered KvPool."""
    from oracle import cachetune_oracle as O
    from paper_2605_24022_b200.cachepool import CachePool
    from paper_2605_24022_b200.pipesim import TierConfig
    g = golden("pool_cases")
    tier = TierConfig("ssd" if file_backed else "cpu-mem", read_bw=535e6, write_bw=445e6,
                      backing=str(tmp_path) if file_backed else None)
    pool = CachePool()
    for i in range(int(g["count"])):
        l, n, h, d, layer = (int(x) for x in g[f"p{i}_geom"])
        keys, vals = g[f"p{i}_keys"], g[f"p{i}_vals"]
        chunk = ct.KvChunk(f"p{i}", tuple(ct.SeqTensor(k) for k in keys),
                           tuple(ct.SeqTensor(v) for v in vals))
        scores, orders, agg = O.rank_chunk(list(keys), list(vals))
        rk = ct.ImportanceRanking(per_layer_scores=scores, per_layer_order=orders,
                                  aggregate_order=agg, alpha=0.5, n_tokens=n)
        pool.put_chunk(chunk, rk, tier)
        for r in (0.0, float(g[f"p{i}_r"]), 0.5, 1.0):
            plan = pool.plan_sparse_fetch(f"p{i}", layer, r)
            before = pool.io_stats["bytes_read"]
            K, V, keep = pool.fetch_sparse(plan)
            assert pool.io_stats["bytes_read"] - before == plan.expected_bytes
            if keep.size == 0:
                assert K is None and V is None
                continue
            assert K.is_cuda and K.dtype == torch.float32
            assert np.array_equal(K.cpu().numpy(), keys[layer][keep])
            assert np.array_equal(V.cpu().numpy(), vals[layer][keep])
    # same-geometry chunks -> the engine's importance-ordered pool (f32, HBM)
    ids = [f"p{i}" for i in range(int(g["count"]))]
    geo = {pool.geometry(c) for c in ids}
    c0 = ids[0]
    same = [c for c in ids if pool.geometry(c) == pool.geometry(c0)]
    kvp = pool.to_kv_pool(same, "hbm", dtype=torch.float32)
    for c in same:
        for r in (0.15, 0.5):
            a = pool.fetch_sparse(pool.plan_sparse_fetch(c, 0, r))
            b = kvp.fetch_sparse(kvp.plan_sparse_fetch(c, 0, r))
            assert np.array_equal(a[2], b[2])
            if a[2].size:
                assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    assert len(geo) >= 1


def test_engine_more_chunks_than_one_blend_launch(ct):
    """80 chunks > CT_MAX_SEGMENTS (64): the engine splits each layer's blend
    into launches of at most 64 segments and matches selective_prefill."""
    from paper_2605_24022_b200.pipeline import SelectivePrefillEngine
    from paper_2605_24022_b200.pool import KvPool
    cfg = ct.ModelConfig.llama3_8b(n_layers=2, vocab_size=1024, seed=6)
    m = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
    rng = np.random.default_rng(6)
    chunks = [ct.encode_chunk_isolated(m, rng.integers(0, 1024, size=64), chunk_id=f"s{j}")
              for j in range(80)]
    ranks = ct.rank_chunks(chunks)
    suffix = torch.as_tensor(rng.integers(0, 1024, size=8).astype(np.int32), device="cuda")
    eng = SelectivePrefillEngine(m, KvPool(chunks, ranks, "hbm"), 0.15, 8)
    got = eng.step(suffix).float().cpu()
    ref = ct.selective_prefill(m, chunks, ranks, suffix.cpu().numpy(), 0.15, logits_rows="last",
                               record_attention=False)
    assert torch.equal(ref.logits.float().cpu(), got)
    assert torch.equal(ref.kv[0][0].float().cpu(), eng.cache[0, 0].float().cpu())


def test_ctkv_pool_without_tokens_is_fetch_only(ct):
    """A pool restored from CTKV files without source tokens serves fetches
    but the engine refuses to recompute its chunks (ct/toymodel.py:243-244)
    instead of recomputing token id 0."""
    from paper_2605_24022_b200.ctkv import pool_from_ctkv, write_ctkv
    from paper_2605_24022_b200.errors import InvalidPlan
    from paper_2605_24022_b200.pipeline import SelectivePrefillEngine
    cfg = ct.ModelConfig.llama3_8b(n_layers=2, vocab_size=1024, seed=7)
    m = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
    rng = np.random.default_rng(7)
    toks = [rng.integers(0, 1024, size=128) for _ in range(2)]
    chunks = [ct.encode_chunk_isolated(m, t, chunk_id=f"f{j}") for j, t in enumerate(toks)]
    ranks = ct.rank_chunks(chunks)
    blobs = [write_ctkv(c.to_host(), rk) for c, rk in zip(chunks, ranks)]
    pool = pool_from_ctkv(blobs, "hbm")
    assert pool.has_tokens == [False, False]
    plan = pool.plan_sparse_fetch(pool.chunk_ids[0], 1, 0.15)
    K, V, keep = pool.fetch_sparse(plan)
    assert K.shape[0] == plan.keep_count
    with pytest.raises(InvalidPlan):
        SelectivePrefillEngine(m, pool, 0.15, 8)
    ok = pool_from_ctkv(blobs, "hbm", tokens=toks)
    assert ok.has_tokens == [True, True]
    SelectivePrefillEngine(m, ok, 0.15, 8).step(
        torch.zeros(8, dtype=torch.int32, device="cuda"))


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_pool_permute_batch_and_per_chunk_bit_identical(ct, dtype):
    """ct_pool_permute (offline stage): the importance-ordered image equals
    torch indexing of the chunks' K/V by their aggregate orders, bit for bit,
    whether the chunks are slices of one batch (one launch) or separate
    allocations (one launch per chunk)."""
    import torch
    from paper_2605_24022_b200.kvcore import DeviceChunk
    from paper_2605_24022_b200.pool import KvPool
    torch.manual_seed(0)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    C, L, N, H, D = 3, 4, 200, 2, 64
    keys = torch.randn(C, L, N, H, D, device="cuda").to(tdt)
    vals = torch.randn(C, L, N, H, D, device="cuda").to(tdt)
    orders = [np.random.default_rng(i).permutation(N) for i in range(C)]
    ranks = [ct.ImportanceRanking(per_layer_scores=np.zeros((L, N)),
                                  per_layer_order=np.tile(np.arange(N), (L, 1)),
                                  aggregate_order=o, alpha=0.5, n_tokens=N) for o in orders]
    want = torch.stack([torch.stack([keys[c][:, torch.as_tensor(orders[c], device="cuda")],
                                     vals[c][:, torch.as_tensor(orders[c], device="cuda")]],
                                    dim=2) for c in range(C)])
    batch = [DeviceChunk(f"c{c}", keys[c], vals[c]) for c in range(C)]
    pool = KvPool(batch, ranks, "hbm")
    assert pool.permute_launches == 1
    assert torch.equal(pool.data, want)
    sep = [DeviceChunk(f"c{c}", keys[c].clone(), vals[c].clone()) for c in range(C)]
    pool2 = KvPool(sep, ranks, "pinned")
    assert pool2.permute_launches in (1, C)
    assert torch.equal(pool2.data.cuda(), want)


def test_pool_permute_rejects_bad_geometry(ct):
    """Validation happens before any launch (no pointer is dereferenced)."""
    from paper_2605_24022_b200 import _lib
    with pytest.raises(ct.InvalidParam):   # row bytes not a multiple of 4
        _lib.call("ct_pool_permute", 16, 16, 1, 1, 1, 8, 8, 8, 6, 16, 16, None)
    with pytest.raises(ct.InvalidParam):   # misaligned pointer
        _lib.call("ct_pool_permute", 18, 16, 1, 1, 1, 8, 8, 8, 8, 16, 16, None)
    with pytest.raises(ct.ShapeError):     # rows overlap
        _lib.call("ct_pool_permute", 16, 16, 1, 1, 1, 4, 8, 8, 8, 16, 16, None)


def test_offline_overlapped_scoring_bit_identical(ct):
    """encode_and_rank (chunk c scored on a side stream while chunk c+1 is
    encoded) == encode_batch then one batched score_device, bit for bit, and
    the pools built both ways are identical."""
    import torch
    from paper_2605_24022_b200.offline import encode_and_rank, encode_batch, prepare_pool
    from paper_2605_24022_b200.spectral import score_device
    cfg = ct.ModelConfig.llama3_8b(n_layers=2, vocab_size=1024, seed=8)
    model = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
    rng = np.random.default_rng(3)
    toks = [rng.integers(0, 1024, size=2048) for _ in range(3)]
    k1, v1, _, s1 = encode_and_rank(model, toks)
    k2, v2, _ = encode_batch(model, toks)
    s2 = score_device(k2, v2, 0.5, "f64", want_layer_order=True)
    assert torch.equal(k1, k2) and torch.equal(v1, v2)
    for key in ("layer_scores", "agg", "agg_order", "layer_order"):
        assert torch.equal(s1[key], s2[key]), key
    t1, t2 = {}, {}
    p1 = prepare_pool(model, toks, location="hbm", timings=t1)
    p2 = prepare_pool(model, toks, location="hbm", timings=t2, overlap=False)
    assert torch.equal(p1.data, p2.data) and torch.equal(p1.agg, p2.agg)
