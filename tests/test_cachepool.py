"""CachePool registry (ct/cachepool.py:283-529) on the host side: planning
against the reference's own byte ranges (tests/golden/pool_cases.npz, made by
the live reference), CTKV round trips, errors and I/O accounting.  The
device fetch is covered in tests/test_gpu_pool.py."""

import threading

import numpy as np
import pytest

from conftest import golden
from oracle import cachetune_oracle as O
from paper_2605_24022_b200.cachepool import CachePool, token_row_bytes
from paper_2605_24022_b200.errors import AlreadyExists, InvalidParam, NotFound, ShapeError
from paper_2605_24022_b200.kvcore import KvChunk, SeqTensor
from paper_2605_24022_b200.pipesim import TIER_PRESETS, TierConfig
from paper_2605_24022_b200.spectral import ImportanceRanking


def _case(g, i):
    l, n, h, d, layer = (int(x) for x in g[f"p{i}_geom"])
    keys, vals = g[f"p{i}_keys"], g[f"p{i}_vals"]
    chunk = KvChunk(f"p{i}", tuple(SeqTensor(k) for k in keys), tuple(SeqTensor(v) for v in vals))
    scores, orders, agg = O.rank_chunk(list(keys), list(vals))
    rk = ImportanceRanking(per_layer_scores=scores, per_layer_order=orders,
                           aggregate_order=agg, alpha=0.5, n_tokens=n)
    return chunk, rk, layer, float(g[f"p{i}_r"])


def test_plans_match_reference_byte_ranges():
    g = golden("pool_cases")
    for i in range(int(g["count"])):
        chunk, rk, layer, r = _case(g, i)
        pool = CachePool()
        pool.put_chunk(chunk, rk, TIER_PRESETS["cpu-mem"])
        plan = pool.plan_sparse_fetch(f"p{i}", layer, r)
        assert np.array_equal(plan.keep_indices, g[f"p{i}_keep"]), i
        got = np.array(plan.byte_ranges, dtype=np.int64).reshape(-1, 2)
        assert np.array_equal(got, g[f"p{i}_ranges"]), i
        assert plan.expected_bytes == int(g[f"p{i}_expected"])
        assert pool.file_bytes(f"p{i}") == int(g[f"p{i}_ctkv_len"])


@pytest.mark.parametrize("file_backed", [False, True])
def test_registry_round_trip_and_accounting(tmp_path, file_backed):
    g = golden("pool_cases")
    chunk, rk, layer, r = _case(g, 3)
    tier = TierConfig("ssd" if file_backed else "cpu-mem", read_bw=535e6, write_bw=445e6,
                      backing=str(tmp_path) if file_backed else None)
    pool = CachePool()
    cid = pool.put_chunk(chunk, rk, tier)
    assert pool.chunk_ids() == [cid]
    assert pool.io_stats["writes"] == 1
    assert pool.io_stats["bytes_written"] == pool.file_bytes(cid)
    assert pool.modeled_write_time(cid) == tier.write_time(pool.file_bytes(cid))
    with pytest.raises(AlreadyExists):
        pool.put_chunk(chunk, rk, tier)
    full = pool.get_full(cid)
    for l in range(chunk.n_layers):
        assert np.array_equal(full.keys_raw[l].data, chunk.keys_raw[l].data)
        assert np.array_equal(full.values[l].data, chunk.values[l].data)
    assert pool.io_stats["bytes_read"] == pool.file_bytes(cid)
    assert np.array_equal(pool.get_ranking(cid).aggregate_order, rk.aggregate_order)
    l, n, h, d = pool.geometry(cid)
    sizes = [pool.plan_sparse_fetch(cid, 0, x).expected_bytes for x in np.linspace(0, 1, 11)]
    assert all(a >= b for a, b in zip(sizes, sizes[1:]))
    assert sizes[0] == n * token_row_bytes(h, d) * 2 and sizes[-1] == 0
    plan = pool.plan_sparse_fetch(cid, layer, 1.0)
    assert plan.keep_indices.size == 0 and plan.byte_ranges == ()
    with pytest.raises(InvalidParam):
        pool.plan_sparse_fetch(cid, l, 0.5)
    with pytest.raises(InvalidParam):
        pool.plan_sparse_fetch(cid, 0, 1.5)
    with pytest.raises(NotFound):
        pool.plan_sparse_fetch("nope", 0, 0.5)
    if file_backed:  # re-attach the file in a second pool
        other = CachePool()
        assert other.attach_chunk_file(tmp_path / f"{cid}.ctkv", tier) == cid
        assert other.plan_sparse_fetch(cid, layer, r).byte_ranges == \
            pool.plan_sparse_fetch(cid, layer, r).byte_ranges


def test_put_rejects_mismatched_ranking_and_serialises_writers():
    g = golden("pool_cases")
    chunk, rk, _, _ = _case(g, 0)
    chunk2, rk2, _, _ = _case(g, 1)
    pool = CachePool()
    if chunk.token_count != rk2.n_tokens:
        with pytest.raises(ShapeError):
            pool.put_chunk(chunk, rk2, TIER_PRESETS["cpu-mem"])
    errors = []

    def put():
        try:
            pool.put_chunk(chunk, rk, TIER_PRESETS["cpu-mem"])
        except AlreadyExists as e:
            errors.append(e)

    ts = [threading.Thread(target=put) for _ in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert len(errors) == 7 and pool.io_stats["writes"] == 1
