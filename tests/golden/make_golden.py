"""Generate golden fixtures by running the LIVE reference package.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports `cachetune` read-only from /root/reference/pkg/src, evaluates the
reference on seeded inputs and writes compressed .npz fixtures next to this
script.  The fixtures travel with the repo; nothing at test time on the GPU
box reads /root/reference.  Inputs that are large are regenerated from their
seed at test time (numpy default_rng, same image) and pinned by a checksum
stored in the fixture.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _ref():
    sys.path.insert(0, str(REF))
    import cachetune as ct  # noqa: E402
    return ct


def _chunk(ct, keys, vals, cid="c", src=None):
    return ct.KvChunk(chunk_id=cid,
                      keys_raw=tuple(ct.SeqTensor(k) for k in keys),
                      values=tuple(ct.SeqTensor(v) for v in vals),
                      source_tokens=src)


def spectral_cases(ct):
    """Random small chunks over awkward geometries and cutoffs."""
    rng = np.random.default_rng(20260101)
    geoms = [(1, 1, 2, 1), (2, 1, 2, 2), (3, 2, 2, 1), (7, 2, 4, 3), (16, 2, 4, 3),
             (31, 1, 8, 2), (64, 4, 8, 2), (127, 2, 4, 1), (128, 2, 8, 2),
             (257, 1, 2, 2), (512, 2, 8, 1), (1000, 2, 4, 1), (1024, 2, 4, 1),
             (2048, 1, 4, 1), (96, 2, 64, 1)]
    alphas = [0.0, 0.1, 0.3, 0.5, 0.7, 1.0]
    out = {}
    i = 0
    for (n, h, d, l) in geoms:
        for alpha in (alphas if n <= 128 else [0.5, 0.3]):
            keys = [rng.standard_normal((n, h, d)).astype(np.float32) for _ in range(l)]
            vals = [rng.standard_normal((n, h, d)).astype(np.float32) for _ in range(l)]
            rk = ct.rank_chunk(_chunk(ct, keys, vals), alpha)
            out[f"c{i}_keys"] = np.stack(keys)
            out[f"c{i}_vals"] = np.stack(vals)
            out[f"c{i}_alpha"] = np.float64(alpha)
            out[f"c{i}_scores"] = rk.per_layer_scores
            out[f"c{i}_orders"] = rk.per_layer_order.astype(np.int32)
            out[f"c{i}_agg"] = rk.aggregate_order.astype(np.int32)
            sel = {}
            for r in (0.0, 0.05, 0.15, 0.5, 1.0):
                sel[r] = ct.indices_for_ratio(rk, r)
            out[f"c{i}_sel15"] = sel[0.15].astype(np.int32)
            out[f"c{i}_sel05"] = sel[0.05].astype(np.int32)
            out[f"c{i}_sel50"] = sel[0.5].astype(np.int32)
            i += 1
    # ties: constant chunk, duplicated rows, zero chunk
    specials = {
        "zeros": (np.zeros((16, 2, 4), np.float32), np.zeros((16, 2, 4), np.float32)),
        "const": (np.ones((16, 2, 4), np.float32), np.full((16, 2, 4), 2.0, np.float32)),
    }
    dup = rng.standard_normal((8, 2, 4)).astype(np.float32)
    specials["dup"] = (np.concatenate([dup, dup]), np.concatenate([dup, dup]))
    for name, (k, v) in specials.items():
        rk = ct.rank_chunk(_chunk(ct, [k], [v]), 0.5)
        out[f"c{i}_keys"] = k[None]
        out[f"c{i}_vals"] = v[None]
        out[f"c{i}_alpha"] = np.float64(0.5)
        out[f"c{i}_scores"] = rk.per_layer_scores
        out[f"c{i}_orders"] = rk.per_layer_order.astype(np.int32)
        out[f"c{i}_agg"] = rk.aggregate_order.astype(np.int32)
        out[f"c{i}_sel15"] = ct.indices_for_ratio(rk, 0.15).astype(np.int32)
        out[f"c{i}_sel05"] = ct.indices_for_ratio(rk, 0.05).astype(np.int32)
        out[f"c{i}_sel50"] = ct.indices_for_ratio(rk, 0.5).astype(np.int32)
        i += 1
    out["count"] = np.int64(i)
    np.savez_compressed(OUT / "spectral_cases.npz", **out)
    print("spectral cases", i)


def big_chunks(ct):
    """Config-2-geometry chunks [2048, 8, 128]: inputs regenerated from seed."""
    out = {}
    seeds = [11, 12, 13, 14]
    for s in seeds:
        rng = np.random.default_rng(s)
        keys = [rng.standard_normal((2048, 8, 128)).astype(np.float32) for _ in range(4)]
        vals = [rng.standard_normal((2048, 8, 128)).astype(np.float32) for _ in range(4)]
        rk = ct.rank_chunk(_chunk(ct, keys, vals), 0.5)
        out[f"s{s}_checksum"] = np.float64(sum(float(np.sum(k.astype(np.float64)))
                                               for k in keys + vals))
        out[f"s{s}_scores"] = rk.per_layer_scores
        out[f"s{s}_orders"] = rk.per_layer_order.astype(np.int16)
        out[f"s{s}_agg"] = rk.aggregate_order.astype(np.int16)
        # bf16-rounded inputs (round-to-nearest-even) scored by the reference
        def bf16(x):
            u = x.view(np.uint32).astype(np.uint64)
            u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
            return u.astype(np.uint32).view(np.float32)
        rkb = ct.rank_chunk(_chunk(ct, [bf16(k) for k in keys], [bf16(v) for v in vals]), 0.5)
        out[f"s{s}_bf16_agg"] = rkb.aggregate_order.astype(np.int16)
        out[f"s{s}_bf16_scores"] = rkb.per_layer_scores
    out["seeds"] = np.array(seeds)
    out["geometry"] = np.array([4, 2048, 8, 128])
    np.savez_compressed(OUT / "big_chunks.npz", **out)
    print("big chunks", seeds)


def rope_cases(ct):
    rng = np.random.default_rng(777)
    out = {}
    cases = [(8, 10000.0, 1.0, "adjacent"), (8, 10000.0, 1.0, "split"),
             (128, 10000.0, 1.0, "adjacent"), (128, 500000.0, 1.0, "split"),
             (64, 10000.0, 0.25, "adjacent"), (2, 10000.0, 1.0, "adjacent")]
    for i, (d, base, scaling, pairing) in enumerate(cases):
        x = rng.standard_normal((300, 2, d)).astype(np.float32)
        pos = rng.integers(0, 70000, size=300)
        pos[:3] = [0, 1, 65535]
        p = ct.RopeParams(head_dim=d, base=base, scaling=scaling, pairing=pairing)
        y = ct.rope_apply(ct.SeqTensor(x), pos, p).data
        out[f"r{i}_x"], out[f"r{i}_pos"], out[f"r{i}_y"] = x, pos, y
        out[f"r{i}_params"] = np.array([d, base, scaling, 0 if pairing == "adjacent" else 1])
    out["count"] = np.int64(len(cases))
    np.savez_compressed(OUT / "rope_cases.npz", **out)


def toy_cfg1(ct):
    """BASELINE config 1: ToyModel(seed=0, n_layers=2), 4 x 512 chunks, r=0.15, S=32."""
    from cachetune import toymodel as tm
    out = {}
    for tag, mlp in (("cfg1", False), ("cfg1mlp", True)):
        model = tm.ToyModel(tm.ToyModelConfig(seed=0, n_layers=2, mlp=mlp))
        tok_rng = np.random.default_rng([0, 1])
        chunk_ids = [tok_rng.integers(0, 256, size=512) for _ in range(4)]
        suffix = tok_rng.integers(0, 256, size=32)
        chunks = [tm.encode_chunk_isolated(model, t, chunk_id=f"c{j}")
                  for j, t in enumerate(chunk_ids)]
        rankings = [ct.rank_chunk(c) for c in chunks]
        sel = tm.selective_prefill(model, chunks, rankings, suffix, 0.15)
        out[f"{tag}_tokens"] = np.stack(chunk_ids)
        out[f"{tag}_suffix"] = suffix
        for j, c in enumerate(chunks):
            out[f"{tag}_chunk{j}_keys"] = np.stack([k.data for k in c.keys_raw])
            out[f"{tag}_chunk{j}_vals"] = np.stack([v.data for v in c.values])
            out[f"{tag}_chunk{j}_agg"] = rankings[j].aggregate_order.astype(np.int32)
        out[f"{tag}_logits"] = sel.logits
        out[f"{tag}_qpos"] = sel.query_positions
        for l, (k, v) in enumerate(sel.kv):
            out[f"{tag}_kv{l}_k"] = k.data
            out[f"{tag}_kv{l}_v"] = v.data
        hist = 4 * 512
        sv = sel.attention.suffix_view(hist)
        for l, m in enumerate(sv.matrices):
            out[f"{tag}_attn{l}_suffix"] = m[:, -4:, :].astype(np.float64)
        full = tm.full_prefill(model, np.concatenate(chunk_ids + [suffix]))
        out[f"{tag}_full_logits_last"] = full.logits[-1]
        sel1 = tm.selective_prefill(model, chunks, rankings, suffix, 1.0)
        out[f"{tag}_r1_logits_last"] = sel1.logits[-1]
        sel0 = tm.selective_prefill(model, chunks, rankings, suffix, 0.0)
        out[f"{tag}_r0_logits_last"] = sel0.logits[-1]
    np.savez_compressed(OUT / "toy_cfg1.npz", **out)
    print("toy cfg1 done")


def fuse_cases(ct):
    from cachetune.pipesim import fuse_layer
    rng = np.random.default_rng(4242)
    out = {}
    for i, (n, h, d) in enumerate([(16, 2, 4), (100, 3, 8), (513, 2, 16)]):
        perm = rng.permutation(n)
        m = int(rng.integers(0, n + 1))
        keep, rec = np.sort(perm[m:]), np.sort(perm[:m])
        kr = rng.standard_normal((keep.size, h, d)).astype(np.float32)
        vr = rng.standard_normal((keep.size, h, d)).astype(np.float32)
        kn = rng.standard_normal((rec.size, h, d)).astype(np.float32)
        vn = rng.standard_normal((rec.size, h, d)).astype(np.float32)
        p = ct.RopeParams(head_dim=d)
        K, V = fuse_layer(
            (ct.SeqTensor(kr) if keep.size else None, ct.SeqTensor(vr) if keep.size else None, keep),
            (ct.SeqTensor(kn) if rec.size else None, ct.SeqTensor(vn) if rec.size else None, rec),
            positions=keep, rope_params=p, n=n)
        for name, a in dict(keep=keep, rec=rec, kr=kr, vr=vr, kn=kn, vn=vn,
                            K=K.data, V=V.data).items():
            out[f"f{i}_{name}"] = a
    out["count"] = np.int64(3)
    np.savez_compressed(OUT / "fuse_cases.npz", **out)


def scheduler_cases(ct):
    from cachetune.scheduler import (HardwareProfile, SearchConfig, gss_optimize,
                                     roofline_r0, ttft_model, calibrate)
    from cachetune.pipesim import (RequestSpec, make_sim_evaluator, simulate,
                                   synthetic_plan, timeline_to_csv)
    rng = np.random.default_rng(909)
    out = {}
    for i in range(20):
        p = HardwareProfile(t_c=float(rng.uniform(0.1e-6, 100e-6)),
                            t_i=float(rng.uniform(0.1e-6, 100e-6)),
                            t_o=float(rng.uniform(0.0, 1e-3)))
        cfg = SearchConfig() if i % 2 == 0 else SearchConfig(r_min=0.05, r_max=0.5)
        r0 = roofline_r0(p, cfg)
        r_star, evals, trace = gss_optimize(lambda r: ttft_model(r, 1000, 8, p), r0, cfg)
        out[f"g{i}_p"] = np.array([p.t_c, p.t_i, p.t_o])
        out[f"g{i}_cfg"] = np.array([cfg.r_min, cfg.r_max, cfg.epsilon])
        out[f"g{i}_r0"] = np.float64(r0)
        out[f"g{i}_rstar"] = np.float64(r_star)
        out[f"g{i}_trace"] = np.array(trace, dtype=np.float64)
        plan = synthetic_plan([100, 37, 64], 6, float(rng.uniform(0, 1)), 2, 8)
        tl = simulate(plan, p)
        out[f"g{i}_sim_ratio"] = np.float64(plan.ratio)
        out[f"g{i}_sim"] = np.array([[e.start_s, e.end_s] for e in tl.events])
        out[f"g{i}_sim_ttft"] = np.float64(tl.ttft_s)
        tier = ct.TIER_PRESETS["hdd" if i % 3 == 0 else "cpu-mem"]
        tl2 = simulate(plan, p, tier=tier)
        out[f"g{i}_sim_tier"] = np.array([[e.start_s, e.end_s] for e in tl2.events])
        out[f"g{i}_tier"] = np.array([tier.read_bw, tier.fixed_latency])
        ev = make_sim_evaluator(p, tier=tier)
        cal = [RequestSpec(chunk_tokens=(128, 128, 128), n_layers=4)] * 3
        rep = calibrate(None, None, ev, cal, cfg, profile=p)
        out[f"g{i}_cal_rstar"] = np.float64(rep.r_star)
        out[f"g{i}_cal_trace"] = np.array(rep.trace, dtype=np.float64)
    out["count"] = np.int64(20)
    np.savez_compressed(OUT / "scheduler_cases.npz", **out)


def pool_cases(ct):
    rng = np.random.default_rng(5151)
    out = {}
    for i in range(12):
        n = int(rng.integers(4, 64))
        h = int(rng.integers(1, 4))
        d = 2 * int(rng.integers(1, 5))
        layers = int(rng.integers(1, 4))
        r = float(rng.uniform(0, 1))
        keys = [rng.standard_normal((n, h, d)).astype(np.float32) for _ in range(layers)]
        vals = [rng.standard_normal((n, h, d)).astype(np.float32) for _ in range(layers)]
        chunk = _chunk(ct, keys, vals, cid=f"p{i}")
        rk = ct.rank_chunk(chunk)
        pool = ct.CachePool()
        pool.put_chunk(chunk, rk, ct.TIER_PRESETS["cpu-mem"])
        layer = int(rng.integers(0, layers))
        plan = pool.plan_sparse_fetch(f"p{i}", layer, r)
        out[f"p{i}_geom"] = np.array([layers, n, h, d, layer])
        out[f"p{i}_r"] = np.float64(r)
        out[f"p{i}_keys"] = np.stack(keys)
        out[f"p{i}_vals"] = np.stack(vals)
        out[f"p{i}_keep"] = plan.keep_indices
        out[f"p{i}_ranges"] = np.array(plan.byte_ranges, dtype=np.int64).reshape(-1, 2)
        out[f"p{i}_expected"] = np.int64(plan.expected_bytes)
        out[f"p{i}_ctkv_len"] = np.int64(pool.file_bytes(f"p{i}"))
    out["count"] = np.int64(12)
    np.savez_compressed(OUT / "pool_cases.npz", **out)


def ctkv_cases(ct):
    """Reference-written CTKV files (ranked and bare) for format parity."""
    rng = np.random.default_rng(6161)
    keys = [rng.standard_normal((32, 2, 8)).astype(np.float32) for _ in range(4)]
    vals = [rng.standard_normal((32, 2, 8)).astype(np.float32) for _ in range(4)]
    chunk = _chunk(ct, keys, vals, cid="fmt")
    rk = ct.rank_chunk(chunk, 0.5)
    (OUT / "fmt_ranked.ctkv").write_bytes(ct.write_ctkv(chunk, rk))
    (OUT / "fmt_bare.ctkv").write_bytes(ct.write_ctkv(chunk))


def highband_cases(ct):
    """high_freq_scores / the highfreq strategy ranking (ct/spectral.py:93-96,
    ct/toymodel.py:356-363) over awkward geometries and cutoffs."""
    from cachetune import toymodel
    rng = np.random.default_rng(20261017)
    geoms = [(1, 1, 2, 1), (7, 2, 4, 2), (16, 2, 4, 3), (33, 1, 8, 2), (64, 4, 8, 2),
             (100, 2, 4, 2), (128, 2, 8, 2), (257, 1, 2, 2), (1024, 2, 4, 1), (96, 2, 64, 1)]
    out = {}
    i = 0
    for (n, h, d, l) in geoms:
        for alpha in (0.0, 0.3, 0.5, 1.0):
            keys = [rng.standard_normal((n, h, d)).astype(np.float32) for _ in range(l)]
            vals = [rng.standard_normal((n, h, d)).astype(np.float32) for _ in range(l)]
            rk = toymodel.strategy_ranking(_chunk(ct, keys, vals), "highfreq", alpha)
            out[f"c{i}_keys"] = np.stack(keys)
            out[f"c{i}_vals"] = np.stack(vals)
            out[f"c{i}_alpha"] = np.float64(alpha)
            out[f"c{i}_scores"] = rk.per_layer_scores
            out[f"c{i}_orders"] = np.asarray(rk.per_layer_order).astype(np.int32)
            out[f"c{i}_agg"] = np.asarray(rk.aggregate_order).astype(np.int32)
            i += 1
    out["count"] = np.int64(i)
    np.savez_compressed(OUT / "highband_cases.npz", **out)


def experiment_cases(ct):
    """Per-seed suffix-attention deviations of run_selection_experiment
    (ct/toymodel.py:374-419) for every strategy on the acceptance suite's
    committed seeds (pkg/tests/test_acceptance.py:28,187-201), plus the
    reference's random-strategy permutations for seed 0."""
    from cachetune import toymodel
    seeds = list(range(25))
    out = {"seeds": np.array(seeds)}
    for strategy in toymodel.STRATEGIES:
        res = toymodel.run_selection_experiment(seeds, r=0.15, strategy=strategy)
        out[f"dev_{strategy}"] = np.array([d for _, d in res])
    for strategy in ("lowfreq", "none"):
        res = toymodel.run_selection_experiment([0, 1, 2], 0.25, strategy,
                                                chunk_tokens=(24, 24), suffix_len=6)
        out[f"small_{strategy}"] = np.array([d for _, d in res])
    res = toymodel.run_selection_experiment([3, 4], r=0.3, strategy="lowfreq", mlp=True)
    out["mlp_lowfreq"] = np.array([d for _, d in res])
    np.savez_compressed(OUT / "experiment_cases.npz", **out)


def spectrum_cases(ct):
    """spectrum_report (ct/toymodel.py:315-341) on seeded chunks, incl. odd N."""
    from cachetune import toymodel
    rng = np.random.default_rng(4242)
    out = {}
    for i, (n, h, d, l, nb) in enumerate([(64, 2, 8, 2, 10), (33, 1, 4, 3, 4),
                                          (256, 2, 16, 1, 10), (2, 1, 2, 1, 1)]):
        keys = [rng.standard_normal((n, h, d)).astype(np.float32) for _ in range(l)]
        vals = [(rng.standard_normal((n, h, d)) + 3.0).astype(np.float32) for _ in range(l)]
        rep = toymodel.spectrum_report(_chunk(ct, keys, vals), nb)
        out[f"s{i}_keys"], out[f"s{i}_vals"] = np.stack(keys), np.stack(vals)
        out[f"s{i}_bands"] = np.int64(nb)
        out[f"s{i}_key"], out[f"s{i}_value"] = rep["key"], rep["value"]
    out["count"] = np.int64(4)
    np.savez_compressed(OUT / "spectrum_cases.npz", **out)


def main():
    ct = _ref()
    if len(sys.argv) > 1:  # regenerate only the named fixtures
        for name in sys.argv[1:]:
            globals()[name](ct)
        return
    highband_cases(ct)
    experiment_cases(ct)
    spectrum_cases(ct)
    ctkv_cases(ct)
    spectral_cases(ct)
    big_chunks(ct)
    rope_cases(ct)
    fuse_cases(ct)
    scheduler_cases(ct)
    pool_cases(ct)
    toy_cfg1(ct)


if __name__ == "__main__":
    main()
