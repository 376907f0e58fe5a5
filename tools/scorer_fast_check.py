#!/usr/bin/env python
"""Fast (single-precision, certified-boundary) scorer vs the exact float64
scorer on config-2-size chunks: accuracy calibration, selection equality and
timing.

    python tools/scorer_fast_check.py [--batches 64] [--gauss 8] [--out FILE]

Each batch = 16 chunks x 32 layers x [2048, 8, 128] bf16 K/V encoded by the
Llama-3-8B-geometry model (random init, seeded) from random token ids; --gauss
adds batches of N(0,1) chunks (the reference CLI's synthetic data).  Per
chunk: max relative error of the single-precision aggregate scores (guard 0
run), the certified top-k set (default guard) == the float64 top-k set at
k = 308 (r = 0.15), window statistics.  Times both scorers per request."""

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_24022_b200 as ct  # noqa: E402
from paper_2605_24022_b200.spectral import (FAST_GUARD, score_device,  # noqa: E402
                                            score_select_fast, selection_count)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=4)
    ap.add_argument("--gauss", type=int, default=2)
    ap.add_argument("--r", type=float, default=0.15)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    C, N = 16, 2048
    k = selection_count(args.r, N)
    cfg = ct.ModelConfig.llama3_8b(n_layers=32, seed=11)
    model = ct.GpuModel.random(cfg, dtype=torch.bfloat16) if args.batches else None
    stats = {"chunks": 0, "model_chunks": 0, "gauss_chunks": 0, "set_mismatch": 0,
             "max_rel_err": 0.0, "rel_err_p999": [], "window_hist": {}, "fallback": 0,
             "guard": FAST_GUARD, "k": k}
    times = {"fast": [], "exact": []}
    errs = []
    for b in range(args.batches + args.gauss):
        if b < args.batches:
            rng = np.random.default_rng(1000 + b)
            chunks = [ct.encode_chunk_isolated(model, rng.integers(0, cfg.vocab_size, size=N),
                                               chunk_id=f"b{b}c{j}") for j in range(C)]
            kk = torch.stack([torch.stack(list(c.keys)) for c in chunks])
            vv = torch.stack([torch.stack(list(c.values)) for c in chunks])
            del chunks
            stats["model_chunks"] += C
        else:
            g = torch.Generator(device="cuda").manual_seed(b)
            kk = torch.randn((C, 32, N, 8, 128), device="cuda", generator=g).to(torch.bfloat16)
            vv = torch.randn((C, 32, N, 8, 128), device="cuda", generator=g).to(torch.bfloat16)
            stats["gauss_chunks"] += C
        ex = score_device(kk, vv, 0.5, "f64", want_layer_order=False)
        raw = score_select_fast(kk, vv, k, guard=0.0)
        fa = score_select_fast(kk, vv, k)
        a = ex["agg"].cpu().numpy()
        rel = np.abs(raw["agg"].cpu().numpy() - a) / np.maximum(a, 1e-300)
        errs.append(rel.max(axis=1))
        eo = ex["agg_order"].cpu().numpy()
        fo = fa["agg_order"].cpu().numpy()
        for c in range(C):
            if not np.array_equal(np.sort(eo[c, :k]), np.sort(fo[c, :k])):
                stats["set_mismatch"] += 1
        wc = fa["wcount"].cpu().numpy()
        for w in wc:
            stats["window_hist"][int(w)] = stats["window_hist"].get(int(w), 0) + 1
        stats["fallback"] += int((wc < 0).sum())
        stats["chunks"] += C
        if b in (0, args.batches):  # time one model batch and one Gaussian batch
            times["fast"].append(timed(lambda: score_select_fast(kk, vv, k)))
            times["exact"].append(timed(lambda: score_device(kk, vv, 0.5, "f64",
                                                             want_layer_order=False)))
        del kk, vv, ex, raw, fa
        print(f"batch {b}: chunks {stats['chunks']} mismatches {stats['set_mismatch']} "
              f"max rel err {np.concatenate(errs).max():.3e}", flush=True)
    allerr = np.concatenate(errs)
    stats["max_rel_err"] = float(allerr.max())
    stats["rel_err_p999"] = float(np.quantile(allerr, 0.999))
    stats["guard_over_max_err"] = float(FAST_GUARD / allerr.max())
    stats["ms_per_request_fast"] = times["fast"]
    stats["ms_per_request_exact"] = times["exact"]
    nbytes = 2 * C * 32 * N * 1024 * 2
    stats["hbm_gbs_fast"] = [nbytes / (t * 1e-3) / 1e9 for t in times["fast"]]
    stats["window_hist"] = {str(kk_): v for kk_, v in sorted(stats["window_hist"].items())}
    print(json.dumps(stats))
    if args.out:
        Path(args.out).write_text(json.dumps(stats, indent=1))


if __name__ == "__main__":
    main()
