#!/usr/bin/env python
"""Exact (float64) GPU scorer vs the float64 numpy oracle at full config-2
chunk size: every per-layer order and the aggregate order bit-exact, scores
within 1e-11 relative, on many model-encoded chunks.

    python tools/scorer_exact_check.py [--chunks 64] [--seed 0] [--out FILE]

Chunks: 2048 tokens each, encoded by the Llama-3-8B-geometry model (32
layers, random init, seeded) from random token ids.  The GPU side is
`rank_chunks` (fft2_energy_kernel + device orders); the oracle is
oracle/cachetune_oracle.rank_chunk (numpy pocketfft in float64, the
reference's own arithmetic, ct/spectral.py:69-101,149-159), run in a process
pool over the host cores.  Test infrastructure: the oracle is the checker."""

import argparse
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def _oracle(args):
    keys, vals = args
    from oracle import cachetune_oracle as O
    return O.rank_chunk(list(keys), list(vals), 0.5)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunks", type=int, default=64)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import torch
    import paper_2605_24022_b200 as ct
    cfg = ct.ModelConfig.llama3_8b(n_layers=32, vocab_size=128256, seed=args.seed + 100)
    model = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
    rng = np.random.default_rng(args.seed)
    gpu_s = cpu_s = 0.0
    workers = max(1, (os.cpu_count() or 2) - 1)
    agg_bad = lay_bad = n_done = 0
    worst = 0.0
    with ProcessPoolExecutor(workers) as ex:
        for b in range(0, args.chunks, 16):  # batches of 16: bounded host memory
            tg = time.time()
            chunks = [ct.encode_chunk_isolated(model, rng.integers(0, cfg.vocab_size, size=2048),
                                               chunk_id=f"c{b + j}")
                      for j in range(min(16, args.chunks - b))]
            ranks = ct.rank_chunks(chunks)
            host = [(c.keys.float().cpu().numpy(), c.values.float().cpu().numpy()) for c in chunks]
            del chunks
            gpu_s += time.time() - tg
            tc = time.time()
            want = list(ex.map(_oracle, host, chunksize=1))
            cpu_s += time.time() - tc
            for rk, (scores, orders, agg) in zip(ranks, want):
                agg_bad += int(not np.array_equal(rk.aggregate_order, agg))
                lay_bad += int(sum(not np.array_equal(a, c) for a, c in zip(rk.per_layer_order, orders)))
                worst = max(worst, float(np.max(np.abs(rk.per_layer_scores - scores) / scores)))
            n_done += len(ranks)
            print(f"{n_done} chunks: agg mismatches {agg_bad}, layer mismatches {lay_bad}, "
                  f"max rel score diff {worst:.2e}", file=sys.stderr, flush=True)
            del host, want, ranks
    out = {"chunks": n_done, "layers_per_chunk": 32, "tokens_per_chunk": 2048,
           "aggregate_order_mismatch": agg_bad, "per_layer_order_mismatch": lay_bad,
           "max_rel_score_diff": worst, "gpu_encode_and_score_s": round(gpu_s, 1),
           "oracle_cpu_s": round(cpu_s, 1), "oracle_workers": workers}
    print(json.dumps(out))
    if args.out:
        Path(args.out).write_text(json.dumps(out, indent=1))
    assert agg_bad == 0 and lay_bad == 0 and worst < 1e-11, out


if __name__ == "__main__":
    main()
