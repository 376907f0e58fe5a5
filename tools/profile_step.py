#!/usr/bin/env python
"""One profiled request of the bench workload, for ncu.

    ncu --profile-from-start off ... python tools/profile_step.py [--what step|scorer|full]

Builds the config-2 engine exactly like bench.py, runs one warm-up request,
then brackets ONE request (or one scorer pass / full prefill) with
cudaProfilerStart/Stop so ncu sees only that launch list.
"""

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2605_24022_b200 as ct  # noqa: E402
from paper_2605_24022_b200.pipeline import FullPrefillEngine, SelectivePrefillEngine  # noqa: E402
from paper_2605_24022_b200.pool import KvPool  # noqa: E402
from paper_2605_24022_b200.spectral import score_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="step", choices=["step", "scorer", "scorer32", "full"])
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--chunks", type=int, default=16)
    args = ap.parse_args()
    cfg = ct.ModelConfig.llama3_8b(n_layers=args.layers, seed=1234)
    model = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
    rng = np.random.default_rng([0, 7])
    toks = [rng.integers(0, cfg.vocab_size, size=2048) for _ in range(args.chunks)]
    suffix = torch.as_tensor(rng.integers(0, cfg.vocab_size, size=64).astype(np.int32),
                             device="cuda")
    chunks = [ct.encode_chunk_isolated(model, t, chunk_id=f"c{j}") for j, t in enumerate(toks)]
    keys = torch.stack([c.keys for c in chunks])
    vals = torch.stack([c.values for c in chunks])
    if args.what.startswith("scorer"):
        prec = "f32" if args.what == "scorer32" else "f64"
        score_device(keys, vals, 0.5, prec, want_layer_order=False)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        score_device(keys, vals, 0.5, prec, want_layer_order=False)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return
    ranks = ct.rank_chunks(chunks)
    del keys, vals
    if args.what == "full":
        full = FullPrefillEngine(model, args.chunks * 2048 + 64)
        tok = torch.cat([torch.cat([c.tokens for c in chunks]), suffix])
        full.step(tok)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        full.step(tok)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return
    pool = KvPool(chunks, ranks, "hbm")
    del chunks
    eng = SelectivePrefillEngine(model, pool, 0.15, 64)
    eng.step(suffix)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    eng.step(suffix)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
