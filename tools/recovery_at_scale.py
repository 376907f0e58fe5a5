"""Attention-recovery check at config-2 geometry.

    python tools/recovery_at_scale.py [--layers 32] [--chunks 16] [--tokens 2048]
        [--suffix 64] [--r 0.15] [--out profiles/round1_recovery_cfg2.json]

Random-init Llama-3-8B-geometry weights (bf16), chunks encoded in isolation,
every strategy at the same recompute budget; suffix-row attention recorded on
the device against a full recompute of the same prompt.
"""

import argparse
import json
import time

import numpy as np
import torch

import paper_2605_24022_b200 as ct
from paper_2605_24022_b200.experiments import attention_recovery_at_scale


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--chunks", type=int, default=16)
    ap.add_argument("--tokens", type=int, default=2048)
    ap.add_argument("--suffix", type=int, default=64)
    ap.add_argument("--r", type=float, nargs="+", default=[0.15])
    ap.add_argument("--seed", type=int, default=5)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = ct.ModelConfig.llama3_8b(n_layers=a.layers, seed=a.seed)
    m = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
    rng = np.random.default_rng(a.seed)
    toks = [rng.integers(0, cfg.vocab_size, size=a.tokens) for _ in range(a.chunks)]
    suffix = rng.integers(0, cfg.vocab_size, size=a.suffix)
    res = {"geometry": f"llama3_8b layers={a.layers} chunks={a.chunks}x{a.tokens} "
                       f"suffix={a.suffix} bf16", "seed": a.seed, "by_r": {}}
    for r in a.r:
        t0 = time.time()
        dev = attention_recovery_at_scale(m, toks, suffix, r, seed=a.seed)
        res["by_r"][str(r)] = dev
        print(f"r={r}: {json.dumps(dev)} ({time.time() - t0:.1f}s)", flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
