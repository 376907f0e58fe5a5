#!/usr/bin/env python
"""Time the fast scorer on one config-2 request (16 chunks x 32 layers x
[2048, 8, 128] bf16 K/V, Gaussian) -- for A/B runs, ncu launch lists and
captures.

    python tools/scorer_fast_bench.py [iters] [--lib other.so] [--dump f.pt]

k = 0 times the energy kernel + combine + order alone (no boundary window);
k = 308 adds the certified boundary (window re-scores)."""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_24022_b200 import _lib  # noqa: E402
from paper_2605_24022_b200.spectral import score_select_fast  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("iters", nargs="?", type=int, default=3)
    ap.add_argument("--lib", default="")
    ap.add_argument("--dump", default="")
    args = ap.parse_args()
    if args.lib:
        _lib._lib = _lib.load(args.lib)
    g = torch.Generator(device="cuda").manual_seed(0)
    k = torch.randn((16, 32, 2048, 8, 128), device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn((16, 32, 2048, 8, 128), device="cuda", generator=g).to(torch.bfloat16)
    for ksel in (0, 308):
        out = score_select_fast(k, v, ksel)
        torch.cuda.synchronize()
        times = []
        for _ in range(args.iters):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            out = score_select_fast(k, v, ksel)
            e.record()
            torch.cuda.synchronize()
            times.append(s.elapsed_time(e))
        times.sort()
        ms = times[len(times) // 2]
        print(f"fast scorer k={ksel}: {ms:.3f} ms per request (median of {args.iters})  "
              f"{2 * k.numel() * 2 / ms / 1e6:.0f} GB/s  windows {out['wcount'].tolist()}")
    if args.dump:
        torch.save({"agg": out["agg"].cpu(), "order": out["agg_order"].cpu()}, args.dump)


if __name__ == "__main__":
    main()
