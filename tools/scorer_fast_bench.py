#!/usr/bin/env python
"""Time the fast scorer on one config-2 request (16 chunks x 32 layers x
[2048, 8, 128] bf16 K/V, Gaussian) -- for ncu launch lists / captures."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_24022_b200.spectral import score_select_fast  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    g = torch.Generator(device="cuda").manual_seed(0)
    k = torch.randn((16, 32, 2048, 8, 128), device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn((16, 32, 2048, 8, 128), device="cuda", generator=g).to(torch.bfloat16)
    score_select_fast(k, v, 308)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        score_select_fast(k, v, 308)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    print(f"fast scorer: {ms:.3f} ms per request  {2 * k.numel() * 2 / ms / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
