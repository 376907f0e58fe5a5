#!/usr/bin/env python
"""Microbenchmark of the scorer (ct_score_chunks) on one config-2 request:
16 chunks x 32 layers x [2048, 8, 128] bf16 K and V (4.29 GB read)."""

import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_24022_b200.spectral import score_device  # noqa: E402


def main():
    C = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
    gen = torch.Generator(device="cuda").manual_seed(0)
    k = torch.randn((C, 32, N, 8, 128), device="cuda", generator=gen).to(torch.bfloat16)
    v = torch.randn((C, 32, N, 8, 128), device="cuda", generator=gen).to(torch.bfloat16)
    nbytes = 2 * k.numel() * 2
    for prec in ("f64", "f32"):
        score_device(k, v, 0.5, prec, want_layer_order=False)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(3):
            score_device(k, v, 0.5, prec, want_layer_order=False)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 3
        print(f"scorer {prec}: {C} chunks {ms:.2f} ms  {nbytes / ms / 1e6:.0f} GB/s  "
              f"({ms / C:.3f} ms per {N}-token chunk of 32 layers)")


if __name__ == "__main__":
    main()
