#!/usr/bin/env python
"""Microbenchmark of ct_selective_attention at the config-2 layer shape.

    python tools/attn_bench.py [--qscale 1.0] [--full]

Queries: 4992 rows (16 x 308 selected positions spread over 16 x 2048 chunks
+ 64 suffix rows), 32 q-heads / 8 kv-heads, D=128, n_ctx 32832.  Reports the
mean launch time (CUDA events) and TFLOP/s against the algorithmic
4*Hq*D*sum(pos+1).  --full times the dense-causal full-prefill shape.
"""

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_24022_b200 import _dev, _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--qscale", type=float, default=1.0)
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--lib", default="", help="alternative libcachetune_b200.so (A/B)")
    ap.add_argument("--dump", default="", help="save the output tensor (bit-identity A/B)")
    ap.add_argument("--rows", type=int, default=0,
                    help="only the last ROWS query rows (the few-row split-key path)")
    args = ap.parse_args()
    if args.lib:
        _lib._lib = _lib.load(args.lib)
    hq, hkv, d = 32, 8, 128
    rng = np.random.default_rng(0)
    if args.full:
        n = 32832
        pos = np.arange(n)
    else:
        pos = np.concatenate([np.sort(rng.choice(2048, 308, replace=False)) + c * 2048
                              for c in range(16)] + [np.arange(32768, 32832)])
        n = 32832
    if args.rows:
        pos = pos[-args.rows:]
    a = pos.size
    gen = torch.Generator(device="cuda").manual_seed(0)
    q = (args.qscale * torch.randn((a, hq, d), device="cuda", generator=gen)).to(torch.bfloat16)
    k = torch.randn((n, hkv, d), device="cuda", generator=gen).to(torch.bfloat16)
    v = torch.randn((n, hkv, d), device="cuda", generator=gen).to(torch.bfloat16)
    p = torch.as_tensor(pos.astype(np.int32), device="cuda")
    out = torch.empty_like(q)
    flops = 4.0 * hq * d * float(np.sum(pos + 1.0))

    wsb = _lib.load().ct_attention_workspace_bytes(a, hq, n, hkv, d, _lib.CT_BF16)
    ws = _dev.workspace(wsb, "bench")

    def run():
        _lib.call("ct_selective_attention", _dev.ptr(q), _dev.ptr(p), a, hq, _dev.ptr(k),
                  _dev.ptr(v), n, hkv, d, hkv * d, 1 / d ** 0.5, _lib.CT_BF16, _dev.ptr(out),
                  _lib.CT_BF16, None, _dev.ptr(ws), wsb, _dev.stream_handle())
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.iters):
        run()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / args.iters
    kv_gbs = 2 * n * hkv * d * 2 / ms / 1e6
    if args.dump:
        torch.save(out.cpu(), args.dump)
    print(f"attention {'full' if args.full else 'selective'} A={a} n_ctx={n} qscale={args.qscale}: "
          f"{ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s  (K+V once: {kv_gbs:.0f} GB/s)")


if __name__ == "__main__":
    main()
