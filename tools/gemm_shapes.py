#!/usr/bin/env python
"""cuBLAS time of the four per-layer projections of the config-2 step vs the
row count M (active rows), to see wave-quantisation effects.  bf16 A/B; the
O / down projections accumulate into an f32 residual (beta = 1) like the step."""
import sys

import torch

def t(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / it

hid, inter, qkv = 4096, 14336, 6144
W = {"qkv": torch.randn(hid, qkv, device="cuda").bfloat16(),
     "o": torch.randn(hid, hid, device="cuda").bfloat16(),
     "gu": torch.randn(hid, 2 * inter, device="cuda").bfloat16(),
     "d": torch.randn(inter, hid, device="cuda").bfloat16()}
for M in [int(x) for x in (sys.argv[1:] or [4864, 4992, 5120, 5248, 5376])]:
    x = torch.randn(M, hid, device="cuda").bfloat16()
    a = torch.randn(M, inter, device="cuda").bfloat16()
    h = torch.zeros(M, hid, device="cuda")
    o_qkv = torch.empty(M, qkv, device="cuda", dtype=torch.bfloat16)
    o_gu = torch.empty(M, 2 * inter, device="cuda", dtype=torch.bfloat16)
    r = {
        "qkv": t(lambda: torch.mm(x, W["qkv"], out=o_qkv)),
        "o": t(lambda: torch.ops.aten.addmm.dtype_out(h, x, W["o"], torch.float32, beta=1, alpha=1, out=h)),
        "gu": t(lambda: torch.mm(x, W["gu"], out=o_gu)),
        "d": t(lambda: torch.ops.aten.addmm.dtype_out(h, a, W["d"], torch.float32, beta=1, alpha=1, out=h)),
    }
    tot = sum(r.values())
    fl = 2 * M * (hid * qkv + hid * hid + hid * 2 * inter + inter * hid)
    print(f"M={M}: " + " ".join(f"{k} {v*1e3:.0f}us" for k, v in r.items())
          + f"  total {tot:.3f} ms  {fl / tot / 1e9:.0f} TFLOP/s  per-row {tot / M * 1e3:.2f} us")
