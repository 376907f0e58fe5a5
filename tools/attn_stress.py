#!/usr/bin/env python
"""Repeatedly launch the tcgen05 attention at a given shape and check each run
(used to chase intermittent failures).  python tools/attn_stress.py A N ITERS [QSCALE] [KSPIKE]"""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_24022_b200 import _dev, _lib  # noqa: E402

A, N, iters = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
qs = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
spike = float(sys.argv[5]) if len(sys.argv) > 5 else 0.0
hq, hkv, d = 32, 8, 128
rng = np.random.default_rng(0)
pos = np.sort(rng.choice(N - 64, A - 64, replace=False))
pos = np.concatenate([pos, np.arange(N - 64, N)])
gen = torch.Generator(device="cuda").manual_seed(0)
q = (qs * torch.randn((A, hq, d), device="cuda", generator=gen)).to(torch.bfloat16)
k = torch.randn((N, hkv, d), device="cuda", generator=gen)
if spike:
    # a ramp of key scale so the running max keeps growing across blocks
    k = k * (1.0 + spike * torch.linspace(0, 1, N, device="cuda")[:, None, None])
k = k.to(torch.bfloat16)
v = torch.randn((N, hkv, d), device="cuda", generator=gen).to(torch.bfloat16)
p = torch.as_tensor(pos.astype(np.int32), device="cuda")
out = torch.empty_like(q)
ref = None
for i in range(iters):
    _lib.call("ct_selective_attention", _dev.ptr(q), _dev.ptr(p), A, hq, _dev.ptr(k), _dev.ptr(v),
              N, hkv, d, hkv * d, 1 / d ** 0.5, 1, _dev.ptr(out), 1, None, None, 0,
              _dev.stream_handle())
    torch.cuda.synchronize()
    if ref is None:
        ref = out.clone()
    elif not torch.equal(ref, out):
        print("iteration", i, "differs: max", (ref.float() - out.float()).abs().max().item())
print("done", A, N, iters, qs, spike)
