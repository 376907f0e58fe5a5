#!/usr/bin/env python
"""Microbenchmark of the HBM-bound row movers at config-2 shapes, one layer:

  blend  ct_gather_rope_blend: 16 chunks x 1740 keep rows, K/V [8,128] bf16,
         read keep rows from an importance-ordered pool + write rotated K / raw V
         into the blended cache (228 MB algorithmic per launch)
  qkv    ct_qkv_rope_scatter: A=4992 rows of q|k|v (48 heads x 128) bf16 in,
         q (rotated) + cache K (rotated) + cache V + raw K out (123 MB + raw K)

Timed with CUDA events on the launching stream, averaged over many launches,
each launch's inputs rotated across several copies so that the working set
exceeds L2 (no cross-launch L2 reuse)."""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_24022_b200 import _dev, _lib  # noqa: E402
from paper_2605_24022_b200.rope import RopeParams, rope_table  # noqa: E402


def ev_time(fn, iters):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(0)
    torch.cuda.synchronize()
    s.record()
    for i in range(iters):
        fn(i)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    dev = torch.device("cuda")
    C, N, k, H, D, S = 16, 2048, 308, 8, 128, 64
    keep = N - k
    n_ctx = C * N + S
    params = RopeParams(head_dim=D, base=500000.0)
    table = rope_table(params, n_ctx, "f32", dev)
    st = _dev.stream_handle()
    COPIES = 4
    # pool [C][N][2][H][D] per layer copy, importance tail = rows k..N
    pools = [torch.randn((C, N, 2, H, D), device=dev).to(torch.bfloat16) for _ in range(COPIES)]
    agg = torch.stack([torch.randperm(N, device=dev) for _ in range(C)]).to(torch.int32)
    caches = [torch.empty((2, n_ctx, H, D), dtype=torch.bfloat16, device=dev)
              for _ in range(COPIES)]
    esz = 2
    segsets = []
    for i in range(COPIES):
        segs = []
        for c in range(C):
            base = pools[i][c, k].data_ptr()
            tok = agg.data_ptr() + (c * N + k) * 4
            segs.append(_lib.Segment(base, base + H * D * esz, tok, keep, c * N, 0))
        segsets.append((_lib.Segment * C)(*segs))

    def blend(i):
        j = i % COPIES
        _lib.call("ct_gather_rope_blend", segsets[j], C, 2 * H * D, H, D, _dev.ct_dtype(torch.bfloat16),
                  params.pairing_code, _dev.ptr(table), _dev.ptr(caches[j][0]),
                  _dev.ptr(caches[j][1]), H * D, st)

    ms = ev_time(blend, 50)
    nbytes = 2 * 2 * C * keep * H * D * esz
    print(f"blend: {ms * 1e3:.1f} us  {nbytes / ms / 1e6:.0f} GB/s  ({nbytes / 1e6:.1f} MB)")

    A, Hq = C * k + S, 32
    hpr = Hq + 2 * H
    qkvs = [torch.randn((A, hpr * D), device=dev).to(torch.bfloat16) for _ in range(COPIES)]
    pos = torch.sort(torch.randperm(n_ctx, device=dev)[:A]).values.to(torch.int32)
    qouts = [torch.empty((A, Hq, D), dtype=torch.bfloat16, device=dev) for _ in range(COPIES)]
    kraws = [torch.empty((A, H, D), dtype=torch.bfloat16, device=dev) for _ in range(COPIES)]

    def qkv(i):
        j = i % COPIES
        _lib.call("ct_qkv_rope_scatter", _dev.ptr(qkvs[j]), hpr * D, _dev.ct_dtype(torch.bfloat16),
                  _dev.ptr(pos), A, Hq, H, D, params.pairing_code, _dev.ptr(table),
                  _dev.ptr(qouts[j]), _dev.ct_dtype(torch.bfloat16), _dev.ptr(caches[j][0]),
                  _dev.ptr(caches[j][1]), _dev.ct_dtype(torch.bfloat16), H * D,
                  _dev.ptr(kraws[j]), st)

    ms = ev_time(qkv, 50)
    nbytes = A * hpr * D * 2 * 2 + A * H * D * 2
    print(f"qkv:   {ms * 1e3:.1f} us  {nbytes / ms / 1e6:.0f} GB/s  ({nbytes / 1e6:.1f} MB)")
    del qkvs, qouts, kraws, pools, caches
    torch.cuda.empty_cache()

    # SwiGLU: gate|up [A, 2*inter] bf16 -> act [A, inter] bf16
    inter, hid = 14336, 4096
    gus = [torch.randn((A, 2 * inter), device=dev).to(torch.bfloat16) for _ in range(COPIES)]
    acts = [torch.empty((A, inter), dtype=torch.bfloat16, device=dev) for _ in range(COPIES)]

    def swiglu(i):
        j = i % COPIES
        _lib.call("ct_mlp_act", _dev.ptr(gus[j]), A, inter, _dev.ct_dtype(torch.bfloat16), 0,
                  _dev.ptr(acts[j]), _dev.ct_dtype(torch.bfloat16), st)

    ms = ev_time(swiglu, 50)
    nbytes = A * inter * 2 * 3
    print(f"swiglu: {ms * 1e3:.1f} us  {nbytes / ms / 1e6:.0f} GB/s  ({nbytes / 1e6:.1f} MB)")
    del gus, acts
    torch.cuda.empty_cache()

    # rmsnorm: h [A, hid] f32 -> x [A, hid] bf16
    hs = [torch.randn((A, hid), device=dev) for _ in range(COPIES * 4)]
    xs = [torch.empty((A, hid), dtype=torch.bfloat16, device=dev) for _ in range(COPIES * 4)]

    def rms(i):
        j = i % (COPIES * 4)
        _lib.call("ct_residual_rmsnorm", _dev.ptr(hs[j]), None, _lib.CT_F32, A, hid, 1e-6,
                  _dev.ptr(xs[j]), _dev.ct_dtype(torch.bfloat16), st)

    ms = ev_time(rms, 100)
    nbytes = A * hid * (4 + 2)
    print(f"rmsnorm: {ms * 1e3:.1f} us  {nbytes / ms / 1e6:.0f} GB/s  ({nbytes / 1e6:.1f} MB)")


if __name__ == "__main__":
    np.random.seed(0)
    main()
