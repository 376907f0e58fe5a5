#!/usr/bin/env python
"""Fused gate/up + SwiGLU (ct_gemm_swiglu) against the unfused pair
(cuBLAS torch.mm -> ct_mlp_act) on the step's shapes, K = 4096, I = 14336
(Llama-3-8B / Mistral-7B MLP).  CUDA events on the launching stream, 3
warm-ups, median of 20; the inputs of every shape exceed L2 except A itself.

    python tools/gemm_swiglu_bench.py [--out FILE]

Rows: 2048 (one chunk encode), 4992 (config-2 selective step), 9920 (config
3 selective step), 32832 (config-2 full prefill).  TFLOP/s counts the GEMM's
2·M·K·2I flops; the fused kernel's HBM floor is x + W + act."""

import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def timed(fn, reps=20):
    st = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    from paper_2605_24022_b200 import _lib
    K, I = 4096, 14336
    st = torch.cuda.current_stream().cuda_stream
    g = torch.Generator(device="cuda").manual_seed(0)
    w = (torch.randn((K, 2 * I), device="cuda", generator=g) / 64).to(torch.bfloat16)
    rows = []
    for M in (2048, 4992, 9920, 32832):
        x = torch.randn((M, K), device="cuda", generator=g).to(torch.bfloat16)
        act = torch.empty((M, I), device="cuda", dtype=torch.bfloat16)
        gu = torch.empty((M, 2 * I), device="cuda", dtype=torch.bfloat16)

        def fused():
            _lib.call("ct_gemm_swiglu", x.data_ptr(), M, K, K, w.data_ptr(), I, 2 * I,
                      act.data_ptr(), I, st)

        def mm():
            torch.mm(x, w, out=gu)

        def unfused():
            torch.mm(x, w, out=gu)
            _lib.call("ct_mlp_act", gu.data_ptr(), M, I, _lib.CT_BF16, 0, act.data_ptr(),
                      _lib.CT_BF16, st)

        tf, tm, tu = timed(fused), timed(mm), timed(unfused)
        flop = 2.0 * M * K * 2 * I
        rows.append({"rows": M, "fused_us": round(tf * 1e3, 1), "cublas_mm_us": round(tm * 1e3, 1),
                     "cublas_mm_plus_act_us": round(tu * 1e3, 1),
                     "fused_tflops": round(flop / tf / 1e9, 1),
                     "cublas_mm_tflops": round(flop / tm / 1e9, 1),
                     "speedup_vs_unfused": round(tu / tf, 3)})
        print(json.dumps(rows[-1]), flush=True)
        del x, act, gu
    if args.out:
        Path(args.out).write_text(json.dumps({"shape": f"[M,{K}] x [{K},{2 * I}] -> SwiGLU [M,{I}]",
                                              "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
