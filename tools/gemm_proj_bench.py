#!/usr/bin/env python
"""ct_gemm_bf16 (CTA-pair tcgen05) against cuBLAS on the step's dense
projections, K / N of Llama-3-8B and Mistral-7B: QKV (bf16 store), O and
down (f32 residual accumulate, cuBLAS addmm beta = 1 with f32 C).  CUDA events
on the launching stream, 3 warm-ups, median of 20.

    python tools/gemm_proj_bench.py [--rows 4992 9920] [--out FILE]"""

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
    ap.add_argument("--rows", type=int, nargs="+", default=[4992, 9920])
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    from paper_2605_24022_b200 import _lib
    st = torch.cuda.current_stream().cuda_stream
    g = torch.Generator(device="cuda").manual_seed(0)
    rows = []
    for M in args.rows:
        for name, K, N, acc in (("qkv", 4096, 6144, 0), ("o", 4096, 4096, 1),
                                ("down", 14336, 4096, 1)):
            x = torch.randn((M, K), device="cuda", generator=g).to(torch.bfloat16)
            w = (torch.randn((K, N), device="cuda", generator=g) / 64).to(torch.bfloat16)
            if acc:
                out = torch.zeros((M, N), device="cuda")

                def ours():
                    _lib.call("ct_gemm_bf16", x.data_ptr(), M, K, K, w.data_ptr(), N, N,
                              out.data_ptr(), N, _lib.CT_F32, 1, st)

                def ref():
                    torch.ops.aten.addmm.dtype_out(out, x, w, torch.float32, beta=1, alpha=1,
                                                   out=out)
            else:
                out = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)

                def ours():
                    _lib.call("ct_gemm_bf16", x.data_ptr(), M, K, K, w.data_ptr(), N, N,
                              out.data_ptr(), N, _lib.CT_BF16, 0, st)

                def ref():
                    torch.mm(x, w, out=out)
            to, tr = timed(ours), timed(ref)
            flop = 2.0 * M * K * N
            rows.append({"rows": M, "proj": name, "ours_us": round(to * 1e3, 1),
                         "cublas_us": round(tr * 1e3, 1), "ours_tflops": round(flop / to / 1e9, 1),
                         "cublas_tflops": round(flop / tr / 1e9, 1), "speedup": round(tr / to, 3)})
            print(json.dumps(rows[-1]), flush=True)
            del x, w, out
    if args.out:
        Path(args.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
