#!/usr/bin/env python
"""ct_gemm_qkv_rope vs torch.mm + ct_qkv_rope_scatter at the step's and the
full prefill's row counts (Llama-3-8B q|k|v: K 4096, 32 q / 8 kv heads),
CUDA events, 3 warm-ups, median of 15.  python tools/qkv_rows_bench.py"""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_24022_b200 import _lib  # noqa: E402
from paper_2605_24022_b200.model import ModelConfig  # noqa: E402
from paper_2605_24022_b200.rope import rope_table  # noqa: E402


def timed(fn, reps=15):
    for _ in range(3):
        fn()
    out = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        out.append(s.elapsed_time(e) * 1e3)
    return statistics.median(out)


def main():
    hq, hkv, d, k = 32, 8, 128, 4096
    n = (hq + 2 * hkv) * d
    params = ModelConfig.llama3_8b(n_layers=1).rope_params
    st = torch.cuda.current_stream().cuda_stream
    for m in (2048, 4992, 9920, 16384, 32832, 65600):
        n_ctx = max(m, 65600)
        table = rope_table(params, n_ctx, "f32", torch.device("cuda"))
        x = torch.randn((m, k), device="cuda").to(torch.bfloat16)
        w = (torch.randn((k, n), device="cuda") / k ** 0.5).to(torch.bfloat16)
        pos = torch.arange(m, device="cuda", dtype=torch.int32)
        q = torch.empty((m, hq, d), device="cuda", dtype=torch.bfloat16)
        kc = torch.empty((n_ctx, hkv, d), device="cuda", dtype=torch.bfloat16)
        vc = torch.empty_like(kc)
        qkv = torch.empty((m, n), device="cuda", dtype=torch.bfloat16)
        lib = _lib.load()

        def fused():
            _lib.call("ct_gemm_qkv_rope", x.data_ptr(), m, k, k, w.data_ptr(), n, pos.data_ptr(),
                      table.data_ptr(), hq, hkv, d, q.data_ptr(), kc.data_ptr(), vc.data_ptr(),
                      hkv * d, st)

        def unfused():
            torch.mm(x, w, out=qkv)
            _lib.check(lib.ct_qkv_rope_scatter(
                qkv.data_ptr(), n, _lib.CT_BF16, pos.data_ptr(), m, hq, hkv, d,
                params.pairing_code, table.data_ptr(), q.data_ptr(), _lib.CT_BF16, kc.data_ptr(),
                vc.data_ptr(), _lib.CT_BF16, hkv * d, None, st), "ct_qkv_rope_scatter")
        tf, tu = timed(fused), timed(unfused)
        fl = 2.0 * m * k * n
        print(json.dumps({"rows": m, "fused_us": round(tf, 1), "unfused_us": round(tu, 1),
                          "fused_tflops": round(fl / tf / 1e6, 1), "speedup": round(tu / tf, 3)}))


if __name__ == "__main__":
    main()
