#!/usr/bin/env python
"""Randomised check of ct_selective_attention (default ping-pong tcgen05 kernel):
random GQA geometry, query count, context length, sorted / unsorted positions,
score scale and a key-scale ramp (forces running-max growth, i.e. the lazy O
rescale), compared on sampled rows with a PyTorch fp32 reference, and every
case launched twice to catch non-deterministic results (races).

    python tools/attn_fuzz.py [CASES] [SEED]
"""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_24022_b200 import _dev, _lib  # noqa: E402


def ref_rows(q, pos, k, v, hq, hkv, rows):
    d = q.shape[-1]
    g = hq // hkv
    out = []
    for a in rows.tolist():
        p = int(pos[a])
        qa = q[a].float()                                  # [hq, d]
        kk = k[: p + 1].float().repeat_interleave(g, dim=1)  # [p+1, hq, d]
        vv = v[: p + 1].float().repeat_interleave(g, dim=1)
        s = torch.einsum("hd,nhd->hn", qa, kk) / d ** 0.5
        out.append(torch.einsum("hn,nhd->hd", torch.softmax(s, -1), vv))
    return torch.stack(out)


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    worst = 0.0
    for c in range(cases):
        hkv = int(rng.choice([1, 2, 4, 8]))
        g = int(rng.choice([1, 2, 4, 8, 16]))
        hq = hkv * g
        n = int(rng.integers(1, 20000))
        a = int(rng.integers(1, min(n, 3000) + 1))
        qs = float(rng.choice([0.3, 1.0, 3.0]))
        spike = float(rng.choice([0.0, 0.0, 4.0, 12.0]))
        pos = np.sort(rng.choice(n, a, replace=False)) if rng.random() < 0.8 else \
            rng.choice(n, a, replace=False)
        gen = torch.Generator(device="cuda").manual_seed(c)
        q = (qs * torch.randn((a, hq, 128), device="cuda", generator=gen)).to(torch.bfloat16)
        k = torch.randn((n, hkv, 128), device="cuda", generator=gen)
        if spike:
            k = k * (1.0 + spike * torch.linspace(0, 1, n, device="cuda")[:, None, None])
        k = k.to(torch.bfloat16)
        v = torch.randn((n, hkv, 128), device="cuda", generator=gen).to(torch.bfloat16)
        p = torch.as_tensor(pos.astype(np.int32), device="cuda")
        outs = []
        for _ in range(2):
            out = torch.empty_like(q)
            wsb = _lib.load().ct_attention_workspace_bytes(a, hq, n, hkv, 128, _lib.CT_BF16)
            ws = _dev.workspace(wsb, "fuzz")
            _lib.call("ct_selective_attention", _dev.ptr(q), _dev.ptr(p), a, hq, _dev.ptr(k),
                      _dev.ptr(v), n, hkv, 128, hkv * 128, 1 / 128 ** 0.5, _lib.CT_BF16,
                      _dev.ptr(out), _lib.CT_BF16, None, _dev.ptr(ws), wsb, _dev.stream_handle())
            torch.cuda.synchronize()
            outs.append(out)
        assert torch.equal(outs[0], outs[1]), f"case {c}: non-deterministic"
        rows = torch.as_tensor(rng.choice(a, min(a, 48), replace=False))
        want = ref_rows(q, pos, k, v, hq, hkv, rows)
        got = outs[0][rows.cuda()].float()
        err = float((got - want).abs().max() / want.abs().max().clamp_min(1e-30))
        worst = max(worst, err)
        assert err < 2e-2, f"case {c}: hq={hq} hkv={hkv} a={a} n={n} qs={qs} spike={spike} err={err}"
    print(f"attn_fuzz: {cases} cases ok, worst max-rel error {worst:.2e}")


if __name__ == "__main__":
    main()
