#!/usr/bin/env python
"""First-token logits of a full-context config-2 request (16 x 2048 chunks +
64 suffix = 32,832 tokens, Llama-3-8B layer geometry, r = 0.15), bf16 mode,
against the float64 oracle's selective prefill (oracle/cachetune_oracle.py,
restating ct/toymodel.py:223-311 with GQA / SwiGLU).

    python tools/fullsize_logits_check.py [--layers 4] [--seed 0] [--torch-bf16] [--out FILE]

Both sides get identical inputs:
- the model's bf16 weights, exact in float64;
- the chunk KV encoded on the GPU (bf16 values, exact in float32);
- the same aggregate orders (the GPU float64 scorer, bit-exact against the
  oracle);
- the same suffix tokens.

The GPU runs the engine of the bench (HBM pool, bf16 mode); the oracle runs
the reference arithmetic in float64.  The check is the north star's bf16
tolerance, normwise relative error of the first-token logits <= 2e-2, plus
the last layer's blended K and V.  The depth is reduced because float64
weights of all 32 layers would need ~64 GB of host memory; every layer has
the full context.  Test infrastructure: the oracle is the checker.

--torch-bf16 adds a third leg: the same request written the usual way in
plain PyTorch bf16 (bf16 residual stream, fp32 RMSNorm, fp32 RoPE, SDPA),
on the same inputs, scored against the same oracle run.  It shows how much
of the deviation is bf16 arithmetic itself."""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default="")
    ap.add_argument("--torch-bf16", action="store_true")
    ap.add_argument("--config", default="cfg2", choices=["cfg2", "cfg3"],
                    help="cfg3: Mistral-7B geometry, 32 x 2048 + 64 = 65,600 tokens, pool in "
                         "pinned host memory (the sparse-H2D path)")
    args = ap.parse_args()
    import torch
    import paper_2605_24022_b200 as ct
    from oracle import cachetune_oracle as O
    from paper_2605_24022_b200.pipeline import SelectivePrefillEngine
    from paper_2605_24022_b200.pool import KvPool

    N, S, R = 2048, 64, 0.15
    if args.config == "cfg3":
        C, where = 32, "pinned"
        cfg = ct.ModelConfig.mistral_7b(n_layers=args.layers, seed=args.seed + 21)
    else:
        C, where = 16, "hbm"
        cfg = ct.ModelConfig.llama3_8b(n_layers=args.layers, seed=args.seed + 21)
    model = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
    rng = np.random.default_rng(args.seed)
    toks = [rng.integers(0, cfg.vocab_size, size=N) for _ in range(C)]
    suffix = rng.integers(0, cfg.vocab_size, size=S).astype(np.int64)
    t0 = time.time()
    chunks = [ct.encode_chunk_isolated(model, t, chunk_id=f"c{j}") for j, t in enumerate(toks)]
    ranks = ct.rank_chunks(chunks)
    eng = SelectivePrefillEngine(model, KvPool(chunks, ranks, where), R, S)
    logits = eng.step(torch.as_tensor(suffix.astype(np.int32), device="cuda"))
    torch.cuda.synchronize()
    got = logits.double().cpu().numpy().reshape(-1)
    kl, vl = eng.caches[-1]
    got_k, got_v = kl.double().cpu().numpy(), vl.double().cpu().numpy()
    gpu_s = time.time() - t0
    tb = torch_bf16_request(model, chunks, ranks, suffix, R) if args.torch_bf16 else None

    t1 = time.time()
    om = O.Model(O.ModelConfig(seed=0, n_layers=args.layers, n_heads=32, head_dim=128,
                               vocab_size=cfg.vocab_size, mlp="swiglu", n_kv_heads=8,
                               intermediate=14336,
                               rope_base=cfg.rope_base),
                 weights=model.to_numpy_weights())
    ochunks = [([c.keys[l].float().cpu().numpy() for l in range(args.layers)],
                [c.values[l].float().cpu().numpy() for l in range(args.layers)], t)
               for c, t in zip(chunks, toks)]
    aggs = [rk.aggregate_order for rk in ranks]
    res = O.selective_prefill(om, ochunks, aggs, suffix, R, want_probs=False,
                              logits_rows="last")
    want = np.asarray(res["logits"]).reshape(-1)
    want_k, want_v = res["kv"][-1]
    cpu_s = time.time() - t1
    geo = "Mistral-7B" if args.config == "cfg3" else "Llama-3-8B"
    out = {"workload": f"{args.config} context ({C} x {N} + {S} = {C * N + S} tokens), {geo} "
                       f"layer geometry, {args.layers} layers, r = 0.15, bf16 mode, pool in {where}",
           "logits_normwise_rel": O.normwise_rel(got, want),
           "last_layer_k_normwise_rel": O.normwise_rel(got_k, want_k),
           "last_layer_v_normwise_rel": O.normwise_rel(got_v, want_v),
           "tolerance": 2e-2, "gpu_s": round(gpu_s, 1), "oracle_cpu_s": round(cpu_s, 1)}
    if tb is not None:
        out["plain_torch_bf16"] = {
            "logits_normwise_rel": O.normwise_rel(tb[0], want),
            "last_layer_k_normwise_rel": O.normwise_rel(tb[1], want_k),
            "last_layer_v_normwise_rel": O.normwise_rel(tb[2], want_v)}
    print(json.dumps(out))
    if args.out:
        Path(args.out).write_text(json.dumps(out, indent=1))
    assert out["logits_normwise_rel"] <= 2e-2, out


def torch_bf16_request(model, chunks, ranks, suffix, r):
    """The same selective prefill in plain PyTorch bf16, the common inference
    recipe: bf16 hidden states and residual adds, RMSNorm and RoPE in fp32
    then cast, bf16 matmuls, SDPA with a position mask.  Returns host float64
    (first-token logits, last layer blended K, last layer blended V)."""
    import torch
    import torch.nn.functional as F
    from paper_2605_24022_b200.spectral import selection_count
    dev, bf = "cuda", torch.bfloat16
    cfg = model.config
    L, hq, hkv, d = cfg.n_layers, cfg.n_heads, cfg.kv_heads, cfg.head_dim
    N = chunks[0].token_count
    k = selection_count(r, N)
    rec = np.concatenate([np.sort(rk.aggregate_order[:k]) + j * N for j, rk in enumerate(ranks)])
    keep = np.concatenate([np.sort(rk.aggregate_order[k:]) + j * N for j, rk in enumerate(ranks)])
    hist = N * len(chunks)
    n_ctx = hist + suffix.size
    pos = np.concatenate([rec, np.arange(hist, n_ctx)])
    toks_all = np.concatenate([np.asarray(c.source_tokens) for c in chunks] + [suffix])
    tok = torch.as_tensor(toks_all[pos], device=dev)
    pos_t = torch.as_tensor(pos, device=dev)
    keep_t = torch.as_tensor(keep, device=dev)
    freqs = torch.as_tensor(cfg.rope_params.freqs(), device=dev, dtype=torch.float64)

    def rope(x, p):  # x [n, h, d] (adjacent pairs), p [n]
        ang = (p.double()[:, None] * cfg.rope_scaling) * freqs[None, :]
        c, s = torch.cos(ang).float()[:, None, :], torch.sin(ang).float()[:, None, :]
        xf = x.float()
        a, b = xf[..., 0::2], xf[..., 1::2]
        out = torch.empty_like(xf)
        out[..., 0::2], out[..., 1::2] = a * c - b * s, a * s + b * c
        return out.to(bf)

    def rms(h):
        hf = h.float()
        return (hf * torch.rsqrt(hf.pow(2).mean(-1, keepdim=True) + 1e-6)).to(bf)

    h = model.embedding[tok].to(bf)
    mask = torch.arange(n_ctx, device=dev)[None, :] <= pos_t[:, None]
    for l, w in enumerate(model.layers):
        x = rms(h)
        qkv = x @ w["wqkv"]
        q = qkv[:, :hq * d].reshape(-1, hq, d)
        kk = qkv[:, hq * d:(hq + hkv) * d].reshape(-1, hkv, d)
        vv = qkv[:, (hq + hkv) * d:].reshape(-1, hkv, d)
        q, kk = rope(q, pos_t), rope(kk, pos_t)
        kc = torch.empty((n_ctx, hkv, d), dtype=bf, device=dev)
        vc = torch.empty_like(kc)
        kraw = torch.cat([c.keys[l] for c in chunks]).to(bf)[keep_t]
        kc[keep_t] = rope(kraw, keep_t)
        vc[keep_t] = torch.cat([c.values[l] for c in chunks]).to(bf)[keep_t]
        kc[pos_t], vc[pos_t] = kk, vv
        ctx = F.scaled_dot_product_attention(
            q.transpose(0, 1)[None], kc.transpose(0, 1)[None], vc.transpose(0, 1)[None],
            attn_mask=mask[None, None], enable_gqa=True)[0].transpose(0, 1)
        h = h + ctx.reshape(-1, hq * d) @ w["wo"]
        xm = rms(h)
        gu = xm @ w["wgu"]
        g, u = gu[:, :cfg.inter], gu[:, cfg.inter:]
        h = h + (F.silu(g) * u) @ w["wd"]
    logits = (h[-1:] @ model.w_out.to(bf)).double().cpu().numpy().reshape(-1)
    return logits, kc.double().cpu().numpy(), vc.double().cpu().numpy()


if __name__ == "__main__":
    main()
