"""tcgen05/TMEM attention kernel (bf16 operands, fp32 accumulation) against a
plain PyTorch fp32 reference of ct/toymodel.py:176-183 on the same bf16
inputs.  Tolerance: normwise 1e-2 (bf16 P rounding), per-row checks for the
masking edge cases."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(q, pos, k, v, hq, hkv):
    a, _, d = q.shape
    n = k.shape[0]
    g = hq // hkv
    kk = k.float().repeat_interleave(g, dim=1).permute(1, 2, 0)
    vv = v.float().repeat_interleave(g, dim=1).permute(1, 0, 2)
    s = torch.bmm(q.float().permute(1, 0, 2), kk) / d ** 0.5
    mask = torch.arange(n, device=q.device)[None, :] <= pos[:, None].long()
    s = s.masked_fill(~mask[None], float("-inf"))
    return torch.bmm(torch.softmax(s, dim=-1), vv).permute(1, 0, 2)


def _run(q, pos, k, v, hq, hkv, out_dtype=torch.bfloat16):
    from paper_2605_24022_b200 import _dev, _lib
    a, _, d = q.shape
    n = k.shape[0]
    out = torch.empty((a, hq, d), device="cuda", dtype=out_dtype)
    wsb = _lib.load().ct_attention_workspace_bytes(a, hq, n, hkv, d, _lib.CT_BF16)
    ws = _dev.workspace(wsb, "test_attention")
    _lib.call("ct_selective_attention", _dev.ptr(q), _dev.ptr(pos), a, hq, _dev.ptr(k),
              _dev.ptr(v), n, hkv, d, k.stride(0), 1.0 / d ** 0.5, _lib.CT_BF16, _dev.ptr(out),
              _dev.ct_dtype(out_dtype), None, _dev.ptr(ws), wsb, _dev.stream_handle())
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("a,hq,hkv,n,sorted_pos", [
    (32, 32, 8, 128, True),       # one tile, one key block
    (300, 32, 8, 2500, True),     # ragged tail, GQA 4
    (1000, 8, 8, 5000, True),     # MHA (G=1), 8 q-blocks
    (77, 16, 2, 3001, False),     # G=8, unsorted positions
    (4992, 32, 8, 32832, True),   # config-2 layer shape (selected + suffix rows)
    (1, 32, 8, 1, True),          # one query, one key
    (5, 64, 4, 700, True),        # G=16 (8 queries per tile), odd tile count
    (129, 8, 8, 129, True),       # MHA, A = n_ctx = 129 (dense causal, ragged)
])
def test_tc_attention_matches_torch(a, hq, hkv, n, sorted_pos):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    gen = torch.Generator(device="cuda").manual_seed(a + n)
    d = 128
    q = torch.randn((a, hq, d), device="cuda", generator=gen).to(torch.bfloat16)
    k = torch.randn((n, hkv, d), device="cuda", generator=gen).to(torch.bfloat16)
    v = torch.randn((n, hkv, d), device="cuda", generator=gen).to(torch.bfloat16)
    pos = torch.randperm(n, device="cuda", generator=gen)[:a]
    if sorted_pos:
        pos = torch.sort(pos)[0]
    pos = pos.to(torch.int32)
    pos[0] = 0 if sorted_pos else pos[0]
    out = _run(q, pos, k, v, hq, hkv)
    if a * hq * n > 2e9:   # keep the torch reference affordable: sample query rows
        idx = torch.randperm(a, device="cuda", generator=gen)[:256]
        want = _ref(q[idx], pos[idx], k, v, hq, hkv)
        got = out[idx].float()
    else:
        want = _ref(q, pos, k, v, hq, hkv)
        got = out.float()
    err = (got - want).abs().max().item() / want.abs().max().item()
    assert err < 1e-2, err


@pytest.mark.parametrize("qscale", [0.3, 3.0, 6.0])
def test_tc_attention_lazy_rescale_many_blocks(qscale):
    """Peaked softmax over 32 key blocks: the running max grows by > 2^8 at
    arbitrary blocks, so O is rescaled in TMEM while later S tiles are in
    flight.  Error must stay at the bf16-P level (a race shows up as O(1))."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    gen = torch.Generator(device="cuda").manual_seed(int(qscale * 10))
    a, hq, hkv, n, d = 512, 32, 8, 4096, 128
    q = (qscale * torch.randn((a, hq, d), device="cuda", generator=gen)).to(torch.bfloat16)
    k = torch.randn((n, hkv, d), device="cuda", generator=gen).to(torch.bfloat16)
    v = torch.randn((n, hkv, d), device="cuda", generator=gen).to(torch.bfloat16)
    pos = torch.sort(torch.randperm(n, device="cuda", generator=gen)[:a])[0].to(torch.int32)
    for _ in range(3):   # repeat: races are intermittent
        out = _run(q, pos, k, v, hq, hkv)
        want = _ref(q, pos, k, v, hq, hkv)
        err = (out.float() - want).abs().max().item() / want.abs().max().item()
        assert err < 5e-3, err


def test_tc_attention_f32_output_and_large_scores():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    gen = torch.Generator(device="cuda").manual_seed(3)
    a, hq, hkv, n, d = 200, 8, 2, 1500, 128
    # large logits exercise the lazy-rescale path (max grows by > 2^8 mid-row)
    q = (4 * torch.randn((a, hq, d), device="cuda", generator=gen)).to(torch.bfloat16)
    k = torch.randn((n, hkv, d), device="cuda", generator=gen)
    k[700:] *= 3
    k = k.to(torch.bfloat16)
    v = torch.randn((n, hkv, d), device="cuda", generator=gen).to(torch.bfloat16)
    pos = torch.sort(torch.randperm(n, device="cuda", generator=gen)[:a])[0].to(torch.int32)
    out = _run(q, pos, k, v, hq, hkv, out_dtype=torch.float32)
    want = _ref(q, pos, k, v, hq, hkv)
    err = (out - want).abs().max().item() / want.abs().max().item()
    assert err < 1e-2, err


def test_tc_attention_randomised_geometries_deterministic():
    """tools/attn_fuzz.py at a CI-sized case count: random GQA group (1-16),
    kv heads, query count, context, sorted/unsorted positions, score scale and a
    key-scale ramp (running-max growth -> lazy O rescale), each launched twice
    (bit-identical) and checked on sampled rows against PyTorch fp32."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    import importlib.util
    from pathlib import Path
    path = Path(__file__).resolve().parents[1] / "tools" / "attn_fuzz.py"
    spec = importlib.util.spec_from_file_location("attn_fuzz", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    import sys
    argv = sys.argv
    try:
        sys.argv = ["attn_fuzz", "12", "7"]
        mod.main()
    finally:
        sys.argv = argv


@pytest.mark.parametrize("a,hq,hkv,n,out_dtype", [
    (1, 32, 8, 32832, torch.bfloat16),   # the last-layer first-token row at config-2 size
    (1, 32, 8, 1, torch.bfloat16),       # one key
    (2, 8, 2, 5000, torch.float32),      # 8 rows (the path's limit), f32 output
    (3, 8, 8, 100, torch.bfloat16),      # MHA, fewer keys than one split
    (4, 16, 4, 70000, torch.bfloat16),   # more than 2048 keys per split needed -> more splits
])
def test_few_row_split_key_attention(monkeypatch, a, hq, hkv, n, out_dtype):
    """A x G <= 8 rows take the split-key path (ct_selective_attention picks it;
    the caller sizes the workspace with ct_attention_workspace_bytes); it must
    agree with the fp32 reference and, for D = 128 bf16, with the tcgen05
    kernel forced on the same rows (CT_ATT_DECODE=0), and be deterministic."""
    gen = torch.Generator(device="cuda").manual_seed(a * 7 + n)
    d = 128
    q = torch.randn((a, hq, d), device="cuda", generator=gen).to(torch.bfloat16)
    k = torch.randn((n, hkv, d), device="cuda", generator=gen).to(torch.bfloat16)
    v = torch.randn((n, hkv, d), device="cuda", generator=gen).to(torch.bfloat16)
    pos = torch.sort(torch.randperm(n, device="cuda", generator=gen)[:a])[0].to(torch.int32)
    pos[-1] = n - 1
    out = _run(q, pos, k, v, hq, hkv, out_dtype)
    again = _run(q, pos, k, v, hq, hkv, out_dtype)
    assert torch.equal(out, again)
    want = _ref(q, pos, k, v, hq, hkv)
    err = (out.float() - want).abs().max().item() / want.abs().max().item()
    assert err < 5e-3, err
    monkeypatch.setenv("CT_ATT_DECODE", "0")
    tc = _run(q, pos, k, v, hq, hkv, out_dtype)
    err_tc = (tc.float() - want).abs().max().item() / want.abs().max().item()
    assert err_tc < 1e-2, err_tc
