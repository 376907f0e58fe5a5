"""ct_gemm_qkv_rope (tcgen05 q|k|v projection with RoPE and the cache scatter
in the epilogue) against a PyTorch fp32 reference of the same op: qkv = x @ W,
q/k rotated at each row's global position with adjacent pairs, k/v written to
their cache rows (ct/toymodel.py:157-163, ct/rope.py), bf16 operands.  Ragged
row counts, scattered positions, untouched cache rows, and the same layer
through the engine with the fused path on and off."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2605_24022_b200 import _lib
    return _lib


def _table(n_ctx):
    from paper_2605_24022_b200.model import ModelConfig
    from paper_2605_24022_b200.rope import rope_table
    params = ModelConfig.llama3_8b(n_layers=1).rope_params
    return rope_table(params, n_ctx, "f32", torch.device("cuda"))


def _rot(x, cs):
    # x [..., 128] f32, cs [..., 64, 2] (cos, sin): adjacent pairs (2j, 2j+1)
    a, b = x[..., 0::2], x[..., 1::2]
    c, s = cs[..., 0], cs[..., 1]
    out = torch.empty_like(x)
    out[..., 0::2] = a * c - b * s
    out[..., 1::2] = a * s + b * c
    return out


@pytest.mark.parametrize("m, k, hq, hkv", [(300, 256, 4, 2), (129, 512, 8, 2),
                                           (4992, 4096, 32, 8), (1, 128, 2, 1)])
def test_gemm_qkv_rope_matches_fp32_reference(lib, m, k, hq, hkv):
    d, n_ctx = 128, 40000
    g = torch.Generator(device="cuda").manual_seed(m + k + hq)
    x = torch.randn((m, k), device="cuda", generator=g).to(torch.bfloat16)
    n = (hq + 2 * hkv) * d
    w = (torch.randn((k, n), device="cuda", generator=g) / k ** 0.5).to(torch.bfloat16)
    pos = torch.randperm(n_ctx, device="cuda", generator=g)[:m].to(torch.int32)
    table = _table(n_ctx)
    q = torch.full((m, hq, d), float("nan"), device="cuda", dtype=torch.bfloat16)
    kc = torch.zeros((n_ctx, hkv, d), device="cuda", dtype=torch.bfloat16)
    vc = torch.zeros_like(kc)
    lib.call("ct_gemm_qkv_rope", x.data_ptr(), m, k, x.stride(0), w.data_ptr(), w.stride(0),
             pos.data_ptr(), table.data_ptr(), hq, hkv, d, q.data_ptr(), kc.data_ptr(),
             vc.data_ptr(), hkv * d, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    qkv = x.float() @ w.float()
    cs = table[pos.long()][:, None]                            # [m, 1, 64, 2]
    q_ref = _rot(qkv[:, :hq * d].view(m, hq, d), cs)
    k_ref = _rot(qkv[:, hq * d:(hq + hkv) * d].view(m, hkv, d), cs)
    v_ref = qkv[:, (hq + hkv) * d:].view(m, hkv, d)
    p = pos.long()
    for got, want in ((q, q_ref), (kc[p], k_ref), (vc[p], v_ref)):
        assert torch.isfinite(got.float()).all()
        err = ((got.float() - want).norm() / want.norm()).item()
        assert err < 8e-3, err  # bf16 output rounding on an fp32-accumulated product
    untouched = torch.ones(n_ctx, dtype=torch.bool, device="cuda")
    untouched[p] = False
    assert not kc[untouched].any() and not vc[untouched].any()


def test_gemm_qkv_rope_rejects_unsupported(lib):
    from paper_2605_24022_b200.errors import CacheTuneError
    x = torch.zeros((4, 128), device="cuda", dtype=torch.bfloat16)
    w = torch.zeros((128, 4 * 64), device="cuda", dtype=torch.bfloat16)
    pos = torch.zeros(4, device="cuda", dtype=torch.int32)
    t = _table(16)
    q = torch.zeros((4, 2, 64), device="cuda", dtype=torch.bfloat16)
    c = torch.zeros((16, 1, 64), device="cuda", dtype=torch.bfloat16)
    with pytest.raises(CacheTuneError):  # head_dim 64
        lib.call("ct_gemm_qkv_rope", x.data_ptr(), 4, 128, 128, w.data_ptr(), 256, pos.data_ptr(),
                 t.data_ptr(), 2, 1, 64, q.data_ptr(), c.data_ptr(), c.data_ptr(), 64,
                 torch.cuda.current_stream().cuda_stream)


def test_engine_layer_fused_qkv_matches_unfused(lib):
    """The same selective request (Llama geometry, 2 layers) with the QKV
    epilogue fused into the GEMM and with cuBLAS + ct_qkv_rope_scatter: logits
    and blended caches agree within bf16 rounding of the q|k|v product."""
    import paper_2605_24022_b200 as ct
    from paper_2605_24022_b200 import prefill
    from paper_2605_24022_b200.pipeline import SelectivePrefillEngine
    from paper_2605_24022_b200.pool import KvPool
    cfg = ct.ModelConfig.llama3_8b(n_layers=2, seed=5)
    model = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
    rng = np.random.default_rng(5)
    chunks = [ct.encode_chunk_isolated(model, rng.integers(0, cfg.vocab_size, size=1024),
                                       chunk_id=f"c{j}") for j in range(4)]
    pool = KvPool(chunks, ct.rank_chunks(chunks), "hbm")
    suffix = torch.as_tensor(rng.integers(0, cfg.vocab_size, size=64).astype(np.int32),
                             device="cuda")
    out = {}
    saved = prefill._QKV_FUSED_ENV
    try:
        for fused in (True, False):
            prefill._QKV_FUSED_ENV = fused
            eng = SelectivePrefillEngine(model, pool, 0.15, 64)
            assert prefill.FUSED_MIN_ROWS <= eng.A <= prefill.FUSED_MAX_ROWS
            logits = eng.step(suffix).float().clone()
            torch.cuda.synchronize()
            out[fused] = (logits, eng.cache.float().clone())
    finally:
        prefill._QKV_FUSED_ENV = saved
    (lf, cf), (lu, cu) = out[True], out[False]
    assert ((lf - lu).norm() / lu.norm()).item() < 2e-2
    assert ((cf - cu).norm() / cu.norm()).item() < 1e-2
