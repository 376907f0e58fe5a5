"""Parity of the bf16 hot-path row movers (blend_bf16_kernel, qkv_bf16_kernel)
against a PyTorch fp32 restatement of the same op on the same bf16 inputs and
the same f32 (cos, sin) table: V rows and raw K rows bit-exact, rotated rows
within one bf16 rounding (the kernel fuses x*c - y*s into one FMA)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ct():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2605_24022_b200 as ct
    return ct


def _rotate_ref(x, pos, table):
    # x [n, H, D] bf16; table [cap, D/2, 2] f32 -> (rotated f32, pair magnitude)
    xf = x.float()
    a, b = xf[..., 0::2], xf[..., 1::2]
    cs = table[pos.long()]                       # [n, D/2, 2]
    c, s = cs[..., 0][:, None, :], cs[..., 1][:, None, :]
    out = torch.empty_like(xf)
    out[..., 0::2] = a * c - b * s
    out[..., 1::2] = a * s + b * c
    mag = torch.empty_like(xf)
    mag[..., 0::2] = a.abs() + b.abs()
    mag[..., 1::2] = a.abs() + b.abs()
    return out, mag


def _close_bf16(got, refmag):
    # one bf16 rounding of the result (2^-9 relative, 2^-8 allowed) plus the
    # f32 FMA-vs-separate-product difference, relative to the pair magnitude
    ref, mag = refmag
    err = (got.float() - ref).abs()
    tol = ref.abs() * 2.0 ** -8 + mag * 2.0 ** -20
    assert bool((err <= tol).all()), float((err - tol).max())


@pytest.mark.parametrize("H,D", [(8, 128), (6, 64), (3, 16)])
@pytest.mark.parametrize("by_tok", [0, 1])
def test_blend_bf16_fast_path(ct, H, D, by_tok):
    from paper_2605_24022_b200 import _dev, _lib
    from paper_2605_24022_b200.rope import RopeParams, rope_table
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(H * 1000 + D + by_tok)
    C, N, k = 3, 300, 45
    keep = N - k
    params = RopeParams(head_dim=D, base=10000.0)
    n_ctx = C * N
    table = rope_table(params, n_ctx, "f32", dev)
    pool = torch.randn((C, N, 2, H, D), device=dev, generator=g).to(torch.bfloat16)
    agg = torch.stack([torch.randperm(N, device=dev, generator=g) for _ in range(C)]).to(torch.int32)
    cache = torch.zeros((2, n_ctx, H, D), dtype=torch.bfloat16, device=dev)
    segs = []
    for c in range(C):
        base = pool[c, 0 if by_tok else k].data_ptr()
        tok = agg.data_ptr() + (c * N + k) * 4
        segs.append(_lib.Segment(base, base + H * D * 2, tok, keep, c * N, by_tok))
    arr = (_lib.Segment * C)(*segs)
    _lib.call("ct_gather_rope_blend", arr, C, 2 * H * D, H, D, _dev.ct_dtype(torch.bfloat16),
              params.pairing_code, _dev.ptr(table), _dev.ptr(cache[0]), _dev.ptr(cache[1]),
              H * D, _dev.stream_handle())
    torch.cuda.synchronize()
    for c in range(C):
        toks = agg[c, k:].long()
        src_rows = toks if by_tok else torch.arange(k, N, device=dev)
        kraw, vraw = pool[c, src_rows, 0], pool[c, src_rows, 1]
        pos = c * N + toks
        assert torch.equal(cache[1, pos], vraw)
        _close_bf16(cache[0, pos], _rotate_ref(kraw, pos, table))
    # rows of recomputed tokens untouched
    mask = torch.ones(n_ctx, dtype=torch.bool, device=dev)
    for c in range(C):
        mask[c * N + agg[c, k:].long()] = False
    assert bool((cache[:, mask] == 0).all())


@pytest.mark.parametrize("Hq,Hkv,D", [(32, 8, 128), (4, 2, 64), (6, 3, 16)])
def test_qkv_bf16_fast_path(ct, Hq, Hkv, D):
    from paper_2605_24022_b200 import _dev, _lib
    from paper_2605_24022_b200.rope import RopeParams, rope_table
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(Hq + Hkv + D)
    A, n_ctx = 777, 5000
    params = RopeParams(head_dim=D, base=500000.0)
    table = rope_table(params, n_ctx, "f32", dev)
    hpr = Hq + 2 * Hkv
    qkv = torch.randn((A, hpr * D), device=dev, generator=g).to(torch.bfloat16)
    pos = torch.sort(torch.randperm(n_ctx, device=dev, generator=g)[:A]).values.to(torch.int32)
    q = torch.empty((A, Hq, D), dtype=torch.bfloat16, device=dev)
    kraw = torch.empty((A, Hkv, D), dtype=torch.bfloat16, device=dev)
    cache = torch.zeros((2, n_ctx, Hkv, D), dtype=torch.bfloat16, device=dev)
    bf = _dev.ct_dtype(torch.bfloat16)
    _lib.call("ct_qkv_rope_scatter", _dev.ptr(qkv), hpr * D, bf, _dev.ptr(pos), A, Hq, Hkv, D,
              params.pairing_code, _dev.ptr(table), _dev.ptr(q), bf, _dev.ptr(cache[0]),
              _dev.ptr(cache[1]), bf, Hkv * D, _dev.ptr(kraw), _dev.stream_handle())
    torch.cuda.synchronize()
    x = qkv.view(A, hpr, D)
    _close_bf16(q, _rotate_ref(x[:, :Hq], pos, table))
    assert torch.equal(kraw, x[:, Hq:Hq + Hkv])
    _close_bf16(cache[0, pos.long()], _rotate_ref(x[:, Hq:Hq + Hkv], pos, table))
    assert torch.equal(cache[1, pos.long()], x[:, Hq + Hkv:])


@pytest.mark.parametrize("A, inter", [(1, 64), (3, 14336), (70000, 64)])
def test_swiglu_and_rmsnorm_kernels_vs_torch(A, inter):
    """ct_mlp_act (SwiGLU, rows on blockIdx.y incl. more rows than one grid
    dimension holds) and ct_residual_rmsnorm (persistent row loop at hid 4096)
    vs PyTorch fp32 of the same op, one bf16 rounding apart."""
    from paper_2605_24022_b200 import _dev, _lib
    torch.manual_seed(A)
    gu = torch.randn((A, 2 * inter), device="cuda").to(torch.bfloat16)
    act = torch.empty((A, inter), dtype=torch.bfloat16, device="cuda")
    _lib.call("ct_mlp_act", gu.data_ptr(), A, inter, _lib.CT_BF16, 0, act.data_ptr(),
              _lib.CT_BF16, _dev.stream_handle())
    g, u = gu[:, :inter].float(), gu[:, inter:].float()
    want = (g * torch.sigmoid(g) * u)
    err = (act.float() - want).abs()
    assert bool((err <= want.abs() * 2.0 ** -7 + 1e-6).all())
    if A <= 3:
        return
    hid = 4096
    h = torch.randn((A // 10, hid), device="cuda")
    x = torch.empty((A // 10, hid), dtype=torch.bfloat16, device="cuda")
    _lib.call("ct_residual_rmsnorm", h.data_ptr(), None, _lib.CT_F32, A // 10, hid, 1e-6,
              x.data_ptr(), _lib.CT_BF16, _dev.stream_handle())
    ref = h.double() / torch.sqrt((h.double() ** 2).mean(dim=1, keepdim=True) + 1e-6)
    assert bool(((x.double() - ref).abs() <= ref.abs() * 2.0 ** -8 + 1e-6).all())
