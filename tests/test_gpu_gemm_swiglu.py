"""ct_gemm_swiglu (tcgen05 gate/up projection with the SwiGLU activation in
the epilogue) against a PyTorch fp32 reference of the same op,
silu(x @ Wg) * (x @ Wu) (the MLP of ct/toymodel.py:186 as SwiGLU), on bf16 operands: ragged
row counts (tail tiles), small and config-2 widths, strided rows."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2605_24022_b200 import _lib
    return _lib


def _run(lib, x, w, inter, act):
    lib.call("ct_gemm_swiglu", x.data_ptr(), x.shape[0], x.shape[1], x.stride(0), w.data_ptr(),
             inter, w.stride(0), act.data_ptr(), act.stride(0),
             torch.cuda.current_stream().cuda_stream)


def _ref(x, w, inter):
    gu = x.float() @ w.float()
    g, u = gu[:, :inter], gu[:, inter:]
    return torch.nn.functional.silu(g) * u


@pytest.mark.parametrize("m, k, inter", [(128, 64, 128), (300, 256, 256), (4992, 4096, 14336),
                                         (9920, 4096, 1024), (1, 128, 128), (129, 512, 384)])
def test_gemm_swiglu_matches_fp32_reference(lib, m, k, inter):
    g = torch.Generator(device="cuda").manual_seed(m + k + inter)
    x = torch.randn((m, k), device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn((k, 2 * inter), device="cuda", generator=g) / k ** 0.5).to(torch.bfloat16)
    act = torch.full((m, inter), float("nan"), device="cuda", dtype=torch.bfloat16)
    _run(lib, x, w, inter, act)
    torch.cuda.synchronize()
    want = _ref(x, w, inter)
    err = ((act.float() - want).norm() / want.norm()).item()
    assert torch.isfinite(act.float()).all()
    assert err < 8e-3, err  # bf16 output rounding (2^-9) on an fp32-accumulated product


def test_gemm_swiglu_strided_rows_and_deterministic(lib):
    g = torch.Generator(device="cuda").manual_seed(5)
    m, k, inter = 700, 1024, 512
    xs = torch.randn((m, k + 64), device="cuda", generator=g).to(torch.bfloat16)
    ws = (torch.randn((k, 2 * inter + 128), device="cuda", generator=g) / 32).to(torch.bfloat16)
    x, w = xs[:, :k], ws[:, :2 * inter]
    outs = []
    for _ in range(2):
        big = torch.zeros((m, inter + 64), device="cuda", dtype=torch.bfloat16)
        _run(lib, x, w, inter, big[:, :inter])
        outs.append(big)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    assert not outs[0][:, inter:].any()  # nothing written past the output columns
    want = _ref(x, w, inter)
    err = ((outs[0][:, :inter].float() - want).norm() / want.norm()).item()
    assert err < 8e-3, err


def test_gemm_swiglu_rejects_unsupported_geometry(lib):
    from paper_2605_24022_b200._lib import Unsupported
    x = torch.zeros((128, 100), device="cuda", dtype=torch.bfloat16)
    w = torch.zeros((100, 256), device="cuda", dtype=torch.bfloat16)
    act = torch.zeros((128, 128), device="cuda", dtype=torch.bfloat16)
    with pytest.raises(Unsupported):
        _run(lib, x, w, 128, act)


def test_gemm_swiglu_single_sm_variant_matches(lib):
    """CT_GEMM_1SM=1 (read once per process) selects the single-SM M128 form;
    run it in a child process on a ragged shape with two L2 bands and compare
    with the default CTA-pair kernel bit for bit (same MMA order per row)."""
    import os
    import subprocess
    import sys
    code = (
        "import torch,sys; sys.path.insert(0, '.');"
        "from paper_2605_24022_b200 import _lib;"
        "g=torch.Generator(device='cuda').manual_seed(3);"
        "m,k,i=5000,4096,256;"
        "x=torch.randn((m,k),device='cuda',generator=g).to(torch.bfloat16);"
        "w=(torch.randn((k,2*i),device='cuda',generator=g)/64).to(torch.bfloat16);"
        "a=torch.empty((m,i),device='cuda',dtype=torch.bfloat16);"
        "_lib.call('ct_gemm_swiglu',x.data_ptr(),m,k,k,w.data_ptr(),i,2*i,a.data_ptr(),i,"
        "torch.cuda.current_stream().cuda_stream);"
        "torch.save(a.cpu(), sys.argv[1])")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for v in ("0", "1"):
        path = os.path.join(root, "gpurun_out", f"gemm_1sm_{v}.pt")
        os.makedirs(os.path.dirname(path), exist_ok=True)
        subprocess.run([sys.executable, "-c", code, path], cwd=root, check=True, timeout=300,
                       env={**os.environ, "CT_GEMM_1SM": v})
        outs.append(torch.load(path))
    assert torch.isfinite(outs[0].float()).all()
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("m, k, n", [(4992, 4096, 6144), (4992, 4096, 4096), (4992, 14336, 4096),
                                     (1, 64, 256), (300, 128, 512), (129, 1024, 768),
                                     (200, 256, 384)])
def test_gemm_bf16_store_and_accumulate_match_fp32_reference(lib, m, k, n):
    """ct_gemm_bf16: the QKV projection (bf16 store) and the O / down
    projections into the f32 residual (out += x @ w), against torch fp32."""
    from paper_2605_24022_b200._lib import CT_BF16, CT_F32
    g = torch.Generator(device="cuda").manual_seed(m + k + n)
    x = torch.randn((m, k), device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn((k, n), device="cuda", generator=g) / k ** 0.5).to(torch.bfloat16)
    want = x.float() @ w.float()
    st = torch.cuda.current_stream().cuda_stream
    out = torch.full((m, n), float("nan"), device="cuda", dtype=torch.bfloat16)
    lib.call("ct_gemm_bf16", x.data_ptr(), m, k, k, w.data_ptr(), n, n, out.data_ptr(), n,
             CT_BF16, 0, st)
    h0 = torch.randn((m, n), device="cuda", generator=g)
    h = h0.clone()
    lib.call("ct_gemm_bf16", x.data_ptr(), m, k, k, w.data_ptr(), n, n, h.data_ptr(), n,
             CT_F32, 1, st)
    torch.cuda.synchronize()
    err = ((out.float() - want).norm() / want.norm()).item()
    assert err < 8e-3, err  # bf16 output rounding
    # f32 output: only the accumulation order differs from the reference
    err_h = ((h - h0 - want).norm() / want.norm()).item()
    assert err_h < 1e-4, err_h


def test_gemm_bf16_strided_views_and_unsupported(lib):
    from paper_2605_24022_b200._lib import CT_BF16, CT_F32, Unsupported
    g = torch.Generator(device="cuda").manual_seed(11)
    m, k, n = 700, 512, 512
    xs = torch.randn((m, k + 64), device="cuda", generator=g).to(torch.bfloat16)
    ws = (torch.randn((k, n + 256), device="cuda", generator=g) / 16).to(torch.bfloat16)
    x, w = xs[:, :k], ws[:, :n]
    big = torch.zeros((m, n + 128), device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(2):  # accumulates twice
        lib.call("ct_gemm_bf16", x.data_ptr(), m, k, x.stride(0), w.data_ptr(), n, w.stride(0),
                 big.data_ptr(), big.stride(0), CT_F32, 1, st)
    torch.cuda.synchronize()
    want = 2 * (x.float() @ w.float())
    assert ((big[:, :n] - want).norm() / want.norm()).item() < 1e-4
    assert not big[:, n:].any()
    with pytest.raises(Unsupported):  # bf16 accumulate is not a supported form
        lib.call("ct_gemm_bf16", x.data_ptr(), m, k, x.stride(0), w.data_ptr(), n, w.stride(0),
                 big.data_ptr(), big.stride(0), CT_BF16, 1, st)
    with pytest.raises(Unsupported):  # N % 128
        lib.call("ct_gemm_bf16", x.data_ptr(), m, k, x.stride(0), w.data_ptr(), 320, w.stride(0),
                 big.data_ptr(), big.stride(0), CT_F32, 1, st)
