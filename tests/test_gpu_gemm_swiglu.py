"""ct_gemm_swiglu (tcgen05 gate/up projection with the SwiGLU activation in
the epilogue) against a PyTorch fp32 reference of the same op,
silu(x @ Wg) * (x @ Wu) (ct/toymodel.py:184-186), on bf16 operands: ragged
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
