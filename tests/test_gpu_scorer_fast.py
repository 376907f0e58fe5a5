"""Fast scorer (ct_score_select_fast): single-precision FFT scores with a
certified top-k boundary.  The selected set at k must equal the float64
scorer's (ct/spectral.py:149-178), which is itself bit-exact against the
oracle (test_gpu_parity.py / test_gpu_fullsize.py)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2605_24022_b200 import spectral
    return spectral


def _sets_equal(ex, fa, k):
    eo = ex["agg_order"].cpu().numpy()
    fo = fa["agg_order"].cpu().numpy()
    return all(np.array_equal(np.sort(eo[c, :k]), np.sort(fo[c, :k])) for c in range(eo.shape[0]))


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_fast_selection_equals_exact_gaussian(lib, dtype):
    g = torch.Generator(device="cuda").manual_seed(7)
    k_ = torch.randn((4, 4, 2048, 8, 128), device="cuda", generator=g).to(dtype)
    v_ = torch.randn((4, 4, 2048, 8, 128), device="cuda", generator=g).to(dtype)
    ex = lib.score_device(k_, v_, 0.5, "f64", want_layer_order=False)
    a = ex["agg"].cpu().numpy()
    raw = lib.score_select_fast(k_, v_, 308, guard=0.0)
    rel = np.abs(raw["agg"].cpu().numpy() - a) / a
    assert rel.max() < lib.FAST_GUARD / 4, rel.max()
    for k in (1, 77, 307, 308, 1024, 2047, 2048):
        fa = lib.score_select_fast(k_, v_, k)
        assert _sets_equal(ex, fa, k), k


def test_fast_selection_model_encoded(lib):
    import paper_2605_24022_b200 as ct
    cfg = ct.ModelConfig.llama3_8b(n_layers=4, vocab_size=4096, seed=5)
    m = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
    rng = np.random.default_rng(5)
    chunks = [ct.encode_chunk_isolated(m, rng.integers(0, 4096, size=2048), chunk_id=f"m{j}")
              for j in range(8)]
    kk = torch.stack([torch.stack(list(c.keys)) for c in chunks])
    vv = torch.stack([torch.stack(list(c.values)) for c in chunks])
    ex = lib.score_device(kk, vv, 0.5, "f64", want_layer_order=False)
    for k in (308, 615):
        fa = lib.score_select_fast(kk, vv, k)
        assert _sets_equal(ex, fa, k), k


def test_fast_window_rescore_and_fallback(lib):
    """Near-ties force the exact re-score; exact ties (a constant chunk, every
    score equal) are wider than the device window and fall back to the
    float64 scorer -- orders then equal the exact ones, index tie-break."""
    g = torch.Generator(device="cuda").manual_seed(3)
    base = torch.randn((1, 2, 2048, 8, 128), device="cuda", generator=g)
    k_ = torch.cat([base, torch.ones_like(base)]).to(torch.bfloat16)
    v_ = torch.cat([base * 0.5, torch.ones_like(base)]).to(torch.bfloat16)
    ex = lib.score_device(k_, v_, 0.5, "f64", want_layer_order=False)
    a = ex["agg"][0].cpu().numpy()
    o = ex["agg_order"][0].cpu().numpy()
    gap = (a[o[307]] - a[o[308]]) / a[o[307]]
    # a guard just wider than chunk 0's boundary gap: a few tokens re-scored
    fa = lib.score_select_fast(k_, v_, 308, guard=max(1.5 * gap, 1e-7))
    w = fa["wcount"].cpu().numpy()
    assert 2 <= w[0] <= lib.FAST_WMAX and w[1] == -1, w
    assert _sets_equal(ex, fa, 308)
    assert np.array_equal(fa["agg_order"][1].cpu().numpy(), ex["agg_order"][1].cpu().numpy())


def test_fast_rejects_unsupported_geometry(lib):
    from paper_2605_24022_b200._lib import Unsupported
    k_ = torch.zeros((1, 1, 1000, 8, 128), device="cuda", dtype=torch.bfloat16)
    with pytest.raises(Unsupported):
        lib.score_select_fast(k_, k_, 10)
