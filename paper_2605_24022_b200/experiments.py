"""Selection-strategy experiment: attention recovery.

Mirrors ct/toymodel.py:344-419 on the device path: every strategy gets the
same recompute budget ceil(r*N) per chunk, the chunks are encoded in
isolation, the selective prefill runs through the CUDA kernels, and the
suffix rows' attention over the history is compared with a full recompute
(mean per-head Frobenius distance, ct/toymodel.py:113-124).

Strategies: "lowfreq" (the CacheTune scorer), "highfreq" (the complementary
band, device scorer with band=1), "random" (a seeded permutation — host
numpy draw identical to the reference's), "none" (reuse everything) and
"full" (recompute everything).  Models come from `GpuModel.reference_init`,
so a seed names the same ToyModel weights the reference draws.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np
import torch

from . import _dev
from .errors import InvalidPlan
from .kvcore import DeviceChunk
from .model import GpuModel, ModelConfig
from .prefill import attention_deviation, encode_chunk_isolated, full_prefill, selective_prefill
from .spectral import ImportanceRanking, rank_chunk

STRATEGIES = ("lowfreq", "highfreq", "random", "none", "full")


def strategy_ranking(chunk, strategy: str, alpha: float = 0.5,
                     rng: np.random.Generator | None = None) -> ImportanceRanking:
    """Token order a selection strategy recomputes first (ct/toymodel.py:351-371)."""
    if strategy in ("lowfreq", "none", "full"):
        return rank_chunk(chunk, alpha)
    if strategy == "highfreq":
        return rank_chunk(chunk, alpha, band="high")
    if strategy == "random":
        if rng is None:
            raise InvalidPlan("random strategy needs an rng")
        n = chunk.token_count
        perm = rng.permutation(n)
        scores = np.tile((n - np.argsort(perm)).astype(np.float64), (chunk.n_layers, 1))
        orders = np.tile(perm, (chunk.n_layers, 1))
        return ImportanceRanking(per_layer_scores=scores, per_layer_order=orders,
                                 aggregate_order=perm, alpha=alpha, n_tokens=n)
    raise InvalidPlan(f"unknown strategy {strategy!r}")


def effective_ratio(strategy: str, r: float) -> float:
    """ct/toymodel.py:374-379."""
    if strategy == "none":
        return 0.0
    if strategy == "full":
        return 1.0
    return r


def run_selection_experiment(seeds: Sequence[int], r: float = 0.15,
                             strategy: str = "lowfreq",
                             chunk_tokens: Sequence[int] = (64, 64, 64),
                             suffix_len: int = 8, alpha: float = 0.5, mlp: bool = False,
                             dtype=torch.float32) -> list[tuple[int, float]]:
    """Suffix-attention deviation from the full recompute, per seed
    (ct/toymodel.py:382-419; same seed-derived token ids and permutations)."""
    if strategy not in STRATEGIES:
        raise InvalidPlan(f"unknown strategy {strategy!r}")
    results = []
    for seed in seeds:
        cfg = ModelConfig(seed=seed, mlp=mlp)
        model = GpuModel.reference_init(cfg, dtype=dtype)
        tok_rng = np.random.default_rng([seed, 1])
        sel_rng = np.random.default_rng([seed, 2])
        chunk_ids = [tok_rng.integers(0, cfg.vocab_size, size=n) for n in chunk_tokens]
        suffix = tok_rng.integers(0, cfg.vocab_size, size=suffix_len)
        history = int(sum(chunk_tokens))
        full = full_prefill(model, np.concatenate(chunk_ids + [suffix]), record_attention=True)
        chunks = [encode_chunk_isolated(model, t, chunk_id=f"s{seed}-c{j}")
                  for j, t in enumerate(chunk_ids)]
        rankings = [strategy_ranking(c, strategy, alpha, rng=sel_rng) for c in chunks]
        sel = selective_prefill(model, chunks, rankings, suffix, effective_ratio(strategy, r),
                                record_attention=True)
        dev = attention_deviation(full.attention.suffix_view(history),
                                  sel.attention.suffix_view(history))
        results.append((seed, dev))
    return results


def attention_recovery_at_scale(model: GpuModel, chunk_tokens: Sequence, suffix: Sequence[int],
                                r: float = 0.15,
                                strategies: Sequence[str] = ("lowfreq", "highfreq", "random",
                                                             "none"),
                                alpha: float = 0.5, seed: int = 0) -> dict:
    """The recovery check of run_selection_experiment on a BASELINE geometry
    (SURVEY.md §8(f) row 4): one request, chunks encoded in isolation, every
    strategy at the same budget, suffix-row attention recorded on the device
    (record_attention=<history>: the selective pass stays on the tensor-core
    kernel, only the suffix rows' probabilities are materialised).  Returns
    {strategy: deviation}."""
    for s in strategies:
        if s not in STRATEGIES:
            raise InvalidPlan(f"unknown strategy {s!r}")
    toks = [np.asarray(t, dtype=np.int64) for t in chunk_tokens]
    suffix = np.asarray(suffix, dtype=np.int64)
    history = int(sum(t.size for t in toks))
    full = full_prefill(model, np.concatenate(toks + [suffix]), record_attention=history,
                        logits_rows=None)
    chunks = [encode_chunk_isolated(model, t, chunk_id=f"x{j}") for j, t in enumerate(toks)]
    sel_rng = np.random.default_rng([seed, 2])
    out = {}
    for s in strategies:
        rankings = [strategy_ranking(c, s, alpha, rng=sel_rng) for c in chunks]
        sel = selective_prefill(model, chunks, rankings, suffix, effective_ratio(s, r),
                                record_attention=history, logits_rows=None)
        out[s] = attention_deviation(full.attention.suffix_view(history),
                                     sel.attention.suffix_view(history))
        del sel
    return out


def spectrum_report(chunk, n_bands: int = 10) -> dict:
    """Energy fraction per frequency band for the chunk's Keys and Values
    (ct/toymodel.py:315-341): conjugate-symmetric interior bins double-weighted,
    bands [floor(b*F/n_bands), floor((b+1)*F/n_bands)).  A reporting helper,
    off the hot path: the per-bin spectra come from cuFFT (torch.fft) in f64."""
    if isinstance(chunk, DeviceChunk):
        sides = (("key", chunk.keys), ("value", chunk.values))
    else:
        dev = _dev.require_cuda()
        sides = (("key", torch.from_numpy(np.stack([np.asarray(t.data, np.float32)
                                                    for t in chunk.keys_raw])).to(dev)),
                 ("value", torch.from_numpy(np.stack([np.asarray(t.data, np.float32)
                                                      for t in chunk.values])).to(dev)))
    n = chunk.token_count
    n_freqs = n // 2 + 1
    weights = np.full(n_freqs, 2.0)
    weights[0] = 1.0
    if n % 2 == 0:
        weights[-1] = 1.0
    edges = [int(np.floor(b * n_freqs / n_bands)) for b in range(n_bands + 1)]
    out = {}
    for name, t in sides:
        per_bin = np.zeros(n_freqs)
        for l in range(t.shape[0]):  # layer by layer, in the reference's order
            spec = torch.fft.rfft(t[l].double(), dim=0)
            per_bin += (spec.abs() ** 2).reshape(n_freqs, -1).sum(dim=1).cpu().numpy()
        per_bin *= weights
        total = per_bin.sum()
        bands = np.array([per_bin[edges[b]:edges[b + 1]].sum() for b in range(n_bands)])
        out[name] = bands / total if total > 0 else bands
    return out
