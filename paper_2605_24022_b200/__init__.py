"""B200-native CacheTune online selective-recompute prefill (sm_100a).

Drop-in surface of the reference package's selection, recompute and blend
entry points (ct/__init__.py:6-28); every hot-path op is a kernel of the
in-tree libcachetune_b200.so reached through the C ABI in
include/cachetune_b200.h.  Importing needs no GPU; the first kernel call
needs the .so and a CUDA device (there is no CPU fallback).
"""

from .errors import (AlreadyExists, CacheTuneError, InvalidParam, InvalidPlan,
                     IoError, NotFound, ObjectiveError, ProfileError, ShapeError)
from .kvcore import (DeviceChunk, DtypeCode, KvChunk, SeqTensor,
                     tensor_slice_tokens)

__version__ = "0.1.0"

_LAZY = {
    "ImportanceRanking": "spectral", "rank_chunk": "spectral", "rank_chunks": "spectral",
    "low_freq_scores": "spectral", "high_freq_scores": "spectral",
    "indices_for_ratio": "spectral",
    "complement_for_ratio": "spectral", "selection_count": "spectral",
    "cutoff_index": "spectral", "rfft_seq": "spectral", "irfft_seq": "spectral",
    "lowpass": "spectral", "highpass": "spectral", "jaccard_overlap": "spectral",
    "selection_stability": "spectral", "ComplexSpectrum": "kvcore", "score_device": "spectral", "select_device": "spectral",
    "RopeParams": "rope", "rope_apply": "rope", "rope_rotate": "rope",
    "fuse_layer": "blend", "tensor_scatter_tokens": "blend",
    "ModelConfig": "model", "GpuModel": "model", "ToyModel": "model", "ToyModelConfig": "model",
    "selective_prefill": "prefill", "full_prefill": "prefill",
    "encode_chunk_isolated": "prefill", "PrefillResult": "prefill",
    "AttentionRecord": "prefill", "attention_deviation": "prefill",
    "STRATEGIES": "experiments", "strategy_ranking": "experiments",
    "effective_ratio": "experiments", "run_selection_experiment": "experiments",
    "FrequencyTokenRanker": "estimators", "RatioCalibrator": "estimators",
    # serving surface: resident pool + preallocated per-request engine
    "CachePool": "cachepool", "token_row_bytes": "cachepool", "TierConfig": "pipesim",
    "TIER_PRESETS": "pipesim", "save_tier_config": "pipesim", "load_tier_config": "pipesim",
    "resolve_tier": "pipesim", "write_ctkv": "ctkv", "read_ctkv": "ctkv",
    "KvPool": "pool", "SelectivePrefillEngine": "pipeline", "FullPrefillEngine": "pipeline",
    "prepare_pool": "offline", "calibrate": "scheduler", "SearchConfig": "scheduler",
    "HardwareProfile": "scheduler",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f".{mod}", __name__), name)
