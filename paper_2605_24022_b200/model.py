"""Transformer weights resident in HBM for the recompute path.

`ModelConfig` extends the reference's ToyModelConfig (ct/toymodel.py:31-55)
with the knobs the BASELINE geometries need (n_kv_heads for GQA, a SwiGLU
MLP, RoPE base/pairing/scaling); with defaults it is the toy model.
`GpuModel.from_reference` uploads a reference `ToyModel` bit-exactly (f32 or
bf16); `GpuModel.random` draws U(-1,1)/sqrt(hid) weights like
ct/toymodel.py:64-68 directly on the device (for 8B-scale geometries).
QKV projections are fused into one [hid, (Hq+2Hkv)D] matrix; SwiGLU gate and
up into one [hid, 2*inter] matrix.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import ShapeError
from .rope import RopeParams


@dataclass(frozen=True)
class ModelConfig:
    seed: int = 0
    n_layers: int = 4
    n_heads: int = 2
    head_dim: int = 8
    vocab_size: int = 256
    mlp: object = False          # False | True/"relu" (reference) | "swiglu"
    rope_base: float = 10000.0
    n_kv_heads: int | None = None
    intermediate: int | None = None
    rope_pairing: str = "adjacent"
    rope_scaling: float = 1.0

    def __post_init__(self):
        if min(self.n_layers, self.n_heads, self.head_dim, self.vocab_size) < 1:
            raise ShapeError("all model dims must be >= 1")
        if self.head_dim % 2 != 0:
            raise ShapeError("head_dim must be even")
        if self.n_heads % self.kv_heads:
            raise ShapeError("n_heads must be a multiple of n_kv_heads")

    @property
    def hidden_dim(self) -> int:
        return self.n_heads * self.head_dim

    @property
    def kv_heads(self) -> int:
        return self.n_kv_heads or self.n_heads

    @property
    def mlp_kind(self):
        if self.mlp is True:
            return "relu"
        return self.mlp or None

    @property
    def inter(self) -> int:
        return self.intermediate or 4 * self.hidden_dim

    @property
    def rope_params(self) -> RopeParams:
        return RopeParams(head_dim=self.head_dim, base=self.rope_base,
                          scaling=self.rope_scaling, pairing=self.rope_pairing)

    @classmethod
    def llama3_8b(cls, n_layers: int = 32, vocab_size: int = 128256, **kw) -> "ModelConfig":
        """BASELINE configs 2/4/5 geometry (32 layers, 32/8 heads, D=128, SwiGLU 14336)."""
        return cls(n_layers=n_layers, n_heads=32, head_dim=128, vocab_size=vocab_size,
                   mlp="swiglu", n_kv_heads=8, intermediate=14336, **kw)

    @classmethod
    def mistral_7b(cls, n_layers: int = 32, vocab_size: int = 32768, **kw) -> "ModelConfig":
        """BASELINE config 3 geometry."""
        return cls(n_layers=n_layers, n_heads=32, head_dim=128, vocab_size=vocab_size,
                   mlp="swiglu", n_kv_heads=8, intermediate=14336, **kw)


class GpuModel:
    """Weights in HBM.  dtype: torch.float32 (1e-5 mode) or torch.bfloat16."""

    def __init__(self, config: ModelConfig, embedding, layers, w_out, dtype):
        self.config = config
        self.embedding = embedding      # [V, hid] f32 (rows gathered into the f32 residual)
        self.layers = layers            # list of dicts of [in, out] matrices
        self.w_out = w_out              # [hid, V]
        self.dtype = dtype

    @property
    def device(self):
        return self.embedding.device

    @classmethod
    def from_numpy(cls, config: ModelConfig, embedding, layers, w_out,
                   dtype=torch.float32, device="cuda"):
        def up(a):
            return torch.from_numpy(np.require(a, np.float64, ["C", "W"])) \
                .to(device=device, dtype=dtype)
        glayers = []
        for layer in layers:
            g = {"wqkv": up(np.concatenate([layer["wq"], layer["wk"], layer["wv"]], axis=1)),
                 "wo": up(layer["wo"])}
            if "w1" in layer:
                g["w1"], g["w2"] = up(layer["w1"]), up(layer["w2"])
            if "wg" in layer:
                g["wgu"] = up(np.concatenate([layer["wg"], layer["wu"]], axis=1))
                g["wd"] = up(layer["wd"])
            glayers.append(g)
        emb = torch.from_numpy(np.asarray(embedding, dtype=np.float32)).to(device)
        return cls(config, emb, glayers, up(w_out), dtype)

    @classmethod
    def from_reference(cls, ref_model, dtype=torch.float32, device="cuda", **extra):
        """Upload a reference ToyModel (or oracle Model) with identical weights."""
        c = ref_model.config
        cfg = ModelConfig(seed=c.seed, n_layers=c.n_layers, n_heads=c.n_heads,
                          head_dim=c.head_dim, vocab_size=c.vocab_size, mlp=c.mlp,
                          rope_base=c.rope_base,
                          n_kv_heads=getattr(c, "n_kv_heads", None),
                          intermediate=getattr(c, "intermediate", None),
                          rope_pairing=getattr(c, "rope_pairing", "adjacent"),
                          rope_scaling=getattr(c, "rope_scaling", 1.0), **extra)
        return cls.from_numpy(cfg, ref_model.embedding, ref_model.layers, ref_model.w_out,
                              dtype=dtype, device=device)

    @classmethod
    def reference_init(cls, config: ModelConfig, dtype=torch.float32, device="cuda"):
        """The reference ToyModel's seeded weights (ct/toymodel.py:61-79): the same
        numpy default_rng(seed) draw order, so a seed names the same model here as
        in the reference's experiments.  Reference geometry only (MHA, relu MLP)."""
        if config.kv_heads != config.n_heads or config.mlp_kind not in (None, "relu"):
            raise ShapeError("reference_init covers the reference ToyModel geometry only")
        hid = config.hidden_dim
        rng = np.random.default_rng(config.seed)
        scale = 1.0 / np.sqrt(hid)

        def w(*shape):
            return rng.uniform(-1.0, 1.0, size=shape) * scale
        emb = w(config.vocab_size, hid)
        layers = []
        for _ in range(config.n_layers):
            layer = {"wq": w(hid, hid), "wk": w(hid, hid), "wv": w(hid, hid), "wo": w(hid, hid)}
            if config.mlp_kind == "relu":
                layer["w1"] = w(hid, 4 * hid)
                layer["w2"] = w(4 * hid, hid)
            layers.append(layer)
        return cls.from_numpy(config, emb, layers, w(hid, config.vocab_size), dtype=dtype,
                              device=device)

    @classmethod
    def random(cls, config: ModelConfig, dtype=torch.bfloat16, device="cuda", seed=None):
        """U(-1,1)/sqrt(hid) weights drawn on the device (ct/toymodel.py:64-68 law)."""
        gen = torch.Generator(device=device)
        gen.manual_seed(config.seed if seed is None else seed)
        hid, d = config.hidden_dim, config.head_dim
        qkv = (config.n_heads + 2 * config.kv_heads) * d
        scale = 1.0 / float(np.sqrt(hid))

        def w(*shape, dt=dtype):
            t = torch.empty(shape, dtype=torch.float32, device=device)
            t.uniform_(-1.0, 1.0, generator=gen).mul_(scale)
            return t.to(dt)
        emb = w(config.vocab_size, hid, dt=torch.float32)
        layers = []
        for _ in range(config.n_layers):
            g = {"wqkv": w(hid, qkv), "wo": w(hid, hid)}
            if config.mlp_kind == "relu":
                g["w1"], g["w2"] = w(hid, 4 * hid), w(4 * hid, hid)
            elif config.mlp_kind == "swiglu":
                g["wgu"], g["wd"] = w(hid, 2 * config.inter), w(config.inter, hid)
            layers.append(g)
        return cls(config, emb, layers, w(hid, config.vocab_size), dtype)

    def to_numpy_weights(self) -> dict:
        """Host float64 copy (for the CPU oracle in tests)."""
        cfg = self.config
        hd = cfg.n_heads * cfg.head_dim
        kvd = cfg.kv_heads * cfg.head_dim
        layers = []
        for g in self.layers:
            qkv = g["wqkv"].double().cpu().numpy()
            layer = {"wq": qkv[:, :hd], "wk": qkv[:, hd:hd + kvd], "wv": qkv[:, hd + kvd:],
                     "wo": g["wo"].double().cpu().numpy()}
            if "w1" in g:
                layer["w1"], layer["w2"] = g["w1"].double().cpu().numpy(), g["w2"].double().cpu().numpy()
            if "wgu" in g:
                gu = g["wgu"].double().cpu().numpy()
                layer["wg"], layer["wu"] = gu[:, :cfg.inter], gu[:, cfg.inter:]
                layer["wd"] = g["wd"].double().cpu().numpy()
            layers.append(layer)
        return {"embedding": self.embedding.double().cpu().numpy(), "layers": layers,
                "w_out": self.w_out.double().cpu().numpy()}


# Drop-in names of ct/toymodel.py:31-85: the reference's config fields are a
# subset of ModelConfig's (same names and defaults), and a ToyModel is the
# seeded reference geometry with its weights resident in HBM.
ToyModelConfig = ModelConfig


def ToyModel(config: ModelConfig, dtype=torch.float32, device="cuda") -> GpuModel:  # noqa: N802
    """The reference ToyModel (ct/toymodel.py:58-79) on the device: same seed ->
    same weights (GpuModel.reference_init), fp32 by default (the 1e-5 mode)."""
    return GpuModel.reference_init(config, dtype=dtype, device=device)
