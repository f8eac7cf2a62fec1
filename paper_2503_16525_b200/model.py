"""Model configuration and device weights.

Mirrors reference pkg/src/kvlab/model.py (ModelConfig :24-43, ToyModel :54-80,
init_model :83-84): an attention-only residual stack, weights drawn from
Philox(key=seed) as uniform(-1, 1) / sqrt(d_model) in the order embedding,
then per layer W_q, W_k, W_v, W_o.  Two extensions, both off by default so
the reference model is reproduced exactly:

* ``num_kv_heads`` (GQA): W_k / W_v are (d_model, kv_heads * d_k).
* ``rope_theta``: rotate-half rotary embedding of q and k by position.

Device layout (B200): weights live in bf16 on the GPU.  Every head is padded
to HEAD_DIM = 128 lanes so all tcgen05 tiles are 128 wide: the model's first
half-dims sit at [0, d_k/2) and its second half at [64, 64 + d_k/2), so the
kernels' rotate-half pairing (i, i + 64) is the model's (i, i + d_k/2); the
padding columns of W_q/W_k/W_v and rows of W_o are zero, so the padded
computation equals the unpadded one.  ``init="device"`` draws the (large)
throughput-shape weights with a seeded on-GPU generator instead of numpy
Philox - same distribution, different stream (the parity configs always use
``init="philox"``).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from .errors import ConfigError, InputError

HEAD_DIM = 128


@dataclass(frozen=True)
class ModelConfig:
    num_layers: int = 4
    num_heads: int = 4
    d_model: int = 64
    vocab_size: int = 4096
    seed: int = 0
    num_kv_heads: int | None = None
    rope_theta: float | None = None
    max_positions: int = 65536

    def __post_init__(self):
        for name in ("num_layers", "num_heads", "d_model", "vocab_size"):
            if getattr(self, name) < 1:
                raise ConfigError(f"{name} must be positive")
        if self.d_model % self.num_heads != 0:
            raise ConfigError(
                f"d_model={self.d_model} not divisible by num_heads={self.num_heads}")
        if self.num_kv_heads is not None and (
                self.num_kv_heads < 1 or self.num_heads % self.num_kv_heads != 0):
            raise ConfigError("num_heads must be a multiple of num_kv_heads")
        if self.d_k > HEAD_DIM or self.d_k % 2:
            raise ConfigError(f"head dim {self.d_k} must be even and <= {HEAD_DIM}")

    @property
    def d_k(self) -> int:
        return self.d_model // self.num_heads

    @property
    def kv_heads(self) -> int:
        return self.num_kv_heads or self.num_heads

    @property
    def group(self) -> int:
        return self.num_heads // self.kv_heads


# public model-card shapes - attention stack only
LLAMA31_8B = dict(num_layers=32, num_heads=32, num_kv_heads=8, d_model=4096,
                  vocab_size=128256, rope_theta=500000.0)
QWEN25_7B = dict(num_layers=28, num_heads=28, num_kv_heads=4, d_model=3584,
                 vocab_size=152064, rope_theta=1000000.0)
YI15_9B = dict(num_layers=48, num_heads=32, num_kv_heads=4, d_model=4096,
               vocab_size=64000, rope_theta=5000000.0)


def _pad_index(d_k: int) -> np.ndarray:
    """Padded lane of each model dim: first half -> [0, d/2), second -> [64, 64+d/2)."""
    half = d_k // 2
    return np.concatenate([np.arange(half), HEAD_DIM // 2 + np.arange(half)])


def rope_tables(cfg: ModelConfig, device) -> tuple[torch.Tensor, torch.Tensor]:
    """fp32 cos/sin [max_positions][64] in padded-lane order (lanes >= d_k/2
    get angle 0: their inputs are zero)."""
    half = cfg.d_k // 2
    inv = np.zeros(HEAD_DIM // 2)
    inv[:half] = cfg.rope_theta ** (-np.arange(half, dtype=np.float64) * 2.0 / cfg.d_k)
    ang = np.arange(cfg.max_positions, dtype=np.float64)[:, None] * inv[None, :]
    cos = torch.from_numpy(np.cos(ang).astype(np.float32)).to(device)
    sin = torch.from_numpy(np.sin(ang).astype(np.float32)).to(device)
    return cos.contiguous(), sin.contiguous()


def draw_host_weights(cfg: ModelConfig):
    """Reference draw order and distribution (model.py:57-70), float64."""
    gen = np.random.Generator(np.random.Philox(key=cfg.seed))
    scale = 1.0 / np.sqrt(cfg.d_model)

    def draw(rows, cols):
        return gen.uniform(-1.0, 1.0, size=(rows, cols)) * scale

    d, kvd = cfg.d_model, cfg.kv_heads * cfg.d_k
    emb = draw(cfg.vocab_size, d)
    layers = [(draw(d, d), draw(d, kvd), draw(d, kvd), draw(d, d)) for _ in range(cfg.num_layers)]
    return emb, layers


class ToyModel:
    """Device weights (bf16, head-padded) for the attention stack."""

    def __init__(self, config: ModelConfig, device="cuda", init: str = "philox",
                 host_weights=None):
        self.config = cfg = config
        self.device = torch.device(device)
        H, G, dk = cfg.num_heads, cfg.kv_heads, cfg.d_k
        self.qkv_width = (H + 2 * G) * HEAD_DIM
        self.pad_index = _pad_index(dk)
        if init == "philox" or host_weights is not None:
            emb, layers = host_weights if host_weights is not None else draw_host_weights(cfg)
            self.host_weights = (emb, layers)
            self.embedding = torch.from_numpy(np.asarray(emb)).to(self.device, torch.bfloat16)
            self.w_qkv, self.w_o = [], []
            for wq, wk, wv, wo in layers:
                self.w_qkv.append(self._pack_qkv(wq, wk, wv))
                self.w_o.append(self._pack_o(wo))
        elif init == "device":
            self.host_weights = None
            g = torch.Generator(device=self.device)
            g.manual_seed(cfg.seed)
            scale = 1.0 / math.sqrt(cfg.d_model)

            def draw(rows, cols):
                t = torch.empty(rows, cols, device=self.device, dtype=torch.float32)
                t.uniform_(-1.0, 1.0, generator=g)
                return (t * scale).to(torch.bfloat16)

            self.embedding = draw(cfg.vocab_size, cfg.d_model)
            self.w_qkv, self.w_o = [], []
            for _ in range(cfg.num_layers):
                wq, wk, wv, wo = (draw(cfg.d_model, H * dk), draw(cfg.d_model, G * dk),
                                  draw(cfg.d_model, G * dk), draw(cfg.d_model, cfg.d_model))
                self.w_qkv.append(self._pack_qkv(wq, wk, wv))
                self.w_o.append(self._pack_o(wo))
        else:
            raise ConfigError(f"unknown init {init!r}")
        self.rope = rope_tables(cfg, self.device) if cfg.rope_theta is not None else None

    # -- padding helpers -------------------------------------------------
    def _pad_cols(self, w, heads):
        """(d_model, heads*d_k) -> (d_model, heads*128) in padded-lane order."""
        cfg = self.config
        w = torch.as_tensor(np.asarray(w) if not torch.is_tensor(w) else w)
        w = w.to(self.device, torch.float32).reshape(cfg.d_model, heads, cfg.d_k)
        out = torch.zeros(cfg.d_model, heads, HEAD_DIM, device=self.device, dtype=torch.float32)
        out[:, :, torch.as_tensor(self.pad_index, device=self.device)] = w
        return out.reshape(cfg.d_model, heads * HEAD_DIM)

    def _pack_qkv(self, wq, wk, wv):
        cfg = self.config
        return torch.cat([self._pad_cols(wq, cfg.num_heads), self._pad_cols(wk, cfg.kv_heads),
                          self._pad_cols(wv, cfg.kv_heads)], dim=1).to(torch.bfloat16).contiguous()

    def _pack_o(self, wo):
        """(H*d_k, d_model) -> (H*128, d_model) with zero rows at padding lanes."""
        cfg = self.config
        wo = torch.as_tensor(np.asarray(wo) if not torch.is_tensor(wo) else wo)
        wo = wo.to(self.device, torch.float32).reshape(cfg.num_heads, cfg.d_k, cfg.d_model)
        out = torch.zeros(cfg.num_heads, HEAD_DIM, cfg.d_model, device=self.device)
        out[:, torch.as_tensor(self.pad_index, device=self.device), :] = wo
        return out.reshape(cfg.num_heads * HEAD_DIM, cfg.d_model).to(torch.bfloat16).contiguous()

    def unpad_heads(self, x: torch.Tensor) -> torch.Tensor:
        """[..., 128] padded head vectors -> [..., d_k] model order."""
        return x[..., torch.as_tensor(self.pad_index, device=x.device)]

    def check_tokens(self, tokens: np.ndarray):
        """model.py:72-80 (embed) validation, on the host before upload."""
        if tokens.ndim != 1 or tokens.size == 0:
            raise InputError("token sequence must be a non-empty 1-D array")
        if tokens.min() < 0 or tokens.max() >= self.config.vocab_size:
            raise InputError(f"token id outside vocabulary [0, {self.config.vocab_size})")

    def weight_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in [self.embedding, *self.w_qkv, *self.w_o])


def init_model(config: ModelConfig, device="cuda", init: str = "philox") -> ToyModel:
    return ToyModel(config, device=device, init=init)
