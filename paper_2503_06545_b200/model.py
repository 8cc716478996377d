"""Toy-DiT model description for the B200 path (mirror of ditrt.model).

Weights are host NumPy arrays produced by the same seeded draw sequence as the
reference's `init_model` (model.py:101-124), so a given config yields identical
weights; the engine uploads them once.  Block computation itself happens on the
device (engine.py); `block_mac_cost`/`head_mac_cost` reproduce the reference's
MAC accounting (model.py:237-252)."""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass, fields
from typing import Callable, List, Optional

import numpy as np

from .errors import ConfigurationError

QUANT_SITES = ("sta_q", "sta_k", "sta_v", "sta_o", "ca_q", "ca_k", "ca_v", "ca_o",
               "ffn1", "ffn2")
FFN_RATIO = 4


@dataclass(frozen=True)
class DiTConfig:
    """model.py:35-57"""
    num_blocks: int = 8
    model_dim: int = 64
    num_heads: int = 4
    tokens_per_frame: int = 16
    frames: int = 4
    cond_dim: int = 32
    seed: int = 0

    def __post_init__(self):
        if min(self.num_blocks, self.model_dim, self.num_heads, self.tokens_per_frame,
               self.frames, self.cond_dim) <= 0:
            raise ConfigurationError("all model dimensions must be positive")
        if self.model_dim % self.num_heads:
            raise ConfigurationError(
                f"model_dim {self.model_dim} not divisible by num_heads {self.num_heads}")

    @property
    def seq_len(self) -> int:
        return self.tokens_per_frame * self.frames


@dataclass
class BlockWeights:
    """Field order is the snapshot/checksum order of model.py:60-78."""
    ln1_g: np.ndarray
    ln1_b: np.ndarray
    sta_q: np.ndarray
    sta_k: np.ndarray
    sta_v: np.ndarray
    sta_o: np.ndarray
    ln2_g: np.ndarray
    ln2_b: np.ndarray
    ca_q: np.ndarray
    ca_k: np.ndarray
    ca_v: np.ndarray
    ca_o: np.ndarray
    ln3_g: np.ndarray
    ln3_b: np.ndarray
    ffn1: np.ndarray
    ffn2: np.ndarray
    mod: np.ndarray


@dataclass
class LayerHooks:
    """Overridable execution hooks (model.py:81-90); all-None = plain forward."""
    before_block: Optional[Callable] = None
    after_block: Optional[Callable] = None
    gemm: Optional[Callable] = None


@dataclass
class DiTModel:
    cfg: DiTConfig
    blocks: List[BlockWeights]
    head_w: np.ndarray
    head_b: np.ndarray


def _shapes(cfg: DiTConfig):
    d, c, h = cfg.model_dim, cfg.cond_dim, FFN_RATIO * cfg.model_dim
    # (field, shape, fan_in or None for LN constants); draw order = declaration order
    return [("ln1_g", (d,), "one"), ("ln1_b", (d,), "zero"),
            ("sta_q", (d, d), d), ("sta_k", (d, d), d), ("sta_v", (d, d), d),
            ("sta_o", (d, d), d), ("ln2_g", (d,), "one"), ("ln2_b", (d,), "zero"),
            ("ca_q", (d, d), d), ("ca_k", (c, d), c), ("ca_v", (c, d), c),
            ("ca_o", (d, d), d), ("ln3_g", (d,), "one"), ("ln3_b", (d,), "zero"),
            ("ffn1", (d, h), d), ("ffn2", (h, d), h), ("mod", (d, 6), d)]


def init_model(cfg: DiTConfig) -> DiTModel:
    """Seeded N(0, fan_in^-1/2) init; identical draws to the reference."""
    rng = np.random.default_rng(cfg.seed)
    blocks = []
    for _ in range(cfg.num_blocks):
        vals = {}
        for name, shape, fan in _shapes(cfg):
            if fan == "one":
                vals[name] = np.ones(shape, np.float32)
            elif fan == "zero":
                vals[name] = np.zeros(shape, np.float32)
            else:
                vals[name] = rng.normal(0.0, fan ** -0.5, size=shape).astype(np.float32)
        blocks.append(BlockWeights(**vals))
    d = cfg.model_dim
    head_w = rng.normal(0.0, d ** -0.5, size=(d, d)).astype(np.float32)
    head_b = rng.normal(0.0, d ** -0.5, size=(d,)).astype(np.float32)
    return DiTModel(cfg, blocks, head_w, head_b)


def timestep_embedding(t: int, dim: int) -> np.ndarray:
    """Sinusoidal embedding (model.py:127-134); host scalar prep."""
    half = dim // 2
    w = np.exp(-np.log(10000.0) * np.arange(half, dtype=np.float64) / half)
    out = np.zeros(dim, np.float64)
    out[:half] = np.sin(t * w)
    out[half:2 * half] = np.cos(t * w)
    return out.astype(np.float32)


@dataclass
class BlockCost:
    quantizable: int
    fp_always: int


def block_mac_cost(cfg: DiTConfig) -> BlockCost:
    """model.py:237-248"""
    s, d, c = cfg.seq_len, cfg.model_dim, cfg.cond_dim
    return BlockCost(
        quantizable=(6 + 2 * FFN_RATIO) * s * d * d + 2 * c * d,
        fp_always=2 * s * s * d + 2 * s * d + 6 * d)


def head_mac_cost(cfg: DiTConfig) -> int:
    return cfg.seq_len * cfg.model_dim * cfg.model_dim


def _arrays(model: DiTModel):
    for blk in model.blocks:
        for f in fields(BlockWeights):
            yield getattr(blk, f.name)
    yield model.head_w
    yield model.head_b


def weight_checksum(model: DiTModel) -> str:
    """sha256 over the little-endian f32 payload (model.py:288-292)."""
    h = hashlib.sha256()
    for a in _arrays(model):
        h.update(np.ascontiguousarray(a, dtype="<f4").tobytes())
    return h.hexdigest()


def save_weights(model: DiTModel, path):
    """Snapshot: JSON header line + little-endian f32 payload (model.py:268-273)."""
    with open(path, "wb") as fh:
        fh.write(json.dumps(model.cfg.__dict__, sort_keys=True).encode() + b"\n")
        for a in _arrays(model):
            fh.write(np.ascontiguousarray(a, dtype="<f4").tobytes())


def load_weights(path) -> DiTModel:
    with open(path, "rb") as fh:
        model = init_model(DiTConfig(**json.loads(fh.readline().decode())))
        for a in _arrays(model):
            raw = fh.read(a.size * 4)
            if len(raw) != a.size * 4:
                raise ValueError("truncated weight snapshot")
            a[...] = np.frombuffer(raw, dtype="<f4").reshape(a.shape)
    return model
