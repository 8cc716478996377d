"""Per-block forward pass with Python hooks (model.py:159-230), on the device ops.

The fused engine (engine.py) runs the sampling hot path; this module serves the
reference's extensibility seams -- `block_forward`, `predict_noise` and
`generate(..., extra_hooks=..., collect_features=...)` -- where a caller's
`LayerHooks` (before_block / after_block / gemm) must see every block.  Every
operation is the same exact device kernel the engine uses (ascending-k f64
`mm`, f64 LN and attention, the cephes GELU), so with no hooks the result is
bit-identical to the reference.  GEMM hooks receive and may return CUDA f32
tensors (`QuantRuntime.gemm_fn` hooks plug in unchanged); NumPy results are
accepted too."""

from __future__ import annotations

from typing import Dict, Optional

import numpy as np
import torch

from . import device as Dv
from .errors import DimensionError
from .model import DiTModel, LayerHooks, timestep_embedding
from .tensor import Tensor, _cuda

_WCACHE: Dict[int, torch.Tensor] = {}


def _w(a: np.ndarray) -> torch.Tensor:
    """Device copy of a (model-owned, immutable) weight array, made once."""
    t = _WCACHE.get(id(a))
    if t is None or t.shape != tuple(a.shape):
        t = torch.as_tensor(np.ascontiguousarray(a, np.float32)).cuda()
        _WCACHE[id(a)] = t
    return t


def _mm(a: torch.Tensor, w) -> torch.Tensor:
    return Dv.gemm_f64(a.contiguous(), w if isinstance(w, torch.Tensor) else _w(w))


def _as_cuda(y) -> torch.Tensor:
    return y.data if isinstance(y, Tensor) else _cuda(y)


def block_forward(x: Tensor, cond: Tensor, t_emb: Tensor, weights, layer: int = 0,
                  hooks: Optional[LayerHooks] = None, num_heads: int = 1) -> Tensor:
    """One transformer block; residual additions stay in f32 (model.py:159-199)."""
    xv = _as_cuda(x)
    if xv.dim() != 2 or xv.shape[1] != weights.sta_q.shape[0]:
        raise DimensionError(f"block input shape {tuple(xv.shape)}")
    cv = _as_cuda(cond).reshape(1, -1)
    if cv.shape[1] != weights.ca_k.shape[0]:
        raise DimensionError(f"cond shape {tuple(cv.shape)}")
    if hooks and hooks.gemm:
        gemm = lambda l, s, a, w: _as_cuda(hooks.gemm(l, s, a, w))   # noqa: E731
    else:
        gemm = lambda _l, _s, a, w: _mm(a, w)   # noqa: E731
    m = _mm(_as_cuda(t_emb).reshape(1, -1), weights.mod)[0].cpu().numpy()
    sh1, sc1, g1, sh3, sc3, g3 = (np.float32(m[i]) for i in range(6))
    one = np.float32(1.0)

    def ln(v, g, b, scale=one, shift=np.float32(0.0)):
        return Dv.ln_mod(v.contiguous(), _w(g), _w(b), float(scale), float(shift))

    h1 = ln(xv, weights.ln1_g, weights.ln1_b, one + sc1, sh1)
    q = gemm(layer, "sta_q", h1, weights.sta_q)
    k = gemm(layer, "sta_k", h1, weights.sta_k)
    v = gemm(layer, "sta_v", h1, weights.sta_v)
    att = Dv.attention_f64(q.contiguous(), k.contiguous(), v.contiguous(), num_heads)
    xv = xv + float(g1) * gemm(layer, "sta_o", att, weights.sta_o)
    h2 = ln(xv, weights.ln2_g, weights.ln2_b)
    q2 = gemm(layer, "ca_q", h2, weights.ca_q)
    k2 = gemm(layer, "ca_k", cv, weights.ca_k)
    v2 = gemm(layer, "ca_v", cv, weights.ca_v)
    ca = Dv.attention_f64(q2.contiguous(), k2.contiguous(), v2.contiguous(), num_heads)
    xv = xv + gemm(layer, "ca_o", ca, weights.ca_o)
    h3 = ln(xv, weights.ln3_g, weights.ln3_b, one + sc3, sh3)
    hid = gemm(layer, "ffn1", h3, weights.ffn1).contiguous().clone()
    Dv.gelu_inplace(hid)
    xv = xv + float(g3) * gemm(layer, "ffn2", hid, weights.ffn2)
    return Tensor(xv, frame_axis=getattr(x, "frame_axis", None))


def predict_noise(x_t: Tensor, t: int, cond: Tensor, model: DiTModel,
                  hooks: Optional[LayerHooks] = None,
                  total_steps: Optional[int] = None) -> Tensor:
    """Full forward pass: L blocks plus the linear head (model.py:202-230)."""
    if t < 0 or (total_steps is not None and t >= total_steps):
        raise ValueError(f"timestep {t} out of range")
    cfg = model.cfg
    xt = _as_cuda(x_t)
    if tuple(xt.shape) != (cfg.frames, cfg.tokens_per_frame, cfg.model_dim):
        raise DimensionError(f"latent shape {tuple(xt.shape)}")
    x = Tensor(xt.reshape(cfg.seq_len, cfg.model_dim))
    t_emb = Tensor(timestep_embedding(t, cfg.model_dim))
    for l in range(cfg.num_blocks):
        rep = hooks.before_block(l, x) if hooks and hooks.before_block else None
        x = rep if rep is not None else block_forward(x, cond, t_emb, model.blocks[l], l,
                                                      hooks, cfg.num_heads)
        if hooks and hooks.after_block:
            hooks.after_block(l, x)
    out = Dv.gemm_f64(_as_cuda(x).contiguous(), _w(model.head_w)) + _w(model.head_b)
    return Tensor(out.reshape(cfg.frames, cfg.tokens_per_frame, cfg.model_dim), frame_axis=0)


def generate_hooked(model: DiTModel, sched, seed: int = 0, collect_features=None,
                    extra_hooks: Optional[LayerHooks] = None) -> torch.Tensor:
    """The reference generate loop without a scheduler (sampler.py:91-134): NumPy
    RNG order x, cond, one noise draw per t > 0; hooks see every block."""
    from .sampler import final_step, reverse_step
    cfg = model.cfg
    rng = np.random.default_rng(seed)
    shape = (cfg.frames, cfg.tokens_per_frame, cfg.model_dim)
    x = Tensor(rng.standard_normal(shape).astype(np.float32), frame_axis=0)
    cond = Tensor(rng.standard_normal(cfg.cond_dim).astype(np.float32))
    for t in range(sched.steps - 1, -1, -1):
        hooks = extra_hooks
        outs = [] if collect_features is not None else None
        if outs is not None:
            base = hooks

            def after(l, out, base=base, outs=outs):
                if base and base.after_block:
                    base.after_block(l, out)
                outs.append(out)

            hooks = LayerHooks(before_block=base.before_block if base else None,
                               after_block=after, gemm=base.gemm if base else None)
        eps = predict_noise(x, t, cond, model, hooks, total_steps=sched.steps)
        if collect_features is not None:
            collect_features.append((t, x, outs))
        if t > 0:
            noise = Tensor(rng.standard_normal(shape).astype(np.float32), frame_axis=0)
            x = Tensor(reverse_step(x.data, t, eps.data, sched, noise.data), frame_axis=0)
        else:
            x = Tensor(final_step(x.data, eps.data, sched), frame_axis=0)
    return x.data
