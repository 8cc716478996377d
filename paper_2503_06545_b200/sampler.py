"""DDPM schedule and the sampling entry point (mirror of ditrt.sampler).

`generate` keeps the reference's signature (sampler.py:91-98).  With a
`Scheduler` (or none) the whole reverse trajectory runs in the device engine;
`reverse_step` / `final_step` are the device DDPM update (qcb_ddpm_step)."""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

import numpy as np
import torch

from . import device as Dv
from .errors import ConfigurationError, DimensionError


@dataclass
class NoiseSchedule:
    """sampler.py:21-37"""
    alpha_bar: np.ndarray

    def __post_init__(self):
        ab = np.asarray(self.alpha_bar, dtype=np.float64)
        if ab.ndim != 1 or ab.size == 0:
            raise ConfigurationError("alpha_bar must be a nonempty vector")
        if not (np.all(ab > 0) and np.all(ab <= 1)):
            raise ConfigurationError("alpha_bar values must lie in (0, 1]")
        if np.any(np.diff(ab) >= 0):
            raise ConfigurationError("alpha_bar must be strictly decreasing")
        self.alpha_bar = ab

    @property
    def steps(self) -> int:
        return len(self.alpha_bar)


def linear_beta_schedule(steps: int, beta_start: float = 1e-4,
                         beta_end: float = 2e-2) -> NoiseSchedule:
    """sampler.py:40-45"""
    if steps < 1:
        raise ConfigurationError("schedule needs at least one step")
    return NoiseSchedule(np.cumprod(1.0 - np.linspace(beta_start, beta_end, steps,
                                                      dtype=np.float64)))


def _cuda(x):
    x = getattr(x, "data", x)
    if isinstance(x, torch.Tensor):
        return x.float().cuda().contiguous()
    return torch.as_tensor(np.ascontiguousarray(np.asarray(x, np.float32))).cuda()


def reverse_step(x_t, t: int, eps_hat, sched: NoiseSchedule, noise) -> torch.Tensor:
    """Fixed-variance DDPM posterior step, noise only for t > 1 (sampler.py:59-80)."""
    if not 1 <= t < sched.steps:
        raise ValueError(f"reverse step timestep {t} out of range")
    x, e, n = _cuda(x_t), _cuda(eps_hat), _cuda(noise)
    if x.shape != e.shape or x.shape != n.shape:
        raise DimensionError("reverse step operands must share a shape")
    a_t, a_p = sched.alpha_bar[t], sched.alpha_bar[t - 1]
    alpha = a_t / a_p
    beta = 1.0 - alpha
    c3 = float(np.sqrt((1.0 - a_p) / (1.0 - a_t) * beta)) if t > 1 else 0.0
    return Dv.ddpm(x, e, float(beta / np.sqrt(1.0 - a_t)), float(np.sqrt(alpha)),
                   n if t > 1 else None, c3)


def final_step(x0_noisy, eps_hat, sched: NoiseSchedule) -> torch.Tensor:
    """Deterministic t = 0 clean-data estimate (sampler.py:83-88)."""
    ab0 = sched.alpha_bar[0]
    return Dv.ddpm(_cuda(x0_noisy), _cuda(eps_hat), float(np.sqrt(1.0 - ab0)),
                   float(np.sqrt(ab0)))


def forward_noise(x0, t: int, eps, sched: NoiseSchedule) -> torch.Tensor:
    """x_t = sqrt(abar) x0 + sqrt(1-abar) eps (sampler.py:48-56; training side)."""
    if not 0 <= t < sched.steps:
        raise ValueError(f"timestep {t} out of range")
    x, e = _cuda(x0), _cuda(eps)
    if x.shape != e.shape:
        raise DimensionError("x0 and eps must share a shape")
    ab = sched.alpha_bar[t]
    # x_t = (x0 - c1*eps)/c2 with c1 = -sqrt(1-ab)/sqrt(ab), c2 = 1/sqrt(ab) is not
    # bit-identical; do the two products in f64 directly.
    return (np.sqrt(ab) * x.double() + np.sqrt(1.0 - ab) * e.double()).float()


def generate(model, sched: NoiseSchedule, scheduler=None, seed: int = 0,
             collect_features: Optional[List] = None, extra_hooks=None, options=None):
    """Run the full reverse trajectory (sampler.py:91-134) on the device.

    Returns the final latent as a CUDA tensor (frames, tokens, d).  The
    scheduler (schedule.Scheduler) receives the trace like the reference's."""
    from .engine import EngineOptions, QuantCacheEngine
    from .schedule import ThresholdConfig, Toggles
    if scheduler is None and (extra_hooks is not None or collect_features is not None):
        # caller hooks see every block: the per-block device path (forward.py)
        from .forward import generate_hooked
        return generate_hooked(model, sched, seed, collect_features, extra_hooks)
    # with a scheduler the reference uses only the scheduled hooks: extra_hooks
    # is ignored (reference sampler.py:114-119)
    if scheduler is None:
        eng = QuantCacheEngine(model, sched.alpha_bar, Toggles(),
                               ThresholdConfig(delta1=0.0, delta2=0.0), options=options)
    else:
        eng = scheduler.engine(model, sched, options)
    feats = [] if collect_features is not None else None
    out, traces = eng.generate([seed], collect_features=feats)
    if scheduler is not None:
        scheduler.trace.extend(traces[0])
    if feats is not None:   # the reference's (t, x_t, [block outputs]) of video 0
        from .tensor import Tensor
        shp = (model.cfg.frames, model.cfg.tokens_per_frame, model.cfg.model_dim)
        for t, x_now, outs in feats:
            collect_features.append((t, Tensor(x_now[0].reshape(shp), frame_axis=0),
                                     [Tensor(o[0]) for o in outs]))
    return torch.as_tensor(out[0]).cuda()
