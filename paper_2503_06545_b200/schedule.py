"""Decision-engine configuration and host-side policy helpers.

The per-step decisions themselves are made ON DEVICE by the qcb_policy_*
kernels (csrc/qc_reduce.cu) from device reductions; this module holds the
config objects with the reference's names and semantics
(/root/reference/pkg/src/ditrt/schedule.py:22-234) and the scalar piecewise
policies, which the harness uses to audit traces (replay) and which the tests
compare against the device plan."""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from .errors import ConfigurationError

FP_BITS = 32


@dataclass
class ThresholdConfig:
    """schedule.py:22-60"""
    delta1: float
    delta2: float
    tau_max: int = 6
    tau_mid: int = 3
    tau_min: int = 1
    theta1: float = 0.4
    theta2: float = 0.8
    bit_max: int = 8
    bit_mid: int = 6
    bit_min: int = 4
    tau_high: float = 0.98
    tau_low: float = 0.5
    p_base: float = 0.3
    v_low: float = 0.0
    v_high: float = 0.0
    history_k: int = 4
    prune_adjust: float = 2.0

    def validate(self):
        rules = (
            ("delta1/delta2", self.delta1 <= self.delta2),
            ("theta1/theta2", self.theta1 <= self.theta2),
            ("tau_low/tau_high", self.tau_low <= self.tau_high),
            ("v_low/v_high", self.v_low <= self.v_high),
            ("tau_min/tau_mid/tau_max", self.tau_min <= self.tau_mid <= self.tau_max),
            ("bit_min/bit_mid/bit_max", self.bit_min <= self.bit_mid <= self.bit_max),
            ("tau_min", self.tau_min >= 1),
            ("p_base", 0.0 <= self.p_base <= 1.0),
            ("prune_adjust", self.prune_adjust >= 1.0),
            ("history_k", self.history_k >= 1),
        )
        for name, ok in rules:
            if not ok:
                raise ConfigurationError(f"threshold invariant violated: {name}")
        if not (1 <= self.bit_min and self.bit_max <= 8):
            raise ConfigurationError("activation bit-widths must lie in [1, 8] on the u8 path")
        return self


@dataclass
class Toggles:
    """schedule.py:213-221"""
    hlc: bool = False
    aigq_weights: bool = False
    aigq_acts: bool = False
    srap: bool = False

    def any(self) -> bool:
        return self.hlc or self.aigq_weights or self.aigq_acts or self.srap


@dataclass
class TraceRecord:
    """schedule.py:187-210 (JSON field names kept for trace compatibility)."""
    t: int
    layer: object
    action: str
    d: Optional[float]
    s: Optional[float]
    bits: int
    wbits: int
    macs: int
    v: Optional[float] = None

    def to_json_obj(self):
        return {"t": self.t, "layer": self.layer, "action": self.action, "D": self.d,
                "S": self.s, "bits": self.bits, "wbits": self.wbits, "macs": self.macs,
                "V": self.v}


@dataclass
class ScheduleDecision:
    """schedule.py:176-184"""
    t: int
    actions: List[str]
    abits: int
    divergences: List[Optional[float]]
    similarities: List[Optional[float]]
    v: float
    forced_bitmax: bool = False


def billed_macs(cost, wbits: int, abits: int) -> int:
    """FP32xFP32 MAC = 1024 units (schedule.py:232-234)."""
    return cost.quantizable * wbits * abits + cost.fp_always * FP_BITS * FP_BITS


# ---- scalar piecewise policies (the device plan kernel implements the same)

def refresh_interval(d: float, cfg: ThresholdConfig) -> int:
    if d < cfg.delta1:
        return cfg.tau_max
    return cfg.tau_mid if d < cfg.delta2 else cfg.tau_min


def redundancy_metric(d_layers: Sequence[float]) -> float:
    if len(d_layers) == 0:
        raise ValueError("need at least one divergence score")
    return 1.0 / (1.0 + float(np.mean(d_layers)))


def activation_bits(r: float, cfg: ThresholdConfig) -> int:
    if r >= cfg.theta2:
        return cfg.bit_min
    return cfg.bit_mid if r >= cfg.theta1 else cfg.bit_max


def prune_probability(s: float, cfg: ThresholdConfig, p_base: Optional[float] = None) -> float:
    base = cfg.p_base if p_base is None else p_base
    if s > cfg.tau_high:
        return 1.0
    return base if s >= cfg.tau_low else 0.0


def adapt_prune_rate(v: float, cfg: ThresholdConfig) -> float:
    if v < cfg.v_low:
        return min(1.0, cfg.p_base * cfg.prune_adjust)
    if v > cfg.v_high:
        return cfg.p_base / cfg.prune_adjust
    return cfg.p_base


def prune_draw(seed: int, t: int, layer: int) -> float:
    """Counter-keyed uniform (schedule.py:144-146).  NumPy's SeedSequence/PCG64
    is the RNG source; the engine uploads a (t, layer) table of these."""
    return float(np.random.default_rng(np.random.SeedSequence((seed, t, layer))).random())


def prune_draw_table(seed: int, steps: int, layers: int) -> np.ndarray:
    tab = np.empty((steps, layers), np.float64)
    for t in range(steps):
        for l in range(layers):
            tab[t, l] = prune_draw(seed, t, l)
    return tab


# ---------------------------------------------------------------------------
# Scheduler: the per-run decision engine (schedule.py:240-382) with its state
# on the device.  `plan_step` / `observe_block` / `finalize_step` keep the
# reference's call protocol for model-free drivers (tests' drive()); a full
# `generate` hands the same configuration to the fused engine instead.


class Scheduler:
    def __init__(self, num_layers: int, total_steps: int, cfg: ThresholdConfig,
                 toggles: Toggles, block_cost, head_macs: int, prune_seed: int = 0,
                 weight_bits=None):
        cfg.validate()
        from . import _native as N
        self.num_layers, self.total_steps = num_layers, total_steps
        self.cfg, self.toggles = cfg, toggles
        self.block_cost, self.head_macs = block_cost, head_macs
        self.prune_seed = prune_seed
        self.weight_bits = dict(weight_bits or {})
        self.trace: List[TraceRecord] = []
        self.quant_runtime = None
        self._N = N
        self._state = None

    # -- configuration hand-off to the fused engine ------------------------
    def gemm_policy(self, decision: ScheduleDecision):
        if self.quant_runtime is None:
            return None
        return self.quant_runtime.gemm_fn(decision.abits)

    def engine(self, model, sched, options=None):
        from .engine import QuantCacheEngine
        qr = self.quant_runtime
        return QuantCacheEngine(
            model, sched.alpha_bar, self.toggles, self.cfg,
            weight_bits=self.weight_bits if self.toggles.aigq_weights else {},
            act_absmax=(qr.site_act_absmax if qr is not None else None),
            sign_seed=(qr.sign_seed if qr is not None else 0),
            prune_seed=self.prune_seed, max_videos=1, options=options)

    # -- step protocol on device state --------------------------------------
    def _init_state(self):
        import ctypes
        import torch
        from . import device as Dv
        N = self._N
        self._pol = torch.zeros(ctypes.sizeof(N.QcbPolicyVideo), dtype=torch.uint8,
                                device="cuda")
        self._thc = Dv.thresholds_struct(self.cfg, self.toggles)
        self._draws = torch.as_tensor(prune_draw_table(self.prune_seed, self.total_steps,
                                                       self.num_layers)).cuda()
        self._srap = torch.zeros((self.num_layers, 1, 3), dtype=torch.float64, device="cuda")
        self._mask = torch.zeros((self.num_layers, 1), dtype=torch.int32, device="cuda")
        self._hl1 = torch.zeros((self.cfg.history_k + 1, 1), dtype=torch.float64, device="cuda")
        self._hlc = torch.zeros((1, 2), dtype=torch.float64, device="cuda")
        self.cache = {}
        self.prev_features = {}
        self.latent_history = []
        self._state = True

    @staticmethod
    def _flat(x):
        import torch
        x = getattr(x, "data", x)
        t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x, np.float32))
        t = t.float().cuda().contiguous()
        return t.reshape(-1, t.shape[-1]) if t.dim() > 1 else t.reshape(1, -1)

    def _read(self):
        N = self._N
        return N.QcbPolicyVideo.from_buffer_copy(self._pol.cpu().numpy().tobytes())

    def plan_step(self, t: int, x_t) -> ScheduleDecision:
        from . import device as Dv
        if self._state is None:
            self._init_state()
        N, L = self._N, self.num_layers
        lib, sp = N.lib(), N.stream_ptr()
        x = self._flat(x_t)
        rows, cols = x.shape
        for j, h in enumerate(self.latent_history):
            Dv.reduce_l1(Dv.feat(x), Dv.feat(h), rows, cols, 1, self._hl1[j])
        N.check(lib.qcb_policy_plan_reuse(self._pol.data_ptr(), 1, L, t, self._thc, sp), "plan")
        N.check(lib.qcb_policy_sim_mask(self._pol.data_ptr(), 1, L, self._thc,
                                        N.ptr(self._mask), sp), "mask")
        for l in range(1, L):
            a, b = self.prev_features.get(l - 1), self.prev_features.get(l)
            if a is not None and b is not None:
                Dv.reduce_srap(Dv.feat(a), Dv.feat(b), a.shape[0], a.shape[1], 1,
                               self._srap[l], seg_active=self._mask[l])
        N.check(lib.qcb_policy_plan_finish(self._pol.data_ptr(), 1, L, t, self._thc,
                                           N.ptr(self._srap), N.ptr(self._hl1),
                                           len(self.latent_history),
                                           N.ptr(self._draws[t]), 0, sp), "plan_finish")
        p = self._read()
        names = ("recompute", "reuse", "prune")
        return ScheduleDecision(
            t, [names[p.action[l]] for l in range(L)], int(p.abits), [None] * L,
            [float(p.sim[l]) if p.sim_valid[l] else None for l in range(L)], float(p.v),
            bool(p.forced))

    def observe_block(self, t: int, layer: int, out, decision: ScheduleDecision):
        from . import device as Dv
        N = self._N
        o = self._flat(out)
        act = decision.actions[layer]
        prev = self.prev_features.get(layer)
        if act == "recompute":
            ref = self.cache[layer] if layer in self.cache else prev
            if ref is not None and prev is not None:
                Dv.reduce_hlc(Dv.feat(o), Dv.feat(ref), Dv.feat(prev), o.shape[0], o.shape[1],
                              1, self._hlc)
        N.check(N.lib().qcb_policy_observe(self._pol.data_ptr(), 1, layer, t, self._thc,
                                           N.ptr(self._hlc), N.stream_ptr()), "observe")
        if act == "recompute":
            p = self._read()
            if p.d_valid[layer]:
                decision.divergences[layer] = float(p.d_now[layer])
            if t > 0:
                self.cache[layer] = o
        self.prev_features[layer] = o

    def finalize_step(self, t: int, x_t, decision: ScheduleDecision):
        self.latent_history.append(self._flat(x_t).clone())
        if len(self.latent_history) > self.cfg.history_k:
            self.latent_history.pop(0)
        for l in range(self.num_layers):
            a = decision.actions[l]
            wb = self.weight_bits.get(l, FP_BITS) if self.toggles.aigq_weights else FP_BITS
            macs = billed_macs(self.block_cost, wb, decision.abits) if a == "recompute" else 0
            self.trace.append(TraceRecord(t, l, a, decision.divergences[l],
                                          decision.similarities[l], decision.abits, wb, macs,
                                          decision.v))
        self.trace.append(TraceRecord(t, "head", "recompute", None, None, FP_BITS, FP_BITS,
                                      self.head_macs * FP_BITS * FP_BITS))

    # -- accounting (schedule.py:375-382) ------------------------------------
    def executed_macs(self) -> int:
        return sum(r.macs for r in self.trace)

    def baseline_macs(self) -> int:
        per_block = billed_macs(self.block_cost, FP_BITS, FP_BITS)
        return self.total_steps * (self.num_layers * per_block +
                                   self.head_macs * FP_BITS * FP_BITS)
