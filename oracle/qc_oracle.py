"""CPU oracle for the QuantCache hot path -- TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference `ditrt` package's
forward-and-sample path (`/root/reference/pkg/src/ditrt`).  It exists so the
B200 kernels can be checked against the reference algorithm on identical
inputs.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import it; the product package
(`paper_2503_06545_b200`) never does, and fails loudly when its CUDA library
is missing.

Parity is PINNED: `tests/golden/make_golden.py` imports the reference itself
in the build container and records its outputs as fixtures under
`tests/golden/`; `tests/test_oracle_golden.py` checks this restatement
against every fixture bit-for-bit (and the reference's own known-answer
values from `pkg/tests`).

Numerics follow the reference exactly:
  * every FP product accumulates in float64 in ascending-k order and is
    rounded once to float32 (tensor.py:43-60);
  * quantization scales are rounded UP to 16-bit significands and rounding
    is half-away-from-zero (quant.py:24-35, 83-123);
  * the integer GEMM is the exact integer contraction scaled per output
    channel (tensor.py:68-112).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

SIG_BITS = 16                # quant.py:21  SCALE_SIGNIFICAND_BITS
FP_BITS = 32                 # schedule.py:19
FFN_RATIO = 4                # model.py:32
SITES = ("sta_q", "sta_k", "sta_v", "sta_o", "ca_q", "ca_k", "ca_v", "ca_o",
         "ffn1", "ffn2")     # model.py:26-30


# ---------------------------------------------------------------------------
# L0: deterministic dense products (tensor.py)

def _lsb_exp(x64: np.ndarray) -> np.ndarray:
    """Exponent of the lowest set bit of each (f32-representable) value; a
    large sentinel for zeros."""
    m, e = np.frexp(x64)
    mi = np.abs(m * 2.0 ** 24).astype(np.int64)
    low = mi & -mi
    tz = np.where(low > 0, np.log2(np.maximum(low, 1)).astype(np.int64), 0)
    return np.where(x64 != 0, e.astype(np.int64) - 24 + tz, 1 << 20)


def seq_mm(a, b) -> np.ndarray:
    """f32(sum_k f64(a[:,k]) * f64(b[k,:])) accumulated in ascending k.

    Restates tensor.py:43-60 (`mm`).  Shortcut with the same result: for an
    output (i, n) whose every partial sum is exact in f64 -- all terms are
    multiples of 2^L with L >= lsb(a[i,:]) + lsb(b[:,n]) and sum_k |term| <
    2^(L + 53) -- the ascending-k sum is the exact sum, which any exact
    summation (f64 BLAS: each intermediate is such a partial sum) returns too.
    The remaining columns take the explicit loop."""
    a64 = np.asarray(a).astype(np.float64)
    b64 = np.asarray(b).astype(np.float64)
    if a64.ndim != 2 or b64.ndim != 2 or a64.shape[1] != b64.shape[0]:
        raise ValueError(f"matmul shapes {a64.shape} x {b64.shape}")
    out = a64 @ b64
    if a64.size and b64.size:
        L = _lsb_exp(a64).min(axis=1)[:, None] + _lsb_exp(b64).min(axis=0)[None, :]
        bound = (np.abs(a64) @ np.abs(b64)) * (1.0 + 2.0 ** -30)
        ok = (bound < np.ldexp(1.0, np.minimum(L + 53, 1000))) | (bound == 0)
    else:
        ok = np.ones(out.shape, dtype=bool)
    cols = np.nonzero(~ok.all(axis=0))[0]
    if cols.size:
        bc = b64[:, cols]
        acc = np.zeros((a64.shape[0], cols.size), dtype=np.float64)
        for k in range(a64.shape[1]):
            acc += a64[:, k:k + 1] * bc[k:k + 1, :]
        out[:, cols] = acc
    return out.astype(np.float32)


def int_acc(codes_a, za, codes_w, zw) -> np.ndarray:
    """Exact integer accumulator sum_k (a - za)(w - zw[n]) as int64.

    The quantity the device's u8 x u8 -> s32 MMA plus zero-point correction
    must reproduce bit-for-bit (tensor.py:100-101)."""
    a = np.asarray(codes_a, dtype=np.int64) - int(za)
    w = np.asarray(codes_w, dtype=np.int64) - np.asarray(zw, dtype=np.int64)
    return a @ w


def matmul_int_seq(codes_a, sa, za, codes_w, sw, zw) -> np.ndarray:
    """Reference integer GEMM: joint scale applied per k, f64 ascending-k sum.

    Restates tensor.py:100-112.  Shortcut with the same result: when every
    partial sum joint[n] * sum_{k<K'} (a-za)(w-zw) is exact in f64 (the
    integer sum of |terms| below 2^(53 - significand bits of joint[n])), the
    ascending-k f64 sum equals the exact value, which is also the one
    rounding of joint * (exact integer accumulator) -- computed directly."""
    a = np.asarray(codes_a, dtype=np.int64) - int(za)
    w = np.asarray(codes_w, dtype=np.int64) - np.asarray(zw, dtype=np.int64)
    joint = float(sa) * np.atleast_1d(np.asarray(sw, dtype=np.float64))
    m, _ = np.frexp(joint)
    sig = np.array([53 - (int(np.round(v * 2.0 ** 53)) & -int(np.round(v * 2.0 ** 53))).bit_length()
                    + 1 if v != 0 else 0 for v in np.abs(m)], dtype=np.int64)
    # integer products below 2^16 and K < 2^20: f64 BLAS sums are exact here
    bound = np.abs(a).astype(np.float64) @ np.abs(w).astype(np.float64)   # >= |partial sums|
    if a.shape[1] < (1 << 20) and (bound.max(axis=0, initial=0) <
                                   np.left_shift(1, 53 - sig).astype(np.float64)).all():
        acc = a.astype(np.float64) @ w.astype(np.float64)
        return (np.broadcast_to(joint[None, :], acc.shape) * acc).astype(np.float32)
    acc = np.zeros((a.shape[0], w.shape[1]), dtype=np.float64)
    for k in range(a.shape[1]):
        acc += joint[None, :] * (a[:, k:k + 1] * w[k:k + 1, :])
    return acc.astype(np.float32)


def matmul_int_single_rounding(codes_a, sa, za, codes_w, sw, zw) -> np.ndarray:
    """f32(f64(sa*sw[n]) * f64(acc)): the device epilogue's formulation.

    Equal to `matmul_int_seq` whenever the f64 partial sums are exact
    (|acc| < 2^21 for 32-bit joint significands) -- checked in the tests."""
    acc = int_acc(codes_a, za, codes_w, zw).astype(np.float64)
    joint = float(sa) * np.atleast_1d(np.asarray(sw, dtype=np.float64))
    return (joint[None, :] * acc).astype(np.float32)


def overflow_guard(k: int, abits: int, wbits: int, acc_bits: int) -> bool:
    """True when K*(2^ba-1)(2^bw-1) fits the signed accumulator (tensor.py:91-98)."""
    return k * (2 ** abits - 1) * (2 ** wbits - 1) <= 2 ** acc_bits - 1


# ---------------------------------------------------------------------------
# L1: AIGQ quantizer (quant.py)

def rha(x) -> np.ndarray:
    """Round half away from zero in f64 (quant.py:24-27)."""
    x = np.asarray(x, dtype=np.float64)
    return np.sign(x) * np.floor(np.abs(x) + 0.5)


def scale_up16(s) -> np.ndarray:
    """Round positive scales UP to a 16-bit significand (quant.py:30-35)."""
    m, e = np.frexp(np.asarray(s, dtype=np.float64))
    return np.ldexp(np.ceil(m * 65536.0) / 65536.0, e)


def _params_from_range(lo, hi, bits):
    top = 2 ** bits - 1
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    span = hi - lo
    flat = span <= 0
    s = np.where(flat, 1.0, scale_up16(np.where(flat, 1.0, span) / top))
    z = np.clip(rha(-lo / s), 0, top).astype(np.int64)
    z = np.where(flat, 0, z)
    return s, z


def act_params(x, bits: int) -> Tuple[float, int]:
    """Per-tensor dynamic min/max params (quant.py:83-110, granularity per-tensor)."""
    d = np.asarray(x, dtype=np.float64)
    if d.size == 0:
        raise ValueError("cannot calibrate an empty tensor")
    s, z = _params_from_range(d.min(), d.max(), bits)
    return float(s), int(z)


def chan_params(w, bits: int) -> Tuple[np.ndarray, np.ndarray]:
    """Per-output-channel params of a (K, N) weight, axis=1 (quant.py:83-110)."""
    d = np.asarray(w, dtype=np.float64)
    return _params_from_range(d.min(axis=0), d.max(axis=0), bits)


def codes_of(x, s, z, bits: int) -> np.ndarray:
    """clip(rha(f64 x / s) + z, 0, 2^b-1) (quant.py:113-123). s, z broadcast."""
    d = np.asarray(x, dtype=np.float64)
    top = 2 ** bits - 1
    return np.clip(rha(d / s) + z, 0, top).astype(np.int64)


def dequant(codes, s, z) -> np.ndarray:
    """f32(s * (code - z)) (quant.py:126-134)."""
    return (np.asarray(s, dtype=np.float64) *
            (np.asarray(codes, dtype=np.int64) - np.asarray(z, dtype=np.int64)
             ).astype(np.float64)).astype(np.float32)


def pow2_floor(n: int) -> int:
    """Largest power of two <= n (quant.py:172-176)."""
    return 1 << (int(n).bit_length() - 1)


def sign_vector(seed: int, b: int) -> np.ndarray:
    """+-1 signs of the randomized Hadamard block (quant.py:155-158)."""
    u = np.random.default_rng(seed).random(b)
    return np.where(u < 0.5, -1.0, 1.0)


def balance_scales(w, act_absmax) -> np.ndarray:
    """c_j = clip(sqrt(absmax_x/absmax_w), 1e-3, 1e3); 1 for dead channels
    (quant.py:179-200)."""
    wv = np.asarray(w, dtype=np.float64)
    st = np.asarray(act_absmax, dtype=np.float64)
    if wv.ndim != 2 or st.shape != (wv.shape[0],):
        raise ValueError("balance stats shape does not match weight rows")
    wa = np.abs(wv).max(axis=1)
    live = (st > 0) & (wa > 0)
    c = np.ones_like(st)
    c[live] = np.clip(np.sqrt(st[live] / wa[live]), 1e-3, 1e3)
    return c


def sylvester(b: int) -> np.ndarray:
    """Sylvester Hadamard matrix (what scipy.linalg.hadamard returns)."""
    h = np.ones((1, 1), dtype=np.int64)
    while h.shape[0] < b:
        h = np.block([[h, h], [h, -h]])
    return h


def rotation_dense(n: int, seed: int) -> np.ndarray:
    """R = diag(signs) H_b / sqrt(b) (+) I_{n-b} in f64 (quant.py:151-161)."""
    b = pow2_floor(n)
    r = np.eye(n)
    r[:b, :b] = (sign_vector(seed, b)[:, None] * sylvester(b)) / np.sqrt(b)
    return r


def rotate_act(x, c, seed: int) -> np.ndarray:
    """Activation side of the balance transform (quant.py:163-165)."""
    x = np.asarray(x, dtype=np.float32)
    y = (x.astype(np.float64) / np.asarray(c, np.float64)[None, :]).astype(np.float32)
    return seq_mm(y, rotation_dense(x.shape[1], seed).astype(np.float32))


def rotate_weight(w, c, seed: int) -> np.ndarray:
    """Weight side R^T (c (.) W) (quant.py:167-169)."""
    w = np.asarray(w, dtype=np.float32)
    sc = (np.asarray(c, np.float64)[:, None] * w.astype(np.float64)).astype(np.float32)
    return seq_mm(rotation_dense(w.shape[0], seed).T.astype(np.float32), sc)


def fwht_rows(v: np.ndarray) -> np.ndarray:
    """Unnormalized in-place-order Walsh-Hadamard transform along axis 1 (f64)."""
    v = np.array(v, dtype=np.float64, copy=True)
    n = v.shape[1]
    h = 1
    while h < n:
        v = v.reshape(v.shape[0], n // (2 * h), 2, h)
        a = v[:, :, 0, :].copy()
        b = v[:, :, 1, :].copy()
        v[:, :, 0, :] = a + b
        v[:, :, 1, :] = a - b
        v = v.reshape(v.shape[0], n)
        h *= 2
    return v


def rotate_act_fwht(x, c, seed: int) -> np.ndarray:
    """The device formulation of `rotate_act`: f32 scale, sign flip, f64 FWHT
    over the leading power-of-two block, one multiply by f32(1/sqrt(b)).

    Equal to `rotate_act` except when an exact value sits within f64 rounding
    of an f32 rounding boundary (measured: 0 mismatches on the fixtures)."""
    x = np.asarray(x, dtype=np.float32)
    k = x.shape[1]
    b = pow2_floor(k)
    y = (x.astype(np.float64) / np.asarray(c, np.float64)[None, :]).astype(np.float32)
    r = np.float64(np.float32(1.0 / np.sqrt(b)))
    head = fwht_rows(y[:, :b].astype(np.float64) * sign_vector(seed, b)[None, :]) * r
    out = y.copy()
    out[:, :b] = head.astype(np.float32)
    return out


# ---------------------------------------------------------------------------
# L3 policies (schedule.py)

@dataclass
class Thresholds:
    """ThresholdConfig restated (schedule.py:22-60)."""
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


def divergence5(p_now, p_cached, k: int, m_now, m_prev) -> float:
    """D = (sum|p_now-p_cached| / k) * ||m_now-m_prev||_2 (schedule.py:67-82)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    l1 = float(np.abs(np.asarray(p_now, np.float64) - np.asarray(p_cached, np.float64)).sum())
    l2 = float(np.linalg.norm(np.asarray(m_now, np.float64) - np.asarray(m_prev, np.float64)))
    return (l1 / k) * l2


def divergence(out, cached, k: int, prev) -> float:
    """The HLC call site: p_now = m_now = the block output (schedule.py:343)."""
    return divergence5(out, cached, k, out, prev)


def refresh_interval(d: float, th: Thresholds) -> int:
    """schedule.py:85-90"""
    return th.tau_max if d < th.delta1 else (th.tau_mid if d < th.delta2 else th.tau_min)


def redundancy(ds: Sequence[float]) -> float:
    """schedule.py:93-97"""
    return 1.0 / (1.0 + float(np.mean(ds)))


def act_bits_for(r: float, th: Thresholds) -> int:
    """schedule.py:100-105"""
    return th.bit_min if r >= th.theta2 else (th.bit_mid if r >= th.theta1 else th.bit_max)


def similarity(a, b) -> float:
    """Cosine of two flattened feature maps, 0 when a norm is 0 (schedule.py:108-116)."""
    x = np.asarray(a, np.float64).ravel()
    y = np.asarray(b, np.float64).ravel()
    nx, ny = np.linalg.norm(x), np.linalg.norm(y)
    if nx == 0.0 or ny == 0.0:
        return 0.0
    return float(x @ y / (nx * ny))


def prune_p(s: float, th: Thresholds, base: float) -> float:
    """schedule.py:119-125"""
    return 1.0 if s > th.tau_high else (base if s >= th.tau_low else 0.0)


def variation(history: Sequence[np.ndarray], cur) -> float:
    """V = sum_h sum|cur - h| (schedule.py:128-133)."""
    c = np.asarray(cur, np.float64)
    tot = 0.0
    for h in history:
        tot += float(np.abs(c - np.asarray(h, np.float64)).sum())
    return tot


def p_eff(v: float, th: Thresholds) -> float:
    """schedule.py:136-141"""
    if v < th.v_low:
        return min(1.0, th.p_base * th.prune_adjust)
    if v > th.v_high:
        return th.p_base / th.prune_adjust
    return th.p_base


def draw(seed: int, t: int, layer: int) -> float:
    """Counter-keyed uniform draw (schedule.py:144-146)."""
    return float(np.random.default_rng(np.random.SeedSequence((seed, t, layer))).random())


def draw_table(seed: int, steps: int, layers: int) -> np.ndarray:
    """(steps, layers) f64 table of `draw`, the device plan kernel's input."""
    out = np.zeros((steps, layers), dtype=np.float64)
    for t in range(steps):
        for l in range(layers):
            out[t, l] = draw(seed, t, l)
    return out


def billed(quantizable: int, fp_always: int, wbits: int, abits: int) -> int:
    """schedule.py:232-234"""
    return quantizable * wbits * abits + fp_always * FP_BITS * FP_BITS


# ---------------------------------------------------------------------------
# Scheduler state machine (schedule.py:240-382), restated as one object


@dataclass
class Decision:
    t: int
    actions: List[str]
    abits: int
    d: List[Optional[float]]
    s: List[Optional[float]]
    v: float
    forced: bool = False


class PolicyState:
    """Mirror of `Scheduler` (schedule.py:240-382): cache entries, last
    divergences, previous-step features, latent history and the trace."""

    def __init__(self, layers, steps, th: Thresholds, hlc=False, aigq_w=False,
                 aigq_a=False, srap=False, quantizable=0, fp_always=0,
                 head_macs=0, prune_seed=0, weight_bits=None):
        self.L, self.T, self.th = layers, steps, th
        self.hlc, self.aigq_w, self.aigq_a, self.srap = hlc, aigq_w, aigq_a, srap
        self.q_macs, self.fp_macs, self.head_macs = quantizable, fp_always, head_macs
        self.seed = prune_seed
        self.wbits = dict(weight_bits or {})
        self.cache: Dict[int, Tuple[np.ndarray, int, int]] = {}   # l -> (tensor, step, tau)
        self.prev: Dict[int, np.ndarray] = {}
        self.last_d: Dict[int, float] = {}
        self.hist: List[np.ndarray] = []
        self.trace: List[dict] = []
        self.seen = 0

    def _live(self, l, t):
        e = self.cache.get(l)
        return e is not None and (e[1] - t) < e[2]

    def plan(self, t: int, x) -> Decision:
        th = self.th
        boundary = self.seen == 0 or t == 0
        acts, long_skip = [], False
        for l in range(self.L):
            if self.hlc and not boundary and self._live(l, t):
                acts.append("reuse")
                continue
            e = self.cache.get(l)
            if self.hlc and e is not None and not self._live(l, t) and e[2] == th.tau_max:
                long_skip = True
            acts.append("recompute")
        v = variation(self.hist, x)
        sims: List[Optional[float]] = [None] * self.L
        if self.srap and not boundary:
            base = p_eff(v, th)
            for l in range(1, self.L):
                if acts[l] != "recompute" or (l - 1) not in self.prev or l not in self.prev:
                    continue
                s = similarity(self.prev[l - 1], self.prev[l])
                sims[l] = s
                p = prune_p(s, th, base)
                if p >= 1.0 or draw(self.seed, t, l) < p:
                    acts[l] = "prune"
        forced = False
        if not self.aigq_a:
            abits = FP_BITS
        elif boundary or not self.last_d:
            abits = th.bit_max
        elif long_skip:
            abits, forced = th.bit_max, True
        else:
            abits = act_bits_for(redundancy(list(self.last_d.values())), th)
        self.seen += 1
        return Decision(t, acts, abits, [None] * self.L, sims, v, forced)

    def observe(self, t: int, l: int, out, dec: Decision):
        prev = self.prev.get(l)
        if dec.actions[l] == "recompute":
            e = self.cache.get(l)
            if e is not None:
                ref, k = e[0], max(1, e[1] - t)
            elif prev is not None:
                ref, k = prev, 1
            else:
                ref, k = None, 1
            if ref is not None and prev is not None:
                d = divergence(out, ref, k, prev)
                self.last_d[l] = d
                tau = refresh_interval(d, self.th)
                dec.d[l] = d
            else:
                tau = 1
            if t > 0:
                self.cache[l] = (out, t, tau)
        self.prev[l] = out

    def finalize(self, t: int, x, dec: Decision):
        self.hist.append(x)
        if len(self.hist) > self.th.history_k:
            self.hist.pop(0)
        for l in range(self.L):
            wb = self.wbits.get(l, FP_BITS) if self.aigq_w else FP_BITS
            macs = billed(self.q_macs, self.fp_macs, wb, dec.abits) \
                if dec.actions[l] == "recompute" else 0
            self.trace.append(dict(t=t, layer=l, action=dec.actions[l], D=dec.d[l],
                                   S=dec.s[l], bits=dec.abits, wbits=wb, macs=macs,
                                   V=dec.v))
        self.trace.append(dict(t=t, layer="head", action="recompute", D=None, S=None,
                               bits=FP_BITS, wbits=FP_BITS,
                               macs=self.head_macs * FP_BITS * FP_BITS, V=None))


# ---------------------------------------------------------------------------
# L2 toy DiT (model.py) and L4 sampler (sampler.py)


@dataclass
class ModelDims:
    num_blocks: int = 8
    model_dim: int = 64
    num_heads: int = 4
    tokens_per_frame: int = 16
    frames: int = 4
    cond_dim: int = 32
    seed: int = 0

    @property
    def seq_len(self):
        return self.tokens_per_frame * self.frames


BLOCK_FIELDS = ("ln1_g", "ln1_b", "sta_q", "sta_k", "sta_v", "sta_o", "ln2_g",
                "ln2_b", "ca_q", "ca_k", "ca_v", "ca_o", "ln3_g", "ln3_b",
                "ffn1", "ffn2", "mod")   # model.py:60-78 declaration order


def init_weights(dims: ModelDims):
    """Seeded init in the reference's draw order (model.py:101-124).

    Returns (blocks: list of dict, head_w, head_b)."""
    rng = np.random.default_rng(dims.seed)
    d, c, h = dims.model_dim, dims.cond_dim, FFN_RATIO * dims.model_dim

    def nrm(shape, fan):
        return rng.normal(0.0, fan ** -0.5, size=shape).astype(np.float32)

    blocks = []
    for _ in range(dims.num_blocks):
        b = {}
        b["ln1_g"], b["ln1_b"] = np.ones(d, np.float32), np.zeros(d, np.float32)
        b["sta_q"] = nrm((d, d), d)
        b["sta_k"] = nrm((d, d), d)
        b["sta_v"] = nrm((d, d), d)
        b["sta_o"] = nrm((d, d), d)
        b["ln2_g"], b["ln2_b"] = np.ones(d, np.float32), np.zeros(d, np.float32)
        b["ca_q"] = nrm((d, d), d)
        b["ca_k"] = nrm((c, d), c)
        b["ca_v"] = nrm((c, d), c)
        b["ca_o"] = nrm((d, d), d)
        b["ln3_g"], b["ln3_b"] = np.ones(d, np.float32), np.zeros(d, np.float32)
        b["ffn1"] = nrm((d, h), d)
        b["ffn2"] = nrm((h, d), h)
        b["mod"] = nrm((d, 6), d)
        blocks.append(b)
    head_w = nrm((d, d), d)
    head_b = nrm((d,), d)
    return blocks, head_w, head_b


def t_embed(t: int, dim: int) -> np.ndarray:
    """Sinusoidal timestep embedding (model.py:127-134)."""
    half = dim // 2
    fr = np.exp(-np.log(10000.0) * np.arange(half, dtype=np.float64) / half)
    e = np.concatenate([np.sin(t * fr), np.cos(t * fr)])
    if e.size < dim:
        e = np.concatenate([e, np.zeros(dim - e.size)])
    return e.astype(np.float32)


def modulation(t: int, mod_w) -> np.ndarray:
    """The 6 block scalars m = t_emb @ mod (model.py:178-180), f32."""
    return seq_mm(t_embed(t, mod_w.shape[0]).reshape(1, -1), mod_w)[0]


def ln64(x, g, b) -> np.ndarray:
    """f64 layer norm, eps 1e-5, cast to f32 (model.py:137-142)."""
    x64 = np.asarray(x).astype(np.float64)
    mu = x64.mean(axis=-1, keepdims=True)
    var = ((x64 - mu) ** 2).mean(axis=-1, keepdims=True)
    y = (x64 - mu) / np.sqrt(var + 1e-5) * np.asarray(g).astype(np.float64) \
        + np.asarray(b).astype(np.float64)
    return y.astype(np.float32)


def gelu64(x) -> np.ndarray:
    """Exact-erf GELU in f64, cast to f32 (model.py:145-147)."""
    from scipy.special import erf
    x64 = np.asarray(x).astype(np.float64)
    return (0.5 * x64 * (1.0 + erf(x64 / np.sqrt(2.0)))).astype(np.float32)


def attention_heads(q, k, v, heads: int) -> np.ndarray:
    """Per-head softmax(q k^T / sqrt(dh)) v with f64 softmax (model.py:150-156,
    tensor.py:115-132)."""
    dh = q.shape[1] // heads
    outs = []
    for h in range(heads):
        sl = slice(h * dh, (h + 1) * dh)
        sc = seq_mm(q[:, sl], k[:, sl].T).astype(np.float64) / np.sqrt(float(dh))
        sc = np.exp(sc - sc.max(axis=-1, keepdims=True))
        p = sc / sc.sum(axis=-1, keepdims=True)
        outs.append(seq_mm(p, v[:, sl]))
    return np.concatenate(outs, axis=1)


def block(x, cond, t: int, w: dict, layer: int, heads: int, gemm=None) -> np.ndarray:
    """One pre-norm block (model.py:159-199). `gemm(layer, site, a, w)`."""
    g = gemm or (lambda _l, _s, a, wt: seq_mm(a, wt))
    cv = np.asarray(cond, np.float32).reshape(1, -1)
    m = modulation(t, w["mod"])
    sh1, sc1, g1, sh3, sc3, g3 = (np.float32(m[i]) for i in range(6))
    h1 = ln64(x, w["ln1_g"], w["ln1_b"]) * (np.float32(1.0) + sc1) + sh1
    q = g(layer, "sta_q", h1, w["sta_q"])
    k = g(layer, "sta_k", h1, w["sta_k"])
    v = g(layer, "sta_v", h1, w["sta_v"])
    x = x + g1 * g(layer, "sta_o", attention_heads(q, k, v, heads), w["sta_o"])
    h2 = ln64(x, w["ln2_g"], w["ln2_b"])
    q2 = g(layer, "ca_q", h2, w["ca_q"])
    k2 = g(layer, "ca_k", cv, w["ca_k"])
    v2 = g(layer, "ca_v", cv, w["ca_v"])
    x = x + g(layer, "ca_o", attention_heads(q2, k2, v2, heads), w["ca_o"])
    h3 = ln64(x, w["ln3_g"], w["ln3_b"]) * (np.float32(1.0) + sc3) + sh3
    hid = gelu64(g(layer, "ffn1", h3, w["ffn1"]))
    return x + g3 * g(layer, "ffn2", hid, w["ffn2"])


def alpha_bar(steps: int, b0: float = 1e-4, b1: float = 2e-2) -> np.ndarray:
    """Linear-beta cumulative products (sampler.py:40-45)."""
    return np.cumprod(1.0 - np.linspace(b0, b1, steps, dtype=np.float64))


def ddpm_step(x, t: int, eps, ab: np.ndarray, noise) -> np.ndarray:
    """Fixed-variance posterior step, noise only for t > 1 (sampler.py:59-80)."""
    a_t, a_p = ab[t], ab[t - 1]
    alpha = a_t / a_p
    beta = 1.0 - alpha
    mean = (np.asarray(x).astype(np.float64)
            - beta / np.sqrt(1.0 - a_t) * np.asarray(eps).astype(np.float64)) / np.sqrt(alpha)
    if t > 1:
        mean = mean + np.sqrt((1.0 - a_p) / (1.0 - a_t) * beta) * \
            np.asarray(noise).astype(np.float64)
    return mean.astype(np.float32)


def rf_step(x, v, dt: float) -> np.ndarray:
    """Rectified-flow Euler step x - dt * v in f64, one rounding to f32.  An
    EXTENSION (C5): the reference has no flow sampler; it reuses
    the DDPM update's arithmetic with c1 = dt, c2 = 1."""
    return ((np.asarray(x).astype(np.float64) - dt * np.asarray(v).astype(np.float64))
            / 1.0).astype(np.float32)


def ddpm_final(x, eps, ab: np.ndarray) -> np.ndarray:
    """Clean-data estimate at t = 0 (sampler.py:83-88)."""
    a0 = ab[0]
    return ((np.asarray(x).astype(np.float64) - np.sqrt(1.0 - a0) *
             np.asarray(eps).astype(np.float64)) / np.sqrt(a0)).astype(np.float32)


class QuantSites:
    """QuantRuntime restated (runtime.py:31-81): offline per-(layer, site)
    weight prep and the per-step GEMM hook."""

    def __init__(self, blocks, aigq_w: bool, aigq_a: bool, weight_bits: Dict[int, int],
                 act_absmax=None, sign_seed: int = 0):
        self.aigq_w, self.aigq_a = aigq_w, aigq_a
        self.prep = {}
        if not aigq_w:
            return
        for l, w in enumerate(blocks):
            stats = (act_absmax or {}).get(l, {})
            for site in SITES:
                wt = w[site]
                if stats.get(site) is not None:
                    c = balance_scales(wt, stats[site])
                    weff = rotate_weight(wt, c, sign_seed)
                    tr = (c, sign_seed)
                else:
                    weff, tr = wt, None
                s, z = chan_params(weff, weight_bits[l])
                codes = codes_of(weff, s[None, :], z[None, :], weight_bits[l])
                self.prep[(l, site)] = dict(codes=codes, s=s, z=z, bits=weight_bits[l],
                                            deq=dequant(codes, s[None, :], z[None, :]),
                                            tr=tr)

    def hook(self, abits: int):
        if not (self.aigq_w or self.aigq_a):
            return None
        qa = self.aigq_a and abits < FP_BITS

        def gemm(layer, site, x, w):
            if self.aigq_w:
                p = self.prep[(layer, site)]
                xe = rotate_act(x, *p["tr"]) if p["tr"] is not None else x
                if qa:
                    sa, za = act_params(xe, abits)
                    ca = codes_of(xe, sa, za, abits)
                    return matmul_int_seq(ca, sa, za, p["codes"], p["s"], p["z"])
                return seq_mm(xe, p["deq"])
            sa, za = act_params(x, abits)
            return seq_mm(dequant(codes_of(x, sa, za, abits), sa, za), w)

        return gemm


def block_costs(dims: ModelDims) -> Tuple[int, int, int]:
    """(quantizable, fp_always, head) MACs (model.py:237-252)."""
    s, d, c = dims.seq_len, dims.model_dim, dims.cond_dim
    q = 4 * s * d * d + 2 * s * d * d + 2 * c * d + 2 * FFN_RATIO * s * d * d
    return q, 2 * s * s * d + 2 * s * d + 6 * d, s * d * d


def sample(dims: ModelDims, steps: int, th: Optional[Thresholds] = None,
           toggles=(False, False, False, False), seed: int = 0, prune_seed: int = 0,
           weight_bits=None, act_absmax=None, sign_seed: int = 0,
           b0: float = 1e-4, b1: float = 2e-2, weights=None, record=None,
           sampler: str = "ddpm"):
    """`generate` + `run_single` wiring restated (sampler.py:91-162,
    harness.py:416-441). toggles = (hlc, aigq_w, aigq_a, srap).
    sampler="rf": the rectified-flow EXTENSION (C5, no reference sampler):
    the head output is a velocity, one Euler step x - v / steps per timestep,
    no noise draws; every QuantCache policy runs unchanged.

    Returns (final latent f32 (F, T, d), PolicyState)."""
    hlc, aw, aa, srap = toggles
    blocks, head_w, head_b = weights if weights is not None else init_weights(dims)
    ab = alpha_bar(steps, b0, b1)
    q, fp, hm = block_costs(dims)
    st = PolicyState(dims.num_blocks, steps, th or Thresholds(0.0, 0.0), hlc, aw, aa, srap,
                     q, fp, hm, prune_seed, weight_bits if aw else {})
    qs = QuantSites(blocks, aw, aa, weight_bits or {}, act_absmax, sign_seed) \
        if (aw or aa) else None
    rng = np.random.default_rng(seed)
    shape = (dims.frames, dims.tokens_per_frame, dims.model_dim)
    x = rng.standard_normal(shape).astype(np.float32)
    cond = rng.standard_normal(dims.cond_dim).astype(np.float32)
    S, D = dims.seq_len, dims.model_dim
    for t in range(steps - 1, -1, -1):
        dec = st.plan(t, x)
        gemm = qs.hook(dec.abits) if qs is not None else None
        h = x.reshape(S, D)
        outs = []
        for l in range(dims.num_blocks):
            a = dec.actions[l]
            if a == "reuse":
                h = st.cache[l][0]
            elif a == "prune":
                pass
            else:
                h = block(h, cond, t, blocks[l], l, dims.num_heads, gemm)
            st.observe(t, l, h, dec)
            outs.append(h)
        eps = (seq_mm(h, head_w) + head_b).reshape(shape)
        st.finalize(t, x, dec)
        if record is not None:
            record.append((t, x, outs, eps, dec))
        if sampler == "rf":
            x = rf_step(x, eps, 1.0 / steps)
        elif t > 0:
            noise = rng.standard_normal(shape).astype(np.float32)
            x = ddpm_step(x, t, eps, ab, noise)
        else:
            x = ddpm_final(x, eps, ab)
    return x, st


def sample_sync(dims: ModelDims, steps: int, th: Optional[Thresholds] = None,
                toggles=(False, False, False, False), seeds: Sequence[int] = (0,),
                prune_seed: int = 0, weight_bits=None, act_absmax=None, sign_seed: int = 0,
                b0: float = 1e-4, b1: float = 2e-2, weights=None):
    """Synchronised-decision mode (BASELINE north_star: "all-reduce the scalar
    cache and prune decisions so every rank takes the same path").

    The videos of the whole batch (every rank's shard) are sampled in lockstep
    under ONE PolicyState, and the policy statistics are the reference formulas
    applied to the CONCATENATED batch: features are stacked on a leading video
    axis, so `divergence` (schedule.py:67-82), `similarity` (:108-116) and
    `variation` (:128-133) sum over every video.  Blocks, quantizers (per video
    tensor), head and the DDPM update stay per video, each video with its own
    NumPy stream (x0, cond, then one noise draw per t > 0, sampler.py:108-131).
    With a single seed this is exactly `sample`.

    Returns (final latents f32 (B, F, T, d), PolicyState)."""
    hlc, aw, aa, srap = toggles
    blocks, head_w, head_b = weights if weights is not None else init_weights(dims)
    ab = alpha_bar(steps, b0, b1)
    q, fp, hm = block_costs(dims)
    st = PolicyState(dims.num_blocks, steps, th or Thresholds(0.0, 0.0), hlc, aw, aa, srap,
                     q, fp, hm, prune_seed, weight_bits if aw else {})
    qs = QuantSites(blocks, aw, aa, weight_bits or {}, act_absmax, sign_seed) \
        if (aw or aa) else None
    rngs = [np.random.default_rng(s) for s in seeds]
    shape = (dims.frames, dims.tokens_per_frame, dims.model_dim)
    xs, conds = [], []
    for r in rngs:
        xs.append(r.standard_normal(shape).astype(np.float32))
        conds.append(r.standard_normal(dims.cond_dim).astype(np.float32))
    x = np.stack(xs)
    B, S, D = len(rngs), dims.seq_len, dims.model_dim
    for t in range(steps - 1, -1, -1):
        dec = st.plan(t, x)
        gemm = qs.hook(dec.abits) if qs is not None else None
        h = x.reshape(B, S, D)
        for l in range(dims.num_blocks):
            a = dec.actions[l]
            if a == "reuse":
                h = st.cache[l][0]
            elif a != "prune":
                h = np.stack([block(h[v], conds[v], t, blocks[l], l, dims.num_heads, gemm)
                              for v in range(B)])
            st.observe(t, l, h, dec)
        eps = np.stack([seq_mm(h[v], head_w) + head_b for v in range(B)]).reshape(x.shape)
        st.finalize(t, x, dec)
        if t > 0:
            noise = np.stack([r.standard_normal(shape).astype(np.float32) for r in rngs])
            x = ddpm_step(x, t, eps, ab, noise)
        else:
            x = ddpm_final(x, eps, ab)
    return x, st
