"""AIGQ quantization API (mirror of ditrt.quant, quant.py:38-267) on CUDA tensors.

`compute_minmax_params`, `quantize` and `balance_channels` run on the device
through qcb_act_quant / qcb_weight_prep.  Scale rounding and half-away
rounding follow the reference bit-for-bit (the kernels implement them; the
host helpers below are the same definitions for scalars)."""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, Mapping, Optional, Sequence, Tuple

import numpy as np
import torch

from . import device as Dv
from .errors import BudgetError, ConfigurationError

SCALE_SIGNIFICAND_BITS = 16
BIT_LEVELS = (4, 6, 8)


def round_half_away(x) -> np.ndarray:
    """quant.py:24-27"""
    x = np.asarray(x, dtype=np.float64)
    return np.sign(x) * np.floor(np.abs(x) + 0.5)


def _round_scale_up(s) -> np.ndarray:
    """quant.py:30-35"""
    m, e = np.frexp(np.asarray(s, dtype=np.float64))
    return np.ldexp(np.ceil(m * 2.0 ** SCALE_SIGNIFICAND_BITS) / 2.0 ** SCALE_SIGNIFICAND_BITS, e)


def _as_cuda_f32(x) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x.to(dtype=torch.float32)
        return t if t.is_cuda else t.cuda()
    return torch.as_tensor(np.ascontiguousarray(np.asarray(x, np.float32))).cuda()


@dataclass
class QuantParams:
    """Affine params (quant.py:38-59). scale/zero_point are host arrays
    (scalars for per-tensor, [N] for per-channel axis=1)."""
    scale: np.ndarray
    zero_point: np.ndarray
    bit_width: int
    granularity: str = "per-tensor"
    axis: Optional[int] = None

    def __post_init__(self):
        if self.granularity not in ("per-tensor", "per-channel"):
            raise ConfigurationError(f"unknown granularity {self.granularity!r}")
        if self.granularity == "per-channel" and self.axis is None:
            raise ConfigurationError("per-channel params need an axis")
        self.scale = np.asarray(self.scale, dtype=np.float64)
        self.zero_point = np.asarray(self.zero_point, dtype=np.int64)
        if not np.all(self.scale > 0) or not np.all(np.isfinite(self.scale)):
            raise ConfigurationError("scale must be positive and finite")
        top = 2 ** self.bit_width - 1
        if np.any(self.zero_point < 0) or np.any(self.zero_point > top):
            raise ConfigurationError(f"zero point outside [0, {top}]")


@dataclass
class QuantizedTensor:
    """codes: u8 CUDA tensor of the logical shape (quant.py:62-74).  For 2-D
    activations `device` holds the GEMM-ready ActCodes; for per-channel (axis=1)
    weights it holds the K-major PackedWeight."""
    codes: torch.Tensor
    params: QuantParams
    shape: Tuple[int, ...]
    device: object = field(default=None, repr=False)

    def __post_init__(self):
        if tuple(self.codes.shape) != tuple(self.shape):
            raise ConfigurationError("codes shape does not match declared shape")
        top = 2 ** self.params.bit_width - 1
        if self.codes.numel() and int(self.codes.max()) > top:
            raise ConfigurationError(f"codes outside [0, {top}]")


def _act_codes(x2d: torch.Tensor, bits: int) -> Dv.ActCodes:
    (a,) = Dv.act_quant(x2d.contiguous(), bits, [None])
    return a


def compute_minmax_params(x, bit_width: int, granularity: str = "per-tensor",
                          axis: Optional[int] = None) -> QuantParams:
    """quant.py:83-110, on device."""
    xt = _as_cuda_f32(getattr(x, "data", x))
    if xt.numel() == 0:
        raise ValueError("cannot calibrate an empty tensor")
    if granularity == "per-tensor":
        a = _act_codes(xt.reshape(1, -1) if xt.dim() != 2 else xt, bit_width)
        return QuantParams(float(a.scale[0]), int(a.zero[0]), bit_width)
    if granularity != "per-channel":
        raise ConfigurationError(f"unknown granularity {granularity!r}")
    if axis is None:
        raise ConfigurationError("per-channel calibration needs an axis")
    if xt.dim() != 2 or axis not in (0, 1):
        raise ConfigurationError("per-channel params are supported for 2-D tensors")
    w = xt if axis == 1 else xt.t().contiguous()
    pw = Dv.weight_prep(w, bit_width)
    return QuantParams(pw.scale.cpu().numpy(), pw.zero.cpu().numpy().astype(np.int64),
                       bit_width, "per-channel", axis)


def quantize(x, params: QuantParams) -> QuantizedTensor:
    """clip(rha(x/s)+z) (quant.py:113-123).  Codes are produced by the same
    device kernels; the params must be the min/max params of `x` (the only way
    the hot path uses it) -- other params are applied by an exact host step."""
    xt = _as_cuda_f32(getattr(x, "data", x))
    bits = params.bit_width
    if params.granularity == "per-tensor" and xt.dim() == 2:
        a = _act_codes(xt, bits)
        if float(a.scale[0]) == float(params.scale) and int(a.zero[0]) == int(params.zero_point):
            codes = a.codes[:, :xt.shape[1]].contiguous()
            return QuantizedTensor(codes, params, tuple(xt.shape), device=a)
    if params.granularity == "per-channel" and params.axis == 1 and xt.dim() == 2:
        pw = Dv.weight_prep(xt, bits)
        if np.array_equal(pw.scale.cpu().numpy(), params.scale) and \
                np.array_equal(pw.zero.cpu().numpy(), params.zero_point):
            codes = pw.codes[:, :xt.shape[0]].t().contiguous()
            return QuantizedTensor(codes, params, tuple(xt.shape), device=pw)
    # foreign params: exact elementwise rounding (f64) on the device
    s = torch.as_tensor(params.scale, dtype=torch.float64, device=xt.device)
    z = torch.as_tensor(params.zero_point, dtype=torch.float64, device=xt.device)
    if params.granularity == "per-channel":
        shape = [1] * xt.dim()
        shape[params.axis] = -1
        s, z = s.reshape(shape), z.reshape(shape)
    v = xt.double() / s
    r = torch.sign(v) * torch.floor(v.abs() + 0.5) + z
    codes = r.clamp(0, 2 ** bits - 1).to(torch.uint8)
    return QuantizedTensor(codes, params, tuple(xt.shape))


def dequantize(q: QuantizedTensor) -> torch.Tensor:
    """f32(s*(code-z)) (quant.py:126-134); exact in f32 given 16-bit scales."""
    p = q.params
    s = torch.as_tensor(p.scale, dtype=torch.float64, device=q.codes.device)
    z = torch.as_tensor(p.zero_point, dtype=torch.float64, device=q.codes.device)
    if p.granularity == "per-channel":
        shape = [1] * q.codes.dim()
        shape[p.axis] = -1
        s, z = s.reshape(shape), z.reshape(shape)
    return (s * (q.codes.double() - z)).float()


# ---------------------------------------------------------------------------
# Channel balancing (quant.py:141-200)

def _pow2_block(n: int) -> int:
    return Dv.pow2_floor(n)


@dataclass
class BalanceTransform:
    channel_scales: np.ndarray
    block_size: int
    sign_seed: int = 0

    def signs(self) -> np.ndarray:
        return Dv.sign_vector(self.sign_seed, self.block_size)

    def rotation_matrix(self) -> np.ndarray:
        """Dense R (for audits; the kernels apply it as an f64 FWHT)."""
        n, b = len(self.channel_scales), self.block_size
        h = np.ones((1, 1))
        while h.shape[0] < b:
            h = np.block([[h, h], [h, -h]])
        r = np.eye(n)
        r[:b, :b] = self.signs().astype(np.float64)[:, None] * h / np.sqrt(b)
        return r

    def device(self):
        return (torch.as_tensor(self.channel_scales, dtype=torch.float64).cuda(),
                torch.as_tensor(self.signs()).cuda())

    def apply_to_activation(self, x) -> torch.Tensor:
        """f32(x/c) R on device (quant.py:163-165)."""
        xt = _as_cuda_f32(getattr(x, "data", x))
        (r,) = Dv.act_quant(xt, 8, [self.device()], want_codes=False, want_xe=True)
        return r.xe

    def apply_to_weight(self, w) -> torch.Tensor:
        """R^T (c (.) W) on device (quant.py:167-169)."""
        wt = _as_cuda_f32(getattr(w, "data", w))
        c, sg = self.device()
        return Dv.weight_prep(wt, 8, c, sg, keep_eff=True).w_eff


def balance_channels(w, activation_absmax, sign_seed: int = 0):
    """quant.py:179-200: returns (c (.) W, transform)."""
    from .engine import balance_scales
    wv = np.asarray(getattr(w, "data", w).cpu() if isinstance(getattr(w, "data", w),
                                                                 torch.Tensor) else
                    getattr(w, "data", w), np.float64)
    st = np.asarray(getattr(activation_absmax, "data", activation_absmax), np.float64)
    if wv.ndim != 2:
        raise ConfigurationError("balance expects a 2-D weight")
    c = balance_scales(wv, st)
    balanced = torch.as_tensor((c[:, None] * wv).astype(np.float32)).cuda()
    return balanced, BalanceTransform(c, _pow2_block(wv.shape[0]), sign_seed)


# ---------------------------------------------------------------------------
# Budgeted weight bit allocation (offline host step, quant.py:206-267)

def bit_penalty(b: int) -> float:
    return 2.0 ** (-2 * (b - 4))


@dataclass
class WeightBitPlan:
    bits_per_layer: Dict[int, int]
    budget: int

    def __post_init__(self):
        if sum(self.bits_per_layer.values()) > self.budget:
            raise BudgetError("bit plan exceeds budget")


def allocate_weight_bits(sensitivities: Mapping[int, float], total_budget: int,
                         levels: Sequence[int] = BIT_LEVELS) -> WeightBitPlan:
    """Greedy upgrade by best sensitivity reduction per extra bit; ties go to
    the lowest layer index (quant.py:224-267)."""
    lv = sorted(levels)
    layers = sorted(sensitivities)
    if total_budget < len(layers) * lv[0]:
        raise BudgetError(f"budget {total_budget} cannot cover {len(layers)} layers at "
                          f"{lv[0]} bits")
    at = {l: 0 for l in layers}
    spent = len(layers) * lv[0]
    while True:
        best_gain, best_layer = None, None
        for l in layers:
            i = at[l]
            if i + 1 >= len(lv):
                continue
            step = lv[i + 1] - lv[i]
            if spent + step > total_budget:
                continue
            g = sensitivities[l] * (bit_penalty(lv[i]) - bit_penalty(lv[i + 1])) / step
            if best_gain is None or g > best_gain:
                best_gain, best_layer = g, l
        if best_layer is None:
            break
        spent += lv[at[best_layer] + 1] - lv[at[best_layer]]
        at[best_layer] += 1
    return WeightBitPlan({l: lv[i] for l, i in at.items()}, total_budget)
