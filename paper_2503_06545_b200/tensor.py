"""Deterministic dense kernels (mirror of ditrt.tensor, tensor.py:22-145) on CUDA.

`mm` / `matmul_fp` are qcb_gemm_f64 (ascending-k f64 accumulation, one f32
rounding - bit-identical to the reference); `matmul_int` is the tcgen05 u8
GEMM with the reference's operand checks (tensor.py:82-98)."""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _native as N
from . import device as Dv
from .errors import ConfigurationError, DimensionError

ACCUMULATOR_BITS = 63       # reference headroom (tensor.py:19)
DEVICE_ACCUMULATOR_BITS = 31  # s32 TMEM accumulator


def _cuda(x) -> torch.Tensor:
    if isinstance(x, Tensor):
        return x.data
    if isinstance(x, torch.Tensor):
        return x.float().cuda().contiguous()
    return torch.as_tensor(np.ascontiguousarray(np.asarray(x, np.float32))).cuda()


@dataclass
class Tensor:
    """Dense f32 CUDA payload with an optional frame axis (tensor.py:22-40)."""
    data: torch.Tensor
    frame_axis: Optional[int] = None

    def __post_init__(self):
        d = self.data
        self.data = d.float().cuda().contiguous() if isinstance(d, torch.Tensor) else \
            torch.as_tensor(np.asarray(d, np.float32)).cuda()
        if not bool(torch.isfinite(self.data).all()):
            raise ValueError("tensor contains non-finite values")
        if self.frame_axis is not None and not 0 <= self.frame_axis < self.data.dim():
            raise DimensionError(f"frame_axis {self.frame_axis} out of range for ndim "
                                 f"{self.data.dim()}")

    @property
    def shape(self):
        return tuple(self.data.shape)


def mm(a, b) -> torch.Tensor:
    a, b = _cuda(a), _cuda(b)
    if a.dim() != 2 or b.dim() != 2 or a.shape[1] != b.shape[0]:
        raise DimensionError(f"matmul shapes {tuple(a.shape)} x {tuple(b.shape)}")
    return Dv.gemm_f64(a, b)


def matmul_fp(a: Tensor, b: Tensor) -> Tensor:
    return Tensor(mm(a.data, b.data))


def matmul_int(aq, wq, acc_bits: int = ACCUMULATOR_BITS) -> Tensor:
    """Integer GEMM on quantized operands (tensor.py:68-112)."""
    from .quant import QuantizedTensor
    if not isinstance(aq, QuantizedTensor) or not isinstance(wq, QuantizedTensor):
        raise TypeError("matmul_int expects QuantizedTensor operands")
    if len(aq.shape) != 2 or len(wq.shape) != 2 or aq.shape[1] != wq.shape[0]:
        raise DimensionError(f"matmul shapes {aq.shape} x {wq.shape}")
    if aq.params.granularity != "per-tensor":
        raise ConfigurationError("activation operand must be per-tensor quantized")
    if wq.params.granularity == "per-channel" and wq.params.axis != 1:
        raise ConfigurationError("per-channel weights must be quantized along axis 1")
    K = aq.shape[1]
    mag = K * (2 ** aq.params.bit_width - 1) * (2 ** wq.params.bit_width - 1)
    if mag > 2 ** min(acc_bits, DEVICE_ACCUMULATOR_BITS) - 1:
        raise ConfigurationError(f"integer accumulator overflow risk: K={K} at "
                                 f"b={aq.params.bit_width}x{wq.params.bit_width} exceeds "
                                 f"{min(acc_bits, DEVICE_ACCUMULATOR_BITS)}-bit headroom")
    M, Nn = aq.shape[0], wq.shape[1]
    dev = aq.codes.device
    # activation operand: [M][ldc] codes + row sums, one segment
    a = aq.device if isinstance(aq.device, Dv.ActCodes) else None
    if a is None:
        buf = torch.zeros((M, Dv.round16(K)), dtype=torch.uint8, device=dev)
        buf[:, :K] = aq.codes
        a = Dv.ActCodes(buf, aq.codes.to(torch.int32).sum(1, dtype=torch.int32),
                        torch.tensor([float(aq.params.scale)], dtype=torch.float64, device=dev),
                        torch.tensor([int(aq.params.zero_point)], dtype=torch.int32, device=dev),
                        K)
    w = wq.device if isinstance(wq.device, Dv.PackedWeight) else None
    if w is None:
        buf = torch.zeros((Nn, Dv.round16(K)), dtype=torch.uint8, device=dev)
        buf[:, :K] = wq.codes.t()
        s = np.broadcast_to(np.atleast_1d(wq.params.scale), (Nn,)).astype(np.float64)
        z = np.broadcast_to(np.atleast_1d(wq.params.zero_point), (Nn,)).astype(np.int32)
        w = Dv.PackedWeight(buf, torch.as_tensor(s).to(dev), torch.as_tensor(z).to(dev),
                            wq.codes.to(torch.int32).sum(0, dtype=torch.int32), K, Nn,
                            wq.params.bit_width)
    return Tensor(Dv.gemm_u8(a, w))


def attention(q: Tensor, k: Tensor, v: Tensor) -> Tensor:
    """Single-head softmax attention, f64 softmax (tensor.py:121-132)."""
    qd, kd, vd = _cuda(q), _cuda(k), _cuda(v)
    if qd.dim() != 2 or kd.dim() != 2 or vd.dim() != 2:
        raise DimensionError("attention expects 2-D q, k, v")
    if qd.shape[1] != kd.shape[1] or kd.shape[0] != vd.shape[0]:
        raise DimensionError(f"attention shapes q={tuple(qd.shape)} k={tuple(kd.shape)} "
                             f"v={tuple(vd.shape)}")
    if vd.shape[1] != qd.shape[1]:
        raise DimensionError("value width must equal the head width on the device kernel")
    return Tensor(Dv.attention_f64(qd, kd, vd, 1))


def layernorm(x: Tensor, gamma: Tensor, beta: Tensor) -> Tensor:
    """Per-row f64 layer norm, then affine (tensor.py:135-145)."""
    xd = _cuda(x)
    g, b = _cuda(gamma), _cuda(beta)
    if g.shape != (xd.shape[-1],) or b.shape != (xd.shape[-1],):
        raise DimensionError("layernorm affine shape mismatch")
    shape = xd.shape
    x2 = xd.reshape(-1, shape[-1])
    out = Dv.ln_mod(x2, g, b)
    return Tensor(out.reshape(shape), frame_axis=getattr(x, "frame_axis", None))


# ---------------------------------------------------------------------------
# Policy statistics (schedule.py:67-133) on the device reduction kernels: the
# same f64 sums the engine's HLC / SRAP / V paths use, over one flat segment.

def _shape(x):
    return tuple(x.shape) if hasattr(x, "shape") else np.shape(x)


def _flat(x) -> torch.Tensor:
    return _cuda(x).reshape(1, -1)


def _res(n: int) -> torch.Tensor:
    return torch.zeros(n, dtype=torch.float64, device="cuda")


def divergence_score(p_now, p_cached, k: int, m_now, m_prev) -> float:
    """(sum|p_now - p_cached| / k) * ||m_now - m_prev||_2 (schedule.py:67-82)."""
    if _shape(p_now) != _shape(p_cached) or _shape(m_now) != _shape(m_prev):
        raise DimensionError("divergence operands must share shapes")
    if k < 1:
        raise ValueError("k must be >= 1")
    a, b, m, mp = _flat(p_now), _flat(p_cached), _flat(m_now), _flat(m_prev)
    r1, r2 = _res(1), _res(2)
    Dv.reduce_l1(Dv.feat(a), Dv.feat(b), 1, a.shape[1], 1, r1)
    Dv.reduce_hlc(Dv.feat(m), Dv.feat(m), Dv.feat(mp), 1, m.shape[1], 1, r2)
    return (float(r1[0]) / k) * float(np.sqrt(float(r2[1])))


def layer_similarity(p_l, p_l1) -> float:
    """Cosine of two flattened feature maps, 0 when a norm is 0
    (schedule.py:108-116)."""
    if _shape(p_l) != _shape(p_l1):
        raise DimensionError("similarity operands must share shapes")
    a, b = _flat(p_l), _flat(p_l1)
    r = _res(3)
    Dv.reduce_srap(Dv.feat(a), Dv.feat(b), 1, a.shape[1], 1, r.view(1, 3))
    dot, aa, bb = (float(v) for v in r.cpu())
    na, nb = float(np.sqrt(aa)), float(np.sqrt(bb))
    if na == 0.0 or nb == 0.0:
        return 0.0
    return dot / (na * nb)


def cumulative_variation(history, current) -> float:
    """sum over the history of sum|current - h| (schedule.py:128-133)."""
    hist = list(history)
    if not hist:
        return 0.0
    cur = _flat(current)
    hs = [_flat(h) for h in hist]
    for h in hs:
        if h.shape != cur.shape:
            raise DimensionError("variation operands must share shapes")
    total = 0.0
    for i in range(0, len(hs), 8):   # up to 8 history entries per pass over x
        part = hs[i:i + 8]
        r = _res(len(part))
        if cur.shape[1] % 4 == 0:
            Dv.reduce_l1_hist(Dv.feat(cur), [Dv.feat(h) for h in part], 1, cur.shape[1], 1,
                              r.view(len(part), 1))
        else:
            for j, h in enumerate(part):
                Dv.reduce_l1(Dv.feat(cur), Dv.feat(h), 1, cur.shape[1], 1, r[j:j + 1])
        for v in r.cpu().tolist():
            total += v
    return total
