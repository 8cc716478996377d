"""Typed wrappers of the C ABI on CUDA torch tensors.

PyTorch is used only for device memory and streams; every computation below is
one of our sm_100a kernels in libqcb200.so.  Layout conventions:
  * activation codes  u8  [rows][ldc], ldc = K rounded up to 16 (TMA stride)
  * weight codes      u8  [N][ldk]   (K-major, i.e. W^T), ldk = roundup(K, 16)
  * per-tensor activation params are per *segment* (video): f64 scale, i32 zero
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _native as N
from .errors import DimensionError


# Count of libqcb200 kernel launches issued (the bench reports the number issued
# inside its timed region as `gpu_launches`).
LAUNCHES = [0]


def count(n: int = 1):
    LAUNCHES[0] += n


def round16(k: int) -> int:
    return (k + 15) // 16 * 16


def pow2_floor(n: int) -> int:
    return 1 << (int(n).bit_length() - 1)


_DEV = None


def _dev() -> torch.device:
    global _DEV
    if _DEV is None:
        if not torch.cuda.is_available():
            raise RuntimeError("QuantCache B200 kernels need a CUDA device (no CPU fallback)")
        _DEV = torch.device("cuda", torch.cuda.current_device())
    return _DEV


@dataclass
class PackedWeight:
    """Prepared quantized weight of one (layer, site) (runtime.py:40-61)."""
    codes: torch.Tensor      # u8 [N][ldk]
    scale: torch.Tensor      # f64 [N]
    zero: torch.Tensor       # i32 [N]
    colsum: torch.Tensor     # i32 [N]
    K: int
    N: int
    bits: int
    chan_scale: Optional[torch.Tensor] = None   # f64 [K] balance c (None: no transform)
    signs: Optional[torch.Tensor] = None        # f32 [b]
    w_deq: Optional[torch.Tensor] = None        # f32 [K][N] dequantized (weight-only mode)
    w_eff: Optional[torch.Tensor] = None
    chan_recip: Optional[torch.Tensor] = None   # f64 [K] 1/c (quantizer fast path)
    packed: Optional[torch.Tensor] = None       # u8 [N][ldwp] W4 nibbles (bits <= 4)


def pack_w4(codes: torch.Tensor, K: int, stream=None) -> torch.Tensor:
    """Nibble-pack <= 4-bit K-major codes [N][ldk] -> [N][ldwp] (qcb_pack_w4)."""
    Nn = codes.shape[0]
    ldwp = (((K + 1) // 2) + 63) // 64 * 64
    out = torch.zeros((Nn, ldwp), dtype=torch.uint8, device=codes.device)
    N.check(N.lib().qcb_pack_w4(N.ptr(codes), codes.stride(0), Nn, K, N.ptr(out), ldwp,
                                N.stream_ptr(stream)), "pack_w4")
    count(1)
    return out


def weight_prep(w: torch.Tensor, bits: int, chan_scale: Optional[torch.Tensor] = None,
                signs: Optional[torch.Tensor] = None, keep_deq: bool = False,
                keep_eff: bool = False, stream=None, pack4: bool = False) -> PackedWeight:
    """Per-channel weight codes (runtime.py:40-61).  pack4 (bits <= 4) also
    stores the codes nibble-packed; the u8 GEMM then streams half the weight
    bytes and unpacks them in shared memory (slower than the u8 operand when
    the weights are L2-resident, as at STDiT sizes: a memory-footprint option)."""
    dev = _dev()
    w = w.to(dev, torch.float32).contiguous()
    K, Nn = w.shape
    ldk = round16(K)
    codes = torch.zeros((Nn, ldk), dtype=torch.uint8, device=dev)
    scale = torch.empty(Nn, dtype=torch.float64, device=dev)
    zero = torch.empty(Nn, dtype=torch.int32, device=dev)
    colsum = torch.empty(Nn, dtype=torch.int32, device=dev)
    w_deq = torch.empty((K, Nn), dtype=torch.float32, device=dev) if keep_deq else None
    w_eff = torch.empty((K, Nn), dtype=torch.float32, device=dev) if keep_eff else None
    rc = None
    if chan_scale is not None:
        chan_scale = chan_scale.to(dev, torch.float64).contiguous()
        signs = signs.to(dev, torch.float32).contiguous()
        rc = torch.empty(K, dtype=torch.float64, device=dev)
    d = N.QcbWeightPrep(N.ptr(w), K, Nn, bits, N.ptr(chan_scale), N.ptr(signs), N.ptr(codes),
                        ldk, N.ptr(scale), N.ptr(zero), N.ptr(colsum), N.ptr(w_eff),
                        N.ptr(w_deq), N.ptr(rc))
    N.check(N.lib().qcb_weight_prep(C.byref(d), N.stream_ptr(stream)), "weight_prep")
    count(1)
    if pack4 and bits > 4:
        raise ValueError("nibble packing needs codes of at most 4 bits")
    packed = pack_w4(codes, K, stream) if pack4 else None
    return PackedWeight(codes, scale, zero, colsum, K, Nn, bits, chan_scale, signs, w_deq, w_eff,
                        rc, packed)


@dataclass
class ActCodes:
    codes: Optional[torch.Tensor]   # u8 [rows][ldc]
    rowsum: Optional[torch.Tensor]  # i32 [rows]
    scale: torch.Tensor             # f64 [nseg]
    zero: torch.Tensor              # i32 [nseg]
    K: int
    xe: Optional[torch.Tensor] = None
    deq: Optional[torch.Tensor] = None


class Workspace:
    """Grow-only device scratch for min/max keys and reduction partials."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes: int) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.zeros(max(nbytes, 1 << 16), dtype=torch.uint8, device=_dev())
        return self.buf


_WS = Workspace()
_RWS = Workspace()


def act_quant(x: torch.Tensor, bits: int, transforms: Sequence[Optional[tuple]],
              seg_rows: Optional[int] = None, seg_valid: Optional[int] = None,
              nseg: int = 1, x_row0: Optional[torch.Tensor] = None,
              ln: Optional[tuple] = None, mod: tuple = (1.0, 0.0), want_codes: bool = True,
              want_xe: bool = False, want_deq: bool = False,
              out: Optional[List[ActCodes]] = None, gelu: bool = False,
              stream=None) -> List[ActCodes]:
    """Fused [LN+mod] -> balance/rotate -> per-segment min/max -> codes.

    transforms[o] = (chan_scale f64 [K], signs f32 [b]) or None (no transform).
    ln = (gamma, beta) enables the LN prologue (None = raw rows)."""
    dev = _dev()
    assert x.dtype in (torch.float32, torch.bfloat16) and x.is_cuda
    bf16_in = x.dtype == torch.bfloat16   # rows widened exactly (no prologue)
    if bf16_in and (ln is not None or gelu):
        raise ValueError("bf16 input rows take no prologue")
    K = x.shape[-1]
    ldx = x.stride(0) if x.dim() == 2 else K
    rows_total = x.shape[0] if x.dim() == 2 else x.numel() // K
    if seg_rows is None:
        seg_rows = rows_total // nseg
    seg_valid = seg_valid or seg_rows
    if seg_rows * nseg * K == 0:
        raise ValueError("cannot calibrate an empty tensor")
    n_out = len(transforms)
    rows = seg_rows * nseg
    ldc = round16(K)
    res = out or []
    if not res:
        for _ in range(n_out):
            res.append(ActCodes(
                torch.empty((rows, ldc), dtype=torch.uint8, device=dev) if want_codes else None,
                torch.empty(rows, dtype=torch.int32, device=dev) if want_codes else None,
                torch.empty(nseg, dtype=torch.float64, device=dev),
                torch.empty(nseg, dtype=torch.int32, device=dev), K,
                torch.empty((rows, K), dtype=torch.float32, device=dev) if want_xe else None,
                torch.empty((rows, K), dtype=torch.float32, device=dev) if want_deq else None))
    q = N.QcbActQuant()
    q.x, q.ldx, q.x_row0 = N.ptr(x), ldx, N.ptr(x_row0)
    q.K, q.seg_rows, q.seg_valid, q.nseg = K, seg_rows, seg_valid, nseg
    if ln is not None:
        q.prologue = N.PRO_LN_MOD
        q.ln_g, q.ln_b = N.ptr(ln[0]), N.ptr(ln[1])
    elif gelu:
        q.prologue = N.PRO_GELU   # f32(gelu_f64(x)) applied to the input rows
    elif bf16_in:
        q.prologue = N.PRO_BF16
    else:
        q.prologue = N.PRO_NONE
    q.mod_scale1, q.mod_shift = float(mod[0]), float(mod[1])
    q.n_out, q.bits = n_out, bits
    for o, tr in enumerate(transforms):
        if tr is not None:
            q.chan_scale[o], q.signs[o] = N.ptr(tr[0]), N.ptr(tr[1])
            if len(tr) > 2:
                q.chan_recip[o] = N.ptr(tr[2])
        r = res[o]
        q.codes[o], q.rowsum[o] = N.ptr(r.codes), N.ptr(r.rowsum)
        q.scale[o], q.zero[o] = N.ptr(r.scale), N.ptr(r.zero)
        q.xe_out[o], q.deq_out[o] = N.ptr(r.xe), N.ptr(r.deq)
    if res[0].codes is not None:
        ldc = res[0].codes.stride(0)
        assert all(r.codes is None or r.codes.stride(0) == ldc for r in res)
    ldxe = K
    for r in res:
        for buf in (r.xe, r.deq):
            if buf is not None:
                ldxe = buf.stride(0)
    q.ldc, q.ldxe = ldc, ldxe
    q.workspace = N.ptr(_WS.get(int(N.lib().qcb_act_quant_workspace_bytes(K, seg_rows, nseg,
                                                                         n_out))))
    N.check(N.lib().qcb_act_quant(C.byref(q), N.stream_ptr(stream)), "act_quant")
    count(3)
    return res


def gemm_u8(a: ActCodes, w: PackedWeight, M: Optional[int] = None, out=None,
            epilogue: int = N.EPI_STORE, resid=None, gate: float = 1.0,
            seg_rows: Optional[int] = None, seg_valid: Optional[int] = None,
            out_row0=None, resid_row0=None, gate_vec=None, seg_active=None, ldo=None,
            block_n: int = 0, stream=None) -> torch.Tensor:
    """Quantized linear y = epilogue(f32(sa*sw[n] * acc)) on tcgen05."""
    dev = _dev()
    if a.K != w.K:
        raise DimensionError(f"matmul shapes (M,{a.K}) x ({w.K},{w.N})")
    M = M if M is not None else a.codes.shape[0]
    if out is None:
        dt = {N.EPI_ACC: torch.int32, N.EPI_STORE_BF16: torch.bfloat16}.get(epilogue,
                                                                          torch.float32)
        out = torch.empty((M, w.N), dtype=dt, device=dev)
    g = N.QcbGemm()
    g.M, g.N, g.K = M, w.N, w.K
    g.seg_rows, g.seg_valid = seg_rows or 0, seg_valid or 0
    g.a_codes, g.lda = N.ptr(a.codes), a.codes.stride(0)
    g.a_scale, g.a_zero, g.a_rowsum = N.ptr(a.scale), N.ptr(a.zero), N.ptr(a.rowsum)
    g.w_codes, g.ldw = N.ptr(w.codes), w.codes.stride(0)
    if w.packed is not None:
        g.w_packed, g.ldwp = N.ptr(w.packed), w.packed.stride(0)
    g.w_scale, g.w_zero, g.w_colsum = N.ptr(w.scale), N.ptr(w.zero), N.ptr(w.colsum)
    g.out, g.ldo = N.ptr(out), ldo if ldo is not None else out.stride(0)
    g.out_row0, g.resid, g.resid_row0 = N.ptr(out_row0), N.ptr(resid), N.ptr(resid_row0)
    g.ldr = resid.stride(0) if resid is not None else 0
    g.gate, g.gate_scalar = N.ptr(gate_vec), float(gate)
    g.epilogue, g.block_n, g.seg_active = epilogue, block_n, N.ptr(seg_active)
    g.out_rows = out.shape[0]
    g.resid_rows = resid.shape[0] if resid is not None else 0
    N.check(N.lib().qcb_gemm_u8(C.byref(g), N.stream_ptr(stream)), "gemm_u8")
    count(1)
    return out


def gemm_f64(a: torch.Tensor, w: torch.Tensor, out=None, epilogue: int = N.EPI_STORE,
             resid=None, gate: float = 1.0, bias=None, seg_rows=None, seg_valid=None,
             a_row0=None, out_row0=None, resid_row0=None, M=None, stream=None):
    """Reference `mm` on device: ascending-k f64 accumulation, f32 out."""
    dev = _dev()
    K = a.shape[-1]
    if w.shape[0] != K:
        raise DimensionError(f"matmul shapes {tuple(a.shape)} x {tuple(w.shape)}")
    M = M if M is not None else a.shape[0]
    Nn = w.shape[1]
    if out is None:
        out = torch.empty((M, Nn), dtype=torch.float32, device=dev)
    g = N.QcbGemmF64()
    g.M, g.N, g.K = M, Nn, K
    g.seg_rows, g.seg_valid = seg_rows or 0, seg_valid or 0
    g.a, g.lda, g.a_row0 = N.ptr(a), a.stride(0), N.ptr(a_row0)
    g.w, g.ldw = N.ptr(w), w.stride(0)
    g.out, g.ldo, g.out_row0 = N.ptr(out), out.stride(0), N.ptr(out_row0)
    g.resid, g.ldr = N.ptr(resid), resid.stride(0) if resid is not None else 0
    g.resid_row0, g.bias = N.ptr(resid_row0), N.ptr(bias)
    g.gate_scalar, g.epilogue = float(gate), epilogue
    N.check(N.lib().qcb_gemm_f64(C.byref(g), N.stream_ptr(stream)), "gemm_f64")
    count(1)
    return out


class HeadWeights:
    """W [K][N] f32 prepared once for head_gemm (digit planes, column stats, W^T)."""

    def __init__(self, w: torch.Tensor, stream=None):
        assert w.dtype == torch.float32 and w.is_cuda and w.dim() == 2
        self.K, self.N = int(w.shape[0]), int(w.shape[1])
        w = w.contiguous()
        nbytes = int(N.lib().qcb_head_prep_bytes(self.K, self.N))
        self.buf = torch.empty(nbytes, dtype=torch.uint8, device=w.device)
        N.check(N.lib().qcb_head_prep(N.ptr(w), self.K, self.N, N.ptr(self.buf),
                                      N.stream_ptr(stream)), "head_prep")
        count(1)


_HWS = Workspace()


def head_gemm(a: torch.Tensor, hw: HeadWeights, out=None, bias=None, seg_rows=None,
              seg_valid=None, nseg: int = 1, a_row0=None, out_row0=None, stream=None,
              fallback_count: Optional[torch.Tensor] = None):
    """f32(mm(a, W)) + bias bit-exactly via certified int8 tensor-core digit GEMMs
    (exact f64 FMA chains for uncertified elements)."""
    dev = _dev()
    K = a.shape[-1]
    if K != hw.K:
        raise DimensionError(f"matmul shapes {tuple(a.shape)} x ({hw.K}, {hw.N})")
    seg_rows = seg_rows or (a.shape[0] // nseg)
    seg_valid = seg_valid or seg_rows
    rows = nseg * seg_rows
    if out is None:
        out = torch.empty((rows, hw.N), dtype=torch.float32, device=dev)
    elif out_row0 is None and (out.shape[0] < rows or out.shape[-1] < hw.N):
        raise DimensionError(f"head output {tuple(out.shape)} smaller than ({rows}, {hw.N})")
    ws = _HWS.get(int(N.lib().qcb_head_workspace_bytes(rows, K, hw.N)))
    g = N.QcbHeadGemm()
    g.nseg, g.seg_rows, g.seg_valid, g.K, g.N = nseg, seg_rows, seg_valid, K, hw.N
    g.x, g.ldx, g.x_row0 = N.ptr(a), a.stride(0), N.ptr(a_row0)
    g.prep, g.bias = N.ptr(hw.buf), N.ptr(bias)
    g.out, g.ldo, g.out_row0 = N.ptr(out), out.stride(0), N.ptr(out_row0)
    g.workspace, g.fallback_count = N.ptr(ws), N.ptr(fallback_count)
    N.check(N.lib().qcb_head_gemm(C.byref(g), N.stream_ptr(stream)), "head_gemm")
    count(10)
    return out


def ln_mod(x: torch.Tensor, gamma=None, beta=None, scale1: float = 1.0, shift: float = 0.0,
           out=None, seg_rows=None, seg_valid=None, nseg: int = 1, x_row0=None,
           out_row0=None, stream=None):
    dev = _dev()
    K = x.shape[-1]
    rows = seg_rows * nseg if seg_rows else x.shape[0]
    if out is None:
        out = torch.empty((rows, K), dtype=torch.float32, device=dev)
    q = N.QcbLnMod(N.ptr(x), x.stride(0), N.ptr(x_row0), N.ptr(out), out.stride(0),
                   N.ptr(out_row0), K, seg_rows or rows // nseg, seg_valid or 0, nseg,
                   N.ptr(gamma), N.ptr(beta), float(scale1), float(shift))
    N.check(N.lib().qcb_ln_mod(C.byref(q), N.stream_ptr(stream)), "ln_mod")
    count(1)
    return out


def attention_f64(q, k, v, heads: int, out=None, nseg: int = 1, S=None, Skv=None,
                  seg_valid=None, stream=None):
    """Per-head attention with f64 softmax (reference _mha)."""
    dev = _dev()
    d = q.shape[-1]
    S = S or q.shape[0] // nseg
    Skv = Skv or k.shape[0] // nseg
    if out is None:
        out = torch.empty((S * nseg, d), dtype=torch.float32, device=dev)
    a = N.QcbAttention(N.ptr(q), q.stride(0), N.ptr(k), k.stride(0), N.ptr(v), v.stride(0),
                       N.ptr(out), out.stride(0), S, Skv, heads, d // heads, nseg, S, Skv, S,
                       seg_valid or 0)
    N.check(N.lib().qcb_attention_f64(C.byref(a), N.stream_ptr(stream)), "attention")
    count(1)
    return out


def attention_bf16(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, heads: int, S: int,
                   nseg: int = 1, seg_stride: Optional[int] = None, out=None,
                   scale: float = 0.0, stream=None) -> torch.Tensor:
    """Fast attention (bf16 operands, f32 softmax / accumulation) on the
    tcgen05 tensor cores: per segment s and head h, rows [s*seg_stride,
    s*seg_stride + S) of q / k / v (bf16 [rows][heads*dh]) -> out (bf16, same
    layout).  The bench-mode replacement of library SDPA for model.py:150-156."""
    seg_stride = seg_stride or S
    d = q.shape[1]
    if out is None:
        out = torch.empty((nseg * seg_stride, d), dtype=torch.bfloat16, device=q.device)
    for t in (q, k, v, out):
        if t.dtype != torch.bfloat16 or t.stride(1) != 1:
            raise TypeError("attention_bf16 takes row-major bf16 tensors")
        if t.shape[0] < nseg * seg_stride:
            raise DimensionError("attention_bf16: fewer rows than nseg * seg_stride")
    a = N.QcbAttentionBf16(N.ptr(q), q.stride(0), N.ptr(k), k.stride(0), N.ptr(v), v.stride(0),
                           N.ptr(out), out.stride(0), S, heads, d // heads, nseg, seg_stride,
                           float(scale))
    N.check(N.lib().qcb_attention_bf16(C.byref(a), N.stream_ptr(stream)), "attention_bf16")
    count(1)
    return out


def ddpm(x, eps, c1: float, c2: float, noise=None, c3: float = 0.0, out=None, stream=None,
         noise_gen=None):
    """reverse_step / final_step (sampler.py:59-88).  noise: a tensor, or
    noise_gen = (seed, offset) for in-kernel Philox N(0,1) noise."""
    if out is None:
        out = torch.empty_like(x)
    seed, off = noise_gen if noise_gen is not None else (0, 0)
    d = N.QcbDdpm(N.ptr(x), N.ptr(eps), N.ptr(noise), N.ptr(out), x.numel(), c1, c2, c3,
                  1.0 / float(c2), int(seed), int(off), 1 if noise_gen is not None else 0)
    N.check(N.lib().qcb_ddpm_step(C.byref(d), N.stream_ptr(stream)), "ddpm_step")
    count(1)
    return out


def cfg_combine(eps_c: torch.Tensor, eps_u: torch.Tensor, scale: float, out=None,
                stream=None) -> torch.Tensor:
    """Classifier-free guidance eps_u + scale * (eps_c - eps_u) (extension)."""
    if out is None:
        out = torch.empty_like(eps_c)
    n = eps_c.numel()
    if eps_u.numel() != n or out.numel() != n:
        raise DimensionError("cfg_combine operands must share a size")
    N.check(N.lib().qcb_cfg_combine(N.ptr(eps_c), N.ptr(eps_u), float(scale), N.ptr(out), n,
                                    N.stream_ptr(stream)), "cfg_combine")
    count(1)
    return out


def gelu_inplace(x: torch.Tensor, rows: Optional[int] = None, cols: Optional[int] = None,
                 stream=None) -> torch.Tensor:
    """x[:rows, :cols] = f32(gelu_f64(x)) in place (reference _gelu)."""
    rows = rows if rows is not None else x.shape[0]
    cols = cols if cols is not None else x.shape[1]
    N.check(N.lib().qcb_gelu_inplace(N.ptr(x), x.stride(0), rows, cols, N.stream_ptr(stream)),
            "gelu")
    count(1)
    return x


def feat(t: Optional[torch.Tensor], row0=None, ld=None) -> N.QcbFeat:
    if t is None:
        return N.QcbFeat(0, 0, 0)
    return N.QcbFeat(N.ptr(t), ld if ld is not None else t.stride(0), N.ptr(row0))


def _rws(nseg):
    return N.ptr(_RWS.get(int(N.lib().qcb_reduce_workspace_bytes(nseg))))


def reduce_hlc(out: N.QcbFeat, ref: N.QcbFeat, prev: N.QcbFeat, rows: int, cols: int,
               nseg: int, res: torch.Tensor, seg_active=None, stream=None):
    N.check(N.lib().qcb_reduce_hlc(out, ref, prev, rows, cols, nseg, N.ptr(seg_active),
                                   N.ptr(res), _rws(nseg), N.stream_ptr(stream)), "reduce_hlc")
    count(1)
    return res


def reduce_srap(a: N.QcbFeat, b: N.QcbFeat, rows: int, cols: int, nseg: int,
                res: torch.Tensor, seg_active=None, stream=None,
                workspace: Optional[Workspace] = None, dup_src=None):
    """workspace: a dedicated scratch when this runs concurrently with other
    reductions (side stream); default the shared one.  dup_src (int64 [nseg],
    optional): first segment with the same (a, b) rows -- duplicates are copied,
    not re-reduced."""
    ws = N.ptr((workspace or _RWS).get(int(N.lib().qcb_reduce_workspace_bytes(nseg))))
    N.check(N.lib().qcb_reduce_srap(a, b, rows, cols, nseg, N.ptr(seg_active), N.ptr(dup_src),
                                    N.ptr(res), ws, N.stream_ptr(stream)), "reduce_srap")
    count(1)
    return res


def reduce_l1(x: N.QcbFeat, h: N.QcbFeat, rows: int, cols: int, nseg: int,
              res: torch.Tensor, stream=None):
    N.check(N.lib().qcb_reduce_l1(x, h, rows, cols, nseg, N.ptr(res), _rws(nseg),
                                  N.stream_ptr(stream)), "reduce_l1")
    count(1)
    return res


def reduce_l1_hist(x: N.QcbFeat, hist: Sequence[N.QcbFeat], rows: int, cols: int, nseg: int,
                   res: torch.Tensor, stream=None):
    """res[j][seg] = sum|x - hist[j]| for every history entry, x read once."""
    arr = (N.QcbFeat * len(hist))(*hist)
    N.check(N.lib().qcb_reduce_l1_hist(x, arr, len(hist), rows, cols, nseg, N.ptr(res),
                                       _rws(nseg), N.stream_ptr(stream)), "reduce_l1_hist")
    count(1)
    return res


def col_absmax(x: torch.Tensor, K: int, out: torch.Tensor, nseg: int = 1,
               seg_rows: Optional[int] = None, seg_valid: Optional[int] = None, x_row0=None,
               stream=None) -> torch.Tensor:
    """out[k] = max(out[k], max over the valid rows of |x[:, k]|) (f32, in place)."""
    seg_rows = seg_rows or (x.shape[0] // nseg)
    seg_valid = seg_valid or seg_rows
    N.check(N.lib().qcb_col_absmax(N.ptr(x), x.stride(0), N.ptr(x_row0), seg_rows, seg_valid,
                                   nseg, K, N.ptr(out), N.stream_ptr(stream)), "col_absmax")
    count(1)
    return out


def thresholds_struct(th, toggles) -> N.QcbThresholds:
    return N.QcbThresholds(
        float(th.delta1), float(th.delta2), int(th.tau_max), int(th.tau_mid), int(th.tau_min),
        float(th.theta1), float(th.theta2), int(th.bit_max), int(th.bit_mid), int(th.bit_min),
        float(th.tau_high), float(th.tau_low), float(th.p_base), float(th.v_low),
        float(th.v_high), int(th.history_k), float(th.prune_adjust), int(toggles.hlc),
        int(toggles.aigq_weights), int(toggles.aigq_acts), int(toggles.srap))


def sign_vector(seed: int, b: int) -> np.ndarray:
    """+-1 signs of the randomized Hadamard block (reference quant.py:155-158);
    NumPy's PCG64 is the RNG source so the block matches the reference."""
    u = np.random.default_rng(seed).random(b)
    return np.where(u < 0.5, -1.0, 1.0).astype(np.float32)
