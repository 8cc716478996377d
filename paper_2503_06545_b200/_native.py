"""ctypes binding of libqcb200.so (the C ABI in include/qcb200.h).

The library is built in-tree (build_native.py).  There is no fallback: if the
library or a CUDA device is missing, every entry point raises."""

from __future__ import annotations

import ctypes as C
import os

from .errors import ConfigurationError, DimensionError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libqcb200.so")

QCB_OK, QCB_ERR_DIM, QCB_ERR_CONFIG, QCB_ERR_OVERFLOW, QCB_ERR_VALUE, QCB_ERR_TYPE, \
    QCB_ERR_CUDA = range(7)
EPI_STORE, EPI_GELU, EPI_GATE_RESID, EPI_RESID, EPI_ACC, EPI_BIAS, EPI_STORE_BF16 = range(7)
PRO_NONE, PRO_LN_MOD, PRO_GELU, PRO_BF16 = 0, 1, 2, 3
ACT_RECOMPUTE, ACT_REUSE, ACT_PRUNE = 0, 1, 2
MAX_LAYERS = 64

vp = C.c_void_p
i32, i64, f32, f64 = C.c_int, C.c_longlong, C.c_float, C.c_double
u64 = C.c_ulonglong


class QcbGemm(C.Structure):
    _fields_ = [("M", i32), ("N", i32), ("K", i32), ("seg_rows", i32), ("seg_valid", i32),
                ("a_codes", vp), ("lda", i64), ("a_scale", vp), ("a_zero", vp),
                ("a_rowsum", vp), ("w_codes", vp), ("ldw", i64), ("w_scale", vp),
                ("w_zero", vp), ("w_colsum", vp), ("out", vp), ("ldo", i64),
                ("out_row0", vp), ("resid", vp), ("ldr", i64), ("resid_row0", vp),
                ("gate", vp), ("gate_scalar", f32), ("epilogue", i32), ("block_n", i32),
                ("seg_active", vp), ("out_rows", i64), ("resid_rows", i64),
                ("w_packed", vp), ("ldwp", i64)]


class QcbGemmF64(C.Structure):
    _fields_ = [("M", i32), ("N", i32), ("K", i32), ("seg_rows", i32), ("seg_valid", i32),
                ("a", vp), ("lda", i64), ("a_row0", vp), ("w", vp), ("ldw", i64),
                ("out", vp), ("ldo", i64), ("out_row0", vp), ("resid", vp), ("ldr", i64),
                ("resid_row0", vp), ("bias", vp), ("gate_scalar", f32), ("epilogue", i32)]


class QcbHeadGemm(C.Structure):
    _fields_ = [("nseg", i32), ("seg_rows", i32), ("seg_valid", i32), ("K", i32), ("N", i32),
                ("x", vp), ("ldx", i64), ("x_row0", vp), ("prep", vp), ("bias", vp),
                ("out", vp), ("ldo", i64), ("out_row0", vp), ("workspace", vp),
                ("fallback_count", vp)]


class QcbActQuant(C.Structure):
    _fields_ = [("x", vp), ("ldx", i64), ("x_row0", vp), ("K", i32), ("seg_rows", i32),
                ("seg_valid", i32), ("nseg", i32), ("prologue", i32), ("ln_g", vp),
                ("ln_b", vp), ("mod_scale1", f32), ("mod_shift", f32), ("n_out", i32),
                ("bits", i32), ("chan_scale", vp * 3), ("signs", vp * 3), ("codes", vp * 3),
                ("ldc", i64), ("rowsum", vp * 3), ("scale", vp * 3), ("zero", vp * 3),
                ("xe_out", vp * 3), ("ldxe", i64), ("deq_out", vp * 3), ("workspace", vp),
                ("chan_recip", vp * 3)]


class QcbWeightPrep(C.Structure):
    _fields_ = [("w", vp), ("K", i32), ("N", i32), ("bits", i32), ("chan_scale", vp),
                ("signs", vp), ("codes", vp), ("ldk", i64), ("scale", vp), ("zero", vp),
                ("colsum", vp), ("w_eff", vp), ("w_deq", vp), ("chan_recip_out", vp)]


class QcbLnMod(C.Structure):
    _fields_ = [("x", vp), ("ldx", i64), ("x_row0", vp), ("out", vp), ("ldo", i64),
                ("out_row0", vp), ("K", i32), ("seg_rows", i32), ("seg_valid", i32),
                ("nseg", i32), ("ln_g", vp), ("ln_b", vp), ("mod_scale1", f32),
                ("mod_shift", f32)]


class QcbAttention(C.Structure):
    _fields_ = [("q", vp), ("ldq", i64), ("k", vp), ("ldk", i64), ("v", vp), ("ldv", i64),
                ("out", vp), ("ldo", i64), ("S", i32), ("Skv", i32), ("heads", i32),
                ("dh", i32), ("nseg", i32), ("q_seg_stride", i64), ("kv_seg_stride", i64),
                ("o_seg_stride", i64), ("seg_valid", i32)]


class QcbAttentionBf16(C.Structure):
    _fields_ = [("q", vp), ("ldq", i64), ("k", vp), ("ldk", i64), ("v", vp), ("ldv", i64),
                ("out", vp), ("ldo", i64), ("S", i32), ("heads", i32), ("dh", i32),
                ("nseg", i32), ("seg_stride", i64), ("scale", C.c_float)]


class QcbDdpm(C.Structure):
    _fields_ = [("x", vp), ("eps", vp), ("noise", vp), ("out", vp), ("n", i64),
                ("c1", f64), ("c2", f64), ("c3", f64), ("rc2", f64), ("noise_seed", u64),
                ("noise_offset", u64), ("gen_noise", i32)]


class QcbFeat(C.Structure):
    _fields_ = [("base", vp), ("ld", i64), ("row0", vp)]


class QcbThresholds(C.Structure):
    _fields_ = [("delta1", f64), ("delta2", f64), ("tau_max", i32), ("tau_mid", i32),
                ("tau_min", i32), ("theta1", f64), ("theta2", f64), ("bit_max", i32),
                ("bit_mid", i32), ("bit_min", i32), ("tau_high", f64), ("tau_low", f64),
                ("p_base", f64), ("v_low", f64), ("v_high", f64), ("history_k", i32),
                ("prune_adjust", f64), ("hlc", i32), ("aigq_w", i32), ("aigq_a", i32),
                ("srap", i32)]


L = MAX_LAYERS


class QcbPolicyVideo(C.Structure):
    _fields_ = [("seen", i32), ("n_d", i32), ("boundary", i32), ("long_skip", i32),
                ("abits", i32), ("forced", i32), ("pad0", i32), ("pad1", i32),
                ("cache_valid", i32 * L), ("cache_step", i32 * L), ("cache_tau", i32 * L),
                ("prev_valid", i32 * L), ("d_order", i32 * L), ("has_d", i32 * L),
                ("action", i32 * L), ("sim_valid", i32 * L), ("d_valid", i32 * L),
                ("ref_kind", i32 * L), ("last_d", f64 * L), ("sim", f64 * L),
                ("d_now", f64 * L), ("v", f64)]


_lib = None


def lib():
    """Load libqcb200.so once; raise loudly when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"libqcb200.so not built at {LIB_PATH}; run `python -m "
            "paper_2503_06545_b200.build_native` (there is no CPU fallback)")
    h = C.CDLL(LIB_PATH)
    P = C.POINTER
    sigs = {
        "qcb_gemm_u8": [P(QcbGemm), vp],
        "qcb_gemm_f64": [P(QcbGemmF64), vp],
        "qcb_head_gemm": [P(QcbHeadGemm), vp],
        "qcb_head_prep": [vp, i32, i32, vp, vp],
        "qcb_act_quant": [P(QcbActQuant), vp],
        "qcb_weight_prep": [P(QcbWeightPrep), vp],
        "qcb_ln_mod": [P(QcbLnMod), vp],
        "qcb_attention_f64": [P(QcbAttention), vp],
        "qcb_attention_bf16": [P(QcbAttentionBf16), vp],
        "qcb_ddpm_step": [P(QcbDdpm), vp],
        "qcb_cfg_combine": [vp, vp, C.c_float, vp, i64, vp],
        "qcb_pack_w4": [vp, i64, i32, i32, vp, i64, vp],
        "qcb_gelu_inplace": [vp, i64, i32, i32, vp],
        "qcb_reduce_hlc": [QcbFeat, QcbFeat, QcbFeat, i32, i32, i32, vp, vp, vp, vp],
        "qcb_reduce_srap": [QcbFeat, QcbFeat, i32, i32, i32, vp, vp, vp, vp, vp],
        "qcb_reduce_l1": [QcbFeat, QcbFeat, i32, i32, i32, vp, vp, vp],
        "qcb_reduce_l1_hist": [QcbFeat, C.POINTER(QcbFeat), i32, i32, i32, i32, vp, vp, vp],
        "qcb_copy_async": [vp, vp, C.c_size_t, vp],
        "qcb_col_absmax": [vp, i64, vp, i32, i32, i32, i32, vp, vp],
        "qcb_policy_plan_reuse": [vp, i32, i32, i32, QcbThresholds, vp],
        "qcb_policy_sim_mask": [vp, i32, i32, QcbThresholds, vp, vp],
        "qcb_policy_plan_finish": [vp, i32, i32, i32, QcbThresholds, vp, vp, i32, vp, i64, vp],
        "qcb_policy_observe": [vp, i32, i32, i32, QcbThresholds, vp, vp],
        "qcb_policy_observe_all": [vp, i32, i32, i32, QcbThresholds, vp, vp],
    }
    for name, args in sigs.items():
        fn = getattr(h, name)
        fn.argtypes = args
        fn.restype = C.c_int
    h.qcb_act_quant_workspace_bytes.argtypes = [i32, i32, i32, i32]
    h.qcb_act_quant_workspace_bytes.restype = C.c_size_t
    h.qcb_head_prep_bytes.argtypes = [i32, i32]
    h.qcb_head_prep_bytes.restype = C.c_size_t
    h.qcb_head_workspace_bytes.argtypes = [i64, i32, i32]
    h.qcb_head_workspace_bytes.restype = C.c_size_t
    h.qcb_reduce_workspace_bytes.argtypes = [i32]
    h.qcb_reduce_workspace_bytes.restype = C.c_size_t
    h.qcb_device_sm_count.restype = C.c_int
    h.qcb_version.restype = C.c_char_p
    h.qcb_last_error.restype = C.c_char_p
    _lib = h
    return h


EXPORTED = ("qcb_gemm_u8", "qcb_pack_w4", "qcb_gemm_f64", "qcb_head_gemm", "qcb_head_prep",
            "qcb_head_prep_bytes", "qcb_head_workspace_bytes", "qcb_act_quant", "qcb_act_quant_workspace_bytes", "qcb_weight_prep", "qcb_ln_mod",
            "qcb_attention_f64", "qcb_attention_bf16", "qcb_ddpm_step", "qcb_cfg_combine", "qcb_gelu_inplace", "qcb_reduce_hlc", "qcb_reduce_srap",
            "qcb_reduce_l1", "qcb_reduce_l1_hist", "qcb_reduce_workspace_bytes", "qcb_copy_async", "qcb_col_absmax", "qcb_policy_plan_reuse",
            "qcb_policy_sim_mask", "qcb_policy_plan_finish", "qcb_policy_observe",
            "qcb_policy_observe_all",
            "qcb_device_sm_count", "qcb_version", "qcb_last_error")


def check(rc: int, what: str):
    """Map a C-ABI status onto the reference's exception types (errors.py)."""
    if rc == QCB_OK:
        return
    msg = f"{what} failed (status {rc})"
    if rc == QCB_ERR_DIM:
        raise DimensionError(msg)
    if rc in (QCB_ERR_CONFIG, QCB_ERR_OVERFLOW):
        raise ConfigurationError(msg + (": integer accumulator overflow risk"
                                        if rc == QCB_ERR_OVERFLOW else ""))
    if rc == QCB_ERR_VALUE:
        raise ValueError(msg)
    if rc == QCB_ERR_TYPE:
        raise TypeError(msg)
    err = _lib.qcb_last_error().decode() if _lib is not None else "?"
    raise RuntimeError(msg + f" (CUDA error: {err})")


def ptr(t) -> int:
    """Device pointer of a torch tensor (None -> NULL)."""
    return 0 if t is None else int(t.data_ptr())


_dev_index = None


def stream_ptr(stream=None) -> int:
    """cudaStream_t of `stream` (default: the current stream).  The current
    stream is read through the raw accessor: torch.cuda.current_stream() costs
    ~15 us of Python per call, which adds up over thousands of launches."""
    import torch
    global _dev_index
    if stream is not None:
        return int(stream.cuda_stream)
    if _dev_index is None:
        _dev_index = torch.cuda.current_device()
    return int(torch._C._cuda_getCurrentRawStream(_dev_index))
