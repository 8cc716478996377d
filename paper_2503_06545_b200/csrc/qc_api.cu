// extern "C" entry points of libqcb200.so (declared in include/qcb200.h).
// Argument validation mirrors the reference's error behaviour
// (tensor.py:82-98, quant.py:83-93); kernels live in the other units.
#include <cstdio>

#include "qc_api_internal.h"

using namespace qc;

static bool aligned16(long long v) { return (v % 16) == 0; }

extern "C" int qcb_gemm_u8(const QcbGemm* g, void* stream) {
  if (!g || !g->a_codes || (!g->w_codes && !g->w_packed) || !g->out || !g->a_scale ||
      !g->a_zero || !g->a_rowsum || !g->w_scale || !g->w_zero || !g->w_colsum)
    return QCB_ERR_VALUE;
  if (g->M <= 0 || g->N <= 0 || g->K <= 0) return QCB_ERR_DIM;
  if (g->lda < g->K || !aligned16(g->lda)) return QCB_ERR_DIM;
  if (g->w_packed) {   // W4: [N][ldwp] nibbles, rows padded to whole 128-k blocks
    if (g->ldwp % 64 || 2 * g->ldwp < g->K || reinterpret_cast<uintptr_t>(g->w_packed) % 16)
      return QCB_ERR_DIM;
  } else if (g->ldw < g->K || !aligned16(g->ldw) ||
             reinterpret_cast<uintptr_t>(g->w_codes) % 16) {
    return QCB_ERR_DIM;
  }
  if (g->ldo < g->N) return QCB_ERR_DIM;
  // u8 x u8 into a signed 32-bit accumulator: K * 255 * 255 must fit
  // (the reference guards its emulated accumulator the same way, tensor.py:91-98).
  if ((long long)g->K * 255LL * 255LL > 2147483647LL) return QCB_ERR_OVERFLOW;
  if ((g->epilogue == QCB_EPI_GATE_RESID || g->epilogue == QCB_EPI_RESID) && !g->resid)
    return QCB_ERR_VALUE;
  if (g->epilogue < QCB_EPI_STORE || g->epilogue > QCB_EPI_STORE_BF16 ||
      g->epilogue == QCB_EPI_BIAS)
    return QCB_ERR_CONFIG;
  if (reinterpret_cast<uintptr_t>(g->a_codes) % 16) return QCB_ERR_DIM;
  return gemm_u8_launch(g, (cudaStream_t)stream);
}

extern "C" int qcb_pack_w4(const uint8_t* codes, long long ldk, int N, int K, uint8_t* packed,
                           long long ldwp, void* stream) {
  if (!codes || !packed) return QCB_ERR_VALUE;
  if (N <= 0 || K <= 0 || ldk < K || ldwp % 64 || 2 * ldwp < K) return QCB_ERR_DIM;
  return pack_w4_launch(codes, ldk, N, K, packed, ldwp, (cudaStream_t)stream);
}

extern "C" int qcb_head_prep(const float* w, int K, int N, void* prep, void* stream) {
  if (!w || !prep) return QCB_ERR_VALUE;
  if (K <= 0 || N <= 0) return QCB_ERR_DIM;
  if (6LL * K * 255LL * 255LL > 2147483647LL) return QCB_ERR_OVERFLOW;
  return qc::head_prep_launch(w, K, N, prep, (cudaStream_t)stream);
}

extern "C" int qcb_head_gemm(const QcbHeadGemm* g, void* stream) {
  if (!g || !g->x || !g->prep || !g->out || !g->workspace) return QCB_ERR_VALUE;
  if (g->nseg <= 0 || g->seg_rows <= 0 || g->K <= 0 || g->N <= 0) return QCB_ERR_DIM;
  if (g->seg_valid <= 0 || g->seg_valid > g->seg_rows || g->ldo < g->N || g->ldx < g->K)
    return QCB_ERR_DIM;
  if (g->K % 4 || g->N % 4 || g->ldx % 4 || (reinterpret_cast<uintptr_t>(g->x) & 15))
    return QCB_ERR_DIM;   // 16-byte row vectors (digits, outputs, exact fallback)
  if (6LL * g->K * 255LL * 255LL > 2147483647LL) return QCB_ERR_OVERFLOW;
  if ((long long)g->nseg * g->seg_rows * g->N >= (1LL << 31)) return QCB_ERR_DIM;
  return qc::head_gemm_launch(g, (cudaStream_t)stream);
}

extern "C" int qcb_gemm_f64(const QcbGemmF64* g, void* stream) {
  if (!g || !g->a || !g->w || !g->out) return QCB_ERR_VALUE;
  if (g->M <= 0 || g->N <= 0 || g->K <= 0) return QCB_ERR_DIM;
  if (g->lda < g->K || g->ldw < g->N || g->ldo < g->N) return QCB_ERR_DIM;
  if ((g->epilogue == QCB_EPI_GATE_RESID || g->epilogue == QCB_EPI_RESID) && !g->resid)
    return QCB_ERR_VALUE;
  if (g->epilogue == QCB_EPI_BIAS && !g->bias) return QCB_ERR_VALUE;
  if (g->epilogue == QCB_EPI_ACC) return QCB_ERR_CONFIG;
  return gemm_f64_launch(g, (cudaStream_t)stream);
}

extern "C" int qcb_act_quant(const QcbActQuant* q, void* stream) {
  if (!q || !q->x || !q->workspace) return QCB_ERR_VALUE;
  if (q->K <= 0 || q->seg_rows <= 0 || q->nseg <= 0) return QCB_ERR_VALUE;  // empty tensor
  if (q->n_out < 1 || q->n_out > 3) return QCB_ERR_CONFIG;
  if (q->bits < 1 || q->bits > 8) return QCB_ERR_CONFIG;
  if (q->ldx < q->K) return QCB_ERR_DIM;
  for (int o = 0; o < q->n_out; ++o) {
    if (!q->scale[o] || !q->zero[o]) return QCB_ERR_VALUE;
    if (q->codes[o] && (!q->rowsum[o] || q->ldc < q->K)) return QCB_ERR_VALUE;
    if (q->chan_scale[o] && !q->signs[o]) return QCB_ERR_VALUE;
  }
  return act_quant_launch(q, (cudaStream_t)stream);
}

extern "C" int qcb_weight_prep(const QcbWeightPrep* q, void* stream) {
  if (!q || !q->w || !q->codes || !q->scale || !q->zero || !q->colsum) return QCB_ERR_VALUE;
  if (q->K <= 0 || q->N <= 0) return QCB_ERR_VALUE;
  if (q->bits < 1 || q->bits > 8) return QCB_ERR_CONFIG;
  if (q->ldk < q->K) return QCB_ERR_DIM;
  if (q->chan_scale && !q->signs) return QCB_ERR_VALUE;
  return weight_prep_launch(q, (cudaStream_t)stream);
}

extern "C" int qcb_ln_mod(const QcbLnMod* q, void* stream) {
  if (!q || !q->x || !q->out) return QCB_ERR_VALUE;
  if (q->K <= 0 || q->seg_rows <= 0 || q->nseg <= 0) return QCB_ERR_DIM;
  return ln_mod_launch(q, (cudaStream_t)stream);
}

extern "C" int qcb_attention_f64(const QcbAttention* a, void* stream) {
  if (!a || !a->q || !a->k || !a->v || !a->out) return QCB_ERR_VALUE;
  if (a->S <= 0 || a->Skv <= 0 || a->heads <= 0 || a->dh <= 0 || a->nseg <= 0) return QCB_ERR_DIM;
  return attention_f64_launch(a, (cudaStream_t)stream);
}

extern "C" int qcb_attention_bf16(const QcbAttentionBf16* a, void* stream) {
  return attention_bf16_launch(a, (cudaStream_t)stream);
}

extern "C" int qcb_ddpm_step(const QcbDdpm* d, void* stream) {
  if (!d || !d->x || !d->eps || !d->out) return QCB_ERR_VALUE;
  if (d->n <= 0) return QCB_ERR_DIM;
  if (d->rc2 != 0.0 && d->rc2 * d->c2 != 1.0 && fabs(d->rc2 * d->c2 - 1.0) > 1e-15)
    return QCB_ERR_VALUE;   // rc2 must be RN(1 / c2)
  return ddpm_launch(d, (cudaStream_t)stream);
}

extern "C" int qcb_cfg_combine(const float* eps_c, const float* eps_u, float scale, float* out,
                               long long n, void* stream) {
  if (!eps_c || !eps_u || !out) return QCB_ERR_VALUE;
  if (n <= 0) return QCB_ERR_DIM;
  return cfg_combine_launch(eps_c, eps_u, scale, out, n, (cudaStream_t)stream);
}

extern "C" int qcb_gelu_inplace(float* x, long long ld, int rows, int cols, void* stream) {
  if (!x) return QCB_ERR_VALUE;
  if (rows <= 0 || cols <= 0 || ld < cols) return QCB_ERR_DIM;
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (ld % 4)) return QCB_ERR_DIM;
  return gelu_launch(x, ld, rows, cols, (cudaStream_t)stream);
}

extern "C" int qcb_device_sm_count(void) { return num_sms(); }

extern "C" const char* qcb_version(void) { return "qcb200 0.1.0 sm_100a"; }

cudaError_t qc::g_last_err = cudaSuccess;

extern "C" const char* qcb_last_error(void) { return cudaGetErrorString(qc::g_last_err); }

extern "C" int qcb_copy_async(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes == 0) return QCB_OK;
  if (!dst || !src) return QCB_ERR_VALUE;
  return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream) == cudaSuccess
             ? QCB_OK
             : QCB_ERR_CUDA;
}
