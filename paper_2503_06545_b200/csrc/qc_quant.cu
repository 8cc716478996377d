// AIGQ quantizer kernels (the activation side of QuantRuntime.gemm_fn and the
// offline weight preparation of QuantRuntime.__init__).
//
// Activation path (runtime.py:69-75 -> quant.py:163-165, 83-123), fused per row:
//   prologue   h  = f32(LN_f64(x)) * (1+scale) + shift      (model.py:182,189,196)
//   balance    y  = f32(f64(h) / c)                           (quant.py:164)
//   rotation   xe = f32(r * FWHT_f64(signs (.) y[:b])) (+) y[b:]  (quant.py:151-165)
//   params     per-tensor (per video) min/max -> (s, z)       (quant.py:83-110)
//   codes      clip(rha(f64(xe)/s) + z, 0, 2^b-1) -> u8, plus row sums
// Two passes over the input (min/max, then codes) instead of materialising
// xe: 8 B/elem read + 1 B/elem written per output instead of 13 B/elem.
// Up to three outputs (q/k/v sites share h1, each with its own c) per read.
//
// Weight path (runtime.py:40-61): R^T (c (.) W) per output channel, per-channel
// min/max params, u8 codes stored K-major [N][K] for the UMMA B operand, and
// column sums for the zero-point correction.
#include "qc_common.cuh"
#include "qc_api_internal.h"

namespace qc {

constexpr int kQThreads = 256;

// Block-wide f64 sum / min / max via warp shuffles + smem (blockDim == 256).
template <typename T, typename Op>
QC_DEV T block_reduce(T v, T* scratch, Op op) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  T r = scratch[0];
#pragma unroll
  for (int w = 1; w < kQThreads / 32; ++w) r = op(r, scratch[w]);
  return r;
}

// In-place unnormalised Walsh-Hadamard transform of buf[0:b] (b power of 2).
QC_DEV void block_fwht(double* buf, int b) {
  for (int h = 1; h < b; h <<= 1) {
    __syncthreads();
    for (int i = threadIdx.x; i < (b >> 1); i += blockDim.x) {
      const int blk = i / h, off = i - blk * h;
      const int j = blk * 2 * h + off;
      const double u = buf[j], v = buf[j + h];
      buf[j] = u + v;
      buf[j + h] = u - v;
    }
  }
  __syncthreads();
}

struct ActQuantParams {
  const float* x;
  long long ldx;
  const long long* x_row0;
  int K, seg_rows, seg_valid, nseg;
  int prologue;  // QCB_PRO_*
  const float* ln_g;
  const float* ln_b;
  float scale1, shift;
  int n_out, bits, b;  // b: rotation block (power of two <= K), 0 = no rotation
  const double* c[3];
  const float* signs[3];
  float rscale;  // f32(1/sqrt(b))
  uint8_t* codes[3];
  long long ldc;
  int* rowsum[3];
  double* scale[3];
  int* zero[3];
  float* xe_out[3];
  long long ldxe;
  float* deq_out[3];
  uint32_t* keys;  // [n_out][nseg][2]: ordered-float min key, max key
};

// Produce xe (rotated, balanced activations) for output `o` into buf (f64),
// given h in hbuf (f32 row after prologue).
QC_DEV void rotate_row(const ActQuantParams& p, int o, const float* hrow, double* buf) {
  const int K = p.K;
  const double* c = p.c[o];
  if (c == nullptr) {
    for (int j = threadIdx.x; j < K; j += blockDim.x) buf[j] = (double)hrow[j];
    __syncthreads();
    return;
  }
  const float* sg = p.signs[o];
  const int b = p.b;
  for (int j = threadIdx.x; j < K; j += blockDim.x) {
    const float y = __double2float_rn(__ddiv_rn((double)hrow[j], c[j]));
    buf[j] = (j < b) ? (double)y * (double)sg[j] : (double)y;
  }
  block_fwht(buf, b);
  const double r = (double)p.rscale;
  for (int j = threadIdx.x; j < b; j += blockDim.x)
    buf[j] = (double)__double2float_rn(__dmul_rn(buf[j], r));
  __syncthreads();
}

// Prologue: h = f32(LN64(x)) * scale1 + shift (or x itself), into hrow (f32 smem).
QC_DEV void prologue_row(const ActQuantParams& p, const float* xrow, float* hrow,
                         double* red) {
  const int K = p.K;
  if (p.prologue == QCB_PRO_NONE) {
    for (int j = threadIdx.x; j < K; j += blockDim.x) hrow[j] = xrow[j];
    __syncthreads();
    return;
  }
  double s = 0.0;
  for (int j = threadIdx.x; j < K; j += blockDim.x) s += (double)xrow[j];
  const double mean = block_reduce(s, red, [](double a, double b) { return a + b; }) / K;
  double v = 0.0;
  for (int j = threadIdx.x; j < K; j += blockDim.x) {
    const double d = (double)xrow[j] - mean;
    v += d * d;
  }
  const double var = block_reduce(v, red, [](double a, double b) { return a + b; }) / K;
  const double sd = sqrt(var + 1e-5);
  for (int j = threadIdx.x; j < K; j += blockDim.x) {
    const double g = p.ln_g ? (double)p.ln_g[j] : 1.0;
    const double bb = p.ln_b ? (double)p.ln_b[j] : 0.0;
    const double nrm = __dadd_rn(__dmul_rn(__ddiv_rn((double)xrow[j] - mean, sd), g), bb);
    const float f = __double2float_rn(nrm);
    hrow[j] = __fadd_rn(__fmul_rn(f, p.scale1), p.shift);
  }
  __syncthreads();
}

// Grid: one CTA per (segment, row).  kPass 1: min/max; kPass 2: codes.
template <int kPass>
__global__ void __launch_bounds__(kQThreads) act_quant_rows(const ActQuantParams p) {
  extern __shared__ __align__(16) uint8_t sm[];
  double* buf = reinterpret_cast<double*>(sm);
  float* hrow = reinterpret_cast<float*>(buf + p.K);
  __shared__ double red[32];
  __shared__ float fred[32];
  __shared__ int ired[32];
  __shared__ double s_scale[3];
  __shared__ int s_zero[3];

  const int seg = blockIdx.y;
  const int mrow = blockIdx.x;
  if (mrow >= p.seg_valid) return;
  const long long in_row = (p.x_row0 ? p.x_row0[seg] : (long long)seg * p.seg_rows) + mrow;
  const long long out_row = (long long)seg * p.seg_rows + mrow;
  const float* xrow = p.x + in_row * p.ldx;
  const int top = (1 << p.bits) - 1;

  if (kPass == 2 && threadIdx.x < p.n_out) {
    const int o = threadIdx.x;
    const uint32_t* k = p.keys + ((size_t)o * p.nseg + seg) * 2;
    const double lo = (double)key2f(k[0]);
    const double hi = (double)key2f(k[1]);
    const double span = hi - lo;
    double s;
    int z;
    if (span <= 0.0) {
      s = 1.0;
      z = 0;
    } else {
      s = scale_up16(__ddiv_rn(span, (double)top));
      double zr = rha(__ddiv_rn(-lo, s));
      zr = fmin(fmax(zr, 0.0), (double)top);
      z = (int)zr;
    }
    s_scale[o] = s;
    s_zero[o] = z;
    if (mrow == 0) {
      p.scale[o][seg] = s;
      p.zero[o][seg] = z;
    }
  }

  prologue_row(p, xrow, hrow, red);
  for (int o = 0; o < p.n_out; ++o) {
    rotate_row(p, o, hrow, buf);
    if (kPass == 1) {
      float mn = INFINITY, mx = -INFINITY;
      for (int j = threadIdx.x; j < p.K; j += blockDim.x) {
        const float v = (float)buf[j];
        mn = fminf(mn, v);
        mx = fmaxf(mx, v);
      }
      mn = block_reduce(mn, fred, [](float a, float b) { return fminf(a, b); });
      mx = block_reduce(mx, fred, [](float a, float b) { return fmaxf(a, b); });
      if (threadIdx.x == 0) {
        uint32_t* k = p.keys + ((size_t)o * p.nseg + seg) * 2;
        atomicMin(&k[0], f2key(mn));
        atomicMax(&k[1], f2key(mx));
      }
      if (p.xe_out[o]) {
        float* xe = p.xe_out[o] + out_row * p.ldxe;
        for (int j = threadIdx.x; j < p.K; j += blockDim.x) xe[j] = (float)buf[j];
      }
    } else {
      const double s = s_scale[o];
      const double z = (double)s_zero[o];
      uint8_t* crow = p.codes[o] ? p.codes[o] + out_row * p.ldc : nullptr;
      float* drow = p.deq_out[o] ? p.deq_out[o] + out_row * p.ldxe : nullptr;
      int rs = 0;
      for (int j = threadIdx.x; j < p.K; j += blockDim.x) {
        double q = __dadd_rn(rha(__ddiv_rn(buf[j], s)), z);
        q = fmin(fmax(q, 0.0), (double)top);
        const int code = (int)q;
        if (crow) crow[j] = (uint8_t)code;
        if (drow) drow[j] = __double2float_rn(__dmul_rn(s, (double)(code - s_zero[o])));
        rs += code;
      }
      rs = block_reduce(rs, ired, [](int a, int b) { return a + b; });
      if (threadIdx.x == 0 && crow) p.rowsum[o][out_row] = rs;
    }
    __syncthreads();
  }
}

__global__ void init_keys(uint32_t* keys, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) keys[i] = (i & 1) ? 0u : 0xFFFFFFFFu;
}

int act_quant_launch(const QcbActQuant* q, cudaStream_t st) {
  ActQuantParams p{};
  p.x = q->x;
  p.ldx = q->ldx;
  p.x_row0 = q->x_row0;
  p.K = q->K;
  p.seg_rows = q->seg_rows;
  p.seg_valid = q->seg_valid > 0 ? q->seg_valid : q->seg_rows;
  p.nseg = q->nseg;
  p.prologue = q->prologue;
  p.ln_g = q->ln_g;
  p.ln_b = q->ln_b;
  p.scale1 = q->mod_scale1;
  p.shift = q->mod_shift;
  p.n_out = q->n_out;
  p.bits = q->bits;
  p.b = 0;
  for (int o = 0; o < q->n_out; ++o) {
    p.c[o] = q->chan_scale[o];
    p.signs[o] = q->signs[o];
    p.codes[o] = q->codes[o];
    p.rowsum[o] = q->rowsum[o];
    p.scale[o] = q->scale[o];
    p.zero[o] = q->zero[o];
    p.xe_out[o] = q->xe_out[o];
    p.deq_out[o] = q->deq_out[o];
  }
  p.ldc = q->ldc;
  p.ldxe = q->ldxe;
  int b = 1;
  while (b * 2 <= q->K) b *= 2;
  p.b = b;
  p.rscale = (float)(1.0 / sqrt((double)b));
  p.keys = reinterpret_cast<uint32_t*>(q->workspace);
  const int nkeys = 2 * q->n_out * q->nseg;
  init_keys<<<(nkeys + 255) / 256, 256, 0, st>>>(p.keys, nkeys);
  const size_t smem = (size_t)q->K * (sizeof(double) + sizeof(float));
  if (smem > 200 * 1024) return QCB_ERR_DIM;
  static bool attr1 = false, attr2 = false;
  allow_max_smem(act_quant_rows<1>, attr1);
  allow_max_smem(act_quant_rows<2>, attr2);
  dim3 grid(p.seg_valid, p.nseg);
  act_quant_rows<1><<<grid, kQThreads, smem, st>>>(p);
  act_quant_rows<2><<<grid, kQThreads, smem, st>>>(p);
  return launch_status();
}

// ------------------------------------------------------------------ weights

struct WeightPrepParams {
  const float* w;  // [K][N] row-major (reference layout)
  int K, N, bits, b;
  const double* c;     // nullable -> no balance/rotation
  const float* signs;  // [b]
  float rscale;
  uint8_t* codes;  // [N][ldk]
  long long ldk;
  double* scale;  // [N]
  int* zero;      // [N]
  int* colsum;    // [N]
  float* w_eff;   // nullable [K][N] (debug / weight-only FP mode)
  float* w_deq;   // nullable [K][N]: f32(s*(code-z)) (runtime.py:61)
};

// One CTA per output channel n.
__global__ void __launch_bounds__(kQThreads) weight_prep_cols(const WeightPrepParams p) {
  extern __shared__ __align__(16) uint8_t sm[];
  double* buf = reinterpret_cast<double*>(sm);
  __shared__ float fred[32];
  __shared__ int ired[32];
  const int n = blockIdx.x;
  const int K = p.K;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const float wv = p.w[(size_t)k * p.N + n];
    if (p.c) {
      const float u = __double2float_rn(__dmul_rn(p.c[k], (double)wv));
      buf[k] = (k < p.b) ? (double)u * (double)p.signs[k] : (double)u;
    } else {
      buf[k] = (double)wv;
    }
  }
  if (p.c) {
    block_fwht(buf, p.b);
    const double r = (double)p.rscale;
    for (int k = threadIdx.x; k < p.b; k += blockDim.x)
      buf[k] = (double)__double2float_rn(__dmul_rn(buf[k], r));
  }
  __syncthreads();
  float mn = INFINITY, mx = -INFINITY;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const float v = (float)buf[k];
    mn = fminf(mn, v);
    mx = fmaxf(mx, v);
    if (p.w_eff) p.w_eff[(size_t)k * p.N + n] = v;
  }
  mn = block_reduce(mn, fred, [](float a, float b) { return fminf(a, b); });
  mx = block_reduce(mx, fred, [](float a, float b) { return fmaxf(a, b); });
  const int top = (1 << p.bits) - 1;
  const double lo = (double)mn, hi = (double)mx, span = hi - lo;
  double s;
  double z;
  if (span <= 0.0) {
    s = 1.0;
    z = 0.0;
  } else {
    s = scale_up16(__ddiv_rn(span, (double)top));
    z = fmin(fmax(rha(__ddiv_rn(-lo, s)), 0.0), (double)top);
  }
  int cs = 0;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double q = __dadd_rn(rha(__ddiv_rn(buf[k], s)), z);
    q = fmin(fmax(q, 0.0), (double)top);
    const int code = (int)q;
    p.codes[(size_t)n * p.ldk + k] = (uint8_t)code;
    cs += code;
    if (p.w_deq) p.w_deq[(size_t)k * p.N + n] = __double2float_rn(s * (double)(code - (int)z));
  }
  cs = block_reduce(cs, ired, [](int a, int b) { return a + b; });
  if (threadIdx.x == 0) {
    p.scale[n] = s;
    p.zero[n] = (int)z;
    p.colsum[n] = cs;
  }
}

int weight_prep_launch(const QcbWeightPrep* q, cudaStream_t st) {
  WeightPrepParams p{};
  p.w = q->w;
  p.K = q->K;
  p.N = q->N;
  p.bits = q->bits;
  int b = 1;
  while (b * 2 <= q->K) b *= 2;
  p.b = b;
  p.c = q->chan_scale;
  p.signs = q->signs;
  p.rscale = (float)(1.0 / sqrt((double)b));
  p.codes = q->codes;
  p.ldk = q->ldk;
  p.scale = q->scale;
  p.zero = q->zero;
  p.colsum = q->colsum;
  p.w_eff = q->w_eff;
  p.w_deq = q->w_deq;
  const size_t smem = (size_t)q->K * sizeof(double);
  if (smem > 200 * 1024) return QCB_ERR_DIM;
  static bool attr = false;
  allow_max_smem(weight_prep_cols, attr);
  weight_prep_cols<<<q->N, kQThreads, smem, st>>>(p);
  return launch_status();
}

}  // namespace qc
