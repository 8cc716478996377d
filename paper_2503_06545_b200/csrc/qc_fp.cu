// Full-precision pieces of the block that sit around the quantized linears:
// the f64-accumulating GEMM (reference `mm`, tensor.py:43-60, used for FP
// sites, the weight-only / act-only AIGQ modes and the noise head), layer norm
// + modulation (model.py:137-142,182,196), per-head attention with an f64
// softmax (model.py:150-156, tensor.py:115-132) and the DDPM update
// (sampler.py:59-88).  These are the reference-exact ("precise") versions;
// every product of two f32 values is exact in f64, so an ascending-k f64 FMA
// chain reproduces the reference's sequential sum bit-for-bit.
#include "qc_common.cuh"
#include "qc_api_internal.h"

namespace qc {

// ------------------------------------------------------------------ gemm_f64
constexpr int kFT = 64;   // output tile
constexpr int kFK = 16;   // k tile

struct GemmF64P {
  QcbGemmF64 g;
};


__global__ void __launch_bounds__(256) gemm_f64_k(const GemmF64P P) {
  const QcbGemmF64& g = P.g;
  __shared__ float As[kFK][kFT + 1];
  __shared__ float Ws[kFK][kFT + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * kFT, n0 = blockIdx.x * kFT;
  const int seg_rows = g.seg_rows > 0 ? g.seg_rows : g.M;
  const int seg_valid = g.seg_valid > 0 ? g.seg_valid : seg_rows;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int k0 = 0; k0 < g.K; k0 += kFK) {
    for (int i = threadIdx.x; i < kFK * kFT; i += 256) {
      const int kk = i / kFT, mm = i % kFT;
      const int m = m0 + mm, k = k0 + kk;
      float av = 0.f;
      if (m < g.M && k < g.K) {
        const int seg = m / seg_rows, r = m - seg * seg_rows;
        const long long row = g.a_row0 ? g.a_row0[seg] + r : (long long)m;
        if (r < seg_valid) av = g.a[row * g.lda + k];
      }
      As[kk][mm] = av;
      const int n = n0 + mm;
      Ws[kk][mm] = (n < g.N && k < g.K) ? g.w[(long long)k * g.ldw + n] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kFK; ++kk) {
      double a[4], w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = (double)As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) w[j] = (double)Ws[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], w[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= g.M) continue;
    const int seg = m / seg_rows, r = m - seg * seg_rows;
    if (r >= seg_valid) continue;
    const long long orow = g.out_row0 ? g.out_row0[seg] + r : (long long)m;
    const long long rrow = g.resid_row0 ? g.resid_row0[seg] + r : (long long)m;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= g.N) continue;
      float y = __double2float_rn(acc[i][j]);
      switch (g.epilogue) {
        case QCB_EPI_GELU: y = __double2float_rn(gelu_ref((double)y)); break;
        case QCB_EPI_GATE_RESID:
          y = __fadd_rn(g.resid[rrow * g.ldr + n], __fmul_rn(g.gate_scalar, y));
          break;
        case QCB_EPI_RESID: y = __fadd_rn(g.resid[rrow * g.ldr + n], y); break;
        case QCB_EPI_BIAS: y = __fadd_rn(y, g.bias[n]); break;
        default: break;
      }
      g.out[orow * g.ldo + n] = y;
    }
  }
}

int gemm_f64_launch(const QcbGemmF64* g, cudaStream_t st) {
  GemmF64P P{*g};
  dim3 grid((g->N + kFT - 1) / kFT, (g->M + kFT - 1) / kFT);
  gemm_f64_k<<<grid, 256, 0, st>>>(P);
  return launch_status();
}

// ------------------------------------------------------------------ ln + mod
template <typename T, typename Op>
QC_DEV T block_reduce256(T v, T* scratch, Op op) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  T r = scratch[0];
  for (int w = 1; w < 8; ++w) r = op(r, scratch[w]);
  return r;
}

__global__ void __launch_bounds__(256) ln_mod_k(const QcbLnMod q) {
  __shared__ double red[32];
  const int seg = blockIdx.y, r = blockIdx.x;
  if (r >= (q.seg_valid > 0 ? q.seg_valid : q.seg_rows)) return;
  const long long irow = (q.x_row0 ? q.x_row0[seg] : (long long)seg * q.seg_rows) + r;
  const long long orow = (q.out_row0 ? q.out_row0[seg] : (long long)seg * q.seg_rows) + r;
  const float* x = q.x + irow * q.ldx;
  float* o = q.out + orow * q.ldo;
  const int K = q.K;
  double s = 0.0;
  for (int j = threadIdx.x; j < K; j += 256) s += (double)x[j];
  const double mean = block_reduce256(s, red, [](double a, double b) { return a + b; }) / K;
  double v = 0.0;
  for (int j = threadIdx.x; j < K; j += 256) {
    const double d = (double)x[j] - mean;
    v += d * d;
  }
  const double var = block_reduce256(v, red, [](double a, double b) { return a + b; }) / K;
  const double sd = sqrt(var + 1e-5);
  for (int j = threadIdx.x; j < K; j += 256) {
    const double g = q.ln_g ? (double)q.ln_g[j] : 1.0;
    const double b = q.ln_b ? (double)q.ln_b[j] : 0.0;
    const float f = __double2float_rn(__dadd_rn(__dmul_rn(__ddiv_rn((double)x[j] - mean, sd), g), b));
    o[j] = __fadd_rn(__fmul_rn(f, q.mod_scale1), q.mod_shift);
  }
}

int ln_mod_launch(const QcbLnMod* q, cudaStream_t st) {
  dim3 grid(q->seg_valid > 0 ? q->seg_valid : q->seg_rows, q->nseg);
  ln_mod_k<<<grid, 256, 0, st>>>(*q);
  return launch_status();
}

// ------------------------------------------------------------------ attention
// numpy pairwise summation (np.add.reduce on a contiguous f64 vector,
// block size 128), so the softmax denominator matches the reference exactly.
QC_DEV double np_pw_sum(const double* a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return np_pw_sum(a, n2) + np_pw_sum(a + n2, n - n2);
}

// One CTA per (query row, head, segment). Scores in smem (f64).
__global__ void __launch_bounds__(128) attention_f64_k(const QcbAttention a) {
  extern __shared__ __align__(16) uint8_t sm[];
  double* sc = reinterpret_cast<double*>(sm);
  __shared__ double qv[256];
  __shared__ double red[32];
  const int i = blockIdx.x, h = blockIdx.y, seg = blockIdx.z;
  if (i >= (a.seg_valid > 0 ? a.seg_valid : a.S)) return;
  const int dh = a.dh;
  const float* qrow = a.q + ((long long)seg * a.q_seg_stride + i) * a.ldq + h * dh;
  for (int d = threadIdx.x; d < dh; d += blockDim.x) qv[d] = (double)qrow[d];
  __syncthreads();
  const double rs = sqrt((double)dh);
  const float* kb = a.k + (long long)seg * a.kv_seg_stride * a.ldk + h * dh;
  for (int j = threadIdx.x; j < a.Skv; j += blockDim.x) {
    const float* kr = kb + (long long)j * a.ldk;
    double s = 0.0;
    for (int d = 0; d < dh; ++d) s = fma(qv[d], (double)kr[d], s);
    sc[j] = (double)__double2float_rn(s) / rs;
  }
  __syncthreads();
  double mx = -INFINITY;
  for (int j = threadIdx.x; j < a.Skv; j += blockDim.x) mx = fmax(mx, sc[j]);
  {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) red[w] = mx;
    __syncthreads();
    mx = red[0];
    for (int k = 1; k < (int)(blockDim.x / 32); ++k) mx = fmax(mx, red[k]);
    __syncthreads();
  }
  for (int j = threadIdx.x; j < a.Skv; j += blockDim.x) sc[j] = exp(sc[j] - mx);
  __syncthreads();
  if (threadIdx.x == 0) red[0] = np_pw_sum(sc, a.Skv);
  __syncthreads();
  const double tot = red[0];
  for (int j = threadIdx.x; j < a.Skv; j += blockDim.x) sc[j] = sc[j] / tot;
  __syncthreads();
  const float* vb = a.v + (long long)seg * a.kv_seg_stride * a.ldv + h * dh;
  float* orow = a.out + ((long long)seg * a.o_seg_stride + i) * a.ldo + h * dh;
  for (int d = threadIdx.x; d < dh; d += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < a.Skv; ++j) s = fma(sc[j], (double)vb[(long long)j * a.ldv + d], s);
    orow[d] = __double2float_rn(s);
  }
}

// Cross-attention on the single cond token (model.py:190-193): the softmax over
// one key is exactly 1 (exp(0)/exp(0)), and mm(p, v) = f32(0 + 1.0*v) = v, so
// every query row's output is the value row -- identical bits, one copy.
__global__ void attention_single_key_k(const QcbAttention a) {
  const int seg = blockIdx.y;
  const int d = a.heads * a.dh;
  const float* vrow = a.v + (long long)seg * a.kv_seg_stride * a.ldv;
  const int valid = a.seg_valid > 0 ? a.seg_valid : a.S;
  for (int i = blockIdx.x; i < valid; i += gridDim.x) {
    float* orow = a.out + ((long long)seg * a.o_seg_stride + i) * a.ldo;
    for (int j = threadIdx.x; j < d; j += blockDim.x) orow[j] = vrow[j];
  }
}

int attention_f64_launch(const QcbAttention* a, cudaStream_t st) {
  if (a->Skv == 1) {
    dim3 grid((unsigned)min(a->S, 1024), a->nseg);
    attention_single_key_k<<<grid, 128, 0, st>>>(*a);
    return launch_status();
  }
  if (a->dh > 256) return QCB_ERR_DIM;
  const size_t smem = (size_t)a->Skv * sizeof(double);
  if (smem > 200 * 1024) return QCB_ERR_DIM;
  static bool attr = false;
  allow_max_smem(attention_f64_k, attr);
  dim3 grid(a->seg_valid > 0 ? a->seg_valid : a->S, a->heads, a->nseg);
  attention_f64_k<<<grid, 128, smem, st>>>(*a);
  return launch_status();
}

// ------------------------------------------------------------------ ddpm
__global__ void ddpm_k(const QcbDdpm d) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.n) return;
  double m = __ddiv_rn(__dsub_rn((double)d.x[i], __dmul_rn(d.c1, (double)d.eps[i])), d.c2);
  if (d.noise) m = __dadd_rn(m, __dmul_rn(d.c3, (double)d.noise[i]));
  d.out[i] = __double2float_rn(m);
}

int ddpm_launch(const QcbDdpm* d, cudaStream_t st) {
  const int th = 256;
  ddpm_k<<<(unsigned)((d->n + th - 1) / th), th, 0, st>>>(*d);
  return launch_status();
}

}  // namespace qc
