// The noise head out = f32(mm(x, W)) + b (reference model.py:228, `mm` =
// tensor.py:43-60: ascending-k f64 accumulation of exact f32*f32 products),
// on the int8 tensor cores with an exactness certificate.
//
// Digit planes.  Each x row i is scaled by 2^-e_i (max|x_i| < 2^e_i) and split
// into kHeadDigits balanced base-128 digits D_s in [-64, 64] of weight
// 2^(e_i - 6 - 7 s); each W column j likewise (E_t, 2^(f_j - 6 - 7 t)).  Digits
// are stored as u8 codes D + 64, so the existing tcgen05 u8 GEMM with zero
// point 64 yields exact integer sums.  The products with s + t = d share the
// weight 2^(e+f-12-7d): one GEMM per diagonal d = 0..kHeadDigits-1 with A =
// [X_0 .. X_d] (a prefix of the row's planes) and B_d = [E_d .. E_0] per column,
// K' = (d+1) K, accumulates them exactly in s32 (|sum| <= 7 K 64^2 < 2^31).
//
// Certificate.  S^ = 2^(e+f-12) sum_d acc_d 2^-7d (f64) differs from the exact
// sum S by at most T1 (diagonals d >= kHeadDigits dropped) + T2 (digit
// truncation) + T3 (f64 combination rounding); the reference's sequential sum
// differs from S by at most T4 = (K-1) 2^-53 sum|x w| <= (K-1) 2^-53 |x|_2 |w|_2.
// When [S^ - E, S^ + E] (E = T1+T2+T3+T4, padded) holds no f32 rounding
// boundary, RN32(S^) == RN32(reference); other elements are listed and
// recomputed with the reference's ascending-k f64 FMA chain (bit-exact).
#include <cudaTypedefs.h>

#include "qc_common.cuh"
#include "qc_api_internal.h"

namespace qc {

constexpr int kHeadDigits = 7;
constexpr int kHeadSliceWarps = 8;

__host__ __device__ inline size_t a16(size_t x) { return (x + 15) & ~size_t(15); }
static size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

// ------------------------------------------------------------------ layouts
struct HeadPrepLayout {   // one-time weight side
  size_t bstack;            // B_d codes stacked [kHeadDigits N][ldb], ldb = a16(kHeadDigits K):
                            // row d N + n = [E_d .. E_0] of column n (zero padded)
  size_t csum;              // s32 [kHeadDigits][N]
  size_t cstat;             // f64 [N][8]: certificate column factors (head_prep_cols)
  size_t wt;                // f32 [N][K] (W^T for the exact fallback)
  size_t ones;              // f64 [N] = 1.0 (w_scale), s32 [N] = 64 (w_zero) after it
  size_t zeros64;
  size_t total;
};

static HeadPrepLayout prep_layout(int K, int N) {
  HeadPrepLayout L{};
  size_t off = 0;
  L.bstack = off;
  off = a256(off + (size_t)kHeadDigits * N * a16((size_t)kHeadDigits * K));
  L.csum = off;
  off = a256(off + (size_t)4 * kHeadDigits * N);
  L.cstat = off;
  off = a256(off + (size_t)8 * 8 * N);
  L.wt = off;
  off = a256(off + (size_t)4 * N * K);
  L.ones = off;
  off = a256(off + (size_t)8 * kHeadDigits * N);
  L.zeros64 = off;
  off = a256(off + (size_t)4 * kHeadDigits * N);
  L.total = off;
  return L;
}

struct HeadWsLayout {     // per call
  size_t planes;  // u8 [M][ldp], ldp = a16(kHeadDigits K)
  size_t rsum;    // s32 [kHeadDigits][M] (prefix over planes)
  size_t rstat;   // f64 [M][8]: certificate row factors (head_slice_rows)
  size_t acc;     // s32 [M][kHeadDigits N] (diagonal d at columns d N ..)
  size_t list;    // s32 [M*N] flagged elements (i*N + j)
  size_t count;   // s32
  size_t one;     // f64 1.0, s32 64
  size_t total;
};

static HeadWsLayout ws_layout(long long M, int K, int N) {
  HeadWsLayout L{};
  size_t off = 0;
  L.planes = off;
  off = a256(off + (size_t)M * a16((size_t)kHeadDigits * K));
  L.rsum = off;
  off = a256(off + (size_t)4 * kHeadDigits * M);
  L.rstat = off;
  off = a256(off + (size_t)8 * 8 * M);
  L.acc = off;
  off = a256(off + (size_t)4 * kHeadDigits * M * N);
  L.list = off;
  off = a256(off + (size_t)4 * M * N);
  L.count = off;
  off = a256(off + 4);
  L.one = off;
  off = a256(off + 16);
  L.total = off;
  return L;
}

// Balanced base-128 digits of r in (-1, 1): r = sum_s D_s 2^(-6-7s) + rest,
// |D_s| <= 64, |rest| <= 2^-(6 + 7 kHeadDigits) / 2.  Every step is exact in f64.
QC_DEV void head_digits(double r, int (&D)[kHeadDigits]) {
  double v = r * 64.0;
#pragma unroll
  for (int s = 0; s < kHeadDigits; ++s) {
    const double q = (v + 6755399441055744.0) - 6755399441055744.0;   // rint, |v| <= 64
    D[s] = (int)q;
    v = (v - q) * 128.0;
  }
}

QC_DEV double up(double v) { return v * (1.0 + 0x1p-40); }   // generous upward padding

// 2^n as f64 for |n| < 1000 (exact, no library call)
QC_DEV double pow2(int n) { return __longlong_as_double((long long)(1023 + n) << 52); }

// max|v| -> exponent e with max|v| < 2^e (0 for an all-zero vector)
QC_DEV int head_exponent(double amax) {
  if (amax == 0.0) return 0;
  int e;
  frexp(amax, &e);   // amax = m 2^e, m in [0.5, 1)
  return e;
}

// ------------------------------------------------------------------ weights
// One warp per output column j (one-time, strided column reads are fine).
__global__ void head_prep_cols(const float* __restrict__ w, int K, int N, uint8_t* base,
                               HeadPrepLayout L) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= N) return;
  const int j = warp;
  double amax = 0.0, l1 = 0.0, l2 = 0.0;
  float* wt = reinterpret_cast<float*>(base + L.wt) + (size_t)j * K;
  for (int k = lane; k < K; k += 32) {
    const float v = w[(size_t)k * N + j];
    wt[k] = v;
    const double a = fabs((double)v);
    amax = fmax(amax, a);
    l1 += a;
    l2 += a * a;
  }
  for (int o = 16; o > 0; o >>= 1) {
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    l2 += __shfl_xor_sync(0xffffffffu, l2, o);
  }
  const int f = head_exponent(amax);
  int cs[kHeadDigits] = {0, 0, 0, 0, 0, 0, 0};
  double sq[kHeadDigits] = {0, 0, 0, 0, 0, 0, 0};
  for (int k = lane; k < K; k += 32) {
    int E[kHeadDigits];
    head_digits((double)w[(size_t)k * N + j] * pow2(-f), E);
#pragma unroll
    for (int t = 0; t < kHeadDigits; ++t) {
      cs[t] += E[t] + 64;
      sq[t] += (double)(E[t] * E[t]);
    }
    const size_t ldb = a16((size_t)kHeadDigits * K);
#pragma unroll
    for (int d = 0; d < kHeadDigits; ++d) {
      uint8_t* bd = base + L.bstack + ((size_t)d * N + j) * ldb;
#pragma unroll
      for (int t = 0; t <= d; ++t) bd[(size_t)(d - t) * K + k] = (uint8_t)(E[t] + 64);
    }
  }
#pragma unroll
  for (int t = 0; t < kHeadDigits; ++t)
    for (int o = 16; o > 0; o >>= 1) {
      cs[t] += __shfl_xor_sync(0xffffffffu, cs[t], o);
      sq[t] += __shfl_xor_sync(0xffffffffu, sq[t], o);
    }
  double rho = 0.0;   // max over digit planes t >= 1 of |E_t|_2 (exact integer sums)
#pragma unroll
  for (int t = 1; t < kHeadDigits; ++t) rho = fmax(rho, sq[t]);
  if (lane == 0) {
    int* csum = reinterpret_cast<int*>(base + L.csum);
    int pre = 0;
    for (int d = 0; d < kHeadDigits; ++d) {
      pre += cs[d];   // B_d holds E_0..E_d
      csum[(size_t)d * N + j] = pre;
    }
    // certificate column factors (see head_combine): 2^f, |E|_2 2^f, |w|_1, 2^(f-49), |w|_2
    double* cst = reinterpret_cast<double*>(base + L.cstat) + (size_t)j * 8;
    cst[0] = pow2(f);
    cst[1] = up(sqrt(rho)) * pow2(f);
    cst[2] = up(l1);
    cst[3] = pow2(f - 49);
    cst[4] = up(sqrt(l2));
    cst[5] = cst[6] = cst[7] = 0.0;
    for (int d = 0; d < kHeadDigits; ++d) {
      reinterpret_cast<double*>(base + L.ones)[(size_t)d * N + j] = 1.0;
      reinterpret_cast<int*>(base + L.zeros64)[(size_t)d * N + j] = 64;
    }
  }
}

// ------------------------------------------------------------------ per call
struct HeadRows {
  const float* x;
  long long ldx;
  const long long* x_row0;   // nullable: first x row per segment
  int seg_rows, seg_valid, K;
  long long M;
};

// One warp per output row i: statistics, digits, planes, prefix rowsums.
__global__ void __launch_bounds__(32 * kHeadSliceWarps)
    head_slice_rows(const HeadRows h, uint8_t* ws, HeadWsLayout L) {
  pdl_wait();
  pdl_trigger();
  const long long i = (long long)blockIdx.x * kHeadSliceWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= h.M) return;
  const int K = h.K;
  const size_t ldp = a16((size_t)kHeadDigits * K);
  uint8_t* prow = ws + L.planes + (size_t)i * ldp;
  int* rsum = reinterpret_cast<int*>(ws + L.rsum);
  double* rst = reinterpret_cast<double*>(ws + L.rstat) + (size_t)i * 8;
  const int seg = (int)(i / h.seg_rows), r = (int)(i - (long long)seg * h.seg_rows);
  if (r >= h.seg_valid) {   // padding row: zero digits
    for (int k = lane; k < kHeadDigits * K; k += 32) prow[k] = 64;
    if (lane == 0) {
      for (int d = 0; d < kHeadDigits; ++d) rsum[(size_t)d * h.M + i] = 64 * (d + 1) * K;
      for (int u = 0; u < 8; ++u) rst[u] = 0.0;
    }
    return;
  }
  const float* xr = h.x + ((h.x_row0 ? h.x_row0[seg] : (long long)seg * h.seg_rows) + r) * h.ldx;
  double amax = 0.0, l1 = 0.0, l2 = 0.0;
  for (int k = lane; k < K; k += 32) {
    const double a = fabs((double)xr[k]);
    amax = fmax(amax, a);
    l1 += a;
    l2 += a * a;
  }
  for (int o = 16; o > 0; o >>= 1) {
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    l2 += __shfl_xor_sync(0xffffffffu, l2, o);
  }
  const int e = head_exponent(amax);
  int cs[kHeadDigits] = {0, 0, 0, 0, 0, 0, 0};
  int sq[kHeadDigits] = {0, 0, 0, 0, 0, 0, 0};   // per-lane sum D^2 <= 36 * 4096: fits
  const double sc = pow2(-e);
  // 4 consecutive k per lane -> one 32-bit store per plane (K % 4 == 0)
  for (int k0 = 4 * lane; k0 < K; k0 += 128) {
    uint32_t pk[kHeadDigits] = {0, 0, 0, 0, 0, 0, 0};
    const float4 x4 = *reinterpret_cast<const float4*>(xr + k0);
    const float xv[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int D[kHeadDigits];
      head_digits((double)xv[u] * sc, D);
#pragma unroll
      for (int s = 0; s < kHeadDigits; ++s) {
        pk[s] |= (uint32_t)(D[s] + 64) << (8 * u);
        cs[s] += D[s] + 64;
        sq[s] += D[s] * D[s];
      }
    }
#pragma unroll
    for (int s = 0; s < kHeadDigits; ++s)
      *reinterpret_cast<uint32_t*>(prow + (size_t)s * K + k0) = pk[s];
  }
#pragma unroll
  for (int s = 0; s < kHeadDigits; ++s)
    for (int o = 16; o > 0; o >>= 1) {
      cs[s] += __shfl_xor_sync(0xffffffffu, cs[s], o);
      sq[s] += __shfl_xor_sync(0xffffffffu, sq[s], o);
    }
  int rho = 0;   // max over digit planes s >= 1 of |D_s|_2^2 (<= 4096 K)
#pragma unroll
  for (int s = 1; s < kHeadDigits; ++s) rho = max(rho, sq[s]);
  if (lane == 0) {
    int pre = 0;
    for (int d = 0; d < kHeadDigits; ++d) {
      pre += cs[d];
      rsum[(size_t)d * h.M + i] = pre;
    }
    // certificate row factors (see head_combine)
    const double Kd = (double)K;
    rst[0] = pow2(e - 12);
    rst[1] = 6.04 * up(sqrt((double)rho)) * pow2(e - 61);
    rst[2] = pow2(e - 49);
    rst[3] = up(l1) + Kd * pow2(e - 49);
    rst[4] = (double)kHeadDigits * pow2(e - 65);
    rst[5] = (Kd - 1.0) * 0x1p-53 * up(sqrt(l2));
    rst[6] = rst[7] = 0.0;
  }
}

struct HeadCombine {
  long long M;
  int N, K, seg_rows, seg_valid;
  const double* rstat;
  const double* cstat;
  const int* acc;   // [kHeadDigits][M][N]
  const float* bias;
  float* out;
  long long ldo;
  const long long* out_row0;   // nullable
  int* list;
  int* count;
};

// 4 consecutive columns per thread over kCombineRows rows.  With the per-row
// (r*) and per-column (c*) factors prepared by the slicing kernels:
//   S^ = s r0 c0 with s = sum_d acc_d 2^-7d             (r0 c0 = 2^(e+f-12), exact)
//   T1 = r1 c1      dropped pairs: 6.04 |D|_2 |E|_2 2^(e+f-61)  (Cauchy-Schwarz)
//   T2 = r2 c2 + r3 c3    truncation: 2^(e-49) |w|_1 + 2^(f-49) (|x|_1 + K 2^(e-49))
//   T3 = r4 c0 (|acc_0| + 65 K)    combination: 7 2^(e+f-65) sum_d |acc_d| 2^-7d
//   T4 = r5 c4      the reference's rounding: (K-1) 2^-53 |x|_2 |w|_2
constexpr int kCombineRows = 16;   // rows per thread (column factors stay in registers)

__global__ void __launch_bounds__(128) head_combine(const HeadCombine c) {
  pdl_wait();
  pdl_trigger();
  const int j0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (j0 >= c.N) return;
  // the thread's 4 columns: certificate factors once
  double c0[4], c1[4], c2[4], c3[4], c4[4];
  float bj[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const double* cf = c.cstat + (size_t)(j0 + u) * 8;
    c0[u] = cf[0];
    c1[u] = cf[1];
    c2[u] = cf[2];
    c3[u] = cf[3];
    c4[u] = cf[4];
    bj[u] = c.bias ? c.bias[j0 + u] : 0.0f;
  }
  const size_t ldacc = (size_t)kHeadDigits * c.N;
  const double k65 = 65.0 * (double)c.K;
  const long long i_end = min((long long)(blockIdx.y + 1) * kCombineRows, c.M);
  for (long long i = (long long)blockIdx.y * kCombineRows; i < i_end; ++i) {
    const int seg = (int)(i / c.seg_rows), r = (int)(i - (long long)seg * c.seg_rows);
    if (r >= c.seg_valid) continue;
    const size_t base = (size_t)i * ldacc + j0;
    int4 a4[kHeadDigits];
#pragma unroll
    for (int d = 0; d < kHeadDigits; ++d)
      a4[d] = __ldcs(reinterpret_cast<const int4*>(c.acc + base + (size_t)d * c.N));
    const double* rf = c.rstat + i * 8;
    const double r0 = rf[0], r1 = rf[1], r2 = rf[2], r3 = rf[3], r4 = rf[4], r5 = rf[5];
    const long long orow = c.out_row0 ? c.out_row0[seg] + r : i;
    float res[4];
    bool all_ok = true;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      double s = 0.0;
#pragma unroll
      for (int d = kHeadDigits - 1; d >= 0; --d) {   // small terms first
        const int av = u == 0 ? a4[d].x : u == 1 ? a4[d].y : u == 2 ? a4[d].z : a4[d].w;
        s = fma(i2d_alu(av), pow2(-7 * d), s);   // exact products, rounded sums (T3)
      }
      const int a0 = u == 0 ? a4[0].x : u == 1 ? a4[0].y : u == 2 ? a4[0].z : a4[0].w;
      const double S = (s * r0) * c0[u];
      const double E = (r1 * c1[u] + r2 * c2[u] + r3 * c3[u] +
                        r4 * c0[u] * (fabs(i2d_alu(a0)) + k65) + r5 * c4[u]) * (1.0 + 0x1p-20);
      const double aS = fabs(S);
      bool ok = aS < 0x1p126 && aS > 0x1p-125;
      float y = 0.0f;
      if (ok) {
        y = __double2float_rn(S);
        const uint32_t yb = __float_as_uint(y);
        const float dn = __uint_as_float(y > 0.0f ? yb - 1u : yb + 1u);   // toward -inf
        const float upn = __uint_as_float(y > 0.0f ? yb + 1u : yb - 1u);  // toward +inf
        const double lo = 0.5 * ((double)y + (double)dn);
        const double hi = 0.5 * ((double)y + (double)upn);
        ok = (S - E > lo) && (S + E < hi);
      }
      if (ok) {
        res[u] = c.bias ? __fadd_rn(y, bj[u]) : y;
      } else {
        all_ok = false;
        res[u] = 0.0f;
        const int slot = atomicAdd(c.count, 1);
        c.list[slot] = (int)(i * c.N + j0 + u);
      }
    }
    float* op = c.out + orow * c.ldo + j0;
    if (all_ok && ((reinterpret_cast<uintptr_t>(op) & 15) == 0)) {
      *reinterpret_cast<float4*>(op) = make_float4(res[0], res[1], res[2], res[3]);
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) op[u] = res[u];   // flagged ones are rewritten by the fallback
    }
  }
}

struct HeadFallback {
  const float* x;
  long long ldx;
  const long long* x_row0;
  int seg_rows, N, K;
  const float* wt;   // [N][K]
  const float* bias;
  float* out;
  long long ldo;
  const long long* out_row0;
  const int* list;
  const int* count;
  int* total;   // nullable running total of exact recomputations
};

// The reference's ascending-k f64 FMA chain for the listed elements.
__global__ void __launch_bounds__(256) head_fallback(const HeadFallback h) {
  pdl_wait();
  pdl_trigger();
  const int n = *h.count;
  if (h.total && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(h.total, n);
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const long long idx = h.list[t];
    const long long i = idx / h.N;
    const int j = (int)(idx - i * h.N);
    const int seg = (int)(i / h.seg_rows), r = (int)(i - (long long)seg * h.seg_rows);
    const float* xr = h.x + ((h.x_row0 ? h.x_row0[seg] : (long long)seg * h.seg_rows) + r) * h.ldx;
    const float* wr = h.wt + (size_t)j * h.K;
    double s = 0.0;
    // ascending k in batches of 16 through a register ring of kFbDepth batches:
    // each batch's 16-byte loads are issued kFbDepth batches ahead of its FMAs
    // (K % 4 == 0, rows 16-byte aligned)
    constexpr int kFbDepth = 4;
    float4 xq[kFbDepth][4], wq[kFbDepth][4];
#pragma unroll
    for (int b = 0; b < kFbDepth; ++b)
      if (16 * b + 16 <= h.K) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          xq[b][u] = __ldg(reinterpret_cast<const float4*>(xr + 16 * b) + u);
          wq[b][u] = __ldg(reinterpret_cast<const float4*>(wr + 16 * b) + u);
        }
      }
    int k = 0;
    for (; k + 16 * kFbDepth <= h.K; k += 16 * kFbDepth) {
#pragma unroll
      for (int b = 0; b < kFbDepth; ++b) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          s = fma((double)xq[b][u].x, (double)wq[b][u].x, s);
          s = fma((double)xq[b][u].y, (double)wq[b][u].y, s);
          s = fma((double)xq[b][u].z, (double)wq[b][u].z, s);
          s = fma((double)xq[b][u].w, (double)wq[b][u].w, s);
        }
        const int kn = k + 16 * (b + kFbDepth);
        if (kn + 16 <= h.K) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            xq[b][u] = __ldg(reinterpret_cast<const float4*>(xr + kn) + u);
            wq[b][u] = __ldg(reinterpret_cast<const float4*>(wr + kn) + u);
          }
        }
      }
    }
    // full batches left in the ring, then the scalar tail
#pragma unroll
    for (int b = 0; b < kFbDepth; ++b)
      if (k + 16 <= h.K) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          s = fma((double)xq[b][u].x, (double)wq[b][u].x, s);
          s = fma((double)xq[b][u].y, (double)wq[b][u].y, s);
          s = fma((double)xq[b][u].z, (double)wq[b][u].z, s);
          s = fma((double)xq[b][u].w, (double)wq[b][u].w, s);
        }
        k += 16;
      }
    for (; k < h.K; ++k) s = fma((double)xr[k], (double)wr[k], s);
    const float y = __double2float_rn(s);
    const long long orow = h.out_row0 ? h.out_row0[seg] + r : i;
    h.out[orow * h.ldo + j] = h.bias ? __fadd_rn(y, h.bias[j]) : y;
  }
}

int head_prep_launch(const float* w, int K, int N, void* prep, cudaStream_t st) {
  const HeadPrepLayout L = prep_layout(K, N);
  cudaMemsetAsync(prep, 0, L.total, st);   // code padding beyond K stays 0 (never read)
  const int threads = 256;
  head_prep_cols<<<(N * 32 + threads - 1) / threads, threads, 0, st>>>(
      w, K, N, reinterpret_cast<uint8_t*>(prep), L);
  return launch_status();
}

int head_gemm_launch(const QcbHeadGemm* g, cudaStream_t st) {
  const int K = g->K, N = g->N;
  const long long M = (long long)g->nseg * g->seg_rows;
  const HeadPrepLayout P = prep_layout(K, N);
  const HeadWsLayout W = ws_layout(M, K, N);
  uint8_t* prep = reinterpret_cast<uint8_t*>(const_cast<void*>(g->prep));
  uint8_t* ws = reinterpret_cast<uint8_t*>(g->workspace);
  // constants: a_scale = 1.0, a_zero = 64
  static const double kOne = 1.0;
  static const int k64 = 64;
  cudaMemcpyAsync(ws + W.one, &kOne, 8, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(ws + W.one + 8, &k64, 4, cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(ws + W.count, 0, 4, st);
  HeadRows hr{g->x, g->ldx, g->x_row0, g->seg_rows, g->seg_valid, K, M};
  head_slice_rows<<<(unsigned)((M + kHeadSliceWarps - 1) / kHeadSliceWarps), 32 * kHeadSliceWarps,
                    0, st>>>(hr, ws, W);
  int rc = launch_status();
  if (rc) return rc;
  {   // every digit diagonal in one grouped launch: column group d reduces K_d = (d+1) K
    QcbGemm q{};
    q.M = (int)M;
    q.N = kHeadDigits * N;
    q.K = kHeadDigits * K;
    q.seg_rows = (int)M;
    q.seg_valid = (int)M;
    q.a_codes = ws + W.planes;
    q.lda = (long long)a16((size_t)kHeadDigits * K);
    q.a_scale = reinterpret_cast<const double*>(ws + W.one);
    q.a_zero = reinterpret_cast<const int*>(ws + W.one + 8);
    q.a_rowsum = reinterpret_cast<const int*>(ws + W.rsum);
    q.w_codes = prep + P.bstack;
    q.ldw = (long long)a16((size_t)kHeadDigits * K);
    q.w_scale = reinterpret_cast<const double*>(prep + P.ones);
    q.w_zero = reinterpret_cast<const int*>(prep + P.zeros64);
    q.w_colsum = reinterpret_cast<const int*>(prep + P.csum);
    q.out = reinterpret_cast<float*>(ws + W.acc);
    q.ldo = (long long)kHeadDigits * N;
    q.epilogue = QCB_EPI_ACC;
    if (N % 32 == 0) {
      const GemmGroup grp{N, K, M};
      rc = gemm_u8_launch(&q, st, &grp);
      if (rc) return rc;
    } else {   // no tile width divides N: one launch per diagonal on the same layout
      const long long ldb = q.ldw;
      for (int d = 0; d < kHeadDigits; ++d) {
        QcbGemm qd = q;
        qd.N = N;
        qd.K = (d + 1) * K;
        qd.a_rowsum = reinterpret_cast<const int*>(ws + W.rsum) + (size_t)d * M;
        qd.w_codes = prep + P.bstack + (size_t)d * N * ldb;
        qd.w_scale = reinterpret_cast<const double*>(prep + P.ones) + (size_t)d * N;
        qd.w_zero = reinterpret_cast<const int*>(prep + P.zeros64) + (size_t)d * N;
        qd.w_colsum = reinterpret_cast<const int*>(prep + P.csum) + (size_t)d * N;
        qd.out = reinterpret_cast<float*>(ws + W.acc) + (size_t)d * N;
        rc = gemm_u8_launch(&qd, st);
        if (rc) return rc;
      }
    }
  }
  HeadCombine c{M, N, K, g->seg_rows, g->seg_valid,
                reinterpret_cast<const double*>(ws + W.rstat),
                reinterpret_cast<const double*>(prep + P.cstat),
                reinterpret_cast<const int*>(ws + W.acc), g->bias, g->out, g->ldo, g->out_row0,
                reinterpret_cast<int*>(ws + W.list), reinterpret_cast<int*>(ws + W.count)};
  head_combine<<<dim3((unsigned)((N / 4 + 127) / 128),
                     (unsigned)((M + kCombineRows - 1) / kCombineRows)), 128, 0, st>>>(c);
  rc = launch_status();
  if (rc) return rc;
  HeadFallback fb{g->x, g->ldx, g->x_row0, g->seg_rows, N, K,
                  reinterpret_cast<const float*>(prep + P.wt), g->bias, g->out, g->ldo,
                  g->out_row0, reinterpret_cast<const int*>(ws + W.list),
                  reinterpret_cast<const int*>(ws + W.count), g->fallback_count};
  head_fallback<<<num_sms() * 4, 256, 0, st>>>(fb);
  rc = launch_status();
  if (rc) return rc;
  return launch_status();
}

}  // namespace qc

extern "C" size_t qcb_head_prep_bytes(int K, int N) { return qc::prep_layout(K, N).total; }

extern "C" size_t qcb_head_workspace_bytes(long long M, int K, int N) {
  return qc::ws_layout(M, K, N).total;
}
