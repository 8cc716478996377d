// The noise head out = f32(mm(x, W)) + b (reference model.py:228, `mm` =
// tensor.py:43-60: ascending-k f64 accumulation of exact f32*f32 products),
// on the int8 tensor cores with an exactness certificate.
//
// Digit planes.  Each x row i is scaled by 2^-e_i (max|x_i| < 2^e_i), r = x 2^-e
// in (-1, 1), and split into kHeadDigits = 6 base-256 floor digits, stored as
// u8 codes U_s in [0, 255]:
//   r = (U_0 - 128) 2^-7 + sum_{s>=1} U_s 2^(-7-8s) + tau,   0 <= tau < 2^-47.
// Read with zero point 128 on every plane, B_s = U_s - 128 in [-128, 127] is a
// balanced digit (mean ~0, so the dropped digit pairs stay small) and
//   r = rho + c + tau,  rho = sum_s B_s 2^(-7-8s),  c = 128 sum_{s=1..5} 2^(-7-8s).
// Each W column j likewise (V_t, C_t, sigma, exponent f_j).  Then
//   sum_k r q = sum_d 2^(-14-8d) A_d + c (sum rho + sum sigma) + c^2 K + (tau terms)
// with the diagonal sums A_d = sum_{s+t=d} sum_k B_s C_t.  All six diagonals run
// as ONE grouped tcgen05 u8 GEMM (zero point 128, which it removes exactly):
// column group d has A = [U_0 .. U_d] (a prefix of the row's planes), B_d =
// [V_d .. V_0] per column and K' = (d+1) K; |A_d| <= 6 K 128^2 and the raw code
// sums <= 6 K 255^2 < 2^31.  Against 7 balanced base-128 planes (28 digit pairs)
// this is 21 pairs: a quarter less tensor-core work.  The row and column offset
// terms R_i = c sum rho_i and Q_j = c (sum sigma_j + c K) come from exact integer
// plane sums.
//
// Certificate.  S^ = 2^(e+f) (2^-14 sum_d A_d 2^-8d + R_i + Q_j) (f64) differs
// from the exact sum S by at most T1 (diagonals d >= kHeadDigits dropped) + T2
// (digit truncation) + T3 (f64 rounding of the combination and of R, Q); the
// reference's sequential sum differs from S by at most
// T4 = (K-1) 2^-53 sum|x w| <= (K-1) 2^-53 |x|_2 |w|_2.
// When [S^ - E, S^ + E] (E = T1+T2+T3+T4, padded) holds no f32 rounding
// boundary, RN32(S^) == RN32(reference); other elements are listed and
// recomputed with the reference's ascending-k f64 FMA chain (bit-exact).
#include <cudaTypedefs.h>

#include "qc_common.cuh"
#include "qc_api_internal.h"

namespace qc {

constexpr int kHeadDigits = 6;
constexpr int kZp = 128;   // code zero point of every digit plane
constexpr int kHeadSliceWarps = 8;
// c = sum_{s=1..5} 128 2^(-7-8s) = sum_{s=1..5} 2^-8s;  c 2^40 = 2^32 + 2^24 + 2^16 + 2^8 + 1
constexpr double kC = 4311810305.0 * 0x1p-40;

__host__ __device__ inline size_t a16(size_t x) { return (x + 15) & ~size_t(15); }
static size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

// ------------------------------------------------------------------ layouts
struct HeadPrepLayout {   // one-time weight side
  size_t bstack;            // B_d codes stacked [kHeadDigits N][ldb], ldb = a16(kHeadDigits K):
                            // row d N + n = [V_d .. V_0] of column n (zero padded)
  size_t csum;              // s32 [kHeadDigits][N]: prefix code sums of B_d's row
  size_t cstat;             // f64 [N][8]: certificate column factors (head_prep_cols)
  size_t wt;                // f32 [N][K] (W^T for the exact fallback)
  size_t ones;              // f64 [kHeadDigits N] = 1.0 (w_scale)
  size_t wzero;             // s32 [kHeadDigits N] = 128 (w_zero)
  size_t one;               // f64 1.0 (a_scale), s32 128 (a_zero)
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
  L.wzero = off;
  off = a256(off + (size_t)4 * kHeadDigits * N);
  L.one = off;
  off = a256(off + 16);
  L.total = off;
  return L;
}

struct HeadWsLayout {     // per call
  size_t planes;  // u8 [M][ldp], ldp = a16(kHeadDigits K)
  size_t rsum;    // s32 [kHeadDigits][M]: prefix code sums over planes 0..d
  size_t rstat;   // f64 [M][8]: certificate row factors (head_slice_rows)
  size_t acc;     // s32 [M][kHeadDigits N] (diagonal d at columns d N ..)
  size_t list;    // s32 [M*N] flagged elements (i*N + j)
  size_t count;   // s32
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
  L.total = off;
  return L;
}

// Codes of r in (-1, 1) (see the header).  floor() by a round-down add of a
// magic constant on the FP64 pipe; the integer is the sum's low word (no
// conversion-pipe instructions).  Every step is exact.
QC_DEV void head_digits(double r, int (&U)[kHeadDigits]) {
  constexpr double kM0 = 6755399441055744.0;   // 1.5 2^52: floor for |v| < 2^51
  constexpr double kM1 = 4503599627370496.0;   // 2^52: floor for 0 <= v < 2^52
  double v = r * 128.0;   // (-128, 128)
  double t = __dadd_rd(v, kM0);
  U[0] = __double2loint(t) + kZp;
  v = (v - (t - kM0)) * 256.0;   // [0, 256)
#pragma unroll
  for (int s = 1; s < kHeadDigits; ++s) {
    t = __dadd_rd(v, kM1);
    U[s] = __double2loint(t);
    v = (v - (t - kM1)) * 256.0;
  }
}

// The same codes from the f32 bits on the integer pipe: F = floor(x 2^(47-e))
// (|x| < 2^e, so |F| < 2^47) in two's complement; U_0 = (F >> 40) + 128 is byte 5
// with its sign bit flipped and U_s (s >= 1) is byte 5 - s -- the base-256 floor
// expansion head_digits forms for r = x 2^-e.  Returns F's low 48 bits.
QC_DEV unsigned long long head_fixed(float x, int e) {
  const unsigned b = __float_as_uint(x);
  const int ex = (int)((b >> 23) & 0xFFu);
  const long long m = (long long)((b & 0x7FFFFFu) | (ex ? 0x800000u : 0u));
  // x = +-m 2^(max(ex,1) - 150); sh <= 23 for finite rows (the clamp only keeps a
  // non-finite row's codes defined: its certificate is not finite -> fallback)
  const int sh = max(ex, 1) - 103 - e;
  const long long sm = (b >> 31) ? -m : m;
  const long long f = sh >= 0 ? (long long)((unsigned long long)sm << min(sh, 23))
                                : sm >> min(-sh, 40);   // floor
  return (unsigned long long)f;
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

// sum_k rho_k 2^47 = sum_s (plane sum_s - 128 K) 2^(40-8s): exact in int64
// (|plane sum - 128 K| <= 128 K < 2^20)
QC_DEV long long rho_sum_2p47(const long long (&ps)[kHeadDigits], int K) {
  long long t = 0;
#pragma unroll
  for (int s = 0; s < kHeadDigits; ++s) t += (ps[s] - (long long)kZp * K) << (40 - 8 * s);
  return t;
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
  long long cs[kHeadDigits] = {0, 0, 0, 0, 0, 0};
  long long sq[kHeadDigits] = {0, 0, 0, 0, 0, 0};   // sum (V - 128)^2
  const size_t ldb = a16((size_t)kHeadDigits * K);
  for (int k = lane; k < K; k += 32) {
    int V[kHeadDigits];
    head_digits((double)w[(size_t)k * N + j] * pow2(-f), V);
#pragma unroll
    for (int t = 0; t < kHeadDigits; ++t) {
      cs[t] += V[t];
      sq[t] += (long long)((V[t] - kZp) * (V[t] - kZp));
    }
#pragma unroll
    for (int d = 0; d < kHeadDigits; ++d) {
      uint8_t* bd = base + L.bstack + ((size_t)d * N + j) * ldb;
#pragma unroll
      for (int t = 0; t <= d; ++t) bd[(size_t)(d - t) * K + k] = (uint8_t)V[t];
    }
  }
#pragma unroll
  for (int t = 0; t < kHeadDigits; ++t)
    for (int o = 16; o > 0; o >>= 1) {
      cs[t] += __shfl_xor_sync(0xffffffffu, cs[t], o);
      sq[t] += __shfl_xor_sync(0xffffffffu, sq[t], o);
    }
  long long rho = 0;   // max over digit planes t >= 1 of |C_t|_2^2
#pragma unroll
  for (int t = 1; t < kHeadDigits; ++t) rho = sq[t] > rho ? sq[t] : rho;
  if (lane == 0) {
    int* csum = reinterpret_cast<int*>(base + L.csum);
    long long pre = 0;
    for (int d = 0; d < kHeadDigits; ++d) {
      pre += cs[d];   // B_d holds V_0..V_d
      csum[(size_t)d * N + j] = (int)pre;
    }
    // certificate column factors (see head_combine)
    double* cst = reinterpret_cast<double*>(base + L.cstat) + (size_t)j * 8;
    cst[0] = pow2(f);
    cst[1] = up(sqrt((double)rho)) * pow2(f);
    cst[2] = up(l1);
    cst[3] = pow2(f - 47);
    cst[4] = up(sqrt(l2));
    cst[5] = kC * ((double)rho_sum_2p47(cs, K) * 0x1p-47 + kC * (double)K);   // Q_j
    cst[6] = cst[7] = 0.0;
    for (int d = 0; d < kHeadDigits; ++d) {
      reinterpret_cast<double*>(base + L.ones)[(size_t)d * N + j] = 1.0;
      reinterpret_cast<int*>(base + L.wzero)[(size_t)d * N + j] = kZp;
    }
    if (j == 0) {   // the activation side's scale / zero point (one segment)
      *reinterpret_cast<double*>(base + L.one) = 1.0;
      *reinterpret_cast<int*>(base + L.one + 8) = kZp;
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

// One warp per output row i: statistics, digit codes, planes, prefix code sums.
__global__ void __launch_bounds__(32 * kHeadSliceWarps, 6)
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
  if (r >= h.seg_valid) {   // padding row (never combined): the codes of 0
    for (int k = lane; k < kHeadDigits * K; k += 32) prow[k] = k < K ? kZp : 0;
    if (lane == 0) {
      for (int d = 0; d < kHeadDigits; ++d) rsum[(size_t)d * h.M + i] = kZp * K;
      for (int u = 0; u < 8; ++u) rst[u] = 0.0;
    }
    return;
  }
  const float* xr = h.x + ((h.x_row0 ? h.x_row0[seg] : (long long)seg * h.seg_rows) + r) * h.ldx;
  double amax = 0.0, l1 = 0.0, l2 = 0.0;
#pragma unroll 3
  for (int k = 4 * lane; k < K; k += 128) {
    const float4 x4 = *reinterpret_cast<const float4*>(xr + k);
    const double a0 = fabs((double)x4.x), a1 = fabs((double)x4.y);
    const double a2 = fabs((double)x4.z), a3 = fabs((double)x4.w);
    amax = fmax(amax, fmax(fmax(a0, a1), fmax(a2, a3)));
    l1 += (a0 + a1) + (a2 + a3);
    l2 += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
  }
  for (int o = 16; o > 0; o >>= 1) {
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    l2 += __shfl_xor_sync(0xffffffffu, l2, o);
  }
  const int e = head_exponent(amax);
  int cs[kHeadDigits] = {0, 0, 0, 0, 0, 0};
  int sq[kHeadDigits] = {0, 0, 0, 0, 0, 0};   // sum (U - 128)^2 <= 128^2 K < 2^31
  // 4 consecutive k per lane -> one 32-bit store per plane (K % 4 == 0); the
  // codes are bytes of the fixed-point words (head_fixed), packed by PRMT, and
  // the plane sums / squared balanced norms are byte dot products
  for (int k0 = 4 * lane; k0 < K; k0 += 128) {
    const float4 x4 = *reinterpret_cast<const float4*>(xr + k0);
    const unsigned long long f0 = head_fixed(x4.x, e), f1 = head_fixed(x4.y, e);
    const unsigned long long f2 = head_fixed(x4.z, e), f3 = head_fixed(x4.w, e);
    const uint32_t lo01 = __byte_perm((uint32_t)f0, (uint32_t)f1, 0x5140);   // b0 b0' b1 b1'
    const uint32_t lo23 = __byte_perm((uint32_t)f2, (uint32_t)f3, 0x5140);
    const uint32_t mid01 = __byte_perm((uint32_t)f0, (uint32_t)f1, 0x7362);  // b2 b2' b3 b3'
    const uint32_t mid23 = __byte_perm((uint32_t)f2, (uint32_t)f3, 0x7362);
    const uint32_t top01 = __byte_perm((uint32_t)(f0 >> 32), (uint32_t)(f1 >> 32), 0x5140);
    const uint32_t top23 = __byte_perm((uint32_t)(f2 >> 32), (uint32_t)(f3 >> 32), 0x5140);
    uint32_t pk[kHeadDigits];
    pk[0] = __byte_perm(top01, top23, 0x7632) ^ 0x80808080u;   // byte 5
    pk[1] = __byte_perm(top01, top23, 0x5410);                 // byte 4
    pk[2] = __byte_perm(mid01, mid23, 0x7632);                 // byte 3
    pk[3] = __byte_perm(mid01, mid23, 0x5410);                 // byte 2
    pk[4] = __byte_perm(lo01, lo23, 0x7632);                   // byte 1
    pk[5] = __byte_perm(lo01, lo23, 0x5410);                   // byte 0
#pragma unroll
    for (int s = 0; s < kHeadDigits; ++s) {
      cs[s] = (int)__dp4a(pk[s], 0x01010101u, (unsigned)cs[s]);
      const int bal = (int)(pk[s] ^ 0x80808080u);   // B = U - 128 as s8 lanes
      sq[s] = __dp4a(bal, bal, sq[s]);
      *reinterpret_cast<uint32_t*>(prow + (size_t)s * K + k0) = pk[s];
    }
  }
#pragma unroll
  for (int s = 0; s < kHeadDigits; ++s)
    for (int o = 16; o > 0; o >>= 1) {
      cs[s] += __shfl_xor_sync(0xffffffffu, cs[s], o);
      sq[s] += __shfl_xor_sync(0xffffffffu, sq[s], o);
    }
  int rho = 0;   // max over digit planes s >= 1 of |B_s|_2^2
#pragma unroll
  for (int s = 1; s < kHeadDigits; ++s) rho = max(rho, sq[s]);
  if (lane == 0) {
    long long ps[kHeadDigits], pre = 0;
    for (int d = 0; d < kHeadDigits; ++d) {
      ps[d] = cs[d];
      pre += cs[d];
      rsum[(size_t)d * h.M + i] = (int)pre;   // A = planes 0..d for diagonal d
    }
    // certificate row factors (see head_combine)
    const double Kd = (double)K;
    rst[0] = pow2(e);
    rst[1] = 5.03 * up(sqrt((double)rho)) * pow2(e - 62);
    rst[2] = pow2(e - 47);
    rst[3] = up(l1) + Kd * pow2(e - 47);
    rst[4] = pow2(e - 64);
    rst[5] = (Kd - 1.0) * 0x1p-53 * up(sqrt(l2));
    rst[6] = kC * ((double)rho_sum_2p47(ps, K) * 0x1p-47);   // R_i
    rst[7] = pow2(e - 50);
  }
}

struct HeadCombine {
  long long M;
  int N, K, seg_rows, seg_valid;
  const double* rstat;
  const double* cstat;
  const int* acc;    // [M][kHeadDigits N] diagonal sums A_d (zero points removed)
  const float* bias;
  float* out;
  long long ldo;
  const long long* out_row0;   // nullable
  int* list;
  int* count;
};

// int32 -> f64 on the FP64 pipe: the word under exponent 2^52, biased by 2^31
QC_DEV double i2d_magic(int v) {
  return __hiloint2double(0x43300000, v ^ (int)0x80000000) - 4503601774854144.0;
}

// kCombineCols consecutive columns per thread over kCombineRows rows.  With the per-row
// (r*) and per-column (c*) factors prepared by the slicing kernels:
//   S^ = ((2^-14 s + R_i) + Q_j) r0 c0,  s = sum_d A_d 2^-8d,  r0 c0 = 2^(e+f)
//   T1 = r1 c1      dropped pairs (s, t >= 1, s + t >= 6; 5 + 4 2^-8 + ... <= 5.03 of
//                   weight 2^-62): 5.03 |B|_2 |C|_2 2^(e+f-62)   (Cauchy-Schwarz)
//   T2 = r2 c2 + r3 c3    truncation: 2^(e-47) |w|_1 + 2^(f-47) (|x|_1 + K 2^(e-47))
//   T3 = c0 (r4 (|A_0| + 130 K) + r7 (|R_i| + |Q_j|))    combination: six FMA
//                   roundings of at most 2^-53 sum_d |A_d| 2^-8d (sum_{d>=1} <= 16384 K
//                   (2 2^-8 + 3 2^-16 + ...) < 129 K), two more adds, and R, Q
//                   (each within 2^-51 relative): <= 2^(e+f) (2^-64 (|A_0| + 130 K)
//                   + 2^-50 (|R| + |Q|))
//   T4 = r5 c4      the reference's rounding: (K-1) 2^-53 |x|_2 |w|_2
// The nearest f32 rounding boundary of S^ is the midpoint T of its f32 bracket
// (bits: low 29 cleared, bit 28 set) as long as E < 2^-26 |S^| (the next
// boundary is >= 2^27 ulp64 away): accept when |S^ - T| > E (exact subtraction).
constexpr int kCombineRows = 16;   // rows per thread (column factors stay in registers)
constexpr int kCombineCols = 2;    // consecutive columns per thread (int2 loads)

__global__ void __launch_bounds__(256) head_combine(const HeadCombine c) {
  pdl_wait();
  pdl_trigger();
  const int j0 = (blockIdx.x * blockDim.x + threadIdx.x) * kCombineCols;
  if (j0 >= c.N) return;
  // the thread's columns: certificate factors once
  double c0[kCombineCols], c1[kCombineCols], c2[kCombineCols], c3[kCombineCols],
      c4[kCombineCols], qj[kCombineCols];
  float bj[kCombineCols];
#pragma unroll
  for (int u = 0; u < kCombineCols; ++u) {
    const double* cf = c.cstat + (size_t)(j0 + u) * 8;
    c0[u] = cf[0];
    c1[u] = cf[1];
    c2[u] = cf[2];
    c3[u] = cf[3];
    c4[u] = cf[4];
    qj[u] = cf[5];
    bj[u] = c.bias ? c.bias[j0 + u] : 0.0f;
  }
  const size_t ldacc = (size_t)kHeadDigits * c.N;
  const double k130 = 130.0 * (double)c.K;
  const long long i0 = (long long)blockIdx.y * kCombineRows;
  const long long i_end = min(i0 + kCombineRows, c.M);
  // the next row's six diagonal sums are in flight while this row is combined
  int2 nx[kHeadDigits];
  auto load_row = [&](long long i, int2 (&dst)[kHeadDigits]) {
    const size_t base = (size_t)i * ldacc + j0;
#pragma unroll
    for (int d = 0; d < kHeadDigits; ++d)
      dst[d] = __ldcs(reinterpret_cast<const int2*>(c.acc + base + (size_t)d * c.N));
  };
  if (i0 < i_end) load_row(i0, nx);
  for (long long i = i0; i < i_end; ++i) {
    int2 a2[kHeadDigits];
#pragma unroll
    for (int d = 0; d < kHeadDigits; ++d) a2[d] = nx[d];
    if (i + 1 < i_end) load_row(i + 1, nx);
    const int seg = (int)(i / c.seg_rows), r = (int)(i - (long long)seg * c.seg_rows);
    if (r >= c.seg_valid) continue;
    const double* rf = c.rstat + i * 8;
    const double r0 = rf[0], r1 = rf[1], r2 = rf[2], r3 = rf[3], r4 = rf[4], r5 = rf[5];
    const double ri = rf[6], r7 = rf[7];
    const long long orow = c.out_row0 ? c.out_row0[seg] + r : i;
    float res[kCombineCols];
    bool all_ok = true;
#pragma unroll
    for (int u = 0; u < kCombineCols; ++u) {
      double s = 0.0;
#pragma unroll
      for (int d = kHeadDigits - 1; d >= 0; --d) {   // small terms first
        const int av = u == 0 ? a2[d].x : a2[d].y;
        s = fma(i2d_magic(av), pow2(-8 * d), s);   // exact products, rounded sums (T3)
      }
      const int a0 = u == 0 ? a2[0].x : a2[0].y;
      const double S = ((fma(s, 0x1p-14, ri) + qj[u]) * r0) * c0[u];
      const double E = (r1 * c1[u] + r2 * c2[u] + r3 * c3[u] + r5 * c4[u] +
                        c0[u] * (r4 * (fabs(i2d_magic(a0)) + k130) +
                                 r7 * (fabs(ri) + fabs(qj[u])))) * (1.0 + 0x1p-20);
      const double aS = fabs(S);
      const long long sb = __double_as_longlong(S);
      const double T = __longlong_as_double((sb & ~0x1FFFFFFFLL) | 0x10000000LL);
      const bool ok = aS < 0x1p126 && aS > 0x1p-125 && E < aS * 0x1p-26 && fabs(S - T) > E;
      if (ok) {
        const float y = __double2float_rn(S);
        res[u] = c.bias ? __fadd_rn(y, bj[u]) : y;
      } else {
        all_ok = false;
        res[u] = 0.0f;
        const int slot = atomicAdd(c.count, 1);
        c.list[slot] = (int)(i * c.N + j0 + u);
      }
    }
    float* op = c.out + orow * c.ldo + j0;
    if (all_ok && ((reinterpret_cast<uintptr_t>(op) & 7) == 0)) {
      *reinterpret_cast<float2*>(op) = make_float2(res[0], res[1]);
    } else {
#pragma unroll
      for (int u = 0; u < kCombineCols; ++u) op[u] = res[u];   // flagged: rewritten by the fallback
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

// The reference's ascending-k f64 FMA chain for the listed elements.  A warp
// takes 32 listed elements (one chain per lane).  Their x / W^T row segments of
// kFbChunk k are staged into shared memory by cp.async (one coalesced
// 128-byte row segment per 8 lanes and instruction, double-buffered), and
// each lane then runs its chain from its own staged rows (LDS.128,
// bank-conflict free with the padded stride).  Per-lane streaming of private
// rows instead costs one L1 wavefront per lane and instruction.
constexpr int kFbWarps = 8;
constexpr int kFbChunk = 32;                 // k per stage
constexpr int kFbStride = kFbChunk + 4;      // floats per staged row

struct FbSmem {
  float buf[kFbWarps][2][2][32][kFbStride];  // [warp][stage][x | w][element][k]
  const float* ptr[kFbWarps][2][32];         // [warp][x | w][element] row pointers
};

QC_DEV void cp_async16(void* dst, const void* src, bool full) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(full ? 16 : 0)
               : "memory");
}
QC_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
QC_DEV void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

__global__ void __launch_bounds__(32 * kFbWarps) head_fallback(const HeadFallback h) {
  extern __shared__ __align__(16) uint8_t fb_smem[];
  FbSmem& sm = *reinterpret_cast<FbSmem*>(fb_smem);
  pdl_wait();
  pdl_trigger();
  const int n = *h.count;
  if (h.total && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(h.total, n);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = h.K;
  const int nchunks = (K + kFbChunk - 1) / kFbChunk;
  for (int base = (blockIdx.x * kFbWarps + warp) * 32; base < n;
       base += gridDim.x * kFbWarps * 32) {
    const int t = base + lane;
    const bool act = t < n;
    const long long idx = h.list[act ? t : base];
    const long long i = idx / h.N;
    const int j = (int)(idx - i * h.N);
    const int seg = (int)(i / h.seg_rows), r = (int)(i - (long long)seg * h.seg_rows);
    __syncwarp();   // the previous group's staged rows are consumed
    sm.ptr[warp][0][lane] =
        h.x + ((h.x_row0 ? h.x_row0[seg] : (long long)seg * h.seg_rows) + r) * h.ldx;
    sm.ptr[warp][1][lane] = h.wt + (size_t)j * K;
    __syncwarp();
    // stage chunk c: lane group g = lane / 8 copies row segments of elements
    // g, g + 4, ...
    auto stage = [&](int c) {
      const int k0 = c * kFbChunk;
      const int kk = 4 * (lane & 7);
      const bool ok = k0 + kk < K;
      for (int e = lane >> 3; e < 32; e += 4) {
        const float* px = sm.ptr[warp][0][e];
        const float* pw = sm.ptr[warp][1][e];
        cp_async16(&sm.buf[warp][c & 1][0][e][kk], ok ? px + k0 + kk : px, ok);
        cp_async16(&sm.buf[warp][c & 1][1][e][kk], ok ? pw + k0 + kk : pw, ok);
      }
      cp_async_commit();
    };
    stage(0);
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) {
      if (c + 1 < nchunks) stage(c + 1);
      else cp_async_commit();   // an empty group keeps wait_group(1) uniform
      cp_async_wait1();
      __syncwarp();             // every lane's copies of chunk c have landed
      const float* xs = sm.buf[warp][c & 1][0][lane];
      const float* ws = sm.buf[warp][c & 1][1][lane];
      const int kn = min(kFbChunk, K - c * kFbChunk);
      if (kn == kFbChunk) {
#pragma unroll
        for (int kk = 0; kk < kFbChunk; kk += 4) {
          const float4 a4 = *reinterpret_cast<const float4*>(xs + kk);
          const float4 b4 = *reinterpret_cast<const float4*>(ws + kk);
          s = fma((double)a4.x, (double)b4.x, s);
          s = fma((double)a4.y, (double)b4.y, s);
          s = fma((double)a4.z, (double)b4.z, s);
          s = fma((double)a4.w, (double)b4.w, s);
        }
      } else {
        for (int kk = 0; kk < kn; ++kk) s = fma((double)xs[kk], (double)ws[kk], s);
      }
      __syncwarp();             // buffer c & 1 is refilled by stage(c + 2)
    }
    if (act) {
      const float y = __double2float_rn(s);
      const long long orow = h.out_row0 ? h.out_row0[seg] + r : i;
      h.out[orow * h.ldo + j] = h.bias ? __fadd_rn(y, h.bias[j]) : y;
    }
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
    q.a_scale = reinterpret_cast<const double*>(prep + P.one);
    q.a_zero = reinterpret_cast<const int*>(prep + P.one + 8);
    q.a_rowsum = reinterpret_cast<const int*>(ws + W.rsum);
    q.w_codes = prep + P.bstack;
    q.ldw = (long long)a16((size_t)kHeadDigits * K);
    q.w_scale = reinterpret_cast<const double*>(prep + P.ones);
    q.w_zero = reinterpret_cast<const int*>(prep + P.wzero);
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
        qd.w_zero = reinterpret_cast<const int*>(prep + P.wzero) + (size_t)d * N;
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
  // threads per block: a multiple of 32 dividing the column groups when one
  // exists (no idle tail block), else 128
  const int quads = N / kCombineCols;
  int cb = 128;
  for (int t = 256; t >= 64; t -= 32)
    if (quads % t == 0) {
      cb = t;
      break;
    }
  head_combine<<<dim3((unsigned)((quads + cb - 1) / cb),
                     (unsigned)((M + kCombineRows - 1) / kCombineRows)), cb, 0, st>>>(c);
  rc = launch_status();
  if (rc) return rc;
  HeadFallback fb{g->x, g->ldx, g->x_row0, g->seg_rows, N, K,
                  reinterpret_cast<const float*>(prep + P.wt), g->bias, g->out, g->ldo,
                  g->out_row0, reinterpret_cast<const int*>(ws + W.list),
                  reinterpret_cast<const int*>(ws + W.count), g->fallback_count};
  static bool fb_attr = false;
  if (!fb_attr) {
    if (cudaFuncSetAttribute(head_fallback, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(FbSmem)) != cudaSuccess)
      return QCB_ERR_CUDA;
    fb_attr = true;
  }
  head_fallback<<<num_sms(), 32 * kFbWarps, sizeof(FbSmem), st>>>(fb);
  rc = launch_status();
  if (rc) return rc;
  return launch_status();
}

}  // namespace qc

extern "C" size_t qcb_head_prep_bytes(int K, int N) { return qc::prep_layout(K, N).total; }

extern "C" size_t qcb_head_workspace_bytes(long long M, int K, int N) {
  return qc::ws_layout(M, K, N).total;
}
