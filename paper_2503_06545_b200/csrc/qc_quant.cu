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
#include "qc_gelu.cuh"
#include "qc_api_internal.h"

namespace qc {

constexpr int kQThreads = 256;

#include "qc_pairwise.cuh"

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
                         double* red, const PairwisePlan& pl, double* pw_scr) {
  const int K = p.K;
  if (p.prologue == QCB_PRO_NONE) {
    for (int j = threadIdx.x; j < K; j += blockDim.x) hrow[j] = xrow[j];
    __syncthreads();
    return;
  }
  if (p.prologue == QCB_PRO_GELU) {
    for (int j = threadIdx.x; j < K; j += blockDim.x) hrow[j] = gelu_f32_ref(xrow[j]);
    __syncthreads();
    return;
  }
  // mean / variance in numpy's pairwise order (qc_pairwise.cuh) by warp 0
  if (threadIdx.x < 32) {
    const double mean_w = __ddiv_rn(np_pairwise_row<false>(xrow, 0.0, pl, pw_scr, threadIdx.x),
                                    (double)K);
    const double var_w = __ddiv_rn(np_pairwise_row<true>(xrow, mean_w, pl, pw_scr, threadIdx.x),
                                   (double)K);
    if (threadIdx.x == 0) {
      red[0] = mean_w;
      red[1] = var_w;
    }
  }
  __syncthreads();
  const double mean = red[0];
  const double sd = __dsqrt_rn(__dadd_rn(red[1], 1e-5));
  __syncthreads();
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
__global__ void __launch_bounds__(kQThreads)
    act_quant_rows(const ActQuantParams p, const PairwisePlan pl) {
  extern __shared__ __align__(16) uint8_t sm[];
  double* buf = reinterpret_cast<double*>(sm);
  float* hrow = reinterpret_cast<float*>(buf + p.K);
  __shared__ double red[32];
  __shared__ double pw_scr[608];
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

  prologue_row(p, xrow, hrow, red, pl, pw_scr);
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
  pdl_wait();
  pdl_trigger();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) keys[i] = (i & 1) ? 0u : 0xFFFFFFFFu;
}

// ------------------------------------------------------------------ v2 path
// Register FWHT for rotation blocks b = 1024 * WPR (STDiT: K = 1152 -> b = 1024,
// K = 4608 -> b = 4096).  One warp owns 1024 elements of a row:
//   load layout  e = lane + 32 r      (coalesced; r = register 0..31)
//   stages on e bits 5..9 in registers, padded-smem transpose to
//   e = 32 lane + r', stages on bits 0..4 in registers, then WPR-1 cross-warp
//   stages through shared memory for bits 10, 11.
// Pass 1 (LN / GELU prologue, balance, rotation, min/max) stashes xe as f32 so
// pass 2 (codes) does no FP64 transform work.  Divisions take an exact
// reciprocal fast path and fall back to IEEE division within a few ulps of a
// rounding boundary, so results equal the reference's f64 division.

constexpr int kV2Threads = 128;

// true when the f64 value q is close enough to an f32 rounding boundary that a
// multiply-by-reciprocal estimate may round differently from exact division.
QC_DEV bool f64_near_f32_tie(double q) { return f64_near_f32_tie_dev(q); }

// f32(f64(h) / c) (quant.py:164): h * (1/c) is within 2 ulp64 of the exact
// division, so its f32 rounding agrees unless it sits near a tie.
QC_DEV float div_to_f32(float h, double c, double rc) {
  const double q = __dmul_rn((double)h, rc);
  if (f64_near_f32_tie(q)) return __double2float_rn(__ddiv_rn((double)h, c));
  return __double2float_rn(q);
}

// clip(rha(f64(xe)/s) + z, 0, top) (quant.py:113-123).  f32 estimate: |q| <
// 512, so the estimate of |q| + 0.5 is within 2^-14 of the exact value; when
// it is further than 2^-12 from an integer the floor is certain, otherwise the
// reference's f64 sequence is evaluated exactly.
QC_DEV int code_of(float xe, float inv_sf, double s, float z, float top) {
  const float qf = __fmul_rn(xe, inv_sf);
  const float t = __fadd_rn(fabsf(qf), 0.5f);
  float n = floorf(t);
  const float fr = t - n;
  float sgn = qf;
  if (fr < 0x1p-12f || fr > 1.0f - 0x1p-12f) {
    const double q = __ddiv_rn((double)xe, s);
    n = (float)floor(__dadd_rn(fabs(q), 0.5));
    sgn = (float)q;
  }
  float v = __fadd_rn(sgn < 0.0f ? -n : n, z);
  v = fminf(fmaxf(v, 0.0f), top);
  return (int)v;
}

struct AQ2 {
  const double* rc[3];  // 1 / chan_scale (v4: rotation signs folded in, see recip_k)
  float* stash[3];      // xe [nseg*seg_rows][K]
  long long ld_stash;
  int total_rows;       // nseg * seg_valid
};

template <int WPR>
struct V2Smem {
  double xbuf[4][32 * 33];  // per-warp transpose / exchange buffer
  float hbuf[4][1024 + 8 * 32];  // per-warp prologue output (block part + tail)
  double red[4][2];         // cross-warp LN partial sums
  float run_mn[4][3][32];   // per-lane running min / max per output (smem: dynamic o)
  float run_mx[4][3][32];
};

QC_DEV void v2_row_index(const ActQuantParams& p, int gr, int& seg, int& mrow,
                         long long& in_row, long long& out_row) {
  seg = gr / p.seg_valid;
  mrow = gr - seg * p.seg_valid;
  in_row = (p.x_row0 ? p.x_row0[seg] : (long long)seg * p.seg_rows) + mrow;
  out_row = (long long)seg * p.seg_rows + mrow;
}

template <int WPR>
QC_DEV double v2_row_sum(double v, double* red_slot, int rowslot, int part) {
  v = warp_sum(v);
  if (WPR == 1) return v;
  if ((threadIdx.x & 31) == 0) red_slot[part] = v;
  named_bar_sync(1 + rowslot, 32 * WPR);
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < WPR; ++i) t += red_slot[i];
  named_bar_sync(1 + rowslot, 32 * WPR);
  return t;
}

// f32(f32(((x - mean) / sd) * g + b) * scale1 + shift), the LN prologue of
// model.py:137-142 + modulation, via x * (1/sd) with an exact fallback.
// w = u + b with u = xm * (1/sd) * g carrying a few ulp64(u) of error against
// the reference's (xm / sd) * g: w's f32 rounding is certain unless w lies
// within 64 (1 + |u| / |w|) ulp64(w) of an f32 tie (covers cancellation
// without a separate test; w == 0 and the f32 range edges always qualify).
// Integer-only and conservative: |u| / |w| < 2^(e_u - e_w + 1) from the binary
// exponents, so the window is below 2^(7 + max(0, e_u - e_w + 1)) ulp64.
QC_DEV bool ln_near_tie(double w, double u) {
  const uint32_t hw = (uint32_t)__double2hiint(w), lw = (uint32_t)__double2loint(w);
  const int ew = (int)((hw >> 20) & 0x7FFu);
  const int eu = (int)(((uint32_t)__double2hiint(u) >> 20) & 0x7FFu);
  const bool range = (uint32_t)(ew - (1023 - 125)) > 251u;   // outside [-125, 126] (w == 0 too)
  const int sh = 7 + max(0, eu - ew + 1);
  const uint32_t d = (uint32_t)abs((int)(lw & 0x1FFFFFFFu) - (1 << 28));
  return range || sh >= 29 || d < (1u << sh);
}

// rare exact paths, kept out of line so they cost no registers in the hot loops
__device__ __noinline__ float ln_exact(double xm, double sd, double g, double b, float scale1,
                                       float shift) {
  const double vv = __dadd_rn(__dmul_rn(__ddiv_rn(xm, sd), g), b);
  return __fadd_rn(__fmul_rn(__double2float_rn(vv), scale1), shift);
}
__device__ __noinline__ double div_exact_f32(double hd, double c) {
  return (double)__double2float_rn(__ddiv_rn(hd, c));
}

QC_DEV float ln_from_xm(double xm, double sd, double rsd, double g, double b, float scale1,
                        float shift) {
  const double u = __dmul_rn(__dmul_rn(xm, rsd), g);
  const double v = __dadd_rn(u, b);
  double vv;
  if (!ln_near_tie(v, u)) {
    vv = v;
  } else {
    vv = __dadd_rn(__dmul_rn(__ddiv_rn(xm, sd), g), b);
  }
  return __fadd_rn(__fmul_rn(__double2float_rn(vv), scale1), shift);
}
QC_DEV float ln_elem(float x, double mean, double sd, double rsd, double g, double b,
                     float scale1, float shift) {
  return ln_from_xm((double)x - mean, sd, rsd, g, b, scale1, shift);
}

template <int WPR, bool kPow2Scale>
__global__ void __launch_bounds__(kV2Threads) aq2_pass1(const ActQuantParams p, const AQ2 a) {
  constexpr int RPC = 4 / WPR;     // rows per CTA iteration
  constexpr int TPL = 8;           // max tail elements per lane
  extern __shared__ __align__(16) uint8_t v2_smem[];
  V2Smem<WPR>& sm = *reinterpret_cast<V2Smem<WPR>*>(v2_smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rowslot = warp / WPR, part = warp % WPR;
  const int K = p.K, b = p.b;
  const int T = K - b;
  double* xb = sm.xbuf[warp];
  float* hb = sm.hbuf[warp];
  float* mn_s = &sm.run_mn[warp][0][0];   // [o*32 + lane]
  float* mx_s = &sm.run_mx[warp][0][0];
  int cur_seg = -1;
#pragma unroll
  for (int o = 0; o < 3; ++o) { mn_s[o * 32 + lane] = INFINITY; mx_s[o * 32 + lane] = -INFINITY; }

  auto flush = [&](int seg) {
#pragma unroll
    for (int o = 0; o < 3; ++o) {
      if (o >= p.n_out) break;
      float lo = mn_s[o * 32 + lane], hi = mx_s[o * 32 + lane];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, off));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, off));
      }
      if (lane == 0 && hi >= lo) {
        uint32_t* k = p.keys + ((size_t)o * p.nseg + seg) * 2;
        atomicMin(&k[0], f2key(lo));
        atomicMax(&k[1], f2key(hi));
      }
      mn_s[o * 32 + lane] = INFINITY;
      mx_s[o * 32 + lane] = -INFINITY;
    }
  };

  for (int base = blockIdx.x * RPC; base < a.total_rows; base += gridDim.x * RPC) {
    const int gr = base + rowslot;
    const bool active = gr < a.total_rows;   // uniform across the row's warps
    int seg = 0, mrow = 0;
    long long in_row = 0, out_row = 0;
    if (active) v2_row_index(p, gr, seg, mrow, in_row, out_row);
    if (active && seg != cur_seg) {
      if (cur_seg >= 0) flush(cur_seg);
      cur_seg = seg;
    }
    // ---- load this warp's share of the row: e = lane + 32 r, tail t = (i*WPR+part)*32+lane
    {
      const float* xr = p.x + in_row * p.ldx;
      float xv[32], xt[TPL];
#pragma unroll
      for (int r = 0; r < 32; ++r) xv[r] = active ? __ldg(xr + part * 1024 + lane + 32 * r) : 0.f;
#pragma unroll
      for (int i = 0; i < TPL; ++i) {
        const int t = (i * WPR + part) * 32 + lane;
        xt[i] = (active && t < T) ? __ldg(xr + b + t) : 0.f;
      }
      // ---- prologue (model.py:182,189,196 LN+mod; model.py:197 GELU) -> smem
      if (p.prologue == QCB_PRO_LN_MOD) {
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < 32; ++r) s += (double)xv[r];
#pragma unroll
        for (int i = 0; i < TPL; ++i) s += (double)xt[i];
        const double mean = v2_row_sum<WPR>(s, sm.red[rowslot], rowslot, part) / K;
        double v = 0.0;
#pragma unroll
        for (int r = 0; r < 32; ++r) { const double d = (double)xv[r] - mean; v += d * d; }
#pragma unroll
        for (int i = 0; i < TPL; ++i) {
          const int t = (i * WPR + part) * 32 + lane;
          if (t < T) { const double d = (double)xt[i] - mean; v += d * d; }
        }
        const double var = v2_row_sum<WPR>(v, sm.red[rowslot], rowslot, part) / K;
        const double sd = sqrt(var + 1e-5);
        const double rsd = 1.0 / sd;
        // branch-free fast path for the whole slab, exact fix-up after a vote
        uint32_t slow = 0;
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          const int col = part * 1024 + lane + 32 * r;
          const double g = p.ln_g ? (double)__ldg(p.ln_g + col) : 1.0;
          const double bb = p.ln_b ? (double)__ldg(p.ln_b + col) : 0.0;
          const double u = __dmul_rn(__dmul_rn((double)xv[r] - mean, rsd), g);
          const double v = __dadd_rn(u, bb);
          slow |= (uint32_t)ln_near_tie(v, u) << r;
          hb[lane + 32 * r] = __fadd_rn(__fmul_rn(__double2float_rn(v), p.scale1), p.shift);
        }
        if (__any_sync(0xffffffffu, slow != 0)) {
#pragma unroll
          for (int r = 0; r < 32; ++r)
            if ((slow >> r) & 1u) {
              const int col = part * 1024 + lane + 32 * r;
              const double g = p.ln_g ? (double)p.ln_g[col] : 1.0;
              const double bb = p.ln_b ? (double)p.ln_b[col] : 0.0;
              hb[lane + 32 * r] = ln_elem(xv[r], mean, sd, rsd, g, bb, p.scale1, p.shift);
            }
        }
#pragma unroll
        for (int i = 0; i < TPL; ++i) {
          const int t = (i * WPR + part) * 32 + lane;
          if (t < T) {
            const double g = p.ln_g ? (double)__ldg(p.ln_g + b + t) : 1.0;
            const double bb = p.ln_b ? (double)__ldg(p.ln_b + b + t) : 0.0;
            hb[1024 + 32 * i + lane] = ln_elem(xt[i], mean, sd, rsd, g, bb, p.scale1, p.shift);
          }
        }
      } else if (p.prologue == QCB_PRO_GELU) {
#pragma unroll
        for (int r = 0; r < 32; ++r) hb[lane + 32 * r] = gelu_f32_ref(xv[r]);
#pragma unroll
        for (int i = 0; i < TPL; ++i) hb[1024 + 32 * i + lane] = gelu_f32_ref(xt[i]);
      } else {
#pragma unroll
        for (int r = 0; r < 32; ++r) hb[lane + 32 * r] = xv[r];
#pragma unroll
        for (int i = 0; i < TPL; ++i) hb[1024 + 32 * i + lane] = xt[i];
      }
    }
    __syncwarp();
    // ---- per output: balance, rotation, min/max, stash
    for (int o = 0; o < p.n_out; ++o) {
      const double* c = p.c[o];
      const double* rc = a.rc[o];
      const uint32_t* sgb = reinterpret_cast<const uint32_t*>(p.signs[o]);
      double w[32];
      if (c) {
        uint32_t slow = 0;
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          const int col = part * 1024 + lane + 32 * r;
          const double q = __dmul_rn((double)hb[lane + 32 * r], __ldg(rc + col));
          slow |= (uint32_t)f64_near_f32_tie(q) << r;
          const float y = __double2float_rn(q);
          w[r] = (double)__uint_as_float(__float_as_uint(y) ^ (__ldg(sgb + col) & 0x80000000u));
        }
        if (__any_sync(0xffffffffu, slow != 0)) {
#pragma unroll
          for (int r = 0; r < 32; ++r)
            if ((slow >> r) & 1u) {
              const int col = part * 1024 + lane + 32 * r;
              const float y = __double2float_rn(__ddiv_rn((double)hb[lane + 32 * r], c[col]));
              w[r] = (double)__uint_as_float(__float_as_uint(y) ^ (sgb[col] & 0x80000000u));
            }
        }
      } else {
#pragma unroll
        for (int r = 0; r < 32; ++r) w[r] = (double)hb[lane + 32 * r];
      }
      float xe[32];
      if (c) {
        // stages on e bits 5..9 (register index bits 0..4)
#pragma unroll
        for (int h = 1; h < 32; h <<= 1)
#pragma unroll
          for (int r = 0; r < 32; ++r)
            if ((r & h) == 0) {
              const double u = w[r], v = w[r + h];
              w[r] = u + v;
              w[r + h] = u - v;
            }
        // transpose e = lane + 32 r  ->  e = 32 lane + r
#pragma unroll
        for (int r = 0; r < 32; ++r) xb[lane + 33 * r] = w[r];
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 32; ++r) w[r] = xb[33 * lane + r];
        __syncwarp();
#pragma unroll
        for (int h = 1; h < 32; h <<= 1)
#pragma unroll
          for (int r = 0; r < 32; ++r)
            if ((r & h) == 0) {
              const double u = w[r], v = w[r + h];
              w[r] = u + v;
              w[r + h] = u - v;
            }
        // cross-warp stages (bits 10, 11)
#pragma unroll
        for (int hbit = 1; hbit < WPR; hbit <<= 1) {
#pragma unroll
          for (int r = 0; r < 32; ++r) xb[33 * lane + r] = w[r];
          named_bar_sync(1 + rowslot, 32 * WPR);
          const double* pb = sm.xbuf[rowslot * WPR + (part ^ hbit)];
          const bool lower = (part & hbit) == 0;
#pragma unroll
          for (int r = 0; r < 32; ++r) {
            const double v = pb[33 * lane + r];
            w[r] = lower ? w[r] + v : v - w[r];
          }
          named_bar_sync(1 + rowslot, 32 * WPR);
        }
        if (kPow2Scale) {   // r = 2^-k exactly: f32(w * r) = f32(w) * r
#pragma unroll
          for (int r = 0; r < 32; ++r) xe[r] = __fmul_rn(__double2float_rn(w[r]), p.rscale);
        } else {
          const double rsc = (double)p.rscale;
#pragma unroll
          for (int r = 0; r < 32; ++r) xe[r] = __double2float_rn(__dmul_rn(w[r], rsc));
        }
      } else {
#pragma unroll
        for (int r = 0; r < 32; ++r) xe[r] = (float)w[r];
      }
      float tl[TPL];
#pragma unroll
      for (int i = 0; i < TPL; ++i) {
        const int t = (i * WPR + part) * 32 + lane;
        const float h = hb[1024 + 32 * i + lane];
        tl[i] = (c && t < T) ? div_to_f32(h, __ldg(c + b + t), __ldg(rc + b + t)) : h;
      }
      if (active) {
        float lo = mn_s[o * 32 + lane], hi = mx_s[o * 32 + lane];
#pragma unroll
        for (int r = 0; r < 32; ++r) { lo = fminf(lo, xe[r]); hi = fmaxf(hi, xe[r]); }
#pragma unroll
        for (int i = 0; i < TPL; ++i) {
          const int t = (i * WPR + part) * 32 + lane;
          if (t < T) { lo = fminf(lo, tl[i]); hi = fmaxf(hi, tl[i]); }
        }
        mn_s[o * 32 + lane] = lo;
        mx_s[o * 32 + lane] = hi;
        float* so = a.stash[o] + out_row * a.ld_stash;
        if (c) {   // rotated layout: this lane owns e = 32 lane + r (contiguous)
          float4* dst = reinterpret_cast<float4*>(so + part * 1024 + 32 * lane);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            dst[j] = make_float4(xe[4 * j], xe[4 * j + 1], xe[4 * j + 2], xe[4 * j + 3]);
        } else {
#pragma unroll
          for (int r = 0; r < 32; ++r) so[part * 1024 + lane + 32 * r] = xe[r];
        }
#pragma unroll
        for (int i = 0; i < TPL; ++i) {
          const int t = (i * WPR + part) * 32 + lane;
          if (t < T) so[b + t] = tl[i];
        }
      }
    }
    __syncwarp();
  }
  if (cur_seg >= 0) flush(cur_seg);
}

// ------------------------------------------------------------------ v3 pass 1
// CTA-level shared-memory FWHT with radix-16 register passes.  256 threads
// handle R = 4096 / b rows at a time; each thread owns 16 f64 values per pass
// (low register use -> several CTAs per SM).  Element e of a row lives at
// smem index e + (e >> 4) (one pad per 16 keeps f64 accesses ~conflict-free).
constexpr int kV3Threads = 256;

QC_DEV int v3_pad(int e) { return e + (e >> 4); }

// Element index of the j-th value (j < 16) of group gi in a pass over bits
// [sh, sh+q): j's low q bits -> bits [sh, sh+q), j's high 4-q bits -> the
// lowest free bits, gi fills the remaining positions in ascending order.
QC_DEV int v3_elem(int gi, int j, int sh, int q, int nbits) {
  const int lo_bits = 4 - q;   // extra "batch" bits taken from the bottom
  int e = ((j & ((1 << q) - 1)) << sh) | (j >> q);
  int g = gi, pos = 0;
  for (int bit = 0; bit < nbits; ++bit) {
    const bool used = (bit >= sh && bit < sh + q) || (bit < lo_bits && !(sh == 0));
    if (used) continue;
    e |= ((g >> pos) & 1) << bit;
    ++pos;
  }
  return e;
}

template <int B>
struct V3Smem {
  static constexpr int R = 4096 / B;
  double f[R][B + B / 16];
  float h[R][2 * B];      // prologue output (K < 2b)
  double red[8];          // LN partial sums, one per warp
  float run_mn[3][kV3Threads / 32];
  float run_mx[3][kV3Threads / 32];
};

template <int B, bool kPow2Scale>
__global__ void __launch_bounds__(kV3Threads) aq3_pass1(const ActQuantParams p, const AQ2 a) {
  constexpr int R = 4096 / B;           // rows per CTA iteration
  constexpr int TPR = kV3Threads / R;   // threads per row (b / 16)
  constexpr int NB = (B == 1024) ? 10 : (B == 2048 ? 11 : 12);
  extern __shared__ __align__(16) uint8_t v3_smem[];
  V3Smem<B>& sm = *reinterpret_cast<V3Smem<B>*>(v3_smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rl = tid / TPR, lt = tid % TPR;   // row slot, thread within the row
  const int K = p.K, T = K - B;
  double* f = sm.f[rl];
  float* h = sm.h[rl];
  int cur_seg = -1;
  for (int o = 0; o < 3; ++o) {
    if (lane == 0) { sm.run_mn[o][warp] = INFINITY; sm.run_mx[o][warp] = -INFINITY; }
  }
  auto flush = [&](int seg) {
    if (lane != 0) return;
    for (int o = 0; o < p.n_out; ++o) {
      const float lo = sm.run_mn[o][warp], hi = sm.run_mx[o][warp];
      if (hi >= lo) {
        uint32_t* k = p.keys + ((size_t)o * p.nseg + seg) * 2;
        atomicMin(&k[0], f2key(lo));
        atomicMax(&k[1], f2key(hi));
      }
      sm.run_mn[o][warp] = INFINITY;
      sm.run_mx[o][warp] = -INFINITY;
    }
  };

  for (int base = blockIdx.x * R; base < a.total_rows; base += gridDim.x * R) {
    const int gr = base + rl;
    const bool active = gr < a.total_rows;
    int seg = 0, mrow = 0;
    long long in_row = 0, out_row = 0;
    if (active) v2_row_index(p, gr, seg, mrow, in_row, out_row);
    if (active && seg != cur_seg) {
      if (cur_seg >= 0) flush(cur_seg);
      cur_seg = seg;
    }
    // ---- load the row (coalesced) + prologue -> h (f32 smem)
    const float* xr = p.x + in_row * p.ldx;
    if (p.prologue == QCB_PRO_LN_MOD) {
      double s = 0.0;
      for (int j = lt; j < K; j += TPR) {
        const float xv = active ? __ldg(xr + j) : 0.f;
        h[j] = xv;
        s += (double)(xv);
      }
      s = warp_sum(s);
      if (lane == 0) sm.red[warp] = s;
      __syncthreads();
      double tot = 0.0;
      for (int w = rl * (TPR / 32); w < (rl + 1) * (TPR / 32); ++w) tot += sm.red[w];
      const double mean = tot / K;
      double v = 0.0;
      for (int j = lt; j < K; j += TPR) {
        const double d = (double)(h[j]) - mean;
        v += d * d;
      }
      v = warp_sum(v);
      __syncthreads();
      if (lane == 0) sm.red[warp] = v;
      __syncthreads();
      double vt = 0.0;
      for (int w = rl * (TPR / 32); w < (rl + 1) * (TPR / 32); ++w) vt += sm.red[w];
      const double sd = sqrt(vt / K + 1e-5);
      const double rsd = 1.0 / sd;
      for (int j = lt; j < K; j += TPR) {
        const double g = p.ln_g ? (double)(__ldg(p.ln_g + j)) : 1.0;
        const double bb = p.ln_b ? (double)(__ldg(p.ln_b + j)) : 0.0;
        h[j] = ln_elem(h[j], mean, sd, rsd, g, bb, p.scale1, p.shift);
      }
    } else if (p.prologue == QCB_PRO_GELU) {
      for (int j = lt; j < K; j += TPR) h[j] = gelu_f32_ref(active ? __ldg(xr + j) : 0.f);
    } else {
      for (int j = lt; j < K; j += TPR) h[j] = active ? __ldg(xr + j) : 0.f;
    }
    __syncthreads();
    for (int o = 0; o < p.n_out; ++o) {
      const double* c = p.c[o];
      const double* rc = a.rc[o];
      const uint32_t* sgb = reinterpret_cast<const uint32_t*>(p.signs[o]);
      float* so = a.stash[o] + out_row * a.ld_stash;
      float lo = INFINITY, hi = -INFINITY;
      if (c) {
        // balance + sign into f (f64), tail straight to the stash
        for (int e = lt; e < B; e += TPR) {
          const double hd = (double)(h[e]);
          const double q = __dmul_rn(hd, __ldg(rc + e));
          // y = f32(h / c) held exactly in f64 (24-bit rounding on the ALU)
          const double y = f64_near_f32_tie(q) ? (double)__double2float_rn(__ddiv_rn(hd, c[e]))
                                               : d_round24(q);
          f[v3_pad(e)] = __longlong_as_double(
              __double_as_longlong(y) ^ ((long long)(__ldg(sgb + e) & 0x80000000u) << 32));
        }
        for (int t = lt; t < T; t += TPR) {
          const double hd = (double)(h[B + t]);
          const double q = __dmul_rn(hd, __ldg(rc + B + t));
          const float y = f64_near_f32_tie(q) ? __double2float_rn(__ddiv_rn(hd, c[B + t]))
                                              : __double2float_rn(q);
          lo = fminf(lo, y);
          hi = fmaxf(hi, y);
          if (active) so[B + t] = y;
        }
        __syncthreads();
        // radix-16 passes over bits [0,4), [4,8), [8, NB)
#pragma unroll
        for (int pass = 0; pass < 3; ++pass) {
          const int sh = 4 * pass;
          const int q = (NB - sh) < 4 ? (NB - sh) : 4;
          double v[16];
          int idx[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            idx[j] = v3_pad(v3_elem(lt, j, sh, q, NB));
            v[j] = f[idx[j]];
          }
#pragma unroll
          for (int hs = 1; hs < 16; hs <<= 1) {
            if (hs >= (1 << q)) break;
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if ((j & hs) == 0) {
                const double u = v[j], w = v[j + hs];
                v[j] = u + w;
                v[j + hs] = u - w;
              }
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) f[idx[j]] = v[j];
          __syncthreads();
        }
        // scale, min/max, coalesced stash write
        for (int e = lt; e < B; e += TPR) {
          const double v = f[v3_pad(e)];
          const float xe = kPow2Scale ? __fmul_rn(__double2float_rn(v), p.rscale)
                                      : __double2float_rn(__dmul_rn(v, (double)p.rscale));
          lo = fminf(lo, xe);
          hi = fmaxf(hi, xe);
          if (active) so[e] = xe;
        }
      } else {
        for (int e = lt; e < K; e += TPR) {
          const float y = h[e];
          lo = fminf(lo, y);
          hi = fmaxf(hi, y);
          if (active) so[e] = y;
        }
      }
      // per-warp running min/max (all lanes of a warp serve the same row)
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, off));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, off));
      }
      if (lane == 0 && active) {
        sm.run_mn[o][warp] = fminf(sm.run_mn[o][warp], lo);
        sm.run_mx[o][warp] = fmaxf(sm.run_mx[o][warp], hi);
      }
      __syncthreads();   // f reused by the next output
    }
  }
  if (cur_seg >= 0) flush(cur_seg);
}

// ------------------------------------------------------------------ v4 pass 1
// Streaming register-first FWHT.  Each of the R = 4096 / b row slots of a CTA
// is served by TPR = b / 16 threads and walks its own sequence of rows; the
// slot's next row is in flight as a 1-D bulk async copy (TMA engine) into
// the slot's shared-memory row, so HBM reads overlap the FP64 work.  Row slots synchronise only among themselves (named barriers).
// Thread lt of a slot owns, per radix-16 stage:
//   stage A (bits NB-4..NB-1): e = lt + TPR j           (from the smem row)
//   stage B (bits 0..3):       e = 16 lt + j
//   stage C (bits 4..NB-5):    e = (lt & 15) + 16 jj + 16 GS top,
//                              top = (lt >> 4) + (TPR / 16) g
// so every shared access is lane-consecutive (conflict-free) and the final
// registers store coalesced runs of xe.  Element e lives at f[e + (e >> 4)].
constexpr int kV4Threads = 256;
constexpr int kV4Tail = 4;   // max tail elements (K - b) per thread
// Input rows in flight per slot.  One suffices: a row is read into registers
// right after it lands, and computing it takes far longer than the next
// row's HBM latency; the smaller footprint allows 3 CTAs per SM.
constexpr int kV4Bufs = 1;

template <int B>
struct V4Smem {
  static constexpr int R = 4096 / B;
  static constexpr int kRowMax = B + kV4Tail * (B / 16);
  float xrow[R][kV4Bufs][kRowMax];  // input row ring per slot (bulk copies)
  double f[R][B + B / 16];        // FWHT work row
  uint64_t full[R][kV4Bufs];       // bulk-copy completion barriers
  double red[2][kV4Threads / 32]; // LN partial sums (mean, variance)
};

// element e of a bf16 row held in a float-typed shared buffer, widened (exact)
QC_DEV float bf16_at(const float* row, int e) {
  return __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(row)[e] << 16);
}

// Radix-2^Q butterflies over groups of 2^Q consecutive registers.
template <int Q>
QC_DEV void fwht_regs(double (&v)[16]) {
#pragma unroll
  for (int hs = 1; hs < (1 << Q); hs <<= 1)
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if ((j & hs) == 0) {
        const double u = v[j], w = v[j + hs];
        v[j] = u + w;
        v[j + hs] = u - w;
      }
}

QC_DEV double flip_sign(double x, uint32_t bit) {
  return __longlong_as_double(__double_as_longlong(x) ^ ((long long)bit << 63));
}

// kPro: the prologue compiled in (0 none, 1 LN + modulation, 2 GELU), so each
// variant gets its own register allocation.
template <int B, bool kPow2Scale, int kMinCtas, int kPro>
__global__ void __launch_bounds__(kV4Threads, kMinCtas)
    aq4_pass1(const ActQuantParams p, const AQ2 a, const PairwisePlan pl) {
  pdl_wait();   // x rows / keys come from the preceding kernels
  pdl_trigger();
  constexpr int R = 4096 / B;               // row slots per CTA
  constexpr int TPR = B / 16;               // threads per row slot
  constexpr int WPR = TPR / 32;             // warps per row slot (>= 2)
  constexpr int NB = (B == 1024) ? 10 : (B == 2048 ? 11 : 12);
  constexpr int Q = NB - 8;                 // bits of stage C
  constexpr int GS = 1 << Q;                // stage-C group size
  constexpr int G = 16 / GS;                // stage-C groups per thread
  constexpr int SA = 17 * TPR / 16;         // stage-A smem stride
  extern __shared__ __align__(128) uint8_t v4_smem[];
  V4Smem<B>& sm = *reinterpret_cast<V4Smem<B>*>(v4_smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rl = tid / TPR, lt = tid % TPR;
  const int K = p.K, T = K - B;
  // kPro 3: bf16 input rows (the attention output), widened exactly to f32
  const uint32_t row_bytes = (uint32_t)K * (kPro == 3 ? 2u : 4u);
  double* const fa = sm.f[rl] + lt + (lt >> 4);
  double* const fb = sm.f[rl] + 17 * lt;
  double* const fc = sm.f[rl] + (lt & 15) + 17 * GS * (lt >> 4);
  auto row_sync = [&]() { named_bar_sync(1 + rl, TPR); };
  // LN affine parameters as f64, once per CTA (dynamic tail of the smem block)
  double* const ln_g64 = reinterpret_cast<double*>(v4_smem + sizeof(V4Smem<B>));
  double* const ln_b64 = ln_g64 + K;
  if (kPro == 1) {
    for (int i = tid; i < K; i += kV4Threads) {
      ln_g64[i] = p.ln_g ? (double)p.ln_g[i] : 1.0;
      ln_b64[i] = p.ln_b ? (double)p.ln_b[i] : 0.0;
    }
  }

  // per-thread running min / max per output (registers; o is 0..2)
  float mn0 = INFINITY, mn1 = INFINITY, mn2 = INFINITY;
  float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY;
  // input rows stream through L2 (evict first); the stash should survive in L2
  // until pass 2 reads it (evict last)
  const uint64_t pol_stream = l2_policy_evict_first();
  const uint64_t pol_keep = l2_policy_evict_last();
  // the slot's k-th row
  const int stride_rows = gridDim.x * R;
  auto row_of = [&](int k) { return blockIdx.x * R + k * stride_rows + rl; };
  auto issue = [&](int k) {   // lt == 0 only
    const int gr = row_of(k);
    if (gr >= a.total_rows) return;
    int seg, mrow;
    long long in_row, out_row;
    v2_row_index(p, gr, seg, mrow, in_row, out_row);
    mbar_arrive_expect_tx(&sm.full[rl][k % kV4Bufs], row_bytes);
    bulk_load_hint(sm.xrow[rl][k % kV4Bufs],
                   kPro == 3 ? static_cast<const void*>(reinterpret_cast<const uint16_t*>(p.x) +
                                                        in_row * p.ldx)
                             : static_cast<const void*>(p.x + in_row * p.ldx),
                   row_bytes,
                   &sm.full[rl][k % kV4Bufs],
                   pol_stream);
  };
  if (lt == 0) {
    for (int i = 0; i < kV4Bufs; ++i) mbar_init(&sm.full[rl][i], 1);
    fence_barrier_init();
    for (int i = 0; i < kV4Bufs; ++i) issue(i);
  }
  __syncthreads();

  auto flush = [&](int seg) {   // warp-level: running min/max -> the segment's keys
    for (int o = 0; o < p.n_out; ++o) {
      float lo = o == 0 ? mn0 : (o == 1 ? mn1 : mn2);
      float hi = o == 0 ? mx0 : (o == 1 ? mx1 : mx2);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, off));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, off));
      }
      if (lane == 0 && hi >= lo) {
        uint32_t* k = p.keys + ((size_t)o * p.nseg + seg) * 2;
        atomicMin(&k[0], f2key(lo));
        atomicMax(&k[1], f2key(hi));
      }
    }
    mn0 = mn1 = mn2 = INFINITY;
    mx0 = mx1 = mx2 = -INFINITY;
  };
  auto slot_sum = [&](double v, double* red) {   // sum over the slot's warps
    v = warp_sum(v);
    if (lane == 0) red[warp] = v;
    row_sync();
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < WPR; ++w) t += red[rl * WPR + w];
    return t;
  };

  int cur_seg = -1;
  for (int k = 0;; ++k) {
    const int gr = row_of(k);
    if (gr >= a.total_rows) break;   // uniform per slot
    int seg, mrow;
    long long in_row, out_row;
    v2_row_index(p, gr, seg, mrow, in_row, out_row);
    if (seg != cur_seg) {
      if (cur_seg >= 0) flush(cur_seg);
      cur_seg = seg;
    }
    // ---- row from shared memory + prologue, in registers
    mbar_wait(&sm.full[rl][k % kV4Bufs], (k / kV4Bufs) & 1);
    const float* xs = sm.xrow[rl][k % kV4Bufs];
    float h[16], ht[kV4Tail];
#pragma unroll
    for (int j = 0; j < 16; ++j) h[j] = kPro == 3 ? bf16_at(xs, lt + TPR * j) : xs[lt + TPR * j];
#pragma unroll
    for (int i = 0; i < kV4Tail; ++i) {
      const int t = lt + TPR * i;
      ht[i] = (t < T) ? (kPro == 3 ? bf16_at(xs, B + t) : xs[B + t]) : 0.f;
    }
    if (kPro == 1) {
      // mean and variance in numpy's pairwise order (qc_pairwise.cuh) by the
      // slot's threads on the row in shared memory, the FWHT work row as scratch
      const double mean = __ddiv_rn(
          np_pairwise_group<false>(xs, 0.0, pl, sm.f[rl], lt, TPR, row_sync), (double)K);
      const double var = __ddiv_rn(
          np_pairwise_group<true>(xs, mean, pl, sm.f[rl], lt, TPR, row_sync), (double)K);
      const double sd = __dsqrt_rn(__dadd_rn(var, 1e-5));
#pragma unroll
      for (int i = 0; i < 16; ++i) fa[SA * i] = __dsub_rn((double)h[i], mean);   // x - mean
      const double rsd = 1.0 / sd;
      // fast path x*(1/sd) for all 16, one sticky flag; exact division only
      // for elements next to an f32 tie or with cancellation (ln_from_xm)
      uint32_t lslow = 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int col = lt + TPR * j;
        const double u = __dmul_rn(__dmul_rn(fa[SA * j], rsd), ln_g64[col]);
        const double w = __dadd_rn(u, ln_b64[col]);
        lslow |= (uint32_t)ln_near_tie(w, u) << j;
        h[j] = __fadd_rn(__fmul_rn(__double2float_rn(w), p.scale1), p.shift);
      }
      if (lslow) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if ((lslow >> j) & 1u) {
            const int col = lt + TPR * j;
            h[j] = ln_exact(fa[SA * j], sd, ln_g64[col], ln_b64[col], p.scale1, p.shift);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < kV4Tail; ++i) {
        const int t = lt + TPR * i;
        if (t < T)
          ht[i] = ln_elem(ht[i], mean, sd, rsd, ln_g64[B + t], ln_b64[B + t], p.scale1, p.shift);
      }
    } else if (kPro == 2) {
      // f32(gelu_f64(x)) (model.py:197): the branch-free certified phase A on
      // 8-element groups; the exact-erfc phase B, then the cephes replica, only
      // for what phase A cannot certify (qc_gelu.cuh)
      uint32_t hard = 0;
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        float a8[8], y8[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) a8[j] = h[8 * g + j];
        const uint32_t hg = gelu_phase_a8(a8, y8, 0xFFu);
        hard |= hg << (8 * g);
#pragma unroll
        for (int j = 0; j < 8; ++j) h[8 * g + j] = ((hg >> j) & 1u) ? a8[j] : y8[j];
      }
      if (hard) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if ((hard >> j) & 1u) {
            float yv;
            if (!gelu_fast_b(h[j], yv)) yv = gelu_f32_ref(h[j]);
            h[j] = yv;
          }
      }
#pragma unroll
      for (int i = 0; i < kV4Tail; ++i) {
        if (lt + TPR * i < T) {
          float yv;
          if (!gelu_fast_a(ht[i], yv) && !gelu_fast_b(ht[i], yv)) yv = gelu_f32_ref(ht[i]);
          ht[i] = yv;
        }
      }
    }
    // every thread of the slot has read the smem row: refill it with row k+2
    row_sync();
    if (lt == 0) issue(k + kV4Bufs);

    for (int o = 0; o < p.n_out; ++o) {
      const double* c = p.c[o];
      float* so = a.stash[o] + out_row * a.ld_stash;
      float lo = INFINITY, hi = -INFINITY;
      if (c) {
        const double* rc = a.rc[o];
        // ---- balance (exact f32(h / c), held in f64) + sign, stage A
        double v[16];
        bool slow = false;
#pragma unroll
        for (int j = 0; j < 16; ++j) {   // rc carries the rotation sign
          const double q = __dmul_rn((double)h[j], __ldg(rc + lt + TPR * j));
          slow |= f32_round_risk_z(q);
          v[j] = d_round24_fast(q);
        }
        if (slow) {   // exact IEEE division next to an f32 rounding boundary (rare)
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const double r = __ldg(rc + lt + TPR * j);
            if (f32_round_risk_z(__dmul_rn((double)h[j], r)))
              v[j] = flip_sign(div_exact_f32((double)h[j], c[lt + TPR * j]),
                               r < 0.0);   // rc carries the sign
          }
        }
        fwht_regs<4>(v);
#pragma unroll
        for (int j = 0; j < 16; ++j) fa[SA * j] = v[j];
        // tail (unrotated): y = f32(h / c) straight to the stash
#pragma unroll
        for (int i = 0; i < kV4Tail; ++i) {
          const int t = lt + TPR * i;
          if (t < T) {
            const double hd = (double)ht[i];
            const double q = __dmul_rn(hd, __ldg(rc + B + t));
            const float y = f64_near_f32_tie(q) ? __double2float_rn(__ddiv_rn(hd, c[B + t]))
                                                : __double2float_rn(q);
            lo = fminf(lo, y);
            hi = fmaxf(hi, y);
            st_f32_hint(so + B + t, y, pol_keep);
          }
        }
        row_sync();
        // ---- stage B (bits 0..3), in place
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = fb[j];
        fwht_regs<4>(v);
#pragma unroll
        for (int j = 0; j < 16; ++j) fb[j] = v[j];
        row_sync();
        // ---- stage C (bits 4..NB-5) -> scale, min/max, stash
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
          for (int jj = 0; jj < GS; ++jj) v[g * GS + jj] = fc[g * (TPR / 16) * 17 * GS + 17 * jj];
        fwht_regs<Q>(v);
        float mn[2] = {lo, INFINITY};   // 2 min/max chains
        float mx[2] = {hi, -INFINITY};
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
          for (int jj = 0; jj < GS; ++jj) {
            const int r = g * GS + jj;
            const double vv = v[r];
            const float x1 = kPow2Scale ? __fmul_rn(__double2float_rn(vv), p.rscale)
                                        : __double2float_rn(__dmul_rn(vv, (double)p.rscale));
            mn[r & 1] = fminf(mn[r & 1], x1);
            mx[r & 1] = fmaxf(mx[r & 1], x1);
            const int e = (lt & 15) + 16 * jj + 16 * GS * ((lt >> 4) + (TPR / 16) * g);
            st_f32_hint(so + e, x1, pol_keep);
          }
        lo = fminf(mn[0], mn[1]);
        hi = fmaxf(mx[0], mx[1]);
        row_sync();   // f is rewritten by the next output / row
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          lo = fminf(lo, h[j]);
          hi = fmaxf(hi, h[j]);
          st_f32_hint(so + lt + TPR * j, h[j], pol_keep);
        }
#pragma unroll
        for (int i = 0; i < kV4Tail; ++i) {
          const int t = lt + TPR * i;
          if (t < T) {
            lo = fminf(lo, ht[i]);
            hi = fmaxf(hi, ht[i]);
            st_f32_hint(so + B + t, ht[i], pol_keep);
          }
        }
      }
      if (o == 0) {
        mn0 = fminf(mn0, lo);
        mx0 = fmaxf(mx0, hi);
      } else if (o == 1) {
        mn1 = fminf(mn1, lo);
        mx1 = fmaxf(mx1, hi);
      } else {
        mn2 = fminf(mn2, lo);
        mx2 = fmaxf(mx2, hi);
      }
    }
  }
  if (cur_seg >= 0) flush(cur_seg);
}

// Pass 2: codes (+ optional dequantized copy) from the f32 stash; warp per row.
// Each lane keeps kP2Batch 16-byte loads in flight; the per-segment (s, z)
// derivation (two f64 divisions) is cached per warp in shared memory.
constexpr int kP2Batch = 4;

__global__ void __launch_bounds__(kV2Threads) aq2_pass2(const ActQuantParams p, const AQ2 a) {
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = p.K;
  const double top = (double)((1 << p.bits) - 1);
  __shared__ int c_seg[kV2Threads / 32][3];
  __shared__ double c_s[kV2Threads / 32][3];
  __shared__ double c_z[kV2Threads / 32][3];
  if (lane < 3) c_seg[warp][lane] = -1;
  __syncwarp();
  for (int gr = blockIdx.x * 4 + warp; gr < a.total_rows; gr += gridDim.x * 4) {
    int seg, mrow;
    long long in_row, out_row;
    v2_row_index(p, gr, seg, mrow, in_row, out_row);
    for (int o = 0; o < p.n_out; ++o) {
      double s, z;
      if (c_seg[warp][o] == seg) {
        s = c_s[warp][o];
        z = c_z[warp][o];
      } else {
        const uint32_t* k = p.keys + ((size_t)o * p.nseg + seg) * 2;
        const double lo = (double)key2f(k[0]), hi = (double)key2f(k[1]);
        const double span = hi - lo;
        if (span <= 0.0) {
          s = 1.0;
          z = 0.0;
        } else {
          s = scale_up16(__ddiv_rn(span, top));
          z = fmin(fmax(rha(__ddiv_rn(-lo, s)), 0.0), top);
        }
        // every warp serving the segment writes the same values
        if (lane == 0) {
          p.scale[o][seg] = s;
          p.zero[o][seg] = (int)z;
          c_s[warp][o] = s;
          c_z[warp][o] = z;
          c_seg[warp][o] = seg;
        }
        __syncwarp();
      }
      const float inv_sf = (float)(1.0 / s);
      const float zf = (float)z, topf = (float)top;
      const int zi = (int)z;
      const float* xr = a.stash[o] + out_row * a.ld_stash;
      uint8_t* cr = p.codes[o] ? p.codes[o] + out_row * p.ldc : nullptr;
      float* dr = p.deq_out[o] ? p.deq_out[o] + out_row * p.ldxe : nullptr;
      int rs = 0;
      auto proc = [&](int j, const float4 t4) {
        const float v4[4] = {t4.x, t4.y, t4.z, t4.w};
        uint32_t packed = 0;
        int code[4];
        bool slow = false;
#pragma unroll
        for (int e = 0; e < 4; ++e) {   // f32 estimate of rha(xe/s), branch-free
          // magic-number rounding (FP32 pipe) instead of FRND/F2I on the XU pipe
          const float qf = __fmul_rn(v4[e], inv_sf);
          const float aq = fabsf(qf);
          const float n = __fsub_rn(__fadd_rn(aq, 12582912.0f), 12582912.0f);  // rint, aq < 2^22
          slow |= fabsf(__fsub_rn(aq, n)) > 0.5f - 0x1p-12f;                   // near a .5 tie
          const float v = fminf(fmaxf(__fadd_rn(qf < 0.0f ? -n : n, zf), 0.0f), topf);
          code[e] = __float_as_int(__fadd_rn(v, 8388608.0f)) - 0x4B000000;    // (int)v in [0, 255]
        }
        if (slow) {
#pragma unroll
          for (int e = 0; e < 4; ++e) code[e] = code_of(v4[e], inv_sf, s, zf, topf);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (j + e < K) {
            rs += code[e];
            packed |= (uint32_t)code[e] << (8 * e);
            if (dr) dr[j + e] = __double2float_rn(__dmul_rn(s, i2d_alu(code[e] - zi)));
          }
        }
        if (cr) {
          if (j + 3 < K) *reinterpret_cast<uint32_t*>(cr + j) = packed;
          else
            for (int e = 0; e < 4 && j + e < K; ++e) cr[j + e] = (uint8_t)(packed >> (8 * e));
        }
      };
      if ((K & 3) == 0 && cr && !dr && (p.ldc & 3) == 0) {
        // hot path: packed f32x2 estimate of clip(rha(xe/s) + z) per float4,
        // one near-tie test per float4, bytes packed with PRMT, row sum by DP4A
        const float2 inv2 = make_float2(inv_sf, inv_sf), z2 = make_float2(zf, zf);
        const float2 mg = make_float2(12582912.0f, 12582912.0f);
        const float2 nmg = make_float2(-12582912.0f, -12582912.0f);
        const float2 m1 = make_float2(-1.0f, -1.0f);
        const float2 b23 = make_float2(8388608.0f, 8388608.0f);
        auto codes2 = [&](float2 x, float& dmax) -> uint32_t {
          const float2 q = __fmul2_rn(x, inv2);
          const float2 n = __fadd2_rn(__fadd2_rn(q, mg), nmg);   // rint(q), |q| < 2^22
          const float2 d = __ffma2_rn(n, m1, q);                  // q - n, exact
          dmax = fmaxf(dmax, fmaxf(fabsf(d.x), fabsf(d.y)));
          float2 v = __fadd2_rn(n, z2);
          v.x = fminf(fmaxf(v.x, 0.0f), topf);
          v.y = fminf(fmaxf(v.y, 0.0f), topf);
          const float2 k = __fadd2_rn(v, b23);                    // code in the low byte
          return __byte_perm(__float_as_uint(k.x), __float_as_uint(k.y), 0x0040);
        };
        for (int j0 = lane * 4; j0 < K; j0 += 128 * kP2Batch) {
          float4 v[kP2Batch];
#pragma unroll
          for (int b = 0; b < kP2Batch; ++b)
            if (j0 + 128 * b < K) v[b] = __ldcs(reinterpret_cast<const float4*>(xr + j0 + 128 * b));
#pragma unroll
          for (int b = 0; b < kP2Batch; ++b) {
            const int j = j0 + 128 * b;
            if (j >= K) break;
            float dmax = 0.0f;
            const uint32_t lo2 = codes2(make_float2(v[b].x, v[b].y), dmax);
            const uint32_t hi2 = codes2(make_float2(v[b].z, v[b].w), dmax);
            uint32_t packed = __byte_perm(lo2, hi2, 0x5410);
            if (dmax > 0.5f - 0x1p-12f) {   // near a .5 tie: the reference's f64 sequence
              const float e4[4] = {v[b].x, v[b].y, v[b].z, v[b].w};
              packed = 0;
#pragma unroll
              for (int e = 0; e < 4; ++e)
                packed |= (uint32_t)code_of(e4[e], inv_sf, s, zf, topf) << (8 * e);
            }
            rs = __dp4a(packed, 0x01010101u, (unsigned)rs);
            *reinterpret_cast<uint32_t*>(cr + j) = packed;
          }
        }
        rs = warp_sum(rs);
        if (lane == 0) p.rowsum[o][out_row] = rs;
        continue;
      }
      for (int j0 = lane * 4; j0 < K; j0 += 128 * kP2Batch) {
        float4 v[kP2Batch];
#pragma unroll
        for (int b = 0; b < kP2Batch; ++b) {
          const int j = j0 + 128 * b;
          if (j + 3 < K) {
            v[b] = __ldcs(reinterpret_cast<const float4*>(xr + j));
          } else {
            v[b].x = (j < K) ? xr[j] : 0.f;
            v[b].y = (j + 1 < K) ? xr[j + 1] : 0.f;
            v[b].z = (j + 2 < K) ? xr[j + 2] : 0.f;
            v[b].w = 0.f;
          }
        }
#pragma unroll
        for (int b = 0; b < kP2Batch; ++b)
          if (j0 + 128 * b < K) proc(j0 + 128 * b, v[b]);
      }
      rs = warp_sum(rs);
      if (lane == 0 && cr) p.rowsum[o][out_row] = rs;
    }
  }
}

// Pass 2, common case (codes only, K % 4 == 0, n_out * nseg <= kP2Pairs): the
// (output, segment) -> (s, z) table is built once per block in shared memory
// while the warp's first row segment is already in flight, and each warp then
// streams its rows as a sequence of (row, output, batch) items with the next
// item's loads issued before the current one is coded.  A persistent grid
// (resident blocks only) lets every warp serve several rows.
constexpr int kP2Pairs = 128;
constexpr int kP2HBatch = 4;   // float4 per lane per item

__global__ void __launch_bounds__(kV2Threads) aq2_pass2_hot(const ActQuantParams p, const AQ2 a) {
  pdl_wait();
  pdl_trigger();
  __shared__ float t_inv[kP2Pairs], t_z[kP2Pairs];
  __shared__ double t_s[kP2Pairs];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = p.K, n_out = p.n_out;
  const float topf = (float)((1 << p.bits) - 1);
  const int nb = (K + 128 * kP2HBatch - 1) / (128 * kP2HBatch);   // items per (row, output)
  const int W = gridDim.x * (kV2Threads / 32);
  const int w = blockIdx.x * (kV2Threads / 32) + warp;
  // the warp's items in order: rows gr = w, w + W, ...; per row the outputs o;
  // per output the batches b of 128 * kP2HBatch columns.  Advanced
  // incrementally (one 32-bit division per new row, none per item).
  int it_gr = w, it_o = 0, it_b = 0, it_seg = 0;
  long long it_orow = 0;
  auto row_setup = [&]() {
    it_seg = it_gr / p.seg_valid;
    it_orow = (long long)it_seg * p.seg_rows + (it_gr - it_seg * p.seg_valid);
  };
  if (it_gr < a.total_rows) row_setup();
  // the current item's stash pointer etc.; false past the warp's last row
  auto item_src = [&](const float*& src, int& jbase, long long& orow, int& o, int& b,
                      int& seg) -> bool {
    if (it_gr >= a.total_rows) return false;
    o = it_o;
    b = it_b;
    seg = it_seg;
    orow = it_orow;
    jbase = lane * 4 + b * 128 * kP2HBatch;
    src = a.stash[o] + orow * a.ld_stash;
    if (++it_b == nb) {
      it_b = 0;
      if (++it_o == n_out) {
        it_o = 0;
        it_gr += W;
        if (it_gr < a.total_rows) row_setup();
      }
    }
    return true;
  };
  auto load_item = [&](const float* src, int jbase, float4 (&v)[kP2HBatch]) {
#pragma unroll
    for (int i = 0; i < kP2HBatch; ++i) {
      const int j = jbase + 128 * i;
      if (j < K) v[i] = __ldcs(reinterpret_cast<const float4*>(src + j));
    }
  };
  float4 cur[kP2HBatch], nxt[kP2HBatch];
  const float* src;
  int jb, o, b, seg;
  long long orow;
  bool have = item_src(src, jb, orow, o, b, seg);
  if (have) load_item(src, jb, cur);
  // (s, z) per (output, segment): quantize's minmax parameters (quant.py:83-123)
  const double top = (double)((1 << p.bits) - 1);
  for (int t = threadIdx.x; t < n_out * p.nseg; t += blockDim.x) {
    const int to = t / p.nseg, ts = t - to * p.nseg;
    const uint32_t* kk = p.keys + ((size_t)to * p.nseg + ts) * 2;
    const double lo = (double)key2f(kk[0]), hi = (double)key2f(kk[1]);
    const double span = hi - lo;
    double sc, z;
    if (span <= 0.0) {
      sc = 1.0;
      z = 0.0;
    } else {
      sc = scale_up16(__ddiv_rn(span, top));
      z = fmin(fmax(rha(__ddiv_rn(-lo, sc)), 0.0), top);
    }
    t_inv[t] = (float)(1.0 / sc);
    t_z[t] = (float)z;
    t_s[t] = sc;
    if (blockIdx.x == 0) {
      p.scale[to][ts] = sc;
      p.zero[to][ts] = (int)z;
    }
  }
  __syncthreads();
  const float2 mg = make_float2(12582912.0f, 12582912.0f);
  const float2 nmg = make_float2(-12582912.0f, -12582912.0f);
  const float2 m1 = make_float2(-1.0f, -1.0f);
  const float2 b23 = make_float2(8388608.0f, 8388608.0f);
  int rs = 0;
  while (have) {
    const float* nsrc;
    int njb, no, nbb, nseg_;
    long long norow;
    const bool nhave = item_src(nsrc, njb, norow, no, nbb, nseg_);
    if (nhave) load_item(nsrc, njb, nxt);
    const int t = o * p.nseg + seg;
    const float inv_sf = t_inv[t], zf = t_z[t];
    const float2 inv2 = make_float2(inv_sf, inv_sf), z2 = make_float2(zf, zf);
    uint8_t* cr = p.codes[o] + orow * p.ldc;
    if (b == 0) rs = 0;
#pragma unroll
    for (int i = 0; i < kP2HBatch; ++i) {
      const int j = jb + 128 * i;
      if (j >= K) break;
      // packed f32x2 estimate of clip(rha(xe/s) + z), one near-tie test per float4
      float dmax = 0.0f;
      auto codes2 = [&](float2 x) -> uint32_t {
        const float2 q = __fmul2_rn(x, inv2);
        const float2 n = __fadd2_rn(__fadd2_rn(q, mg), nmg);   // rint(q), |q| < 2^22
        const float2 d = __ffma2_rn(n, m1, q);                  // q - n, exact
        dmax = fmaxf(dmax, fmaxf(fabsf(d.x), fabsf(d.y)));
        float2 v = __fadd2_rn(n, z2);
        v.x = fminf(fmaxf(v.x, 0.0f), topf);
        v.y = fminf(fmaxf(v.y, 0.0f), topf);
        const float2 kq = __fadd2_rn(v, b23);                   // code in the low byte
        return __byte_perm(__float_as_uint(kq.x), __float_as_uint(kq.y), 0x0040);
      };
      const uint32_t lo2 = codes2(make_float2(cur[i].x, cur[i].y));
      const uint32_t hi2 = codes2(make_float2(cur[i].z, cur[i].w));
      uint32_t packed = __byte_perm(lo2, hi2, 0x5410);
      if (dmax > 0.5f - 0x1p-12f) {   // near a .5 tie: the reference's f64 sequence
        const float e4[4] = {cur[i].x, cur[i].y, cur[i].z, cur[i].w};
        const double sc = t_s[t];
        packed = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e)
          packed |= (uint32_t)code_of(e4[e], inv_sf, sc, zf, topf) << (8 * e);
      }
      rs = __dp4a(packed, 0x01010101u, (unsigned)rs);
      *reinterpret_cast<uint32_t*>(cr + j) = packed;
    }
    if (b == nb - 1) {
      const int tot = warp_sum(rs);
      if (lane == 0) p.rowsum[o][orow] = tot;
    }
#pragma unroll
    for (int i = 0; i < kP2HBatch; ++i) cur[i] = nxt[i];
    have = nhave;
    src = nsrc;
    jb = njb;
    orow = norow;
    o = no;
    b = nbb;
    seg = nseg_;
  }
}

// reciprocal table 1/c; with `signs`, the rotation signs of the first b
// columns are folded in (s_j / c_j), which is what the v4 kernel consumes
__global__ void recip_k(const double* c, const float* signs, int b, double* rc, int K) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= K) return;
  const double r = 1.0 / c[i];
  rc[i] = (signs && i < b && signs[i] < 0.f) ? -r : r;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// codes-only calls that the streaming pass 2 serves
static bool pass2_hot_ok(const qc::ActQuantParams& p, const qc::AQ2& a) {
  bool hot = (p.K & 3) == 0 && (p.ldc & 3) == 0 && p.n_out * p.nseg <= qc::kP2Pairs &&
             a.ld_stash % 4 == 0;
  for (int o = 0; o < p.n_out; ++o)
    if (!p.codes[o] || p.deq_out[o] || (reinterpret_cast<uintptr_t>(p.codes[o]) & 3)) hot = false;
  return hot;
}

// pass 2 launch: the streaming kernel for codes-only calls, else the general one
static void launch_pass2(const qc::ActQuantParams& p, const qc::AQ2& a, cudaStream_t st) {
  const bool hot = pass2_hot_ok(p, a);
  if (hot) {
    static int resident = 0;
    if (!resident) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, qc::aq2_pass2_hot, qc::kV2Threads, 0);
      if (resident < 1) resident = 1;
    }
    int b2 = (a.total_rows + 3) / 4;
    if (b2 > num_sms() * resident) b2 = num_sms() * resident;
    launch_pdl(qc::aq2_pass2_hot, dim3(b2), dim3(qc::kV2Threads), 0, st, p, a);
  } else {
    int b2 = (a.total_rows + 3) / 4;
    if (b2 > num_sms() * 16) b2 = num_sms() * 16;
    launch_pdl(qc::aq2_pass2, dim3(b2), dim3(qc::kV2Threads), 0, st, p, a);
  }
}

}  // namespace qc

extern "C" size_t qcb_act_quant_workspace_bytes(int K, int seg_rows, int nseg, int n_out) {
  return qc::align256((size_t)8 * 3 * nseg) + qc::align256((size_t)8 * 3 * K) +
         (size_t)3 * qc::align256((size_t)4 * K * seg_rows * nseg) + 256;
}

namespace qc {

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
  // the LN prologue's numpy pairwise-sum plan over K (qc_pairwise.cuh)
  PairwisePlan pl{};
  if (q->prologue == QCB_PRO_LN_MOD && !pairwise_plan(q->K, pl)) return QCB_ERR_DIM;
  const int nkeys = 2 * q->n_out * q->nseg;
  launch_pdl(init_keys, dim3((nkeys + 255) / 256), dim3(256), 0, st, p.keys, nkeys);
  // v2: register FWHT for b in {1024, 2048, 4096} with a short tail
  const int wpr = b / 1024;
  const bool v2 = (b == 1024 || b == 2048 || b == 4096) && (q->K - b) <= 8 * 32 * wpr &&
                  (q->K % 4 == 0) && (q->ldx % 4 == 0) && (q->ldc % 4 == 0 || !q->codes[0]);
  if (q->prologue == QCB_PRO_BF16 && !v2) return QCB_ERR_CONFIG;
  if (v2) {
    uint8_t* ws = reinterpret_cast<uint8_t*>(q->workspace);
    size_t off = align256((size_t)8 * 3 * q->nseg);
    AQ2 a{};
    a.total_rows = p.seg_valid * p.nseg;
    double* rcbuf = reinterpret_cast<double*>(ws + off);
    off += align256((size_t)8 * 3 * q->K);
    const size_t stash_bytes = align256((size_t)4 * q->K * q->seg_rows * q->nseg);
    a.ld_stash = q->K;
    // v4 (register-first FWHT): 16-byte aligned rows, short tail; it takes the
    // signed reciprocal table (qcb_weight_prep's chan_recip_out), v3 the plain one
    const bool v4 = (q->K - b) <= kV4Tail * (b / 16) &&
                    (reinterpret_cast<uintptr_t>(q->x) & 15) == 0;
    if (q->prologue == QCB_PRO_BF16 && !v4) return QCB_ERR_CONFIG;
    for (int o = 0; o < q->n_out; ++o) {
      a.rc[o] = rcbuf + (size_t)o * q->K;
      if (q->chan_scale[o] && q->chan_recip[o] && v4) {
        a.rc[o] = q->chan_recip[o];
      } else if (q->chan_scale[o]) {
        recip_k<<<(q->K + 255) / 256, 256, 0, st>>>(q->chan_scale[o], v4 ? q->signs[o] : nullptr,
                                                     b, rcbuf + (size_t)o * q->K, q->K);
      }
      if (q->xe_out[o] && q->ldxe == q->K) {
        a.stash[o] = q->xe_out[o];
      } else {
        a.stash[o] = reinterpret_cast<float*>(ws + off);
        off += stash_bytes;
      }
    }
    const int rpc = 4 / wpr;
    int blocks = (a.total_rows + rpc - 1) / rpc;
    const int cap = num_sms() * 4;
    if (blocks > cap) blocks = cap;
    // pass 1: CTA shared-memory FWHT (v3); 1/sqrt(b) is a power of two for b = 1024, 4096
    (void)blocks;
    static bool at1 = false, at2 = false, at4 = false;
    static bool a41 = false, a42 = false, a44 = false, a41l = false, a42l = false, a44l = false;
    const int rows_per_cta = 4096 / b;
    int b1 = (a.total_rows + rows_per_cta - 1) / rows_per_cta;
    if (b1 > num_sms() * 3) b1 = num_sms() * 3;
    if (v4) {
      // 2 CTAs per SM (128 registers) for every prologue: at 3 CTAs per SM the
      // 85-register cap spills (measured 10-15% slower)
      const bool ln = q->prologue == QCB_PRO_LN_MOD;
      const int pro = ln ? 1 : (q->prologue == QCB_PRO_GELU ? 2 :
                                (q->prologue == QCB_PRO_BF16 ? 3 : 0));
      if (pro == 3 && (b != 1024 || (q->ldx % 8))) return QCB_ERR_CONFIG;
      const size_t ln_bytes = ln ? (size_t)16 * q->K : 0;
      const int cap = num_sms() * 2;
      if (b1 > cap) b1 = cap;
      static bool a41g = false, a42g = false, a44g = false, a41b = false;
      switch (b * 4 + pro) {
#define QC_AQ4(BB, P2, MC, PRO, FLAG)                                                          \
  allow_max_smem(aq4_pass1<BB, P2, MC, PRO>, FLAG);                                            \
  launch_pdl(aq4_pass1<BB, P2, MC, PRO>, dim3(b1), dim3(kV4Threads),                           \
             sizeof(V4Smem<BB>) + ln_bytes, st, p, a, pl);                                     \
  break;
        case 4096: QC_AQ4(1024, true, 2, 0, a41)
        case 4097: QC_AQ4(1024, true, 2, 1, a41l)
        case 4098: QC_AQ4(1024, true, 2, 2, a41g)
        case 4099: QC_AQ4(1024, true, 2, 3, a41b)
        case 8192: QC_AQ4(2048, false, 2, 0, a42)
        case 8193: QC_AQ4(2048, false, 2, 1, a42l)
        case 8194: QC_AQ4(2048, false, 2, 2, a42g)
        case 16384: QC_AQ4(4096, true, 2, 0, a44)
        case 16385: QC_AQ4(4096, true, 2, 1, a44l)
        default: QC_AQ4(4096, true, 2, 2, a44g)
#undef QC_AQ4
      }
    } else switch (b) {
      case 1024:
        allow_max_smem(aq3_pass1<1024, true>, at1);
        aq3_pass1<1024, true><<<b1, kV3Threads, sizeof(V3Smem<1024>), st>>>(p, a);
        break;
      case 2048:
        allow_max_smem(aq3_pass1<2048, false>, at2);
        aq3_pass1<2048, false><<<b1, kV3Threads, sizeof(V3Smem<2048>), st>>>(p, a);
        break;
      default:
        allow_max_smem(aq3_pass1<4096, true>, at4);
        aq3_pass1<4096, true><<<b1, kV3Threads, sizeof(V3Smem<4096>), st>>>(p, a);
        break;
    }
    launch_pass2(p, a, st);
    if (q->xe_out[0] && q->ldxe != q->K) return QCB_ERR_DIM;  // debug copy layout unsupported
    return launch_status();
  }
  const size_t smem = (size_t)q->K * (sizeof(double) + sizeof(float));
  if (smem > 200 * 1024) return QCB_ERR_DIM;
  static bool attr1 = false, attr2 = false;
  allow_max_smem(act_quant_rows<1>, attr1);
  allow_max_smem(act_quant_rows<2>, attr2);
  dim3 grid(p.seg_valid, p.nseg);
  act_quant_rows<1><<<grid, kQThreads, smem, st>>>(p, pl);
  act_quant_rows<2><<<grid, kQThreads, smem, st>>>(p, pl);
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
  double* rc_out;  // nullable [K]: 1/c
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
  if (n == 0 && p.rc_out && p.c)   // signed reciprocal table (see recip_k)
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
      const double r = 1.0 / p.c[k];
      p.rc_out[k] = (k < p.b && p.signs[k] < 0.f) ? -r : r;
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
  p.rc_out = q->chan_recip_out;
  const size_t smem = (size_t)q->K * sizeof(double);
  if (smem > 200 * 1024) return QCB_ERR_DIM;
  static bool attr = false;
  allow_max_smem(weight_prep_cols, attr);
  weight_prep_cols<<<q->N, kQThreads, smem, st>>>(p);
  return launch_status();
}

}  // namespace qc
