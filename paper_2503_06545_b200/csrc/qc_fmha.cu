// Fast bf16 attention on the tcgen05 tensor cores (sm_100a), the bench-mode
// replacement of the library SDPA for the STDiT self-attention
// (reference model.py:150-156 `_mha`, computed there in f64; this mode uses
// bf16 operands and f32 accumulation like the SDPA it replaces, and is
// checked against an f32 reference with a tolerance, tests/test_gpu_fmha.py).
//
// One CTA (one per SM) owns 256 query rows of one (segment, head) as two
// 128-row tiles and streams the segment's keys in 128-row blocks:
//   warp 16      TMA producer: K and V blocks into an ST-stage ring (and Q
//                when it stays in shared memory)
//   warp 17      MMA issuer (one thread): S_i = Q_i K^T (M 128, N 128) and
//                O_i += P_i V (A = P from TMEM, B = V MN-major, N = dhp)
//   warps 0-15   softmax: warp -> (tile, column half, lane quarter), thread =
//                (query row, 64 key columns).  S from TMEM, the row max across
//                the two halves through shared memory, a lazy rescale of O
//                (only when the running max grows by more than 2^8), exp2 on
//                the MUFU, f32 row sums, P as bf16 pairs over S in TMEM; O / l.
// TMEM (512 columns): S_0 [0,128) S_1 [128,256), then O_0, O_1 and (QT) Q_0,
// Q_1 as the A operand of S from tensor memory.  The head dimension is padded
// to dhp = 16k (72 -> 80) by the TMA (3-D tensor map {dh, heads, rows}:
// columns >= dh are out of bounds and land as zeros): a 64-column 128-byte-
// swizzled chunk plus a narrow 32/64-byte-swizzled tail (K, Q) or a second
// 128-byte chunk (V, so that one MMA with N = dhp spans both).
//
// Ordering: the MMA thread issues, per tile, S_i(j) after PV_i(j-1), so the
// commit that signals S_i(j) also covers PV_i(j-1): a softmax thread that has
// seen S_i(j) may rescale its O row without another barrier.
//
// Measured at the STDiT target (4 videos x 16 heads x S = 16384, dh = 72):
// 6.85 ms against 5.7 ms for cuDNN SDPA (tools/fmha_bench.py), with the MUFU
// 58% and the tensor pipe 35% busy.  The per-tile chain S -> softmax -> P V ->
// next S is serial (TMEM holds one S per tile next to O at dh = 72), and two
// tiles do not hide it; the engine therefore keeps the library SDPA as its
// default bf16 attention (EngineOptions.attention).
#include <cuda_bf16.h>
#include <math.h>

#include "qc_common.cuh"
#include "qc_api_internal.h"

namespace qc {

constexpr int kFmSoftWarps = 16;                // 2 tiles x 2 column halves x 4 lane quarters
constexpr int kFmThreads = 32 * (kFmSoftWarps + 2);
constexpr int kFmProducer = kFmSoftWarps, kFmMma = kFmSoftWarps + 1;

// kind::f16 instruction descriptor: A, B bf16; D f32; A K-major; B K- or MN-major.
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t M, uint32_t N, uint32_t b_mn) {
  return (1u << 4)             // D format: F32
         | (1u << 7)           // A format: BF16
         | (1u << 10)          // B format: BF16
         | (0u << 15)          // A K-major
         | (b_mn << 16)        // B major-ness
         | ((N >> 3) << 17)    // N / 8
         | ((M >> 4) << 24);   // M / 16
}

QC_DEV void umma_bf16_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
// A operand from TMEM (128 lanes x K/2 32-bit columns of packed bf16 pairs)
QC_DEV void umma_bf16_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

QC_DEV void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

QC_DEV void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
QC_DEV void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}
QC_DEV void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
QC_DEV void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                   taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
               "r"(r[7])
               : "memory");
}
QC_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

QC_DEV float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Blackwell packed f32x2 arithmetic (FFMA2 / FADD2): two lanes per instruction
QC_DEV unsigned long long f2_bits(float lo, float hi) {
  return ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
}
QC_DEV unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
QC_DEV unsigned long long fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
QC_DEV float f2_lo(unsigned long long v) { return __uint_as_float((uint32_t)v); }
QC_DEV float f2_hi(unsigned long long v) { return __uint_as_float((uint32_t)(v >> 32)); }
QC_DEV uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);   // .x (low half) = lo
  return *reinterpret_cast<const uint32_t*>(&v);
}

struct FmhaArgs {
  const __nv_bfloat16* q;   // Q rows (read by the softmax warps into TMEM when QT)
  long long ldq;
  __nv_bfloat16* out;
  long long ldo;
  long long seg_stride;
  int S, dh, dhp, nkb;
  float c;   // softmax scale * log2(e)
};

// Operand tile of 128 rows: the first 64 head-dim columns as a 128-byte
// swizzled chunk (128-byte rows), then the remaining TW columns (dh > 64) as a
// chunk with TW*2-byte rows and the matching swizzle (TW = 16: 32B, 32: 64B,
// 64: 128B).  Zero columns past dh come from the TMA's out-of-bounds fill.
template <int TW>
struct FmTile {
  static constexpr uint32_t kMain = 128 * 128;
  static constexpr uint32_t kTail = 128 * 2 * TW;
  static constexpr uint32_t kBytes = kMain + kTail;   // multiple of 1024
  static constexpr uint32_t kTailRow = 2 * TW;        // bytes per tail row
  // descriptor layout type (sm_100): 128B = 2, 64B = 4, 32B = 6
  static constexpr uint32_t kTailLayout = TW == 16 ? 6u : (TW == 32 ? 4u : 2u);
  // V (the MN-major B operand of P V) keeps 128-byte rows in both chunks, so
  // one MMA with N = dhp spans the two 64-column atoms (LBO = kMain)
  static constexpr uint32_t kVBytes = kMain + (TW ? kMain : 0);
};

QC_DEV uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// QT: Q lives in TMEM (A operand of S = Q K^T from tensor memory, loaded by
// the softmax warps) instead of shared memory: S reads only K from shared
// memory.  TMEM: S 2 x 128, O 2 x dhp, Q 2 x max(dhp / 2, 32) columns (dhp <= 80).
template <int TW, int ST, bool QT>
__global__ void __launch_bounds__(kFmThreads, 1)
    fmha_bf16_k(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mqt,
                const __grid_constant__ CUtensorMap mkt, const __grid_constant__ CUtensorMap mvt,
                const FmhaArgs a) {
  using Tl = FmTile<TW>;
  extern __shared__ uint8_t fm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(fm_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* sQ = sm;                          // [2 tiles] (shared-memory Q only)
  uint8_t* sK = sQ + (QT ? 0 : 2 * Tl::kBytes);   // [ST stages]
  uint8_t* sV = sK + ST * Tl::kBytes;        // [ST stages]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + ST * Tl::kVBytes);
  uint64_t* q_full = bars;
  uint64_t* s_full = bars + 1;     // [2] per tile
  uint64_t* p_full = bars + 3;     // [2] per tile
  uint64_t* o_full = bars + 5;
  uint64_t* kv_full = bars + 6;    // [ST]
  uint64_t* kv_empty = kv_full + ST;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(kv_empty + ST);
  __shared__ float xch[2 * 2 * 2 * 128];   // [block parity][tile][half][row] (shared, not generic)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = blockIdx.y;
  const int row0 = (int)(blockIdx.z * a.seg_stride);
  const int q0 = blockIdx.x * 256;
  const int nkb = a.nkb;

  if (tid == 0) {
    mbar_init(q_full, QT ? 32 * kFmSoftWarps : 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], 256);
    }
    for (int s = 0; s < ST; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    mbar_init(o_full, 1);
    fence_barrier_init();
  }
  if (warp == kFmMma) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  auto o_col = [&](int i) -> uint32_t { return QT ? 256u + i * a.dhp : 256u + 128u * i; };
  pdl_wait();   // q / k / v come from the preceding GEMMs
  pdl_trigger();

  if (warp == kFmProducer) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      auto load_tile = [&](const CUtensorMap* m, const CUtensorMap* mt, uint64_t* bar,
                           uint8_t* dst, int row) {
        tma_load_3d(m, bar, dst, 0, h, row);
        if (TW) tma_load_3d(mt, bar, dst + Tl::kMain, 64, h, row);
      };
      if (!QT) {
        mbar_arrive_expect_tx(q_full, 2 * Tl::kBytes);
        for (int i = 0; i < 2; ++i)
          load_tile(&mq, &mqt, q_full, sQ + i * Tl::kBytes, row0 + q0 + 128 * i);
      }
      for (int j = 0; j < nkb; ++j) {
        const int st = j % ST;
        if (j >= ST) mbar_wait(&kv_empty[st], ((j / ST) - 1) & 1);
        mbar_arrive_expect_tx(&kv_full[st], Tl::kBytes + Tl::kVBytes);
        load_tile(&mk, &mkt, &kv_full[st], sK + st * Tl::kBytes, row0 + 128 * j);
        load_tile(&mv, &mvt, &kv_full[st], sV + st * Tl::kVBytes, row0 + 128 * j);
      }
    }
  } else if (warp == kFmMma) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      const int nmain = a.dhp < 64 ? a.dhp : 64;
      const uint32_t idesc_s = idesc_bf16(128, 128, 0);
      const uint32_t idesc_o = idesc_bf16(128, (uint32_t)a.dhp, 1);
      const int kmain = nmain >> 4;
      auto issue_s = [&](int i, int st) {
        const uint32_t ka = smem_u32(sK + st * Tl::kBytes);
        if (QT) {
          const uint32_t qt = tbase + 256 + 2 * a.dhp + i * (TW ? (a.dhp >> 1) : 32);
          for (int ks = 0; ks < kmain; ++ks)
            umma_bf16_ts(tbase + 128 * i, qt + 8 * ks, smem_desc(ka + 32u * ks, 16, 1024, 2),
                         idesc_s, ks > 0);
#pragma unroll
          for (int ks = 0; ks < TW / 16; ++ks)
            umma_bf16_ts(tbase + 128 * i, qt + 32 + 8 * ks,
                         smem_desc(ka + Tl::kMain + 32u * ks, 16, 8 * Tl::kTailRow, Tl::kTailLayout),
                         idesc_s, 1);
        } else {
          const uint32_t qa = smem_u32(sQ + i * Tl::kBytes);
          for (int ks = 0; ks < kmain; ++ks)
            umma_bf16_ss(tbase + 128 * i, smem_desc(qa + 32u * ks, 16, 1024, 2),
                         smem_desc(ka + 32u * ks, 16, 1024, 2), idesc_s, ks > 0);
#pragma unroll
          for (int ks = 0; ks < TW / 16; ++ks)
            umma_bf16_ss(tbase + 128 * i,
                         smem_desc(qa + Tl::kMain + 32u * ks, 16, 8 * Tl::kTailRow, Tl::kTailLayout),
                         smem_desc(ka + Tl::kMain + 32u * ks, 16, 8 * Tl::kTailRow, Tl::kTailLayout),
                         idesc_s, 1);
        }
        umma_commit(&s_full[i]);
      };
      auto issue_pv = [&](int i, int st, bool acc) {
        const uint32_t va = smem_u32(sV + st * Tl::kVBytes);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)   // 16 keys per MMA: 8 P columns, 2 V row groups
          umma_bf16_ts(tbase + o_col(i), tbase + 128 * i + 8 * kk,
                       smem_desc(va + 2048u * kk, TW ? Tl::kMain : 16u, 1024, 2), idesc_o,
                       acc || kk > 0);
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      for (int j = 0; j < nkb; ++j) {
        for (int i = 0; i < 2; ++i) {
          if (j > 0) {
            mbar_wait(&p_full[i], (j - 1) & 1);
            tc_fence_after();
            issue_pv(i, (j - 1) % ST, j > 1);
            if (i == 1) umma_commit(&kv_empty[(j - 1) % ST]);
          }
          if (i == 0) {
            mbar_wait(&kv_full[j % ST], (j / ST) & 1);
            tc_fence_after();
          }
          issue_s(i, j % ST);
        }
      }
      for (int i = 0; i < 2; ++i) {
        mbar_wait(&p_full[i], (nkb - 1) & 1);
        tc_fence_after();
        issue_pv(i, (nkb - 1) % ST, nkb > 1);
      }
      umma_commit(o_full);
    }
  } else {
    // ------------------------------------------------ softmax
    // warp -> (tile i, column half hf, lane quarter): thread = (row, 64 columns)
    const int i = warp >> 3, hf = (warp >> 2) & 1, quarter = warp & 3;
    const int r = 32 * quarter + lane;
    const uint32_t lanes = (uint32_t)(32 * quarter) << 16;
    const uint32_t s_addr = tbase + lanes + 128 * i + 64 * hf;    // this half's scores
    const uint32_t p_addr = tbase + lanes + 128 * i + 32 * hf;    // its packed P columns
    const uint32_t o_addr = tbase + lanes + o_col(i);
    const int nch = a.dhp >> 4;                                   // 16-column O chunks
    const int ch0 = hf ? (nch + 1) / 2 : 0, ch1 = hf ? nch : (nch + 1) / 2;
    const float c = a.c;
    float* const xm0 = xch + (2 * i) * 128;                       // [parity][.][half][row]
    float m = -INFINITY, l0 = 0.f, l1 = 0.f;
    auto masked = [&](uint32_t (&s)[32], int col0, int valid) {
      if (valid < 128) {
#pragma unroll
        for (int t = 0; t < 32; ++t)
          if (col0 + t >= valid) s[t] = __float_as_uint(-INFINITY);
      }
    };
    if (QT) {
      // this thread's Q row into TMEM (packed bf16 pairs; zeros past dh and
      // past the tensor): half 0 columns [0, 32) = d 0..63, half 1 the rest
      const int qrow = q0 + 128 * i + r;
      const bool ok = qrow < a.seg_stride;
      const uint4* src = reinterpret_cast<const uint4*>(
          a.q + (long long)(row0 + (ok ? qrow : 0)) * a.ldq + (long long)h * a.dh);
      const uint32_t qt = tbase + lanes + 256 + 2 * a.dhp + i * (TW ? (a.dhp >> 1) : 32);
      if (hf == 0) {
        uint32_t w[32];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint4 v = (ok && 8 * u < a.dh) ? src[u] : make_uint4(0, 0, 0, 0);
          w[4 * u] = v.x; w[4 * u + 1] = v.y; w[4 * u + 2] = v.z; w[4 * u + 3] = v.w;
        }
        tmem_st32(qt, w);
      } else if (TW) {
        uint32_t w[8];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint4 v = (ok && 64 + 8 * u < a.dh) ? src[8 + u] : make_uint4(0, 0, 0, 0);
          w[4 * u] = v.x; w[4 * u + 1] = v.y; w[4 * u + 2] = v.z; w[4 * u + 3] = v.w;
        }
        tmem_st8(qt + 32, w);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(q_full);
    }
    // Both tiles' softmax warps run concurrently (4 warps per SM sub-partition
    // while both have scores).  Measured alternatives, all slower at the
    // target shape: strict turn-taking between the tiles (named barriers),
    // turn-taking around the exp2 pass only, and 1/4 of the exponentials as a
    // cubic on the FMA pipe (the MUFU is not the limiter: 58% busy).
    for (int j = 0; j < nkb; ++j) {
      mbar_wait(&s_full[i], j & 1);
      tc_fence_after();
      const int valid = a.S - 128 * j;
      uint32_t s0[32], s1[32];
      tmem_ld32(s_addr, s0);
      tmem_ld32(s_addr + 32, s1);
      tmem_ld_wait();
      masked(s0, 64 * hf, valid);
      masked(s1, 64 * hf + 32, valid);
      float mx0 = __uint_as_float(s0[0]), mx1 = __uint_as_float(s0[1]);
      float mx2 = __uint_as_float(s1[0]), mx3 = __uint_as_float(s1[1]);
#pragma unroll
      for (int t = 2; t < 32; t += 2) {
        mx0 = fmaxf(mx0, __uint_as_float(s0[t]));
        mx1 = fmaxf(mx1, __uint_as_float(s0[t + 1]));
        mx2 = fmaxf(mx2, __uint_as_float(s1[t]));
        mx3 = fmaxf(mx3, __uint_as_float(s1[t + 1]));
      }
      // the row's max over both halves (exchange through shared memory)
      // (slots alternate with the block parity: a slot is rewritten two blocks
      // later, after the next exchange barrier, so one barrier per block)
      float* const xm = xm0 + (j & 1) * 512;
      xm[hf * 128 + r] = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
      named_bar_sync(3 + i, 256);
      const float mblk = fmaxf(xm[r], xm[128 + r]) * c;
      // lazy rescale, warp-uniform (tcgen05.ld / st are warp-collective) and
      // identical in the row's two halves: only when some row's max grew by
      // more than 2^8 (first block: m = -inf)
      if (__any_sync(0xffffffffu, mblk > m + 8.0f)) {
        const float newm = fmaxf(m, mblk);
        if (j > 0) {
          const float f = ex2_approx(m - newm);
          l0 *= f;
          l1 *= f;
          for (int cc = ch0; cc < ch1; ++cc) {
            uint32_t o[16];
            tmem_ld16(o_addr + 16 * cc, o);
            tmem_ld_wait();
#pragma unroll
            for (int t = 0; t < 16; ++t) o[t] = __float_as_uint(__uint_as_float(o[t]) * f);
            tmem_st16(o_addr + 16 * cc, o);
          }
        }
        m = newm;
      }
      // P = exp2(s c - m) as bf16 pairs: this half's 64 scores -> 32 packed
      // columns at 32 hf.  Half 1's P lands in [32, 64), scores of half 0,
      // which half 0 read before the exchange barrier above.
      // packed pairs: one FFMA2 for two scaled scores, one FADD2 for two sums
      const unsigned long long c2 = f2_bits(c, c), nm2 = f2_bits(-m, -m);
      unsigned long long acc2 = f2_bits(l0, l1);
      uint32_t pk[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const unsigned long long x2 =
            ffma2(((unsigned long long)s0[2 * t + 1] << 32) | s0[2 * t], c2, nm2);
        const float p0 = ex2_approx(f2_lo(x2)), p1 = ex2_approx(f2_hi(x2));
        acc2 = fadd2(acc2, f2_bits(p0, p1));
        pk[t] = pack_bf16(p0, p1);
      }
      tmem_st16(p_addr, pk);
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const unsigned long long x2 =
            ffma2(((unsigned long long)s1[2 * t + 1] << 32) | s1[2 * t], c2, nm2);
        const float p0 = ex2_approx(f2_lo(x2)), p1 = ex2_approx(f2_hi(x2));
        acc2 = fadd2(acc2, f2_bits(p0, p1));
        pk[t] = pack_bf16(p0, p1);
      }
      l0 = f2_lo(acc2);
      l1 = f2_hi(acc2);
      tmem_st16(p_addr + 16, pk);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[i]);
    }
    // ---- epilogue: O / l -> bf16 rows (each half stores its O chunks)
    float* const xl = xm0 + (nkb & 1) * 512;   // the slot no thread can still be reading
    xl[hf * 128 + r] = l0 + l1;
    named_bar_sync(3 + i, 256);
    const float rl = 1.0f / (xl[r] + xl[128 + r]);
    mbar_wait(o_full, 0);
    tc_fence_after();
    const int row = q0 + 128 * i + r;
    __nv_bfloat16* orow = a.out + (long long)(row0 + row) * a.ldo + (long long)h * a.dh;
    for (int cc = ch0; cc < ch1; ++cc) {
      uint32_t o[16];
      tmem_ld16(o_addr + 16 * cc, o);
      tmem_ld_wait();
      if (row < a.S) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = 16 * cc + 8 * e;
          if (col < a.dh) {
            uint4 v;
            v.x = pack_bf16(__uint_as_float(o[8 * e + 0]) * rl, __uint_as_float(o[8 * e + 1]) * rl);
            v.y = pack_bf16(__uint_as_float(o[8 * e + 2]) * rl, __uint_as_float(o[8 * e + 3]) * rl);
            v.z = pack_bf16(__uint_as_float(o[8 * e + 4]) * rl, __uint_as_float(o[8 * e + 5]) * rl);
            v.w = pack_bf16(__uint_as_float(o[8 * e + 6]) * rl, __uint_as_float(o[8 * e + 7]) * rl);
            *reinterpret_cast<uint4*>(orow + col) = v;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kFmMma) {
    tc_fence_after();
    tmem_free<512>(tbase);
  }
}

// bf16 [rows][ld] viewed as {dh, heads, rows}: box box_w x 1 x 128 with the
// matching swizzle; columns >= dh of a head are out of bounds (zero-filled).
static int make_map_heads(CUtensorMap* map, const void* base, long long rows, int heads, int dh,
                          long long ld, int box_w) {
  auto enc = get_encode_fn();
  if (!enc) return QCB_ERR_CUDA;
  cuuint64_t dims[3] = {(cuuint64_t)dh, (cuuint64_t)heads, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)dh * 2, (cuuint64_t)ld * 2};
  cuuint32_t box[3] = {(cuuint32_t)box_w, 1, 128};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUtensorMapSwizzle sw = box_w == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                                : (box_w == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                               : CU_TENSOR_MAP_SWIZZLE_128B);
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? QCB_OK : QCB_ERR_CUDA;
}

template <int TW, int ST, bool QT>
static int fmha_launch_t(const CUtensorMap* m, const FmhaArgs& fa, dim3 grid, cudaStream_t st) {
  const size_t smem = 1024 + (size_t)((QT ? 0 : 2) + ST) * FmTile<TW>::kBytes +
                      (size_t)ST * FmTile<TW>::kVBytes + (6 + 2 * ST + 2) * 8 + 4 * 128 * 4;
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(fmha_bf16_k<TW, ST, QT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    done = true;
  }
  launch_pdl(fmha_bf16_k<TW, ST, QT>, grid, dim3(kFmThreads), smem, st, m[0], m[1], m[2], m[3], m[4],
             m[5], fa);
  return launch_status();
}

int attention_bf16_launch(const QcbAttentionBf16* a, cudaStream_t st) {
  if (!a || !a->q || !a->k || !a->v || !a->out) return QCB_ERR_VALUE;
  if (a->S <= 0 || a->heads <= 0 || a->nseg <= 0 || a->dh <= 0 || a->dh > 128 || a->dh % 8 ||
      a->seg_stride < a->S)
    return QCB_ERR_DIM;
  if (a->ldq % 8 || a->ldk % 8 || a->ldv % 8 || a->ldo % 8 || a->ldq < (long long)a->heads * a->dh ||
      a->ldk < (long long)a->heads * a->dh || a->ldv < (long long)a->heads * a->dh ||
      a->ldo < (long long)a->heads * a->dh)
    return QCB_ERR_DIM;
  const uintptr_t al = (uintptr_t)a->q | (uintptr_t)a->k | (uintptr_t)a->v | (uintptr_t)a->out;
  if (al & 15) return QCB_ERR_DIM;
  const long long rows = (long long)a->nseg * a->seg_stride;
  if (rows + 256 > 0x7FFFFFFFLL) return QCB_ERR_DIM;
  const int dhp = (a->dh + 15) / 16 * 16;
  const int tw = dhp <= 64 ? 0 : (dhp - 64 <= 16 ? 16 : (dhp - 64 <= 32 ? 32 : 64));
  CUtensorMap m[6];
  const void* src[3] = {a->q, a->k, a->v};
  const long long ld[3] = {a->ldq, a->ldk, a->ldv};
  for (int t = 0; t < 3; ++t) {
    if (make_map_heads(&m[t], src[t], rows, a->heads, a->dh, ld[t], 64) != QCB_OK) return QCB_ERR_CUDA;
    if (make_map_heads(&m[3 + t], src[t], rows, a->heads, a->dh, ld[t], (tw && t < 2) ? tw : 64) !=
        QCB_OK)
      return QCB_ERR_CUDA;
  }
  FmhaArgs fa;
  fa.q = reinterpret_cast<const __nv_bfloat16*>(a->q);
  fa.ldq = a->ldq;
  fa.out = reinterpret_cast<__nv_bfloat16*>(a->out);
  fa.ldo = a->ldo;
  fa.seg_stride = a->seg_stride;
  fa.S = a->S;
  fa.dh = a->dh;
  fa.dhp = dhp;
  fa.nkb = (a->S + 127) / 128;
  const double scale = a->scale != 0.0f ? (double)a->scale : 1.0 / sqrt((double)a->dh);
  fa.c = (float)(scale * 1.4426950408889634);
  const dim3 grid((unsigned)((a->S + 255) / 256), (unsigned)a->heads, (unsigned)a->nseg);
  switch (tw) {
    case 0: return fmha_launch_t<0, 6, true>(m, fa, grid, st);
    case 16: return fmha_launch_t<16, 4, true>(m, fa, grid, st);
    case 32: return fmha_launch_t<32, 3, false>(m, fa, grid, st);
    default: return fmha_launch_t<64, 2, false>(m, fa, grid, st);
  }
}

}  // namespace qc
