// Shared device primitives for the QuantCache B200 kernels (sm_100a only).
//
// Inline PTX wrappers for mbarrier, TMA (cp.async.bulk.tensor), tcgen05
// (alloc / mma / commit / ld) and a few exact-arithmetic helpers that the
// quantizer and epilogues need to match the reference's numerics.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "QuantCache B200 kernels are sm_100a-only"
#endif

#define QC_DEV __device__ __forceinline__

namespace qc {

// ---------------------------------------------------------------- PDL
// Wait until the preceding grid on the stream completed and its writes are
// visible (no-op when the kernel was launched without the PDL attribute).
QC_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Let the next grid on the stream start launching (its pdl_wait still waits
// for this grid's completion).
QC_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// ---------------------------------------------------------------- smem / barriers
QC_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

QC_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

QC_DEV void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

QC_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

QC_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

QC_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------- TMA
QC_DEV void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// 2-D tiled bulk tensor load into CTA shared memory, completion on `bar`.
QC_DEV void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// 2-D tiled bulk tensor store from CTA shared memory (bulk-group completion).
QC_DEV void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(smem_u32(src))
      : "memory");
}
// 1-D bulk async copy global -> shared (16-byte aligned, size % 16 == 0),
// completion signalled on `bar` as transaction bytes.
QC_DEV void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// L2 eviction-priority policies (createpolicy) and hinted accesses
QC_DEV uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
QC_DEV uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
QC_DEV void st_f32_hint(float* a, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(pol) : "memory");
}
QC_DEV void st_f32x4_hint(float* a, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(a), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}
QC_DEV void bulk_load_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                           uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

QC_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
QC_DEV void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
QC_DEV void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// Generic-proxy shared-memory writes -> visible to the async (TMA) proxy.
QC_DEV void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
QC_DEV void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- tcgen05
QC_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
QC_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Allocate `ncols` TMEM columns (power of two >= 32); one full warp calls.
template <uint32_t kCols>
QC_DEV void tmem_alloc(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

template <uint32_t kCols>
QC_DEV void tmem_free(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
               : "memory");
}

// D[tmem] (+)= A[smem] x B[smem]^T, u8 x u8 -> s32, one elected thread issues.
QC_DEV void umma_u8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                    uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive on `bar` once every previously issued tcgen05.mma of this thread retires.
QC_DEV void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------- CTA pairs
// Two CTAs of a (2,1,1) cluster on one TPC cooperate on M = 256 tiles
// (tcgen05 cta_group::2): each holds its 128 rows of A and half of B's columns
// in shared memory; the leader (rank 0) issues the MMA for both.
QC_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// address of the same shared variable in CTA `rank` of the cluster
QC_DEV uint32_t mapa_shared(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
QC_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
template <uint32_t kCols>
QC_DEV void tmem_alloc2(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
QC_DEV void tmem_free2(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
               : "memory");
}
QC_DEV void umma_u8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                         uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on `bar` (same offset) in both CTAs once the pair's MMAs retire
QC_DEV void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
// TMA tile load whose completion is counted on the leader's barrier
// (`bar_cl`: a shared::cluster address, e.g. mapa_shared(..., 0))
QC_DEV void tma_load_2d_pair(const CUtensorMap* map, uint32_t bar_cl, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cl), "r"(c0), "r"(c1)
      : "memory");
}
QC_DEV void mbar_arrive_cluster(uint32_t bar_cl) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cl)
               : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread.
QC_DEV void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// 32 lanes x 8 consecutive 32-bit columns -> 8 registers per thread.
QC_DEV void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

QC_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor: K-major operand, 128-byte swizzle, rows of
// 128 bytes, 8-row core groups 1024 bytes apart (SBO), LBO unused (=1).
QC_DEV uint64_t smem_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);  // start address
  d |= (uint64_t)1u << 16;                    // leading byte offset (ignored for SW128 K-major)
  d |= (uint64_t)(1024u >> 4) << 32;          // stride byte offset
  d |= (uint64_t)1u << 46;                    // descriptor version (sm_100)
  d |= (uint64_t)2u << 61;                    // layout: SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::i8: A,B unsigned 8-bit, K-major; D s32.
__host__ __device__ constexpr uint32_t idesc_u8(uint32_t M, uint32_t N) {
  return (2u << 4)            // D format: S32
         | (0u << 7)          // A format: unsigned 8-bit
         | (0u << 10)         // B format: unsigned 8-bit
         | (0u << 15)         // A K-major
         | (0u << 16)         // B K-major
         | ((N >> 3) << 17)   // N / 8
         | ((M >> 4) << 24);  // M / 16
}

// ---------------------------------------------------------------- exact arithmetic
// Round half away from zero, f64 (reference quant.py:24-27).
QC_DEV double rha(double v) {
  double a = floor(__dadd_rn(fabs(v), 0.5));
  return v < 0.0 ? -a : (v > 0.0 ? a : 0.0 * v);
}

// Round a positive scale UP to a 16-bit significand (quant.py:30-35).
QC_DEV double scale_up16(double s) {
  int e;
  double m = frexp(s, &e);
  m = ceil(m * 65536.0) / 65536.0;
  return ldexp(m, e);
}

// erf(x) as SciPy evaluates it (cephes ndtr.c rational approximations, odd
// symmetry, 1 - erfc for |x| > 1), which the reference's GELU calls
// (model.py:145-147).  Matching the formulation keeps 1 + erf(x) identical in
// the cancellation region x << 0; only exp() may differ from glibc by an ulp.
// Horner steps as cephes polevl/p1evl evaluate them (separate mul and add, no
// FMA); coefficients are literals so nothing spills to local memory.
#define QC_H(a, x, c) __dadd_rn(__dmul_rn((a), (x)), (c))
QC_DEV double erfc_pos(double x) {  // x >= 1
  const double z0 = -__dmul_rn(x, x);
  if (z0 < -7.09782712893383996843E2) return 0.0;
  const double z = exp(z0);
  double p, q;
  if (x < 8.0) {
    p = 2.46196981473530512524E-10;
    p = QC_H(p, x, 5.64189564831068821977E-1);
    p = QC_H(p, x, 7.46321056442269912687E0);
    p = QC_H(p, x, 4.86371970985681366614E1);
    p = QC_H(p, x, 1.96520832956077098242E2);
    p = QC_H(p, x, 5.26445194995477358631E2);
    p = QC_H(p, x, 9.34528527171957607540E2);
    p = QC_H(p, x, 1.02755188689515710272E3);
    p = QC_H(p, x, 5.57535335369399327526E2);
    q = __dadd_rn(x, 1.32281951154744992508E1);
    q = QC_H(q, x, 8.67072140885989742329E1);
    q = QC_H(q, x, 3.54937778887819891062E2);
    q = QC_H(q, x, 9.75708501743205489753E2);
    q = QC_H(q, x, 1.82390916687909736289E3);
    q = QC_H(q, x, 2.24633760818710981792E3);
    q = QC_H(q, x, 1.65666309194161350182E3);
    q = QC_H(q, x, 5.57535340817727675546E2);
  } else {
    p = 5.64189583547755073984E-1;
    p = QC_H(p, x, 1.27536670759978104416E0);
    p = QC_H(p, x, 5.01905042251180477414E0);
    p = QC_H(p, x, 6.16021097993053585195E0);
    p = QC_H(p, x, 7.40974269950448939160E0);
    p = QC_H(p, x, 2.97886665372100240670E0);
    q = __dadd_rn(x, 2.26052863220117276590E0);
    q = QC_H(q, x, 9.39603524938001434673E0);
    q = QC_H(q, x, 1.20489539808096656605E1);
    q = QC_H(q, x, 1.70814450747565897222E1);
    q = QC_H(q, x, 9.60896809063285878198E0);
    q = QC_H(q, x, 3.36907645100081516050E0);
  }
  return __ddiv_rn(__dmul_rn(z, p), q);
}
QC_DEV double erf_cephes(double x) {
  const double ax = fabs(x);
  double r;
  if (ax > 1.0) {
    r = __dsub_rn(1.0, erfc_pos(ax));
  } else {
    const double z = __dmul_rn(ax, ax);
    double t = 9.60497373987051638749E0;
    t = QC_H(t, z, 9.00260197203842689217E1);
    t = QC_H(t, z, 2.23200534594684319226E3);
    t = QC_H(t, z, 7.00332514112805075473E3);
    t = QC_H(t, z, 5.55923013010394962768E4);
    double u = __dadd_rn(z, 3.35617141647503099647E1);
    u = QC_H(u, z, 5.21357949780152679795E2);
    u = QC_H(u, z, 4.59432382970980127987E3);
    u = QC_H(u, z, 2.26290000613890934246E4);
    u = QC_H(u, z, 4.92673942608635921086E4);
    r = __ddiv_rn(__dmul_rn(ax, t), u);
  }
  return x < 0.0 ? -r : r;
}
// GELU(x) = 0.5 x (1 + erf(x / sqrt 2)) in f64 (model.py:145-147).
QC_DEV double gelu_ref(double x) {
  const double e = erf_cephes(__ddiv_rn(x, 1.4142135623730951));
  return __dmul_rn(__dmul_rn(0.5, x), __dadd_rn(1.0, e));
}
// f32(GELU(x)) for an f32 input.  For x >= 6, erfc(x/sqrt2) < 2^-28 so the f64
// value is within x*2^-29 of x and rounds back to x: return it directly.
QC_DEV float gelu_f32_ref(float x) {
  if (x >= 6.0f) return x;
  return __double2float_rn(gelu_ref((double)x));
}

// ---- conversions without the XU pipe ----------------------------------------
// On this B200 an f32<->f64 convert issues at ~8/clk/SM (measured), an f64 add
// at ~61/clk/SM.  These exact bit-level equivalents run on the ALU / FP64 pipes
// and fall back to the hardware conversion only for rare special values.

// exact (double)f
QC_DEV double f2d_alu(float f) {
  const uint32_t u = __float_as_uint(f);
  const uint32_t e = (u >> 23) & 0xFFu, m = u & 0x7FFFFFu;
  if (e == 0xFFu || (e == 0u && m != 0u)) return (double)f;   // inf/nan/subnormal
  const unsigned long long s = (unsigned long long)(u & 0x80000000u) << 32;
  const unsigned long long body =
      e == 0u ? 0ull : ((unsigned long long)(e + 896u) << 52) | ((unsigned long long)m << 29);
  return __longlong_as_double((long long)(s | body));
}

// exact (double)i for any int32 (magic-number add on the FP64 pipe)
QC_DEV double i2d_alu(int i) {
  return __longlong_as_double(0x4338000000000000LL + (long long)i) - 6755399441055744.0;
}

// round-to-nearest-even of d to f32; integer path when the result is a normal
// f32 (or zero), hardware conversion otherwise.
QC_DEV float d2f_alu(double d) {
  unsigned long long u = (unsigned long long)__double_as_longlong(d);
  const unsigned long long s = u & 0x8000000000000000ull;
  u &= 0x7FFFFFFFFFFFFFFFull;
  if (u == 0ull) return __uint_as_float((uint32_t)(s >> 32));
  const int ex = (int)(u >> 52);
  if (ex < 1023 - 126 || ex > 1023 + 126) return __double2float_rn(d);   // f32 range edge
  u += 0x0FFFFFFFull + ((u >> 29) & 1ull);   // RNE at bit 29; carries bump the exponent
  const uint32_t bits = (uint32_t)(s >> 32) |
                        ((uint32_t)((int)(u >> 52) - 1023 + 127) << 23) |
                        (uint32_t)((u >> 29) & 0x7FFFFFull);
  return __uint_as_float(bits);
}

// Branch-free d2f_alu for batches: sets `bad` when d needs the hardware path
// (f32 range edge); the caller redoes the batch with __double2float_rn then.
QC_DEV float d2f_alu_flag(double d, bool& bad) {
  unsigned long long u = (unsigned long long)__double_as_longlong(d);
  const uint32_t s = (uint32_t)(u >> 32) & 0x80000000u;
  u &= 0x7FFFFFFFFFFFFFFFull;
  const int ex = (int)(u >> 52);
  bad |= (u != 0ull) & ((ex < 1023 - 126) | (ex > 1023 + 126));
  u += 0x0FFFFFFFull + ((u >> 29) & 1ull);
  const uint32_t bits = ((uint32_t)((int)(u >> 52) - 1023 + 127) << 23) |
                        (uint32_t)((u >> 29) & 0x7FFFFFull);
  return __uint_as_float(s | (ex == 0 ? 0u : bits));
}

// d rounded to a 24-bit significand (RNE), kept as f64 == (double)f32(d) for
// values in the f32 normal range (callers guarantee the range).
QC_DEV double d_round24(double d) {
  unsigned long long u = (unsigned long long)__double_as_longlong(d);
  u += 0x0FFFFFFFull + ((u >> 29) & 1ull);
  u &= ~0x1FFFFFFFull;
  return __longlong_as_double((long long)u);
}

// Branch-free companion of d_round24_fast: 1 when q is within 64 ulp64 of an
// f32 rounding tie or outside the f32 normal range (zero is safe), i.e. when
// an estimate of q may round to f32 differently from the exact value.
QC_DEV uint32_t f32_round_risk(double q) {
  const uint32_t lo = (uint32_t)__double2loint(q), hi = (uint32_t)__double2hiint(q);
  const uint32_t ex = (hi >> 20) & 0x7FFu;
  const bool nonzero = ((hi & 0x7FFFFFFFu) | lo) != 0u;
  const bool range = (ex - (1023u - 125u)) > 251u;                // ex - 1023 outside [-125, 126]
  const bool tie = ((lo & 0x1FFFFFFFu) - ((1u << 28) - 63u)) < 127u;  // |t - 2^28| < 64
  return (uint32_t)(nonzero & (range | tie));
}

// f32_round_risk without the zero exemption, in fewer integer instructions
// (the range test on the masked exponent field, no field extraction): zero is
// reported as a risk and takes the exact path, which returns it unchanged.
QC_DEV bool f32_round_risk_z(double q) {
  const uint32_t lo = (uint32_t)__double2loint(q), hi = (uint32_t)__double2hiint(q);
  const bool range = ((hi & 0x7FF00000u) - ((1023u - 125u) << 20)) > (251u << 20);
  const bool tie = ((lo & 0x1FFFFFFFu) - ((1u << 28) - 63u)) < 127u;
  return range | tie;
}

// q rounded to a 24-bit significand by round-half-up on the magnitude: equal
// to (double)(float)q whenever f32_round_risk(q) == 0 (ties never reach it).
QC_DEV double d_round24_fast(double q) {
  unsigned long long u = (unsigned long long)__double_as_longlong(q);
  u = (u + 0x10000000ull) & ~0x1FFFFFFFull;
  return __longlong_as_double((long long)u);
}

// True when rounding the f64 value q to f32 could differ from rounding a value
// a few f64 ulps away: the 29 dropped fraction bits are within 64 units of the
// round-to-nearest midpoint pattern, or q is outside the f32 normal range.
QC_DEV bool f64_near_f32_tie_dev(double q) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(q);
  if ((u << 1) == 0ull) return false;   // +-0 rounds exactly
  const int ex = (int)((u >> 52) & 0x7FF) - 1023;
  if (ex < -125 || ex > 126) return true;
  const int d = (int)((unsigned)u & 0x1FFFFFFFu) - (1 << 28);
  return d > -64 && d < 64;
}

// Float total order as an unsigned key (for atomic min/max on floats).
QC_DEV uint32_t f2key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
QC_DEV float key2f(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  return __uint_as_float(u);
}

template <typename T>
QC_DEV T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace qc
