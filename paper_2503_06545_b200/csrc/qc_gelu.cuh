// Certified fast GELU paths shared by the in-place GELU kernel (qc_fp.cu) and
// the quantizer's GELU prologue (qc_quant.cu): f32(gelu_f64(x)) with the
// reference's SciPy/cephes erf (model.py:145-147).  Each path returns false
// (or flags the element "hard") when it cannot certify the f32 rounding; the
// exact cephes replica (gelu_f32_ref) decides those.
#pragma once

#include "qc_common.cuh"

namespace qc {

// cephes ndtr.c coefficients in constant memory: FP64 instructions read them as
// c[bank][offset] operands instead of re-materialising 64-bit literals with
// uniform moves on every use (a quarter of the kernel's instructions before)
__constant__ double kErfT[5] = {9.60497373987051638749E0, 9.00260197203842689217E1,
                                2.23200534594684319226E3, 7.00332514112805075473E3,
                                5.55923013010394962768E4};
__constant__ double kErfU[5] = {3.35617141647503099647E1, 5.21357949780152679795E2,
                                4.59432382970980127987E3, 2.26290000613890934246E4,
                                4.92673942608635921086E4};
__constant__ double kErfcP[9] = {2.46196981473530512524E-10, 5.64189564831068821977E-1,
                                 7.46321056442269912687E0,  4.86371970985681366614E1,
                                 1.96520832956077098242E2,  5.26445194995477358631E2,
                                 9.34528527171957607540E2,  1.02755188689515710272E3,
                                 5.57535335369399327526E2};
__constant__ double kErfcQ[8] = {1.32281951154744992508E1, 8.67072140885989742329E1,
                                 3.54937778887819891062E2, 9.75708501743205489753E2,
                                 1.82390916687909736289E3, 2.24633760818710981792E3,
                                 1.65666309194161350182E3, 5.57535340817727675546E2};

// ~correctly rounded 1/u: MUFU seed + two Newton steps (within an ulp or two)
QC_DEV double fast_rcp(double u) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(u));
  double e = fma(-u, r, 1.0);
  r = fma(r, e, r);
  e = fma(-u, r, 1.0);
  return fma(r, e, r);
}

// Is the f64 value g at least w ulp64 away from an f32 rounding tie, inside
// the f32 normal range?  (the certificate test of the fast GELU paths)
QC_DEV bool f32_round_safe(double g, double w) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(g);
  const int ex = (int)((bits >> 52) & 0x7FF) - 1023;
  if (ex < -125 || ex > 126) return false;
  const int d = abs((int)((unsigned)bits & 0x1FFFFFFFu) - (1 << 28));
  return (double)d > w;
}

// Phase A, |x / sqrt2| < 1: the cephes T/U rational with FMA Horner steps and
// a Newton reciprocal instead of the reference's separate mul/add and IEEE
// division.  Relative error of erf vs the reference's value: well under
// 20 ulp, amplified at most ~6x in 1 + erf (>= 0.157) -> accepted when g is
// 256 ulp64 clear of an f32 tie.  Returns false for |t| >= 1 or near ties.
QC_DEV bool gelu_fast_a(float xf, float& y) {
  if (xf >= 6.0f) {
    y = xf;
    return true;
  }
  const double x = (double)xf;
  const double t = x * 0.70710678118654752440;
  const double at = fabs(t);
  if (!(at < 1.0 - 0x1p-40)) return false;
  const double z = at * at;
  double tt = kErfT[0];
#pragma unroll
  for (int i = 1; i < 5; ++i) tt = fma(tt, z, kErfT[i]);
  double u = z + kErfU[0];
#pragma unroll
  for (int i = 1; i < 5; ++i) u = fma(u, z, kErfU[i]);
  double r = (at * tt) * fast_rcp(u);
  if (t < 0.0) r = -r;
  const double g = (0.5 * x) * (1.0 + r);
  if (g == 0.0) {   // x == +-0
    y = __double2float_rn(g);
    return true;
  }
  if (!f32_round_safe(g, 256.0)) return false;
  y = __double2float_rn(g);
  return true;
}

// 1/u from the MUFU seed and ONE Newton step: relative error below 2^-40
// (seed error below 2^-20), for the phase-A path whose certificate window is
// widened to match
QC_DEV double fast_rcp1(double u) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(u));
  const double e = fma(-u, r, 1.0);
  return fma(r, e, r);
}

// Phase A for 8 elements without branches: every element runs the same
// straight-line code and the certificate becomes a select (per-element early
// exits cost more than the shared arithmetic).  Returns the hard mask.
QC_DEV uint32_t gelu_phase_a8(const float (&v)[8], float (&y)[8], uint32_t valid) {
  uint32_t hard = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const double x = (double)v[i];
    const double t = x * 0.70710678118654752440;
    const double at = fabs(t);
    const double z = at * at;
    double tt = kErfT[0];
#pragma unroll
    for (int k = 1; k < 5; ++k) tt = fma(tt, z, kErfT[k]);
    double u = z + kErfU[0];
#pragma unroll
    for (int k = 1; k < 5; ++k) u = fma(u, z, kErfU[k]);
    double r = (at * tt) * fast_rcp1(u);
    r = t < 0.0 ? -r : r;
    const double g = (0.5 * x) * (1.0 + r);
    // certificate: f32-normal range and >= 2^14 ulp64 from an f32 tie (the
    // one-step reciprocal's < 2^-40 error amplified at most ~6x by 1 + erf,
    // plus the rational's own error), as integers
    const unsigned long long gb = (unsigned long long)__double_as_longlong(g);
    const unsigned ex = (unsigned)((gb >> 52) & 0x7FF);
    const int dd = abs((int)((unsigned)gb & 0x1FFFFFFFu) - (1 << 28));
    const bool ok = (at < 1.0 - 0x1p-40) && (ex - (1023u - 125u)) <= 251u && dd > 16384;
    const bool big = v[i] >= 6.0f, zero = v[i] == 0.0f;
    y[i] = big ? v[i] : __double2float_rn(g);   // g = +-0 for x = +-0
    if (((valid >> i) & 1u) && !big && !zero && !ok) hard |= 1u << i;
  }
  return hard;
}

// Phase B, 1 <= |x / sqrt2| < 8: cephes erfc(|t|) = exp(-t^2) P(|t|)/Q(|t|)
// with FMA Horner, a Newton reciprocal and CUDA exp, then the reference's own
// structure 1 + erf = 1 +- (1 - erfc).  Error vs the reference's f64 value:
// (~24 + 4 t^2) ulp relative in erfc (exp, Horner, division, the 1-ulp
// argument difference), plus the reference's double rounding of 1 - erfc
// (<= 2^-53 absolute, i.e. <= 1/ope ulp of g) -> window 512 + 32 t^2 + 8/ope.
QC_DEV bool gelu_fast_b(float xf, float& y) {
  const double x = (double)xf;
  const double t = x * 0.70710678118654752440;
  const double at = fabs(t);
  if (!(at >= 1.0 && at < 8.0)) return false;
  const double ez = exp(-(at * at));
  double pp = kErfcP[0];
#pragma unroll
  for (int i = 1; i < 9; ++i) pp = fma(pp, at, kErfcP[i]);
  double qq = at + kErfcQ[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) qq = fma(qq, at, kErfcQ[i]);
  const double ec = (ez * pp) * fast_rcp(qq);
  const double r = 1.0 - ec;                         // erf(|t|), rounded like the reference
  const double ope = t > 0.0 ? 1.0 + r : 1.0 - r;    // 1 + erf(t)
  if (!(ope > 0.0)) return false;
  const double g = (0.5 * x) * ope;
  if (!f32_round_safe(g, 512.0 + 32.0 * (t * t) + 8.0 / ope)) return false;
  y = __double2float_rn(g);
  return true;
}


}  // namespace qc
