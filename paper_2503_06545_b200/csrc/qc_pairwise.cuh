// numpy's pairwise summation of a row, computed by one warp (the LN mean and
// variance of the quantizer's prologue, model.py:137-142).
//
// Included by qc_quant.cu inside namespace qc.  The reference computes
// x64.mean(axis=-1) and ((x64 - mean) ** 2).mean(axis=-1) with numpy's
// pairwise_sum (numpy/_core/src/umath/loops_utils.h.src): ranges of <= 128
// elements are leaves summed by 8 strided accumulators, combined as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus the n % 8 remainder in order;
// longer ranges split at n/2 rounded down to a multiple of 8.  The host builds
// the leaf list and the postfix program of that tree (pairwise_plan); one warp
// evaluates it in exactly that order, so the f64 mean and variance are
// bit-identical to numpy's (not only when the sums happen to be exact).
#pragma once

constexpr int kPwMaxLeaves = 64;

// numpy pairwise_sum over K elements: the leaves in order and the postfix
// program of the tree (bit i of prog: 1 = push the next leaf, 0 = add the top
// two), built on the host by pairwise_plan().  balanced: nleaf is a power of
// two <= 32 and every split halves the leaf range, so the tree is the
// butterfly reduction xor 1, 2, 4, ... over lanes holding the leaf sums.
struct PairwisePlan {
  int nleaf;
  int balanced;
  unsigned short leaf_start[kPwMaxLeaves];
  unsigned char leaf_len[kPwMaxLeaves];
  unsigned long long prog[2];
};

// in-register unnormalised WHT over the 5 register-index bits
QC_DEV void v5_fwht32(double (&v)[32]) {
#pragma unroll
  for (int h = 1; h < 32; h <<= 1)
#pragma unroll
    for (int r = 0; r < 32; ++r)
      if ((r & h) == 0) {
        const double a = v[r], b = v[r + h];
        v[r] = __dadd_rn(a, b);
        v[r + h] = __dsub_rn(a, b);
      }
}

// numpy's pairwise sum over the row of f(x[e]), computed by a group of nthr
// threads (tid = index in the group, the group's first 32 threads form one
// full warp; sync() is the group's barrier):
// kSq = false: f = x (the mean), kSq = true: f = (x - mean)^2 rounded like
// numpy's ((x64 - mean) ** 2).  scr: >= 601 doubles of group scratch.
template <bool kSq, class Sync>
QC_DEV double np_pairwise_group(const float* x, double mean, const PairwisePlan& pl, double* scr,
                                int tid, int nthr, Sync sync) {
  auto val = [&](int e) -> double {
    if (kSq) {
      const double d = __dsub_rn((double)x[e], mean);
      return __dmul_rn(d, d);
    }
    return (double)x[e];
  };
  const int nch = pl.nleaf * 8;
  for (int ch = tid; ch < nch; ch += nthr) {   // chain j of leaf L: x[st + j + 8 m]
    const int L = ch >> 3, len = pl.leaf_len[L];
    const int st = pl.leaf_start[L] + (ch & 7), n8 = len >> 3;
    double r;
    if (len < 8) {   // a short leaf (n < 8 overall) is one sequential sum
      r = 0.0;
      if ((ch & 7) == 0)
        for (int i = 0; i < len; ++i) r = __dadd_rn(r, val(st + i));
    } else {
      r = val(st);
#pragma unroll 4
      for (int m = 1; m < n8; ++m) r = __dadd_rn(r, val(st + 8 * m));
    }
    scr[ch] = r;
  }
  sync();
  if (tid < 32) {
    const int lane = tid;
    double leaf = 0.0;
    for (int L = lane; L < pl.nleaf; L += 32) {
      const double* c = scr + 8 * L;
      const int len = pl.leaf_len[L], st = pl.leaf_start[L];
      double res = c[0];
      if (len >= 8) {
        res = __dadd_rn(__dadd_rn(__dadd_rn(c[0], c[1]), __dadd_rn(c[2], c[3])),
                        __dadd_rn(__dadd_rn(c[4], c[5]), __dadd_rn(c[6], c[7])));
        for (int i = len & ~7; i < len; ++i) res = __dadd_rn(res, val(st + i));
      }
      scr[512 + L] = res;
      leaf = res;
    }
    double tot;
    if (pl.balanced) {
      // lane L holds leaf L: level k of the tree adds siblings 2^k apart
      for (int o = 1; o < pl.nleaf; o <<= 1)
        leaf = __dadd_rn(leaf, __shfl_xor_sync(0xffffffffu, leaf, o));
      tot = leaf;
    } else {
      __syncwarp();
      tot = 0.0;
      if (lane == 0) {
        double stk[8];
        int sp = 0, lf = 0;
        const int nops = 2 * pl.nleaf - 1;
        for (int i = 0; i < nops; ++i) {
          if ((pl.prog[i >> 6] >> (i & 63)) & 1ull) {
            stk[sp++] = scr[512 + lf++];
          } else {
            const double b = stk[--sp];
            stk[sp - 1] = __dadd_rn(stk[sp - 1], b);
          }
        }
        tot = stk[0];
      }
    }
    if (lane == 0) scr[600] = tot;
  }
  sync();
  const double tot = scr[600];
  sync();   // scr is reused
  return tot;
}

// the same by one warp (lane = tid)
template <bool kSq>
QC_DEV double np_pairwise_row(const float* x, double mean, const PairwisePlan& pl, double* scr,
                              int lane) {
  return np_pairwise_group<kSq>(x, mean, pl, scr, lane, 32, [] { __syncwarp(); });
}

// Host: the plan of numpy's pairwise_sum over n elements.  False when n is 0
// or the tree does not fit the plan (n > 8192).
static bool pairwise_plan_rec(int n, int off, PairwisePlan& pl, int& nops) {
  if (n <= 128) {
    if (pl.nleaf >= kPwMaxLeaves || nops >= 128) return false;
    pl.leaf_start[pl.nleaf] = (unsigned short)off;
    pl.leaf_len[pl.nleaf] = (unsigned char)n;
    ++pl.nleaf;
    pl.prog[nops >> 6] |= 1ull << (nops & 63);
    ++nops;
    return true;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  if (!pairwise_plan_rec(n2, off, pl, nops) || !pairwise_plan_rec(n - n2, off + n2, pl, nops))
    return false;
  if (nops >= 128) return false;
  ++nops;   // an add: its program bit stays 0
  return true;
}
static inline bool pairwise_plan(int n, PairwisePlan& pl) {
  pl = PairwisePlan{};
  int nops = 0;
  if (n <= 0 || !pairwise_plan_rec(n, 0, pl, nops)) return false;
  // balanced: 2^j equal leaves (<= 32) from exact halvings -> butterfly tree
  bool bal = pl.nleaf <= 32 && (pl.nleaf & (pl.nleaf - 1)) == 0 && pl.leaf_len[0] >= 8;
  for (int i = 0; i < pl.nleaf && bal; ++i)
    bal = pl.leaf_len[i] == pl.leaf_len[0] && pl.leaf_start[i] == i * pl.leaf_len[0];
  pl.balanced = bal ? 1 : 0;
  return true;
}
