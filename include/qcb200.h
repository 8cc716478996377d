/*
 * qcb200.h -- C ABI of the B200-native QuantCache hot path (libqcb200.so).
 *
 * Plain pointers, sizes and a cudaStream_t passed as void*; no torch types.
 * All pointers are DEVICE pointers unless stated; the caller owns every
 * buffer (no allocation inside hot-path calls; workspaces are passed in).
 * Every entry point returns a status code (QCB_OK == 0).  The Python mirror
 * (paper_2503_06545_b200/_native.py) maps codes onto the reference's
 * exception types (errors.py:4-21):
 *     QCB_ERR_DIM -> DimensionError, QCB_ERR_CONFIG / QCB_ERR_OVERFLOW ->
 *     ConfigurationError, QCB_ERR_VALUE -> ValueError, QCB_ERR_TYPE ->
 *     TypeError, QCB_ERR_CUDA -> RuntimeError.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/ditrt):
 *   qcb_gemm_u8        tensor.py:68-112   matmul_int
 *   qcb_pack_w4        quant.py:206       W4 weights, nibble-packed GEMM operand (+ model.py:187-198 epilogues)
 *   qcb_gemm_f64       tensor.py:43-65    mm / matmul_fp (FP sites)
 *   qcb_head_gemm      model.py:228       mm(x, head_w) + head_b (certified int8)
 *   qcb_act_quant      quant.py:83-123,163-165  compute_minmax_params + quantize
 *                      on BalanceTransform.apply_to_activation, with the
 *                      LN/modulation prologue of model.py:182,189,196
 *   qcb_weight_prep    runtime.py:40-61   QuantRuntime.__init__ weight prep
 *   qcb_attention_f64  model.py:150-156, tensor.py:115-132  _mha / attention
 *   qcb_attention_bf16 model.py:150-156                     _mha, bf16 fast mode
 *   qcb_ln_mod         model.py:137-142 (+182,196)  _ln and modulation
 *   qcb_ddpm_step      sampler.py:59-88   reverse_step / final_step
 *   qcb_cfg_combine    (extension)        classifier-free guidance of eps
 *   qcb_gelu_inplace   model.py:145-147   _gelu
 *   qcb_reduce_hlc     schedule.py:67-82  divergence_score partial sums
 *   qcb_reduce_srap    schedule.py:108-116 layer_similarity partial sums
 *   qcb_reduce_var     schedule.py:128-133 cumulative_variation
 *   qcb_policy_*       schedule.py:281-351 Scheduler.plan_step / observe_block
 */
#ifndef QCB200_H_
#define QCB200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  QCB_OK = 0,
  QCB_ERR_DIM = 1,
  QCB_ERR_CONFIG = 2,
  QCB_ERR_OVERFLOW = 3,
  QCB_ERR_VALUE = 4,
  QCB_ERR_TYPE = 5,
  QCB_ERR_CUDA = 6
};

/* GEMM epilogues (model.py:183-198). */
enum {
  QCB_EPI_STORE = 0,      /* out = y                         (q, k, v, ca_q/k/v)  */
  QCB_EPI_GELU = 1,       /* out = f32(gelu_f64(y))          (ffn1)               */
  QCB_EPI_GATE_RESID = 2, /* out = resid + gate * y (f32)    (sta_o, ffn2)        */
  QCB_EPI_RESID = 3,      /* out = resid + y (f32)           (ca_o)               */
  QCB_EPI_ACC = 4,        /* out = exact s32 accumulator (debug / parity)         */
  QCB_EPI_BIAS = 5,       /* out = y + bias[n] (f32)         (head, gemm_f64 only) */
  QCB_EPI_STORE_BF16 = 6  /* out = bf16(f32 y), out as uint16 [M][ldo] (q, k, v for */
                          /* the bf16 attention path; gemm_u8 only)               */
};

/* Activation prologues. */
enum { QCB_PRO_NONE = 0, QCB_PRO_LN_MOD = 1, QCB_PRO_GELU = 2 /* f32(gelu_f64(x)), model.py:197 */,
       QCB_PRO_BF16 = 3 /* x holds bf16 rows (ldx in bf16 elements), widened exactly;
                           K = 1024 + tail, rows 16-byte aligned */ };

#define QCB_MAX_LAYERS 64
#define QCB_MAX_HIST 8

/* ---------------------------------------------------------------- GEMMs */
typedef struct QcbGemm {
  int M, N, K;            /* K = true reduction length                         */
  int seg_rows;           /* rows per activation segment (video); 0 = M        */
  int seg_valid;          /* valid rows per segment (others are padding); 0=all */
  const uint8_t* a_codes; /* [M][lda] u8, lda % 16 == 0                         */
  long long lda;
  const double* a_scale;  /* [segments] per-tensor activation scale            */
  const int* a_zero;      /* [segments]                                        */
  const int* a_rowsum;    /* [M] sum_k a_codes                                 */
  const uint8_t* w_codes; /* [N][ldw] u8 (K-major, i.e. W^T), ldw % 16 == 0     */
  long long ldw;
  const double* w_scale;  /* [N] per-output-channel scale                      */
  const int* w_zero;      /* [N]                                               */
  const int* w_colsum;    /* [N] sum_k w_codes                                 */
  float* out;             /* [M][ldo] f32 (or s32 for QCB_EPI_ACC)             */
  long long ldo;
  const long long* out_row0;   /* nullable: first output row per segment        */
  const float* resid;          /* residual input for *_RESID (may alias out)   */
  long long ldr;
  const long long* resid_row0; /* nullable: first residual row per segment     */
  const float* gate;           /* nullable: per-segment gate                    */
  float gate_scalar;
  int epilogue;
  int block_n;                 /* 0 = auto                                      */
  const int* seg_active;       /* nullable: per-segment flag, skip inactive     */
  long long out_rows;          /* rows of the output buffer (TMA bounds); 0 = M */
  long long resid_rows;        /* rows of the residual buffer (TMA bounds); 0 =  */
                               /* out_rows when resid == out, else M             */
  const uint8_t* w_packed;     /* nullable: W4 weights, 2 codes per byte (low    */
  long long ldwp;              /* nibble = even k), [N][ldwp], ldwp % 64 == 0,   */
                               /* zero padded; replaces w_codes (qcb_pack_w4)    */
} QcbGemm;

int qcb_gemm_u8(const QcbGemm* g, void* stream);

/* Nibble-pack <= 4-bit weight codes (quant.py:206 BIT_LEVELS 4, the paper's W4):
 * packed[n][k/2] = codes[n][k] | codes[n][k+1] << 4 from the K-major [N][ldk]
 * u8 codes, rows zero padded to ldwp (a multiple of 64 bytes).  The GEMM then
 * streams half the weight bytes and unpacks them to u8 in shared memory in
 * its producer warps (tcgen05 has no 4-bit integer MMA).  QCB_ERR_VALUE if a
 * code exceeds 15. */
int qcb_pack_w4(const uint8_t* codes, long long ldk, int N, int K, uint8_t* packed,
                long long ldwp, void* stream);

/* Plain f64-accumulating FP GEMM, ascending k (tensor.py:43-60), f32 out.
 * A [M][lda] f32 (rows via a_row0 per segment), W [K][ldw] f32 row-major. */
typedef struct QcbGemmF64 {
  int M, N, K;
  int seg_rows, seg_valid;
  const float* a;
  long long lda;
  const long long* a_row0;
  const float* w;
  long long ldw;
  float* out;
  long long ldo;
  const long long* out_row0;
  const float* resid;
  long long ldr;
  const long long* resid_row0;
  const float* bias;
  float gate_scalar;
  int epilogue;
} QcbGemmF64;

int qcb_gemm_f64(const QcbGemmF64* g, void* stream);

/* Noise head out = f32(mm(x, W)) + bias (model.py:228 with tensor.py:43-60) on
 * the int8 tensor cores: x rows and W columns split into 6 base-256 digit planes,
 * one grouped exact u8 GEMM over the digit diagonals, f64 combination with an
 * error bound;
 * elements whose bound straddles an f32 rounding boundary are recomputed with
 * the reference's ascending-k f64 FMA chain, so every output equals mm's.
 * qcb_head_prep writes W's planes / statistics into `prep` once
 * (qcb_head_prep_bytes); qcb_head_gemm runs per call with a workspace of
 * qcb_head_workspace_bytes(nseg * seg_rows, K, N).  K and N must be multiples of 4;
 * K <= 5504 (6 K 255^2 < 2^31, else QCB_ERR_OVERFLOW). */
typedef struct QcbHeadGemm {
  int nseg, seg_rows, seg_valid; /* rows = nseg * seg_rows; rows >= seg_valid of a */
  int K, N;                      /* segment are padding (not written)             */
  const float* x;                /* rows via x_row0 per segment (nullable)        */
  long long ldx;
  const long long* x_row0;
  const void* prep;              /* from qcb_head_prep                            */
  const float* bias;             /* nullable [N]                                  */
  float* out;                    /* [rows][ldo] (rows via out_row0, nullable)     */
  long long ldo;
  const long long* out_row0;
  void* workspace;
  int* fallback_count;           /* nullable device int += exact recomputations   */
} QcbHeadGemm;

size_t qcb_head_prep_bytes(int K, int N);
size_t qcb_head_workspace_bytes(long long rows, int K, int N);
int qcb_head_prep(const float* w, int K, int N, void* prep, void* stream);
int qcb_head_gemm(const QcbHeadGemm* g, void* stream);

/* ---------------------------------------------------------------- quantizer */
typedef struct QcbActQuant {
  const float* x;            /* input rows [.][ldx]                             */
  long long ldx;
  const long long* x_row0;   /* nullable: first input row per segment           */
  int K, seg_rows, seg_valid, nseg;
  int prologue;              /* QCB_PRO_*                                        */
  const float* ln_g;         /* nullable (= ones)                               */
  const float* ln_b;         /* nullable (= zeros)                              */
  float mod_scale1;          /* f32(1 + scale) ; 1 for no modulation             */
  float mod_shift;           /* shift ; 0 for no modulation                      */
  int n_out;                 /* 1..3 outputs sharing the prologue                */
  int bits;                  /* activation bit-width                             */
  const double* chan_scale[3]; /* nullable: balance scales c (no rotation)       */
  const float* signs[3];     /* [b] +-1 of the randomized Hadamard block         */
  uint8_t* codes[3];         /* [nseg*seg_rows][ldc] outputs                     */
  long long ldc;
  int* rowsum[3];            /* [nseg*seg_rows]                                  */
  double* scale[3];          /* [nseg]                                           */
  int* zero[3];              /* [nseg]                                           */
  float* xe_out[3];          /* nullable: rotated activations (debug / FP modes) */
  long long ldxe;
  float* deq_out[3];         /* nullable: f32(s*(code-z)) fake-quant outputs     */
  void* workspace;           /* qcb_act_quant_workspace_bytes(...) bytes         */
  const double* chan_recip[3]; /* nullable: signed reciprocals s_j/c_j (j < b) and   */
                               /* 1/c_j (j >= b), as qcb_weight_prep writes them;    */
                               /* else computed per call                             */
} QcbActQuant;

int qcb_act_quant(const QcbActQuant* q, void* stream);
/* Workspace bytes qcb_act_quant needs (keys, reciprocals, f32 stash of xe). */
size_t qcb_act_quant_workspace_bytes(int K, int seg_rows, int nseg, int n_out);

typedef struct QcbWeightPrep {
  const float* w;            /* [K][N] f32, reference layout                     */
  int K, N, bits;
  const double* chan_scale;  /* nullable: no balance / rotation                  */
  const float* signs;        /* [b]                                              */
  uint8_t* codes;            /* [N][ldk] K-major                                 */
  long long ldk;
  double* scale;             /* [N]                                              */
  int* zero;                 /* [N]                                              */
  int* colsum;               /* [N]                                              */
  float* w_eff;              /* nullable [K][N]: rotated weights                 */
  float* w_deq;              /* nullable [K][N]: dequantized weights             */
  double* chan_recip_out;    /* nullable [K]: signed reciprocals for act_quant    */
} QcbWeightPrep;

int qcb_weight_prep(const QcbWeightPrep* q, void* stream);

/* ---------------------------------------------------------------- FP helpers */
typedef struct QcbLnMod {
  const float* x; long long ldx; const long long* x_row0;
  float* out; long long ldo; const long long* out_row0;
  int K, seg_rows, seg_valid, nseg;
  const float* ln_g; const float* ln_b;
  float mod_scale1, mod_shift;
} QcbLnMod;

int qcb_ln_mod(const QcbLnMod* q, void* stream);

/* Per-head softmax(q k^T / sqrt(dh)) v with f64 softmax; q [S][ldq], k/v [Skv][.]. */
typedef struct QcbAttention {
  const float* q; long long ldq;
  const float* k; long long ldk;
  const float* v; long long ldv;
  float* out; long long ldo;
  int S, Skv, heads, dh, nseg;   /* segments stacked along rows                 */
  long long q_seg_stride, kv_seg_stride, o_seg_stride; /* rows between segments */
  int seg_valid;
} QcbAttention;

int qcb_attention_f64(const QcbAttention* a, void* stream);

/* Fast attention for the benchmarked bf16 path (the reference computes _mha in
 * f64, model.py:150-156; this mode trades that for bf16 operands like any
 * library SDPA it replaces): out = softmax(scale q k^T) v per head and segment
 * on the tcgen05 tensor cores (S and O accumulate in f32 in TMEM, P is bf16).
 * q, k, v, out: bf16 [nseg * seg_stride][ld] with head h at columns
 * [h*dh, (h+1)*dh); segment s owns rows [s*seg_stride, s*seg_stride + S).
 * dh % 8 == 0 and dh <= 128; ld* % 8 == 0; pointers 16-byte aligned;
 * S <= seg_stride.  scale = 0 means 1/sqrt(dh). */
typedef struct QcbAttentionBf16 {
  const void* q; long long ldq;
  const void* k; long long ldk;
  const void* v; long long ldv;
  void* out; long long ldo;
  int S, heads, dh, nseg;
  long long seg_stride;
  float scale;
} QcbAttentionBf16;

int qcb_attention_bf16(const QcbAttentionBf16* a, void* stream);

/* x_{t-1} = f32((x - c1*eps)/c2 + c3*noise) in f64 (c3 = 0: no noise). */
typedef struct QcbDdpm {
  const float* x; const float* eps; const float* noise; float* out;
  long long n;
  double c1, c2, c3;
  double rc2;                /* RN(1 / c2) (host IEEE division) or 0: the quotient by */
                             /* c2 then comes from one FMA correction, else a divide  */
  unsigned long long noise_seed;   /* gen_noise: N(0,1) from Philox4x32-10 in-kernel  */
  unsigned long long noise_offset; /* (key = seed, counter = offset + i / 4) instead  */
  int gen_noise;                   /* of reading `noise` (the device-noise mode)      */
} QcbDdpm;

int qcb_ddpm_step(const QcbDdpm* d, void* stream);

/* Classifier-free guidance (a labelled EXTENSION: the reference has no CFG,
 * SPEC.md:468): out[i] = f32(eps_u[i] + scale * (eps_c[i] - eps_u[i])), one
 * fused multiply-add per element, over n elements (16-byte aligned buffers use
 * vector loads).  Feeds qcb_ddpm_step with the guided noise estimate of a
 * video whose cond / uncond branches ran as two engine slots. */
int qcb_cfg_combine(const float* eps_c, const float* eps_u, float scale, float* out,
                    long long n, void* stream);

/* In-place x = f32(gelu_f64(x)) with SciPy's erf (model.py:145-147) over a
 * [rows][ld] f32 buffer (cols valid columns); ld % 4 == 0, x 16-byte aligned. */
int qcb_gelu_inplace(float* x, long long ld, int rows, int cols, void* stream);

/* ---------------------------------------------------------------- reductions */
/* Segmented f64 reductions over f32 feature maps, one result per segment.
 * A segment is `rows` rows of `cols` floats starting at base + row0[seg]*ld.
 * Results are deterministic (fixed-order two-stage reduction). */
typedef struct QcbFeat {
  const float* base; long long ld; const long long* row0;
} QcbFeat;

/* sum|out-ref| and sum (out-prev)^2 per segment -> res[seg*2 + {0,1}] */
int qcb_reduce_hlc(QcbFeat out, QcbFeat ref, QcbFeat prev, int rows, int cols, int nseg,
                   const int* seg_active, double* res, void* workspace, void* stream);
/* <a,b>, <a,a>, <b,b> per segment -> res[seg*3 + {0,1,2}].  dup_src
 * (nullable, int64 [nseg]): index of the first segment with the same (a, b)
 * rows; only those representatives are reduced and the others copied (results
 * are identical: the reduction order depends only on rows/cols/nseg). */
int qcb_reduce_srap(QcbFeat a, QcbFeat b, int rows, int cols, int nseg,
                    const int* seg_active, const long long* dup_src, double* res,
                    void* workspace, void* stream);
/* sum|x - h| per segment -> res[seg] */
int qcb_reduce_l1(QcbFeat x, QcbFeat h, int rows, int cols, int nseg, double* res,
                  void* workspace, void* stream);

/* cumulative_variation terms for all history entries in one pass
 * (schedule.py:128-133): res[j*nseg + seg] = sum|x - hist[j]| per segment, x read
 * once; 1 <= nh <= 8, every operand's segment rows contiguous (ld == cols),
 * cols % 4 == 0.  Replaces nh qcb_reduce_l1 calls. */
int qcb_reduce_l1_hist(QcbFeat x, const QcbFeat* hist, int nh, int rows, int cols, int nseg,
                       double* res, void* workspace, void* stream);

size_t qcb_reduce_workspace_bytes(int nseg);

/* Calibration statistics (harness.py:305-311): out[k] = max(out[k], max |x[r][k]|)
 * over the seg_valid rows of each of nseg segments (rows via x_row0, nullable);
 * out is f32 [K], initialised by the caller (0 for a fresh record). */
int qcb_col_absmax(const float* x, long long ldx, const long long* x_row0, int seg_rows,
                   int seg_valid, int nseg, int K, float* out, void* stream);

/* Stream-ordered copy of `bytes` (cudaMemcpyAsync, kind inferred from the
 * pointers): the engine's per-step table uploads and decision read-back without
 * a framework dispatch per copy. */
int qcb_copy_async(void* dst, const void* src, size_t bytes, void* stream);

/* ---------------------------------------------------------------- policy */
typedef struct QcbThresholds {  /* schedule.py:22-42 */
  double delta1, delta2;
  int tau_max, tau_mid, tau_min;
  double theta1, theta2;
  int bit_max, bit_mid, bit_min;
  double tau_high, tau_low, p_base, v_low, v_high;
  int history_k;
  double prune_adjust;
  int hlc, aigq_w, aigq_a, srap;  /* Toggles (schedule.py:213-221) */
} QcbThresholds;

/* Device-resident per-video Scheduler state (schedule.py:243-269) plus the
 * current step's decision (ScheduleDecision, schedule.py:176-184). */
typedef struct QcbPolicyVideo {
  int seen, n_d, boundary, long_skip;
  int abits, forced, pad0, pad1;
  int cache_valid[QCB_MAX_LAYERS];
  int cache_step[QCB_MAX_LAYERS];
  int cache_tau[QCB_MAX_LAYERS];
  int prev_valid[QCB_MAX_LAYERS];
  int d_order[QCB_MAX_LAYERS];      /* insertion order of last_divergences   */
  int has_d[QCB_MAX_LAYERS];
  int action[QCB_MAX_LAYERS];       /* 0 recompute, 1 reuse, 2 prune          */
  int sim_valid[QCB_MAX_LAYERS];
  int d_valid[QCB_MAX_LAYERS];      /* D computed this step                   */
  int ref_kind[QCB_MAX_LAYERS];     /* 0 none, 1 cache, 2 prev (this step)    */
  double last_d[QCB_MAX_LAYERS];
  double sim[QCB_MAX_LAYERS];
  double d_now[QCB_MAX_LAYERS];
  double v;
} QcbPolicyVideo;

enum { QCB_ACT_RECOMPUTE = 0, QCB_ACT_REUSE = 1, QCB_ACT_PRUNE = 2 };

/* plan_step part 1: boundary, HLC reuse (cache liveness), long-skip flag. */
int qcb_policy_plan_reuse(QcbPolicyVideo* st, int nvid, int L, int t, QcbThresholds th,
                          void* stream);
/* Which (video, layer) pairs need an SRAP similarity this step:
 * flags[l*nvid + v] = 1 iff srap on, not boundary, l >= 1, action recompute
 * and both previous features exist (schedule.py:296-304). */
int qcb_policy_sim_mask(const QcbPolicyVideo* st, int nvid, int L, QcbThresholds th,
                        int* flags, void* stream);
/* plan_step part 2: SRAP prune decisions from srap sums [L][nvid][3], the
 * variation V = sum_j hist_l1[j*nvid + v] over the n_hist history latents in
 * insertion order (schedule.py:128-133), and the activation bits
 * (schedule.py:293-326).  draws: prune_draw(seed_v, t, l) at
 * draws[v*draws_vid_stride + l]. */
int qcb_policy_plan_finish(QcbPolicyVideo* st, int nvid, int L, int t, QcbThresholds th,
                           const double* srap_sums, const double* hist_l1, int n_hist,
                           const double* draws, long long draws_vid_stride, void* stream);
/* observe_block for layer l: hlc sums [v][2] (valid where ref_kind != 0),
 * k per video from cache step; tau / cache / prev / last_d updates
 * (schedule.py:330-351). */
int qcb_policy_observe(QcbPolicyVideo* st, int nvid, int l, int t, QcbThresholds th,
                       const double* hlc_sums, void* stream);
/* observe_block for every layer of step t in order, hlc sums [L][nvid][2]. */
int qcb_policy_observe_all(QcbPolicyVideo* st, int nvid, int L, int t, QcbThresholds th,
                           const double* hlc_sums, void* stream);

/* ---------------------------------------------------------------- misc */
int qcb_device_sm_count(void);
const char* qcb_version(void);
const char* qcb_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* QCB200_H_ */
