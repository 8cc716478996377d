// Internal launcher declarations shared by the .cu translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "../../include/qcb200.h"

namespace qc {
// Last CUDA error seen by a launcher (reported by qcb_last_error()).
extern cudaError_t g_last_err;

// Status of the launch just issued: QCB_OK or QCB_ERR_CUDA (error recorded).
inline int launch_status() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_last_err = e;
    return QCB_ERR_CUDA;
  }
  return QCB_OK;
}

// Programmatic dependent launch: the kernel may begin (prologue: barrier init,
// TMEM allocation, descriptor prefetch) while the previous kernel on the
// stream drains; it must execute griddepcontrol.wait (pdl_wait()) before
// touching anything that kernel wrote.  Every kernel launched this way does.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// Same, as (2,1,1) clusters (grid.x even).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_pair(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;   // CTA pairs (tcgen05 cta_group::2)
  attr[1].val.clusterDim.x = 2;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// Opt a kernel into the full dynamic shared-memory carve-out once.
template <typename K>
inline void allow_max_smem(K kernel, bool& done) {
  if (!done) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    done = true;
  }
}

int num_sms();
// cuTensorMapEncodeTiled from the driver (nullptr when unavailable)
PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn();
int attention_bf16_launch(const QcbAttentionBf16* a, cudaStream_t st);
int pick_block_n(int N);
// Grouped launch: output column group j (group n columns) reduces over
// K_j = (j+1)*k with row sums a_rowsum + j*rowsum_stride.
struct GemmGroup {
  int n, k;
  long long rowsum_stride;
};
int gemm_u8_launch(const QcbGemm* g, cudaStream_t st, const GemmGroup* grp = nullptr);
int gemm_f64_launch(const QcbGemmF64* g, cudaStream_t st);
int head_prep_launch(const float* w, int K, int N, void* prep, cudaStream_t st);
// 2-D u8 tensor map [rows][ld] (K valid columns), box kBlockK x box_rows, SWIZZLE_128B
int make_map_u8(CUtensorMap* map, const void* base, int rows, int K, long long ld, int box_rows);
int head_gemm_launch(const QcbHeadGemm* g, cudaStream_t st);
int act_quant_launch(const QcbActQuant* q, cudaStream_t st);
int weight_prep_launch(const QcbWeightPrep* q, cudaStream_t st);
int ln_mod_launch(const QcbLnMod* q, cudaStream_t st);
int attention_f64_launch(const QcbAttention* a, cudaStream_t st);
int ddpm_launch(const QcbDdpm* d, cudaStream_t st);
int pack_w4_launch(const uint8_t* codes, long long ldk, int N, int K, uint8_t* packed,
                   long long ldwp, cudaStream_t st);
int cfg_combine_launch(const float* ec, const float* eu, float scale, float* out, long long n,
                       cudaStream_t st);
int gelu_launch(float* x, long long ld, int rows, int cols, cudaStream_t st);
}  // namespace qc
