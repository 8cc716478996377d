// Internal launcher declarations shared by the .cu translation units.
#pragma once
#include <cuda_runtime.h>

#include "../../include/qcb200.h"

namespace qc {
int num_sms();
int pick_block_n(int N);
int gemm_u8_launch(const QcbGemm* g, cudaStream_t st);
int gemm_f64_launch(const QcbGemmF64* g, cudaStream_t st);
int act_quant_launch(const QcbActQuant* q, cudaStream_t st);
int weight_prep_launch(const QcbWeightPrep* q, cudaStream_t st);
int ln_mod_launch(const QcbLnMod* q, cudaStream_t st);
int attention_f64_launch(const QcbAttention* a, cudaStream_t st);
int ddpm_launch(const QcbDdpm* d, cudaStream_t st);
}  // namespace qc
