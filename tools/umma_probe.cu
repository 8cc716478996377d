// tcgen05.mma kind::f16 throughput probe: one CTA per SM issues back-to-back
// MMAs (cta_group::1, operands in shared memory, D in TMEM) and reports
// cycles per instruction for a few (N, A-source) shapes.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2503_06545_b200/csrc/qc_common.cuh"
using namespace qc;
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t M, uint32_t N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(a),
               "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d), "r"(a),
               "l"(b), "r"(id), "r"(acc) : "memory");
}
template <int N, bool TS>
__global__ void probe(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tb = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    const uint32_t id = idesc_bf16(128, N);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (TS) mma_ts(tb + 256, tb + 8 * k, smem_desc_sw128(b + 32 * (k & 3)), id, 1);
        else mma_ss(tb, smem_desc_sw128(a + 32 * (k & 3)), smem_desc_sw128(b + 32 * (k & 3)), id, 1);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x < 32) tmem_free<512>(tb);
}
template <int N, bool TS>
void run(const char* name, long long* d, int sms) {
  const int iters = 2000;
  cudaFuncSetAttribute(probe<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  probe<N, TS><<<sms, 128, 65536>>>(d, iters);
  cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double s = 0; for (int i = 0; i < sms; ++i) s += h[i];
  const double cyc = s / sms / (iters * 8.0);
  const double flop = 2.0 * 128 * N * 16;
  printf("%-22s N=%3d  %.1f cycles/MMA  %.0f flop/clk/SM  (%s)\n", name, N, cyc, flop / cyc,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d; cudaMalloc(&d, 256 * 8);
  for (int r = 0; r < 2; ++r) {
    run<64, false>("SS M128 K16", d, sms);
    run<128, false>("SS M128 K16", d, sms);
    run<256, false>("SS M128 K16", d, sms);
    run<64, true>("TS M128 K16 (A tmem)", d, sms);
    run<128, true>("TS M128 K16 (A tmem)", d, sms);
  }
  return 0;
}
