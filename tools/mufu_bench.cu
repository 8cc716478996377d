// Throughput probe: ex2.approx.f32 (MUFU) and FFMA per SM per clock on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_ex2(float* out, int iters) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  float a4 = a0 + 0.4f, a5 = a0 + 0.5f, a6 = a0 + 0.6f, a7 = a0 + 0.7f;
  for (int i = 0; i < iters; ++i) {
#define E(a) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a))
    E(a0); E(a1); E(a2); E(a3); E(a4); E(a5); E(a6); E(a7);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_ffma(float* out, int iters) {
  float a[16];
  for (int j = 0; j < 16; ++j) a[j] = threadIdx.x * 1e-3f + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 16; ++j) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f3A000000;" : "+f"(a[j]));
  float s = 0; for (int j = 0; j < 16; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_mix(float* out, int iters) {   // 1 ex2 : 4 ffma interleaved
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  float b[16];
  for (int j = 0; j < 16; ++j) b[j] = a0 + j;
  for (int i = 0; i < iters; ++i) {
    E(a0); E(a1); E(a2); E(a3);
#pragma unroll
    for (int j = 0; j < 16; ++j) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f3A000000;" : "+f"(b[j]));
  }
  float s = a0 + a1 + a2 + a3; for (int j = 0; j < 16; ++j) s += b[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* o; cudaMalloc(&o, sms * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0); k_ex2<<<sms * 4, 512>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)sms * 4 * 512 * iters * 8;
    printf("ex2 : %.3f ms  %.1f G/s  per SM %.2f G/s\n", ms, n / ms / 1e6, n / ms / 1e6 / sms);
    cudaEventRecord(e0); k_ffma<<<sms * 4, 512>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    n = (double)sms * 4 * 512 * iters * 16;
    printf("ffma: %.3f ms  %.1f G/s  per SM %.2f G/s\n", ms, n / ms / 1e6, n / ms / 1e6 / sms);
    cudaEventRecord(e0); k_mix<<<sms * 4, 512>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    n = (double)sms * 4 * 512 * iters * 4;
    printf("mix (4 ex2 + 16 ffma): %.3f ms  ex2 %.1f G/s per SM %.2f G/s\n", ms, n / ms / 1e6, n / ms / 1e6 / sms);
  }
  return 0;
}
