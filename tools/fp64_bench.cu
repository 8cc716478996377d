// Microbenchmark: FP64 add / f32<->f64 conversion / FP32 add throughput per SM.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dadd_k(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = a[i] + 1.000001;
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void fadd_k(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = a[i] + 1.000001f;
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void f2f_k(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = (float)((double)a[i] * 1.0000001);  // F2F, DMUL, F2F
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  double* d;
  float* f;
  cudaMalloc(&d, blocks * threads * 8);
  cudaMalloc(&f, blocks * threads * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const double ops = (double)blocks * threads * iters * 8;
  dadd_k<<<blocks, threads>>>(d, 16);
  cudaEventRecord(e0);
  dadd_k<<<blocks, threads>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("DADD: %.1f Gop/s  (%.1f per SM per ns)\n", ops / ms / 1e6, ops / ms / 1e6 / sms);
  fadd_k<<<blocks, threads>>>(f, 16);
  cudaEventRecord(e0);
  fadd_k<<<blocks, threads>>>(f, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("FADD: %.1f Gop/s\n", ops / ms / 1e6);
  f2f_k<<<blocks, threads>>>(f, 16);
  cudaEventRecord(e0);
  f2f_k<<<blocks, threads>>>(f, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("F2F+DMUL+F2F chains: %.1f Gelem/s\n", ops / ms / 1e6);
  return 0;
}
