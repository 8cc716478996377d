// Microbenchmark: per-SM throughput of FP64 add, FP32 add and the f32<->f64 /
// int->f64 conversions (hardware F2F/I2F vs the ALU bit-level versions in
// qc_common.cuh).  Each kernel runs 8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2503_06545_b200/csrc/qc_common.cuh"

using namespace qc;

#define CHAIN_KERNEL(name, T, init, step)                                       \
  __global__ void name(T* out, int iters) {                                     \
    T a[8];                                                                     \
    for (int i = 0; i < 8; ++i) a[i] = init;                                    \
    for (int it = 0; it < iters; ++it) {                                        \
      _Pragma("unroll") for (int i = 0; i < 8; ++i) { step; }                   \
    }                                                                           \
    T s = a[0];                                                                 \
    for (int i = 1; i < 8; ++i) s += a[i];                                      \
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;                             \
  }

CHAIN_KERNEL(dadd_k, double, threadIdx.x * 1e-3 + i, a[i] = a[i] + 1.000001)
CHAIN_KERNEL(fadd_k, float, threadIdx.x * 1e-3f + i, a[i] = a[i] + 1.000001f)
// one F2F.F64.F32 + one F2F.F32.F64 per step (plus a DADD to keep the value moving)
CHAIN_KERNEL(f2f_hw_k, float, threadIdx.x * 1e-3f + i,
             a[i] = __double2float_rn((double)a[i] + 1.0000001))
CHAIN_KERNEL(f2f_alu_k, float, threadIdx.x * 1e-3f + i,
             a[i] = d2f_alu(f2d_alu(a[i]) + 1.0000001))
// f32 -> f64 only (round trip back via bit truncation, an ALU op)
CHAIN_KERNEL(f2d_hw_k, float, threadIdx.x * 1e-3f + i,
             a[i] = __int_as_float((int)__double2hiint((double)a[i] + 1.0000001) << 3))
CHAIN_KERNEL(f2d_alu_k, float, threadIdx.x * 1e-3f + i,
             a[i] = __int_as_float((int)__double2hiint(f2d_alu(a[i]) + 1.0000001) << 3))
// f64 -> f32 only
CHAIN_KERNEL(d2f_hw_k, double, threadIdx.x * 1e-3 + i,
             a[i] = __hiloint2double(__float_as_int(__double2float_rn(a[i])) >> 3, 7) + 1.0)
CHAIN_KERNEL(d2f_alu_k, double, threadIdx.x * 1e-3 + i,
             a[i] = __hiloint2double(__float_as_int(d2f_alu(a[i])) >> 3, 7) + 1.0)
CHAIN_KERNEL(i2d_hw_k, int, threadIdx.x + i,
             a[i] = __double2hiint((double)a[i] + 3.0))
CHAIN_KERNEL(i2d_alu_k, int, threadIdx.x + i,
             a[i] = __double2hiint(i2d_alu(a[i]) + 3.0))

template <typename T>
void run(const char* name, void (*k)(T*, int), T* buf, int blocks, int threads, int iters,
         int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<<<blocks, threads>>>(buf, 16);
  cudaEventRecord(e0);
  k<<<blocks, threads>>>(buf, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double ops = (double)blocks * threads * iters * 8;
  const double per_clk_sm = ops / (ms * 1e-3) / sms / (clk_khz * 1e3);
  printf("%-10s %9.1f Gop/s  %6.1f per SM per clk (at %d MHz nominal)\n", name,
         ops / ms / 1e6, per_clk_sm, clk_khz / 1000);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 2048;
  double* d;
  float* f;
  int* n;
  cudaMalloc(&d, blocks * threads * 8);
  cudaMalloc(&f, blocks * threads * 4);
  cudaMalloc(&n, blocks * threads * 4);
  run("DADD", dadd_k, d, blocks, threads, iters, sms);
  run("FADD", fadd_k, f, blocks, threads, iters, sms);
  run("f2f_hw", f2f_hw_k, f, blocks, threads, iters, sms);
  run("f2f_alu", f2f_alu_k, f, blocks, threads, iters, sms);
  run("f2d_hw", f2d_hw_k, f, blocks, threads, iters, sms);
  run("f2d_alu", f2d_alu_k, f, blocks, threads, iters, sms);
  run("d2f_hw", d2f_hw_k, d, blocks, threads, iters, sms);
  run("d2f_alu", d2f_alu_k, d, blocks, threads, iters, sms);
  run("i2d_hw", i2d_hw_k, n, blocks, threads, iters, sms);
  run("i2d_alu", i2d_alu_k, n, blocks, threads, iters, sms);
  return 0;
}
