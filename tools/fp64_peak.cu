// fp64 peak microbenchmark for the LU roofline: DFMA (vector) and DMMA
// (mma.sync.m8n8k4.f64) issue-bound throughput on every SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}

__global__ void dmma_kernel(double* out, double a0) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = a0 + threadIdx.x, b = a0 - threadIdx.x;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1.2345) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    const int blocks = sms * 4;
    const int threads = warps * 32 / 4;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      dfma_kernel<<<blocks, threads>>>(out, 0.999, 1e-3);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fl = 2.0 * 16 * kIters * (double)blocks * threads;
      if (rep) printf("DFMA warps/SM=%d: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
      cudaEventRecord(e0);
      dmma_kernel<<<blocks, threads>>>(out, 0.5);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double fm = 2.0 * 256 * 8 * kIters * (double)blocks * (threads / 32);
      if (rep) printf("DMMA warps/SM=%d: %.2f TFLOP/s\n", warps, fm / ms / 1e9);
    }
  }
  printf("SMs=%d clock_khz=%d err=%s\n", sms, clk, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
