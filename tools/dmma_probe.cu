// DMMA.8x8x4 latency and per-SM-sub-partition throughput (design probe for lu_cta.cu)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void mma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double* out, long long* cyc, int iters) {
  double c[CH][2];
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = threadIdx.x;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) mma(c[i][0], c[i][1], a, b);
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x % 32 == 0) cyc[blockIdx.x * 32 + threadIdx.x / 32] = t1 - t0;
}
template <int CH>
void run(int warps, const char* tag) {
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 20); cudaMallocManaged(&cyc, 1 << 16);
  const int iters = 1000;
  k<CH><<<1, 32 * warps>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  double mx = 0;
  for (int w = 0; w < warps; ++w) mx = cyc[w] > mx ? cyc[w] : mx;
  printf("%-10s chains/warp=%2d warps/SM=%2d: %.1f cyc per DMMA per warp, %.2f cyc per DMMA per SM\n",
         tag, CH, warps, mx / (iters * CH), mx / (iters * CH * warps));
}
int main() {
  run<1>(1, "latency");
  run<2>(1, "");
  run<4>(1, "");
  run<8>(1, "");
  run<4>(2, "");
  run<4>(4, "");
  run<8>(4, "");
  run<4>(8, "");
  run<8>(8, "");
  run<4>(16, "");
  return 0;
}
