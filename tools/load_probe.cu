// How fast can a persistent CTA (one per SM) pull Q x Q row-major fp64 blocks
// from HBM into swizzled shared-memory tiles?  (design probe for lu_cta.cu)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/load_probe tools/load_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NT = 21;
__device__ __forceinline__ int swz(int r) { return ((r & 2) << 1) | ((r & 4) >> 1); }
__device__ __forceinline__ int tpos(int r, int c) { return 8 * r + (c ^ swz(r)); }

template <int MODE, int W, int UN>
__global__ void __launch_bounds__(W * 32, 1) load_k(const double* A, int Q, int nb, double* out,
                                                     long long* cyc) {
  extern __shared__ __align__(16) double T[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double acc = 0.0;
  long long tl = 0;
  for (int e = blockIdx.x; e < nb; e += gridDim.x) {
    const double* Ae = A + (int64_t)e * Q * Q;
    if (MODE == 2 && threadIdx.x == 0 && e + gridDim.x < nb) {
      const uintptr_t b0 = reinterpret_cast<uintptr_t>(A + (int64_t)(e + gridDim.x) * Q * Q) & ~uintptr_t(15);
      const uintptr_t b1 = (reinterpret_cast<uintptr_t>(A + (int64_t)(e + gridDim.x + 1) * Q * Q) + 15) & ~uintptr_t(15);
      for (uintptr_t b = b0; b < b1; b += 32768) {
        const unsigned n = (unsigned)((b1 - b) < 32768 ? (b1 - b) : 32768);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b), "r"(n) : "memory");
      }
    }
    const long long t0 = clock64();
    if (MODE == 0 || MODE == 2) {  // half tiles, 8-byte loads
      const int rr = lane >> 3, cc = lane & 7;
      for (int h0 = w; h0 < 2 * NT * NT; h0 += UN * W) {
        double v[UN];
#pragma unroll
        for (int k = 0; k < UN; ++k) {
          const int h = h0 + k * W;
          const int t = h >> 1, ti = t % NT, tj = t / NT;
          const int row = 8 * ti + 4 * (h & 1) + rr, col = 8 * tj + cc;
          v[k] = (h < 2 * NT * NT && row < Q && col < Q) ? __ldg(Ae + row * Q + col) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < UN; ++k) {
          const int h = h0 + k * W;
          if (h < 2 * NT * NT) T[(h >> 1) * 64 + tpos(4 * (h & 1) + rr, cc)] = v[k];
        }
      }
    } else if (MODE == 1) {  // row-contiguous: each warp a row, 8-byte loads, scattered stores
      for (int i0 = w; i0 < Q; i0 += W) {
        for (int c = lane; c < Q; c += 32) {
          const double x = __ldg(Ae + i0 * Q + c);
          T[((c >> 3) * NT + (i0 >> 3)) * 64 + tpos(i0 & 7, c & 7)] = x;
        }
      }
    }
    __syncthreads();
    tl += clock64() - t0;
    acc += T[(threadIdx.x * 97) % (NT * NT * 64)];
    __syncthreads();
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = tl;
}

template <int MODE, int W, int UN>
void run(const double* A, int Q, int nb, double* out, long long* cyc, int sms, const char* name) {
  const size_t smem = NT * NT * 64 * 8;
  cudaFuncSetAttribute(load_k<MODE, W, UN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  load_k<MODE, W, UN><<<sms, W * 32, smem>>>(A, Q, nb, out, cyc);
  cudaEventRecord(a);
  load_k<MODE, W, UN><<<sms, W * 32, smem>>>(A, Q, nb, out, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double gb = (double)nb * Q * Q * 8 / 1e9;
  printf("%-28s %7.3f ms  %7.1f GB/s  load cycles/block (CTA 0) %lld  err=%s\n", name, ms, gb / ms * 1e3,
         c / ((nb + sms - 1) / sms), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int Q = 165, nb = 48000;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *A, *out;
  long long* cyc;
  cudaMalloc(&A, (size_t)nb * Q * Q * 8);
  cudaMemset(A, 0, (size_t)nb * Q * Q * 8);
  cudaMalloc(&out, sms * 1024 * 8);
  cudaMalloc(&cyc, sms * 8);
  run<0, 8, 8>(A, Q, nb, out, cyc, sms, "half-tile W8 un8");
  run<0, 8, 16>(A, Q, nb, out, cyc, sms, "half-tile W8 un16");
  run<0, 16, 8>(A, Q, nb, out, cyc, sms, "half-tile W16 un8");
  run<2, 8, 8>(A, Q, nb, out, cyc, sms, "half-tile W8 un8 +prefetch");
  run<2, 8, 16>(A, Q, nb, out, cyc, sms, "half-tile W8 un16 +prefetch");
  run<1, 8, 1>(A, Q, nb, out, cyc, sms, "row per warp");
  return 0;
}
