// Dependent-chain latencies of the instructions on the batched LU's pivot chain
// (one warp, clock64 around 256 dependent operations).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_probe tools/lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(double* out, long long* cyc, double seed) {
  const int lane = threadIdx.x;
  __shared__ double sm[32];
  double x = seed + lane * 1e-3;
  unsigned u = (unsigned)lane;
  long long t0, t1;
  constexpr int N = 256;
#define TIME(k, body)                             \
  t0 = clock64();                                 \
  _Pragma("unroll 1") for (int i = 0; i < N / 8; ++i) { body; body; body; body; body; body; body; body; } \
  t1 = clock64();                                 \
  if (lane == 0) cyc[k] = (t1 - t0);
  TIME(0, x = fma(x, 0.999, 1e-9))
  TIME(1, x = x * 1.0000001)
  TIME(2, x = x + 1e-9)
  TIME(3, x = fabs(x) > 0.5 ? x - 1e-9 : x + 1e-9)
  TIME(4, x = __drcp_rn(x))
  TIME(5, u = __reduce_max_sync(0xffffffffu, u) + (unsigned)lane)
  TIME(6, x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31))
  TIME(7, u = __ballot_sync(0xffffffffu, (u & 1) != 0) + lane)
  TIME(8, u = u * 3u + 1u)
  TIME(9, {
    unsigned long long b = (unsigned long long)__double_as_longlong(x);
    x = __longlong_as_double((long long)(b ^ 1ull));
  })
  TIME(10, x = __ddiv_rn(1.0, x))
  // the substitution / pivot chains alternate pipes: fp64 result -> shuffle -> fp64
  TIME(11, x = __shfl_sync(0xffffffffu, fma(x, 0.999, 1e-9), (lane + 1) & 31))
  TIME(12, {
    sm[lane] = fma(x, 0.999, 1e-9);
    __syncwarp();
    x = sm[(lane + 1) & 31];
    __syncwarp();
  })
  out[lane] = x + u;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  probe<<<1, 32>>>(out, cyc, 1.5);
  probe<<<1, 32>>>(out, cyc, 1.5);
  cudaDeviceSynchronize();
  const char* names[] = {"DFMA", "DMUL", "DADD", "fabs>? sel (DSETP+FSEL+DADD)", "drcp_rn",
                         "REDUX.MAX +IADD", "SHFL.IDX f64", "VOTE.ballot +IADD", "IMAD",
                         "LOP xor (64-bit as 2x32)", "ddiv_rn", "DFMA -> SHFL.IDX f64 (chain)",
                         "DFMA -> STS / LDS f64 (chain)"};
  for (int k = 0; k < 13; ++k) printf("%-32s %6.1f cyc/op\n", names[k], cyc[k] / 256.0);
  return 0;
}
