// Helpers shared by the batched LU kernels (lu.cu, lu_tile.cu).
#pragma once

#include <cfloat>

#include "mh_internal.h"

namespace mh {

struct LuArgs {
  const double* A;   // N x Q x Q row-major input
  double* LU;        // workspace (global variant only)
  double* Lp;        // N x ldL packed strict lower, columns 0..Q-2
  double* Up;        // N x ldL packed strict upper, columns Q-1..1
  double* udiag;     // N x Q
  double* dinv;      // N x Q
  int32_t* piv;      // N x Q
  int32_t* perm;     // N x Q
  int32_t* stat;     // N
  int64_t ldL;
  int64_t nblocks;
  int Q;
  int use_smem;
};

int launch_lu_tile(mh_system* s, const LuArgs& g, cudaEvent_t start, const int64_t* list = nullptr,
                   const int* list_count = nullptr, int64_t nwork = -1);
int launch_lu_pipe(mh_system* s, const LuArgs& g, cudaEvent_t start);
int launch_lu_cta(mh_system* s, const LuArgs& g, cudaEvent_t start);
bool lu_cta_supported(int Q);
bool lu_pipe_supported(int Q);

namespace {


// packed-layout offsets (see element.cu)
__host__ __device__ __forceinline__ int64_t off_lower(int j, int Q) {
  return (int64_t)j * (Q - 1) - (int64_t)j * (j - 1) / 2;
}
__host__ __device__ __forceinline__ int64_t off_upper(int j, int Q) {
  return (int64_t)Q * (Q - 1) / 2 - (int64_t)j * (j + 1) / 2;
}

// opaque select: keeps "for a: if (a == x) r[a] = v" from being turned into
// a dynamically indexed (local-memory) register array access
__device__ __forceinline__ double osel(bool c, double x, double y) {
  double r;
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n selp.f64 %0, %1, %2, q;\n}"
      : "=d"(r) : "d"(x), "d"(y), "r"((int)c));
  return r;
}

template <int RW>
__device__ __forceinline__ double pick_r(const double (&col)[RW], int a_sel) {
  double v = col[0];
#pragma unroll
  for (int a = 1; a < RW; ++a) v = osel(a == a_sel, col[a], v);
  return v;
}

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

}  // namespace
}  // namespace mh
