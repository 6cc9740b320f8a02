// Batched fp64 LU with partial pivoting: one CTA per macro block.
//
// Replaces _factorize_local's dense branch (schur_solver.py:105-111):
// scipy.linalg.lu_factor (LAPACK getrf) + the singularity test
// min|diag U| <= 1e-13 max|A|  ->  SingularLocalBlock(macro_id).
//
// Pivot rule = LAPACK idamax (largest |a_ik|, first index on ties); the pivot
// column is scaled by the reciprocal of the pivot when |pivot| >= DBL_MIN, as
// dgetf2 does; a zero pivot skips the swap/scale (LAPACK info > 0 path).
// Output layout (device): LU column-major packed L\U per block, 1/U_jj,
// LAPACK 0-based pivots, and the composed row permutation used by the
// element kernel (x_perm[i] = x[perm[i]]).
//
// Two variants share one body:
//   * the block lives in shared memory when Q*Q*8 fits the opt-in limit
//     (Q <= 168 on B200);
//   * otherwise the block is factored in place in its HBM output slot
//     (L2-resident working set), e.g. Q = 220 (387 KB).

#include <cfloat>

#include "mh_internal.h"

namespace mh {
namespace {

constexpr int kLuThreads = 256;
constexpr int kLuMaxQ = 256;

__device__ __forceinline__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double r = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, red[w]);
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kLuThreads)
lu_kernel(const double* __restrict__ A, double* __restrict__ LU, double* __restrict__ dinv,
          int32_t* __restrict__ piv, int32_t* __restrict__ perm, int32_t* __restrict__ stat,
          int Q, int use_smem) {
  extern __shared__ double smem[];
  __shared__ double red[kLuThreads / 32];
  __shared__ int s_perm[kLuMaxQ];
  __shared__ int s_p;
  constexpr int NW = kLuThreads / 32;
  const int64_t e = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t QQ = (size_t)Q * Q;
  const double* __restrict__ Ae = A + e * QQ;
  double* W = use_smem ? smem : (LU + e * QQ);

  // load row-major A into column-major W; track max|A| for the singular test
  double amax = 0.0;
  for (size_t idx = tid; idx < QQ; idx += kLuThreads) {
    const int i = (int)(idx / Q), j = (int)(idx - (size_t)i * Q);
    const double v = __ldg(Ae + idx);
    W[(size_t)j * Q + i] = v;
    amax = fmax(amax, fabs(v));
  }
  for (int i = tid; i < Q; i += kLuThreads) s_perm[i] = i;
  amax = block_max(amax, red);  // contains __syncthreads

  for (int k = 0; k < Q; ++k) {
    double* colk = W + (size_t)k * Q;
    if (warp == 0) {  // idamax over rows k..Q-1
      double best = -1.0;
      int bi = k;
      for (int i = k + lane; i < Q; i += 32) {
        const double v = fabs(colk[i]);
        if (v > best) { best = v; bi = i; }
      }
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(kFull, best, o);
        const int oi = __shfl_xor_sync(kFull, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if (lane == 0) {
        s_p = bi;
        piv[e * Q + k] = bi;
        const int tmp = s_perm[k];
        s_perm[k] = s_perm[bi];
        s_perm[bi] = tmp;
      }
    }
    __syncthreads();
    const int p = s_p;
    const double pv = colk[p];
    if (pv != 0.0) {
      if (p != k) {  // dswap of the whole row (dgetf2)
        for (int j = tid; j < Q; j += kLuThreads) {
          double* c = W + (size_t)j * Q;
          const double a = c[k];
          c[k] = c[p];
          c[p] = a;
        }
        __syncthreads();
      }
      if (fabs(pv) >= DBL_MIN) {
        const double r = 1.0 / pv;
        for (int i = k + 1 + tid; i < Q; i += kLuThreads) colk[i] *= r;
      } else {
        for (int i = k + 1 + tid; i < Q; i += kLuThreads) colk[i] /= pv;
      }
      __syncthreads();
    }
    // rank-1 update of the trailing block: warp per column, lanes over rows
    for (int j = k + 1 + warp; j < Q; j += NW) {
      double* cj = W + (size_t)j * Q;
      const double akj = cj[k];
      for (int i = k + 1 + lane; i < Q; i += 32) cj[i] = fma(-colk[i], akj, cj[i]);
    }
    __syncthreads();
  }

  // write back, reciprocal diagonal, permutation, singular flag
  double* LUe = LU + e * QQ;
  if (use_smem)
    for (size_t idx = tid; idx < QQ; idx += kLuThreads) LUe[idx] = W[idx];
  double dmin = DBL_MAX;
  for (int i = tid; i < Q; i += kLuThreads) {
    const double d = W[(size_t)i * Q + i];
    dinv[e * Q + i] = 1.0 / d;
    perm[e * Q + i] = s_perm[i];
    dmin = fmin(dmin, fabs(d));
  }
  for (int o = 16; o; o >>= 1) dmin = fmin(dmin, __shfl_xor_sync(kFull, dmin, o));
  if (lane == 0) red[warp] = dmin;
  __syncthreads();
  if (tid == 0) {
    double m = DBL_MAX;
    for (int w = 0; w < NW; ++w) m = fmin(m, red[w]);
    stat[e] = (m <= 1e-13 * fmax(amax, 1e-300)) ? 1 : 0;
  }
}

}  // namespace

int launch_lu(mh_system* s, float* ms) {
  if (s->Q > kLuMaxQ) {
    set_error("Q > 256 is not supported by the batched LU");
    return MH_E_UNSUPPORTED;
  }
  if (s->N == 0) {
    if (ms) *ms = 0.f;
    return MH_OK;
  }
  const size_t bytes = (size_t)s->Q * s->Q * sizeof(double);
  const int static_smem = (kLuThreads / 32) * 8 + kLuMaxQ * 4 + 16;
  const int use_smem = (int)(bytes + static_smem <= (size_t)s->max_smem_optin);
  const size_t dyn = use_smem ? bytes : 0;
  if (use_smem)
    MH_CHECK_CUDA(cudaFuncSetAttribute(lu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)dyn));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ms) {
    MH_CHECK_CUDA(cudaEventCreate(&e0));
    MH_CHECK_CUDA(cudaEventCreate(&e1));
    MH_CHECK_CUDA(cudaEventRecord(e0, s->stream));
  }
  lu_kernel<<<(unsigned)s->N, kLuThreads, dyn, s->stream>>>(
      s->A.p, s->LU.p, s->dinv.p, s->piv.p, s->perm.p, s->lstat.p, s->Q, use_smem);
  MH_CHECK_CUDA(cudaGetLastError());
  if (ms) {
    MH_CHECK_CUDA(cudaEventRecord(e1, s->stream));
    MH_CHECK_CUDA(cudaEventSynchronize(e1));
    MH_CHECK_CUDA(cudaEventElapsedTime(ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  return MH_OK;
}

}  // namespace mh
