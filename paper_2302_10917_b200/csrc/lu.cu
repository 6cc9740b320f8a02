// Batched fp64 LU with partial pivoting: the dispatcher and the Q <= 32 kernel.
//
// Replaces _factorize_local's dense branch (schur_solver.py:105-111):
// scipy.linalg.lu_factor (LAPACK getrf) + the singularity test
// min|diag U| <= 1e-13 max|A|  ->  SingularLocalBlock(macro_id).
//
// Pivot rule = LAPACK idamax (largest |a_ik|, first index on ties); the pivot
// column is scaled by the reciprocal of the pivot when |pivot| >= DBL_MIN, as
// dgetf2 does; a zero pivot skips the swap/scale (LAPACK info > 0 path).
// Output layout (device): per block the packed streams of the element kernel
// (strict lower L by columns 0..Q-2, strict upper U by columns Q-1..1), diag(U), 1/U_jj,
// LAPACK 0-based pivots, and the composed row permutation used by the
// element kernel (x_perm[i] = x[perm[i]]).
//
// Kernels: Q <= 32 lu_reg_kernel (below, register-resident); 32 < Q <= 256
// lu_tile_kernel (lu_tile.cu, warp per block, DMMA updates); the CTA-resident
// lu_cta_kernel (lu_cta.cu, Q <= 168) with MEHDG_LU=cta.  Earlier variants
// (CTA per block in shared memory / HBM, left-looking DFMA, shared-memory
// right-looking DMMA) were measured slower and removed.

#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <string>

#include "lu_common.cuh"

namespace mh {
namespace {

constexpr int kLuMaxQ = 256;

// ---------------------------------------------------------------------------
// Register-resident variant for Q <= 32 R <= NW NB: the whole block lives in
// registers, lane l of warp w owning rows l + 32 a and columns w + NW b.
// Column k is owned by warp k % NW, so the pivot search is a warp argmax and
// the pivot row's values reach every warp with one shuffle per column; rows
// are exchanged physically (LAPACK dgetf2 semantics) only when the pivot
// actually moves.  One CTA barrier per column step publishes the pivot and
// the multiplier column l (double-buffered in shared memory).
template <int R, int NB, int NW>
__global__ void __launch_bounds__(NW * 32, 512 / (NW * 32)) lu_reg_kernel(LuArgs g) {
  __shared__ double lcol[2][32 * R];
  __shared__ int s_p[2];
  __shared__ int s_perm[32 * R];
  __shared__ double red[NW];
  static_assert(32 % NW == 0 || NW % 32 == 0, "NW must divide 32");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e = blockIdx.x;
  const int Q = g.Q;
  const double* __restrict__ Ae = g.A + e * (int64_t)Q * Q;

  double A[R][NB];
  double amax = 0.0;
#pragma unroll
  for (int a = 0; a < R; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int i = lane + 32 * a, j = w + NW * b;
      const double v = (i < Q && j < Q) ? __ldg(Ae + (int64_t)i * Q + j) : 0.0;
      A[a][b] = v;
      amax = fmax(amax, fabs(v));
    }
  for (int o = 16; o; o >>= 1) amax = fmax(amax, __shfl_xor_sync(kFull, amax, o));
  if (lane == 0) red[w] = amax;
  for (int i = threadIdx.x; i < 32 * R; i += NW * 32) s_perm[i] = i;
  __syncthreads();
  amax = 0.0;
#pragma unroll
  for (int i = 0; i < NW; ++i) amax = fmax(amax, red[i]);
  double dmin = DBL_MAX;  // min |U_kk| (owner lanes 0)

#pragma unroll
  for (int b = 0; b < NB; ++b) {
#pragma unroll 1
    for (int kk = 0; kk < NW; ++kk) {
      const int k = b * NW + kk;
      if (k >= Q) break;
      const int buf = k & 1;
      // row k lives in register a = k / 32 = (NW b) / 32 (static: NW | 32 and
      // kk < NW), lane k % 32
      const int ak = (NW * b) >> 5, lk = k & 31;
      if (w == kk) {
        // ---- owner of column k: idamax over rows k..Q-1 (first index on ties)
        double best = -1.0;
        int bi = Q;
#pragma unroll
        for (int a = 0; a < R; ++a) {
          const int i = lane + 32 * a;
          const double v = fabs(A[a][b]);
          if (i >= k && i < Q && v > best) { best = v; bi = i; }
        }
        for (int o = 16; o; o >>= 1) {
          const double ov = __shfl_xor_sync(kFull, best, o);
          const int oi = __shfl_xor_sync(kFull, bi, o);
          if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
        }
        const int p = bi;
        // swap A[k][k] <-> A[p][k] inside this column
        double colk_p = 0.0, colk_k = 0.0;
#pragma unroll
        for (int a = 0; a < R; ++a) {
          const double vp = __shfl_sync(kFull, A[a][b], p & 31);
          const double vk = __shfl_sync(kFull, A[a][b], lk);
          colk_p = osel(a == (p >> 5), vp, colk_p);
          if (a == ak) colk_k = vk;
        }
        const double pv = colk_p;
        if (p != k && pv != 0.0) {
#pragma unroll
          for (int a = 0; a < R; ++a) {
            if (a == ak) A[a][b] = osel(lane == lk, colk_p, A[a][b]);
            A[a][b] = osel(a == (p >> 5) && lane == (p & 31), colk_k, A[a][b]);
          }
        }
        // multipliers l_i = a_ik / pivot (reciprocal when |pivot| >= DBL_MIN)
        const bool big = fabs(pv) >= DBL_MIN;
        const double rcp = 1.0 / pv;
#pragma unroll
        for (int a = 0; a < R; ++a) {
          const int i = lane + 32 * a;
          double l = 0.0;
          if (i > k && i < Q) {
            if (pv != 0.0) A[a][b] = big ? A[a][b] * rcp : A[a][b] / pv;
            l = A[a][b];
          }
          lcol[buf][i] = l;
        }
        if (lane == 0) {
          s_p[buf] = (pv != 0.0) ? p : k;
          g.piv[e * Q + k] = p;
          if (p != k) {
            const int tmp = s_perm[k];
            s_perm[k] = s_perm[p];
            s_perm[p] = tmp;
          }
          dmin = fmin(dmin, fabs(pv));
        }
      }
      __syncthreads();
      const int p = s_p[buf];
      // ---- physical row exchange k <-> p in this warp's other columns
      if (p != k) {
#pragma unroll
        for (int bb = 0; bb < NB; ++bb) {
          if (w == kk && bb == b) continue;
          double vk = 0.0, vp = 0.0;
#pragma unroll
          for (int a = 0; a < R; ++a) {
            const double xp = __shfl_sync(kFull, A[a][bb], p & 31);
            if (a == ak) vk = __shfl_sync(kFull, A[a][bb], lk);
            vp = osel(a == (p >> 5), xp, vp);
          }
#pragma unroll
          for (int a = 0; a < R; ++a) {
            if (a == ak) A[a][bb] = osel(lane == lk, vp, A[a][bb]);
            A[a][bb] = osel(a == (p >> 5) && lane == (p & 31), vk, A[a][bb]);
          }
        }
      }
      // ---- rank-1 update of the trailing columns j > k owned by this warp
      double l[R];
#pragma unroll
      for (int a = 0; a < R; ++a) l[a] = lcol[buf][lane + 32 * a];
#pragma unroll
      for (int bb = b; bb < NB; ++bb) {
        const int j = w + NW * bb;
        if (j > k && j < Q) {  // warp-uniform
          const double u = __shfl_sync(kFull, A[ak][bb], lk);
#pragma unroll
          for (int a = 0; a < R; ++a)
            if (a >= ak) A[a][bb] = fma(-l[a], u, A[a][bb]);
        }
      }
    }
  }

  // ---- outputs: packed L (columns ascending), packed U (columns
  // descending), diag(U), 1/U_kk, permutation, singular flag
  double* Lpe = g.Lp + e * g.ldL;
  double* Upe = g.Up + e * g.ldL;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int j = w + NW * b;
    if (j >= Q) continue;
    const int64_t ol = off_lower(j, Q), ou = off_upper(j, Q);
#pragma unroll
    for (int a = 0; a < R; ++a) {
      const int i = lane + 32 * a;
      if (i >= Q) continue;
      const double v = A[a][b];
      if (i > j) Lpe[ol + (i - j - 1)] = v;
      else if (i < j) Upe[ou + i] = v;
      else {
        g.udiag[e * Q + i] = v;
        g.dinv[e * Q + i] = 1.0 / v;
      }
    }
  }
  for (int64_t i = (int64_t)Q * (Q - 1) / 2 + threadIdx.x; i < g.ldL; i += NW * 32) {
    Lpe[i] = 0.0;
    Upe[i] = 0.0;
  }
  __syncthreads();  // s_perm complete
  for (int i = threadIdx.x; i < Q; i += NW * 32) g.perm[e * Q + i] = s_perm[i];
  if (lane == 0) red[w] = dmin;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = DBL_MAX;
    for (int i = 0; i < NW; ++i) m = fmin(m, red[i]);
    g.stat[e] = (m <= 1e-13 * fmax(amax, 1e-300)) ? 1 : 0;
  }
}


__global__ void unpack_lu_kernel(const double* __restrict__ Lp, const double* __restrict__ Up,
                                 const double* __restrict__ udiag, int64_t ldL, int Q,
                                 int64_t first, int64_t count, double* __restrict__ out) {
  const int64_t QQ = (int64_t)Q * Q;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < count * QQ;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = idx / QQ, e = first + b;
    const int r = (int)(idx - b * QQ);
    const int i = r / Q, j = r - i * Q;
    double v;
    if (i > j) v = Lp[e * ldL + off_lower(j, Q) + (i - j - 1)];
    else if (i < j) v = Up[e * ldL + off_upper(j, Q) + i];
    else v = udiag[e * Q + i];
    out[idx] = v;
  }
}

}  // namespace

int launch_unpack_lu(mh_system* s, int64_t first, int64_t count, double* out) {
  if (count <= 0) return MH_OK;
  const int64_t total = count * (int64_t)s->Q * s->Q;
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 65535);
  unpack_lu_kernel<<<grid, 256, 0, s->stream>>>(s->Lp.p, s->Up.p, s->udiag.p, s->ldL, s->Q, first,
                                                count, out);
  MH_CHECK_CUDA(cudaGetLastError());
  return MH_OK;
}

int launch_lu(mh_system* s, float* ms) {
  if (s->Q > kLuMaxQ) {
    set_error("Q > 256 is not supported by the batched LU");
    return MH_E_UNSUPPORTED;
  }
  if (s->N == 0) {
    if (ms) *ms = 0.f;
    return MH_OK;
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ms) {
    MH_CHECK_CUDA(cudaEventCreate(&e0));
    MH_CHECK_CUDA(cudaEventCreate(&e1));
  }
  LuArgs g;
  g.A = s->A.p;
  g.LU = nullptr;
  g.Lp = s->Lp.p;
  g.Up = s->Up.p;
  g.udiag = s->udiag.p;
  g.dinv = s->dinv.p;
  g.piv = s->piv.p;
  g.perm = s->perm.p;
  g.stat = s->lstat.p;
  g.ldL = s->ldL;
  g.nblocks = s->N;
  g.Q = s->Q;
  g.use_smem = 1;
  const int Q = s->Q;
  if (Q <= 32) {
    if (e0) MH_CHECK_CUDA(cudaEventRecord(e0, s->stream));
    lu_reg_kernel<1, 4, 8><<<(unsigned)s->N, 256, 0, s->stream>>>(g);
  } else if (s->knobs.lu == 2 && lu_cta_supported(Q)) {
    // the CTA-resident kernel (lu_cta.cu) measured slower than the warp-per-block
    // tile kernel at every BASELINE shape: selectable, not the default
    MH_CHECK(launch_lu_cta(s, g, e0));
  } else if (s->knobs.lu == 3 && lu_pipe_supported(Q)) {
    // one CTA per block, panels pipelined over its warps, L tiles in shared memory;
    // blocks that need row exchanges come back through the tile kernel (lu_pipe.cu)
    MH_CHECK(launch_lu_pipe(s, g, e0));
  } else {
    MH_CHECK(launch_lu_tile(s, g, e0));  // records e0 after its scratch allocation
  }
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
