// Batched fp64 LU with partial pivoting: one CTA per macro block.
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
// Two variants share one body:
//   * the block lives in shared memory when Q*Q*8 fits the opt-in limit
//     (Q <= 168 on B200);
//   * otherwise the block is factored in place in its HBM output slot
//     (L2-resident working set), e.g. Q = 220 (387 KB).

#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <string>

#include "lu_common.cuh"

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



__global__ void __launch_bounds__(kLuThreads) lu_kernel(LuArgs g) {
  const double* __restrict__ A = g.A;
  double* __restrict__ LU = g.LU;
  double* __restrict__ dinv = g.dinv;
  int32_t* __restrict__ piv = g.piv;
  int32_t* __restrict__ perm = g.perm;
  int32_t* __restrict__ stat = g.stat;
  const int Q = g.Q, use_smem = g.use_smem;
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

  // write the packed streams (L columns ascending, U columns descending),
  // diag(U), its reciprocal, the permutation and the singular flag
  double* Lpe = g.Lp + e * g.ldL;
  double* Upe = g.Up + e * g.ldL;
  for (int j = warp; j < Q; j += NW) {
    const double* cj = W + (size_t)j * Q;
    const int64_t ol = off_lower(j, Q), ou = off_upper(j, Q);
    for (int i = lane; i < Q; i += 32) {
      if (i > j) Lpe[ol + (i - j - 1)] = cj[i];
      else if (i < j) Upe[ou + i] = cj[i];
    }
  }
  for (int64_t i = (int64_t)Q * (Q - 1) / 2 + tid; i < g.ldL; i += kLuThreads) {
    Lpe[i] = 0.0;  // zero the pad so it streams clean
    Upe[i] = 0.0;
  }
  double dmin = DBL_MAX;
  for (int i = tid; i < Q; i += kLuThreads) {
    const double d = W[(size_t)i * Q + i];
    g.udiag[e * Q + i] = d;
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

// ---------------------------------------------------------------------------
// Blocked right-looking variant with fp64 tensor-core trailing updates.
//
// The block (padded to QP = 32 RW rows/columns, zeros outside Q) lives in
// shared memory, row-major with leading dimension LD (LD % 16 == 4 keeps the
// DMMA fragment loads bank-conflict free).  Per panel of 8 columns:
//   1. warp 0 factors the panel (rows >= c0) in registers: idamax via REDUX on
//      the bit pattern of |a_ik| (first index on ties), LAPACK row exchange,
//      reciprocal scaling, rank-1 update of the remaining panel columns;
//   2. all threads apply the panel's row exchanges to the other columns and
//      form U12 = L11^-1 A12 (one thread per trailing column);
//   3. the trailing block A22 -= L21 U12 is updated 8x8 tile by tile with
//      mma.sync.m8n8k4.f64 (SASS DMMA), two k-steps per tile.  Look-ahead:
//      warp 0 updates the next panel's tile column first and factors that
//      panel while warps 1..7 update the rest of the trailing block.
// Two CTA barriers per 8 columns.


// one 8x8 tile of A22 -= L21(rows of ti, panel columns) U12(panel rows, cols of tj)
template <int LD>
__device__ __forceinline__ void tile_update(double* Ws, int c0, int ti, int tj, int lane) {
  const int r = lane >> 2, q = lane & 3;
  const int row = ti * 8 + r, col = tj * 8 + 2 * q;
  double d0 = Ws[row * LD + col], d1 = Ws[row * LD + col + 1];
#pragma unroll
  for (int k0 = 0; k0 < 8; k0 += 4) {
    const double av = -Ws[row * LD + c0 + k0 + q];          // A: row r, k = q
    const double bv = Ws[(c0 + k0 + q) * LD + tj * 8 + r];  // B: k = q, col r
    dmma_8x8x4(d0, d1, av, bv);
  }
  Ws[row * LD + col] = d0;
  Ws[row * LD + col + 1] = d1;
}

// Panel factorisation by one warp.  AK = c0 / 32 is static (8 | 32), so the
// pivot row of every step sits in register block AK of some lane.
template <int RW, int LD, int AK>
__device__ __noinline__ double panel_factor(double* Ws, int c0, int Q, int lane, int* s_pv,
                                            int* s_perm, int* piv) {
  double P[8][RW];
#pragma unroll
  for (int jj = 0; jj < 8; ++jj)
#pragma unroll
    for (int a = AK; a < RW; ++a) P[jj][a] = Ws[(lane + 32 * a) * LD + c0 + jj];
  double dmin = DBL_MAX;
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const int k = c0 + jj;
    if (k >= Q) break;
    const int lk = k & 31;
    uint64_t key[RW];
    uint64_t best = 0;
#pragma unroll
    for (int a = AK; a < RW; ++a) {
      const int i = lane + 32 * a;
      key[a] = (i >= k && i < Q) ? (uint64_t)__double_as_longlong(fabs(P[jj][a])) + 1ull : 0ull;
      best = key[a] > best ? key[a] : best;
    }
    const unsigned hi = (unsigned)(best >> 32);
    const unsigned mhi = __reduce_max_sync(kFull, hi);
    const unsigned lo = hi == mhi ? (unsigned)(best & 0xffffffffu) : 0u;
    const unsigned mlo = __reduce_max_sync(kFull, lo);
    const uint64_t mk = ((uint64_t)mhi << 32) | mlo;
    int p = k;
#pragma unroll
    for (int a = RW - 1; a >= AK; --a) {
      const unsigned m = __ballot_sync(kFull, key[a] == mk);
      if (m) p = 32 * a + __ffs(m) - 1;
    }
    const int ap = p >> 5, lp = p & 31;
    double pv;
    if (p == k) {
      pv = __shfl_sync(kFull, P[jj][AK], lk);
    } else {
      pv = __shfl_sync(kFull, pick_r<RW>(P[jj], ap), lp);
      if (pv != 0.0) {  // exchange rows k and p inside the panel
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const double vk = __shfl_sync(kFull, P[c][AK], lk);
          const double vp = __shfl_sync(kFull, pick_r<RW>(P[c], ap), lp);
#pragma unroll
          for (int a = AK; a < RW; ++a) {
            if (a == AK) P[c][a] = osel(lane == lk, vp, P[c][a]);
            P[c][a] = osel(a == ap && lane == lp, vk, P[c][a]);
          }
        }
      }
    }
    const double rcp = __drcp_rn(pv);
    const bool scale = pv != 0.0, big = fabs(pv) >= DBL_MIN;
#pragma unroll
    for (int a = AK; a < RW; ++a) {
      const int i = lane + 32 * a;
      if (i > k && i < Q && scale) P[jj][a] = big ? P[jj][a] * rcp : P[jj][a] / pv;
    }
#pragma unroll
    for (int c = jj + 1; c < 8; ++c) {  // rank-1 update inside the panel
      const double u = __shfl_sync(kFull, P[c][AK], lk);
#pragma unroll
      for (int a = AK; a < RW; ++a)
        if (lane + 32 * a > k) P[c][a] = fma(-P[jj][a], u, P[c][a]);
    }
    if (lane == 0) {
      const int pe = scale ? p : k;
      s_pv[jj] = pe;
      piv[k] = p;
      if (pe != k) {
        const int tmp = s_perm[k];
        s_perm[k] = s_perm[pe];
        s_perm[pe] = tmp;
      }
    }
    dmin = fmin(dmin, fabs(pv));
  }
#pragma unroll
  for (int jj = 0; jj < 8; ++jj)
#pragma unroll
    for (int a = AK; a < RW; ++a) {
      const int i = lane + 32 * a;
      if (i >= c0) Ws[i * LD + c0 + jj] = P[jj][a];
    }
  return dmin;
}

template <int RW, int LD>
__device__ __forceinline__ double panel_dispatch(double* Ws, int c0, int Q, int lane, int* s_pv,
                                                 int* s_perm, int* piv) {
  switch (c0 >> 5) {
    case 0: return panel_factor<RW, LD, 0>(Ws, c0, Q, lane, s_pv, s_perm, piv);
    case 1: if (RW > 1) return panel_factor<RW, LD, (RW > 1 ? 1 : 0)>(Ws, c0, Q, lane, s_pv, s_perm, piv); break;
    case 2: if (RW > 2) return panel_factor<RW, LD, (RW > 2 ? 2 : 0)>(Ws, c0, Q, lane, s_pv, s_perm, piv); break;
    case 3: if (RW > 3) return panel_factor<RW, LD, (RW > 3 ? 3 : 0)>(Ws, c0, Q, lane, s_pv, s_perm, piv); break;
  }
  return DBL_MAX;
}

template <int RW, int LD>
__global__ void __launch_bounds__(256) lu_dmma_kernel(LuArgs g) {
  constexpr int QP = 32 * RW, NTQ = QP / 8;
  constexpr int NT = 256, NW = 8;
  extern __shared__ double Ws[];  // QP x LD row-major
  __shared__ int s_pv[8];
  __shared__ int s_perm[QP];
  __shared__ double red[NW];
  static_assert(LD % 16 == 4 && LD >= QP, "LD");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t e = blockIdx.x;
  const int Q = g.Q;
  const double* __restrict__ Ae = g.A + e * (int64_t)Q * Q;
  int* piv = g.piv + e * Q;

  double amax = 0.0;
  for (int idx = tid; idx < QP * QP; idx += NT) {
    const int i = idx / QP, j = idx - i * QP;
    const double v = (i < Q && j < Q) ? __ldg(Ae + (int64_t)i * Q + j) : 0.0;
    Ws[i * LD + j] = v;
    amax = fmax(amax, fabs(v));
  }
  for (int i = tid; i < QP; i += NT) s_perm[i] = i;
  for (int o = 16; o; o >>= 1) amax = fmax(amax, __shfl_xor_sync(kFull, amax, o));
  if (lane == 0) red[warp] = amax;
  __syncthreads();
  amax = 0.0;
#pragma unroll
  for (int i = 0; i < NW; ++i) amax = fmax(amax, red[i]);
  double dmin = DBL_MAX;
  const int npanel = (Q + 7) / 8;
  if (warp == 0) dmin = panel_dispatch<RW, LD>(Ws, 0, Q, lane, s_pv, s_perm, piv);
  __syncthreads();

  for (int pnl = 0; pnl < npanel; ++pnl) {
    const int c0 = pnl * 8;
    // ---- 2. row exchanges outside the panel + U12 = L11^-1 A12
    const int ncolp = min(8, Q - c0);
    for (int j = tid; j < QP; j += NT) {
      if (j >= c0 && j < c0 + 8) continue;
      for (int jj = 0; jj < ncolp; ++jj) {
        const int k = c0 + jj, p = s_pv[jj];
        if (p != k) {
          const double t = Ws[k * LD + j];
          Ws[k * LD + j] = Ws[p * LD + j];
          Ws[p * LD + j] = t;
        }
      }
      if (j >= c0 + 8) {
        double u[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) u[r] = Ws[(c0 + r) * LD + j];
#pragma unroll
        for (int r = 1; r < 8; ++r)
#pragma unroll
          for (int m = 0; m < r; ++m) u[r] = fma(-Ws[(c0 + r) * LD + c0 + m], u[m], u[r]);
#pragma unroll
        for (int r = 0; r < 8; ++r) Ws[(c0 + r) * LD + j] = u[r];
      }
    }
    __syncthreads();
    // ---- 3. trailing update; warp 0 runs ahead to the next panel
    const int t0 = pnl + 1;
    if (t0 < NTQ) {
      if (warp == 0) {
        for (int ti = t0; ti < NTQ; ++ti) tile_update<LD>(Ws, c0, ti, t0, lane);
        __syncwarp();
        if (pnl + 1 < npanel)
          dmin = fmin(dmin, panel_dispatch<RW, LD>(Ws, c0 + 8, Q, lane, s_pv, s_perm, piv));
      } else {
        const int ncol = NTQ - t0 - 1;  // tile columns t0+1 .. NTQ-1
        if (ncol > 0) {
          int ti = t0, tj = t0 + 1 + (warp - 1);
          while (tj >= NTQ) { tj -= ncol; ++ti; }
          while (ti < NTQ) {
            tile_update<LD>(Ws, c0, ti, tj, lane);
            tj += NW - 1;
            while (tj >= NTQ) { tj -= ncol; ++ti; }
          }
        }
      }
    }
    __syncthreads();
  }

  // ---- outputs (same packed streams as the other variants)
  double* Lpe = g.Lp + e * g.ldL;
  double* Upe = g.Up + e * g.ldL;
  for (int j = warp; j < Q; j += NW) {
    const int64_t ol = off_lower(j, Q), ou = off_upper(j, Q);
    for (int i = lane; i < Q; i += 32) {
      const double v = Ws[i * LD + j];
      if (i > j) Lpe[ol + (i - j - 1)] = v;
      else if (i < j) Upe[ou + i] = v;
      else {
        g.udiag[e * Q + i] = v;
        g.dinv[e * Q + i] = 1.0 / v;
      }
    }
  }
  for (int64_t i = (int64_t)Q * (Q - 1) / 2 + tid; i < g.ldL; i += NT) {
    Lpe[i] = 0.0;
    Upe[i] = 0.0;
  }
  for (int i = tid; i < Q; i += NT) g.perm[e * Q + i] = s_perm[i];
  if (tid == 0) g.stat[e] = (dmin <= 1e-13 * fmax(amax, 1e-300)) ? 1 : 0;
}

// ---------------------------------------------------------------------------
// Left-looking blocked variant: ONE WARP PER BLOCK, no shared-memory copy of
// the matrix, so many blocks are in flight per SM (the limiter of the
// CTA-per-block kernels is the dependent pivot chain of each block).
//
// Rows are tracked by position (prow[i] = original row now at position i, the
// composed LAPACK permutation).  For each 8-column panel (columns c0..c0+7):
//   1. gather the panel rows of the ORIGINAL matrix through prow (each entry
//      of A is read exactly once overall);
//   2. for every previous panel kb: U_kb = L11(kb)^-1 rows(kb) (8x8 solve,
//      lanes over columns, via a per-warp shared 8x8 tile), written to the
//      packed U stream, then rows below -= L(rows, kb) U_kb (L read back from
//      the packed L stream -- L2 resident);
//   3. factor the panel (idamax via REDUX, LAPACK row exchange -- mirrored on
//      the already stored L rows, rare --, reciprocal scaling, rank-1 updates);
//   4. store L (packed, by position), U (packed) and the diagonal.
// The factors land directly in the streams the element kernel reads.
template <int R>
__device__ __forceinline__ double lpk(const double* Lpe, int i, int j, int Q) {
  return Lpe[off_lower(j, Q) + (i - j - 1)];
}

constexpr int kLeftWarps = 4;  // blocks (one per warp) per CTA

template <int R>
__global__ void __launch_bounds__(kLeftWarps * 32) lu_left_kernel(LuArgs g) {
  __shared__ double Ssh[kLeftWarps][64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * kLeftWarps + w;
  const int Q = g.Q;
  if (e >= g.nblocks) return;
  const double* __restrict__ Ae = g.A + e * (int64_t)Q * Q;
  double* Lpe = g.Lp + e * g.ldL;  // L is stored in place (L2 resident while in use)
  double* Upe = g.Up + e * g.ldL;
  int* piv = g.piv + e * Q;
  double* S = Ssh[w];

  int prow[R];
#pragma unroll
  for (int a = 0; a < R; ++a) prow[a] = lane + 32 * a;
  double amax = 0.0, dmin = DBL_MAX;
  const int npanel = (Q + 7) / 8;

  for (int jb = 0; jb < npanel; ++jb) {
    const int c0 = 8 * jb;
    const int ncol = min(8, Q - c0);
    // ---- 1. gather the panel (rows by position)
    double P[8][R];
#pragma unroll
    for (int a = 0; a < R; ++a) {
      const int i = lane + 32 * a;
      const double* row = Ae + (int64_t)prow[a] * Q + c0;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double v = (i < Q && c < ncol) ? __ldg(row + c) : 0.0;
        P[c][a] = v;
        amax = fmax(amax, fabs(v));
      }
    }
    // ---- 2. left-looking update with the previous panels
    for (int kb = 0; kb < jb; ++kb) {
      const int k0 = 8 * kb;
      // (a) rows k0..k0+7 of the panel -> S (8 x 8, row-major)
#pragma unroll
      for (int a = 0; a < R; ++a) {
        const int i = lane + 32 * a;
        if (i >= k0 && i < k0 + 8)
#pragma unroll
          for (int c = 0; c < 8; ++c) S[(i - k0) * 8 + c] = P[c][a];
      }
      __syncwarp();
      if (lane < 8) {  // unit-lower solve, lane = panel column
        double u[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) u[r] = S[r * 8 + lane];
#pragma unroll
        for (int r = 1; r < 8; ++r)
#pragma unroll
          for (int m = 0; m < r; ++m) u[r] = fma(-lpk<R>(Lpe, k0 + r, k0 + m, Q), u[m], u[r]);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          S[r * 8 + lane] = u[r];
          if (lane < ncol) Upe[off_upper(c0 + lane, Q) + k0 + r] = u[r];
        }
      }
      __syncwarp();
      // (b) rows below: P -= L(rows, k0..k0+7) U_kb
#pragma unroll
      for (int a = 0; a < R; ++a) {
        const int i = lane + 32 * a;
        if (i >= k0 + 8 && i < Q) {
          double l[8];
#pragma unroll
          for (int m = 0; m < 8; ++m) l[m] = lpk<R>(Lpe, i, k0 + m, Q);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            double acc = P[c][a];
#pragma unroll
            for (int m = 0; m < 8; ++m) acc = fma(-l[m], S[m * 8 + c], acc);
            P[c][a] = acc;
          }
        }
      }
      __syncwarp();
    }
    // ---- 3. factor the panel (positions >= c0)
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int k = c0 + jj;
      if (jj >= ncol) break;
      const int lk = k & 31, ak = k >> 5;
      uint64_t key[R];
      uint64_t best = 0;
#pragma unroll
      for (int a = 0; a < R; ++a) {
        const int i = lane + 32 * a;
        key[a] = (i >= k && i < Q) ? (uint64_t)__double_as_longlong(fabs(P[jj][a])) + 1ull : 0ull;
        best = key[a] > best ? key[a] : best;
      }
      const unsigned hi = (unsigned)(best >> 32);
      const unsigned mhi = __reduce_max_sync(kFull, hi);
      const unsigned lo = hi == mhi ? (unsigned)(best & 0xffffffffu) : 0u;
      const unsigned mlo = __reduce_max_sync(kFull, lo);
      const uint64_t mk = ((uint64_t)mhi << 32) | mlo;
      int p = k;
#pragma unroll
      for (int a = R - 1; a >= 0; --a) {
        const unsigned m = __ballot_sync(kFull, key[a] == mk);
        if (m) p = 32 * a + __ffs(m) - 1;
      }
      const int ap = p >> 5, lp = p & 31;
      const double pv = __shfl_sync(kFull, pick_r<R>(P[jj], ap), lp);
      if (p != k && pv != 0.0) {
        // exchange positions k and p: panel values, prow, stored L rows
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const double vk = __shfl_sync(kFull, pick_r<R>(P[c], ak), lk);
          const double vp = __shfl_sync(kFull, pick_r<R>(P[c], ap), lp);
#pragma unroll
          for (int a = 0; a < R; ++a) {
            P[c][a] = osel(a == ak && lane == lk, vp, P[c][a]);
            P[c][a] = osel(a == ap && lane == lp, vk, P[c][a]);
          }
        }
        int rk = 0, rp = 0;
#pragma unroll
        for (int a = 0; a < R; ++a) {
          const int xk = __shfl_sync(kFull, prow[a], lk);
          const int xp = __shfl_sync(kFull, prow[a], lp);
          if (a == ak) rk = xk;
          if (a == ap) rp = xp;
        }
#pragma unroll
        for (int a = 0; a < R; ++a) {
          if (a == ak && lane == lk) prow[a] = rp;
          if (a == ap && lane == lp) prow[a] = rk;
        }
        for (int j = lane; j < c0; j += 32) {  // stored L rows k, p (columns < c0)
          double* ck = Lpe + off_lower(j, Q) + (k - j - 1);
          double* cp = Lpe + off_lower(j, Q) + (p - j - 1);
          const double t = *ck;
          *ck = *cp;
          *cp = t;
        }
        __syncwarp();
      }
      const bool scale = pv != 0.0, big = fabs(pv) >= DBL_MIN;
      const double rcp = __drcp_rn(pv);
#pragma unroll
      for (int a = 0; a < R; ++a) {
        const int i = lane + 32 * a;
        if (i > k && i < Q && scale) P[jj][a] = big ? P[jj][a] * rcp : P[jj][a] / pv;
      }
#pragma unroll
      for (int c = jj + 1; c < 8; ++c) {
        const double u = __shfl_sync(kFull, pick_r<R>(P[c], ak), lk);
#pragma unroll
        for (int a = 0; a < R; ++a)
          if (lane + 32 * a > k) P[c][a] = fma(-P[jj][a], u, P[c][a]);
      }
      if (lane == 0) piv[k] = p;
      dmin = fmin(dmin, fabs(pv));
    }
    // ---- 4. store: L below the diagonal, U above (within the panel), diag
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (c >= ncol) break;
      const int j = c0 + c;
      const int64_t ol = off_lower(j, Q), ou = off_upper(j, Q);
#pragma unroll
      for (int a = 0; a < R; ++a) {
        const int i = lane + 32 * a;
        if (i >= Q || i < c0) continue;
        const double v = P[c][a];
        if (i > j) Lpe[ol + (i - j - 1)] = v;
        else if (i < j) Upe[ou + i] = v;
        else {
          g.udiag[e * Q + i] = v;
          g.dinv[e * Q + i] = 1.0 / v;
        }
      }
    }
    __syncwarp();
  }
  for (int64_t i = (int64_t)Q * (Q - 1) / 2 + lane; i < g.ldL; i += 32) {
    Lpe[i] = 0.0;
    Upe[i] = 0.0;
  }
#pragma unroll
  for (int a = 0; a < R; ++a) {
    const int i = lane + 32 * a;
    if (i < Q) g.perm[e * Q + i] = prow[a];
  }
  for (int o = 16; o; o >>= 1) amax = fmax(amax, __shfl_xor_sync(kFull, amax, o));
  if (lane == 0) g.stat[e] = (dmin <= 1e-13 * fmax(amax, 1e-300)) ? 1 : 0;
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
  }
  LuArgs g;
  g.A = s->A.p;
  g.LU = s->LU.p;
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
  g.use_smem = use_smem;
  const int Q = s->Q;
  const unsigned grid = (unsigned)s->N;
  // kernel choice: warp-per-block tile LU with DMMA updates for Q > 32 (lu_tile.cu);
  // MEHDG_LU=left|dmma|reg selects the earlier kernels for comparison
  const char* var = getenv("MEHDG_LU");
  const std::string choice = var ? std::string(var) : std::string();
  // the CTA-resident kernel (lu_cta.cu) measured slower than the warp-per-block
  // tile kernel at every BASELINE shape: selectable, not the default
  const bool cta = choice == "cta" && lu_cta_supported(Q);
  const bool tile = !cta && (choice.empty() || choice == "tile" || choice == "cta") && Q > 32;
  const bool left = choice == "left" || (choice == "dmma" && Q > 96) || (choice == "reg" && Q > 128);
  if (e0 && !tile && !cta) MH_CHECK_CUDA(cudaEventRecord(e0, s->stream));
  if (cta) {
    MH_CHECK(launch_lu_cta(s, g, e0));
  } else if (tile) {
    MH_CHECK(launch_lu_tile(s, g, e0));  // records e0 after its scratch allocation
  } else if (left) {
    const unsigned gw = (unsigned)((s->N + kLeftWarps - 1) / kLeftWarps);
#define MH_LEFT(RR)                                                   \
  case RR:                                                            \
    lu_left_kernel<RR><<<gw, kLeftWarps * 32, 0, s->stream>>>(g);     \
    break;
    switch ((Q + 31) / 32) {
      MH_LEFT(1) MH_LEFT(2) MH_LEFT(3) MH_LEFT(4) MH_LEFT(5) MH_LEFT(6) MH_LEFT(7)
      default: MH_LEFT(8)
    }
#undef MH_LEFT
  } else if (Q <= 32) lu_reg_kernel<1, 4, 8><<<grid, 256, 0, s->stream>>>(g);
  else if (Q <= 64 && choice != "reg") {
    constexpr int LD = 68;
    const size_t sm = (size_t)64 * LD * sizeof(double);
    MH_CHECK_CUDA(cudaFuncSetAttribute(lu_dmma_kernel<2, LD>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    lu_dmma_kernel<2, LD><<<grid, 256, sm, s->stream>>>(g);
  } else if (Q <= 96 && choice != "reg") {
    constexpr int LD = 100;
    const size_t sm = (size_t)96 * LD * sizeof(double);
    MH_CHECK_CUDA(cudaFuncSetAttribute(lu_dmma_kernel<3, LD>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    lu_dmma_kernel<3, LD><<<grid, 256, sm, s->stream>>>(g);
  } else if (Q <= 64) lu_reg_kernel<2, 8, 8><<<grid, 256, 0, s->stream>>>(g);
  else if (Q <= 96) lu_reg_kernel<3, 12, 8><<<grid, 256, 0, s->stream>>>(g);
  else if (Q <= 128) lu_reg_kernel<4, 8, 16><<<grid, 512, 0, s->stream>>>(g);
  else {
    if (!use_smem) {
      MH_CHECK(s->LU.alloc((size_t)s->N * s->Q * s->Q));
      g.LU = s->LU.p;
    }
    lu_kernel<<<grid, kLuThreads, dyn, s->stream>>>(g);
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
