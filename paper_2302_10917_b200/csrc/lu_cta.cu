// Batched fp64 LU with partial pivoting, one CTA per block, the whole block
// resident in shared memory (Q <= 168: 227 KB at Q = 165), DMMA updates.
//
// Replaces _factorize_local's dense branch (schur_solver.py:105-111):
// scipy.linalg.lu_factor (LAPACK getrf, partial pivoting, first index on ties)
// and the singularity test min|diag U| <= 1e-13 max|A|.  Same outputs as the
// other LU kernels: the packed L / U streams the element kernel reads,
// diag(U), 1/U_jj, LAPACK pivots, composed row permutation, status.
//
// Right-looking by panels of 8 columns (one tile column) with a look-ahead of
// one panel.  The block lives in shared memory as NT x NT tiles of 8 x 8
// doubles (tile (ti, tj) at (tj NT + ti) 64), element (r, c) of a tile at
// 8 r + (c ^ swz(r)), swz(r) = 4 bit1(r) + 2 bit2(r).  That swizzle makes every
// access of the kernel conflict-free: the A fragment (8 x 4) and B fragment
// (4 x 8) loads of mma.m8n8k4.f64 (8-byte loads), the C fragment as one
// 16-byte load per lane (the pair (2q, 2q+1) stays adjacent), and the panel
// warp's column-pair loads of 32 consecutive rows.
//
// Per panel p (columns 8p .. 8p+7):
//   F_p  (warp 0) the panel's rows >= 8p in registers (lane l, register a <->
//        row 8p + l + 32 a): idamax = per-lane max, the warp max of the high
//        word of |a| (REDUX), and -- only when several lanes share that word --
//        of the low word and the first position (LAPACK's first index on ties);
//        reciprocal scaling (division below DBL_MIN, as dgetf2), rank-1
//        updates; a row exchange goes out of line through shared memory.  L
//        goes straight to its packed stream, the diagonal block's U too, and
//        -L11^-1 (8 x 8) to shared memory in A-fragment order.
//   W_p  (all, only when F_p exchanged rows) the exchanges on the columns right
//        of the panel (shared memory), on the L stream of the columns left of
//        it (global) and on the composed permutation.
//   U_p  (all) column p+1: -U(p, p+1) = (-L11^-1) A(p, p+1) (2 DMMA, each warp)
//        and C(i, p+1) += L(i, p) (-U(p, p+1)) over the row tiles i > p.
//   then, concurrently:
//        warp 0:      F_{p+1}                              (look-ahead)
//        warps 1..:   -U(p, j) for j >= p+2 (in place; U to its stream), then
//                     C(i, j) += L(i, p) (-U(p, j)) in 2 x 2 tile units.
// The L and U of a finished panel leave shared memory at once (their streams
// in global memory); a later row exchange patches the L stream there.

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "lu_common.cuh"


namespace mh {
namespace {

__device__ __forceinline__ int swz(int r) { return ((r & 2) << 1) | ((r & 4) >> 1); }
__device__ __forceinline__ int tpos(int r, int c) { return 8 * r + (c ^ swz(r)); }

__device__ __forceinline__ void mma_acc(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ uint64_t pol_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void st_ef(double* ptr, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(ptr), "d"(v), "l"(pol));
}

// B fragment k-step kk of an 8 x 8 tile held in C layout (see lu_tile.cu)
__device__ __forceinline__ double bfrag_c(double x0, double x1, int kk, int lane) {
  const int src = 4 * (4 * kk + (lane & 3)) + (lane >> 3);
  const double v0 = __shfl_sync(kFull, x0, src);
  const double v1 = __shfl_sync(kFull, x1, src);
  return ((lane >> 2) & 1) ? v1 : v0;
}

__device__ __forceinline__ int ol(int j, int Q) { return j * (Q - 1) - j * (j - 1) / 2; }
__device__ __forceinline__ int ou(int j, int Q) { return Q * (Q - 1) / 2 - j * (j + 1) / 2; }

__device__ __forceinline__ double div_slow(double x, double y) { return x / y; }

__device__ __forceinline__ unsigned hiabs(double x) {
  return (unsigned)((uint64_t)__double_as_longlong(x) >> 32) & 0x7fffffffu;
}

__device__ __noinline__ int singular_reread(const double* Ae, int n, double dmin, int lane) {
  double m = 0.0;
  for (int i = lane; i < n; i += 32) m = fmax(m, fabs(Ae[i]));
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(kFull, m, o));
  return dmin <= 1e-13 * fmax(m, 1e-300) ? 1 : 0;
}

// min|U_jj| <= 1e-13 max|A| from the block max H of the high words of |a_ij|:
// max|A| lies in [H:0, H:ffffffff]; between the bounds the block is re-read.
__device__ __forceinline__ int singular_of(const double* Ae, int n, unsigned amh, double dmin,
                                           int lane) {
  const double lo = __longlong_as_double((long long)((uint64_t)amh << 32));
  const double hi = __longlong_as_double((long long)(((uint64_t)amh << 32) | 0xffffffffull));
  if (dmin <= 1e-13 * fmax(lo, 1e-300)) return 1;
  if (dmin > 1e-13 * fmax(hi, 1e-300)) return 0;
  return singular_reread(Ae, n, dmin, lane);
}


// panels whose fast path fell back to the pivot search (MEHDG_LU_VERBOSE)
__device__ unsigned long long g_lu_fallbacks[2];

template <int NT>
struct CtaLu {
  static constexpr int kW = NT <= 14 ? 4 : 8;                  // warps per CTA
  // with 8 warps, warp 4 shares warp 0's SM sub-partition: it takes the
  // stores and the next block's copies (no DMMA competing with the panel
  // chain's fp64 instructions); the other six run the trailing updates
  static constexpr int kMover = kW == 8 ? 4 : -1;
  static constexpr int kWorkers = kW - 1 - (kMover >= 0 ? 1 : 0);
  static constexpr int kMinBlocks = NT <= 12 ? 3 : (NT <= 14 ? 2 : 1);
  static constexpr int R = (8 * NT + 31) / 32;                 // panel rows per lane
  static constexpr int kTileDoubles = NT * NT * 64;
  static constexpr size_t smem_bytes() {
    return (size_t)kTileDoubles * 8 + 3 * 64 * 8 + (size_t)(8 * NT + 20) * 4;
  }
};

template <int NT>
__device__ __forceinline__ double* tile_at(double* T, int ti, int tj) {
  return T + (tj * NT + ti) * 64;
}

// Row exchange (relative rows jj, prel of panel p) inside the panel's tile
// column, through shared memory; the caller has written the panel back.
template <int NT>
__device__ __noinline__ void swap_in_panel(double* T, int p, int jj, int prel, int lane) {
  if (lane < 8) {
    const int ra = 8 * p + jj, rb = 8 * p + prel;
    double* a = tile_at<NT>(T, ra >> 3, p) + tpos(ra & 7, lane);
    double* b = tile_at<NT>(T, rb >> 3, p) + tpos(rb & 7, lane);
    const double t = *a;
    *a = *b;
    *b = t;
  }
  __syncwarp();
}

template <int NT, int R>
__device__ __forceinline__ void panel_io(double* T, int p, double (&P)[8][R], int lane, bool store) {
#pragma unroll
  for (int a = 0; a < R; ++a) {
    const int rel = lane + 32 * a;
    if (rel < 8 * (NT - p)) {
      double* tl = tile_at<NT>(T, p + (rel >> 3), p);
      const int r = rel & 7;
#pragma unroll
      for (int cp = 0; cp < 4; ++cp) {
        double2* q = reinterpret_cast<double2*>(tl + tpos(r, 2 * cp));
        if (store) {
          *q = make_double2(P[2 * cp][a], P[2 * cp + 1][a]);
        } else {
          const double2 v = *q;
          P[2 * cp][a] = v.x;
          P[2 * cp + 1][a] = v.y;
        }
      }
    } else if (!store) {
#pragma unroll
      for (int c = 0; c < 8; ++c) P[c][a] = 0.0;
    }
  }
  __syncwarp();
}

// pivot candidate: key = (|x| bit pattern) + 1, 0 = excluded; the larger key
// wins, the earlier (smaller) row on ties -- LAPACK's idamax
__device__ __forceinline__ void cand_max(uint64_t& k0, double& v0, int& p0, uint64_t k1, double v1,
                                         int p1) {
  const bool t = k1 > k0;
  k0 = t ? k1 : k0;
  v0 = t ? v1 : v0;
  p0 = t ? p1 : p0;
}

__device__ __forceinline__ uint64_t cand_key(double x) {
  return ((uint64_t)__double_as_longlong(x) & 0x7fffffffffffffffull) + 1ull;
}

// Panel columns with the pivot search (LAPACK getf2): local candidate by a
// tree of integer compares on the |a| bit patterns, the warp max of the keys'
// high words (REDUX) and a ballot (a second and third REDUX only when several
// lanes share that word), the reciprocal of every lane's candidate computed
// before the reduction, then the exchange (through shared memory), the scaling
// and the rank-1 updates.
template <int NT, int R>
__device__ __forceinline__ void panel_pivot(double* T, double (&P)[8][R], int p, int ncol, int lane,
                                            int* swapped, int& my_prel, double& my_pv,
                                            double& my_rcp) {
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    if (jj >= ncol) break;
    uint64_t kk[R];
    double vv[R];
    int pp[R];
#pragma unroll
    for (int a = 0; a < R; ++a) {
      kk[a] = (a == 0 && lane < jj) ? 0ull : cand_key(P[jj][a]);
      vv[a] = P[jj][a];
      pp[a] = lane + 32 * a;
    }
#pragma unroll
    for (int st = 1; st < R; st *= 2)
#pragma unroll
      for (int a = 0; a + st < R; a += 2 * st)
        cand_max(kk[a], vv[a], pp[a], kk[a + st], vv[a + st], pp[a + st]);
    const uint64_t bk = kk[0];
    const double bv = vv[0];
    const int bpos = pp[0];
    const double brcp = __drcp_rn(bv);
    const unsigned khi = (unsigned)(bk >> 32);
    const unsigned mhi = __reduce_max_sync(kFull, khi);
    const unsigned ball = __ballot_sync(kFull, khi == mhi);
    int src;
    if (__popc(ball) == 1) {
      src = __ffs(ball) - 1;
    } else {  // ties on the high word: low word, then the first position
      const unsigned klo = khi == mhi ? (unsigned)bk : 0u;
      const unsigned mlo = __reduce_max_sync(kFull, klo);
      src = (int)__reduce_min_sync(
                kFull, (unsigned)((khi == mhi && (unsigned)bk == mlo) ? bpos : INT_MAX)) & 31;
    }
    const int prel = __shfl_sync(kFull, bpos, src);
    const double pv = __shfl_sync(kFull, bv, src);
    const double rcp = __shfl_sync(kFull, brcp, src);
    if (prel != jj && pv != 0.0) {  // row exchange through shared memory
      panel_io<NT, R>(T, p, P, lane, true);
      swap_in_panel<NT>(T, p, jj, prel, lane);
      panel_io<NT, R>(T, p, P, lane, false);
      if (lane == 0) *swapped = 1;
    }
    if (lane == jj) {
      my_prel = pv != 0.0 ? prel : jj;
      my_pv = pv;
      my_rcp = rcp;
    }
    if (pv != 0.0) {
      if (fabs(pv) >= DBL_MIN) {
#pragma unroll
        for (int a = 0; a < R; ++a)
          if (a > 0 || lane > jj) P[jj][a] *= rcp;
      } else {
#pragma unroll
        for (int a = 0; a < R; ++a)
          if (a > 0 || lane > jj) P[jj][a] = div_slow(P[jj][a], pv);
      }
    }
#pragma unroll
    for (int c = jj + 1; c < 8; ++c) {
      const double u = __shfl_sync(kFull, P[c][0], jj);
#pragma unroll
      for (int a = 0; a < R; ++a)
        if (a > 0 || lane > jj) P[c][a] = fma(-P[jj][a], u, P[c][a]);
    }
  }
}

// The whole panel p with the pivot search (one warp): the exact LAPACK getf2
// path, taken when the diagonal-block fast path below cannot decide.  Leaves
// the factored panel in shared memory, piv / udiag / dinv stored, -L11^-1 in
// Xd (A-fragment order), the exchanges in psw (*swapped set when there was
// one); dmin (per lane) takes min |U_jj| of the panel.
template <int NT>
__device__ __forceinline__ void factor_panel_pivot(double* T, double* Xd, int* psw, int* swapped,
                                                const LuArgs& g, int64_t e, int p, int lane,
                                                double& dmin) {
  __syncwarp();
  constexpr int R = CtaLu<NT>::R;
  const int Q = g.Q, c0 = 8 * p;
  const int ncol = min(8, Q - c0);
  double P[8][R];
  panel_io<NT, R>(T, p, P, lane, false);
  int my_prel = lane;  // lane jj keeps column jj's pivot / U_jj / 1/U_jj
  double my_pv = 1.0, my_rcp = 1.0;
  panel_pivot<NT, R>(T, P, p, ncol, lane, swapped, my_prel, my_pv, my_rcp);
  if (lane < ncol) {
    const int64_t k = e * Q + c0 + lane;
    g.piv[k] = c0 + my_prel;
    g.udiag[k] = my_pv;
    g.dinv[k] = my_rcp;
    psw[lane] = my_prel;
    dmin = fmin(dmin, fabs(my_pv));
  }
  panel_io<NT, R>(T, p, P, lane, true);
  if (lane < 8) {  // -L11^-1 from the stored diagonal block
    const double* d = tile_at<NT>(T, p, p);
    const int jc = lane;
    double x[8];
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      double s = 0.0;
#pragma unroll
      for (int m = 0; m < rr; ++m) s = fma(-d[tpos(rr, m)], x[m], s);
      x[rr] = rr < jc ? 0.0 : (rr == jc ? 1.0 : s);
      Xd[2 * (4 * rr + (jc & 3)) + (jc >> 2)] = -x[rr];
    }
  }
  __syncwarp();
}

// Fast path of F_p (one warp): the 8 x 8 diagonal block alone, without row
// exchanges.  LAPACK keeps the diagonal as the pivot exactly when no row below
// has a strictly larger |a| (idamax: first index on ties); inside the block
// that is checked exactly, column by column; for the rows below (the tiles of
// L21 = A21 U11^-1, formed by DMMA in the next phase) it is |l| < 1 with a
// margin far above rounding.  Returns false -- nothing written -- when a row
// exchange, a zero or a tiny pivot shows up in the block; else the block's
// L11\U11 goes back to its tile, -L11^-1 to Xd (A-fragment order), U11^-1 to
// Ud (a swizzled tile), and lane jj keeps U_jj, 1/U_jj (pv, rcp) and its
// original row (orig, for a fallback).  The chain per column is shuffle ->
// reciprocal -> scaling -> next column's update on one row per lane.
template <int NT>
__device__ __forceinline__ bool diag_fast(double* T, double* Xd, double* Ud, int* psw,
                                          const LuArgs& g, int64_t e, int p, int ncol,
                                          int lane, double& pv_l, double& rcp_l,
                                          double (&orig)[8]) {
  __syncwarp();  // converged: the shuffles below take their fast form
  double* d = tile_at<NT>(T, p, p);
  double a[8], xr[8];
#pragma unroll
  for (int cp = 0; cp < 4; ++cp) {
    double2 v = make_double2(0.0, 0.0);
    if (lane < 8) v = *reinterpret_cast<const double2*>(d + tpos(lane, 2 * cp));
    a[2 * cp] = v.x;
    a[2 * cp + 1] = v.y;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    orig[k] = a[k];
    xr[k] = k == lane ? 1.0 : 0.0;
  }
  bool bad = false;
  pv_l = DBL_MAX;  // lanes >= ncol: no column (neutral in min |U_jj|)
  rcp_l = 1.0;
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    if (jj >= ncol) break;
    const double pv = __shfl_sync(kFull, a[jj], jj);
    const double rcp = __drcp_rn(pv);
    const double apv = fabs(pv);
    bad |= (lane > jj && fabs(a[jj]) > apv) || !(apv >= DBL_MIN);
    if (lane == jj) {
      pv_l = pv;
      rcp_l = rcp;
    }
    if (lane > jj) a[jj] *= rcp;
#pragma unroll
    for (int c = jj + 1; c < 8; ++c) {
      const double u = __shfl_sync(kFull, a[c], jj);
      if (lane > jj) a[c] = fma(-a[jj], u, a[c]);
    }
    // X = L11^-1 = E_7 ... E_0, E_j = I - l_j e_j^T: rows i > jj -= l_ij X[jj]
#pragma unroll
    for (int k = 0; k <= jj; ++k) {
      const double xk = __shfl_sync(kFull, xr[k], jj);
      if (lane > jj) xr[k] = fma(-a[jj], xk, xr[k]);
    }
  }
  if (__any_sync(kFull, bad)) return false;
  if (lane < ncol) {  // speculative: the pivot path rewrites them on a fallback
    const int64_t k = e * g.Q + 8 * p + lane;
    g.piv[k] = 8 * p + lane;
    g.udiag[k] = pv_l;
    g.dinv[k] = rcp_l;
    psw[lane] = lane;
  }
  __syncwarp();
  if (lane < 8) {
#pragma unroll
    for (int cp = 0; cp < 4; ++cp)
      *reinterpret_cast<double2*>(d + tpos(lane, 2 * cp)) = make_double2(a[2 * cp], a[2 * cp + 1]);
#pragma unroll
    for (int k = 0; k < 8; ++k) Xd[2 * (4 * lane + (k & 3)) + (k >> 2)] = -xr[k];
  }
  __syncwarp();
  // U11^-1 by columns (lane k < ncol): back substitution from the stored block
  double rc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) rc[i] = __shfl_sync(kFull, rcp_l, i);
  if (lane < 8) {
    const int k = lane;
    double x[8];
#pragma unroll
    for (int i = 7; i >= 0; --i) {
      double s = i == k ? 1.0 : 0.0;
#pragma unroll
      for (int m = i + 1; m < 8; ++m) s = fma(-d[tpos(i, m)], x[m], s);
      x[i] = (i > k || k >= ncol) ? 0.0 : s * rc[i];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) Ud[tpos(i, k)] = x[i];
  }
  __syncwarp();
  return true;
}

// The factored panel p (shared memory, tile column p) to the packed streams:
// L below the diagonal, the diagonal block's U above it.  Tiles i >= p are
// spread over the calling warps (index wk of nw); lane (r, q) stores rows
// 8 i + r of columns 8 p + 2 q (+1), whose L-stream bases are fixed per panel.
template <int NT>
__device__ __forceinline__ void store_panel(const double* T, double* Lpe, double* Upe, int Q, int p,
                                            int wk, int nw, int lane, uint64_t pol) {
  const int r = lane >> 2, q = lane & 3;
  const int j0 = 8 * p + 2 * q, j1 = j0 + 1;
  double* L0 = Lpe + ol(j0, Q) - j0 - 1;  // + row
  double* L1 = Lpe + ol(j1, Q) - j1 - 1;
  const double* src = T + p * NT * 64 + tpos(r, 2 * q);
  int i = p + wk;
  if (i == p) {  // the diagonal tile: L below, U above the diagonal
    const double2 v = *reinterpret_cast<const double2*>(src + p * 64);
    const int row = 8 * p + r;
    if (row < Q) {
      if (j0 < Q) {
        if (row > j0) st_ef(L0 + row, v.x, pol);
        else if (row < j0) st_ef(Upe + ou(j0, Q) + row, v.x, pol);
      }
      if (j1 < Q) {
        if (row > j1) st_ef(L1 + row, v.y, pol);
        else if (row < j1) st_ef(Upe + ou(j1, Q) + row, v.y, pol);
      }
    }
    i += nw;
  }
  const bool c0v = j0 < Q, c1v = j1 < Q;
  for (; i < NT; i += nw) {
    const double2 v = *reinterpret_cast<const double2*>(src + i * 64);
    const int row = 8 * i + r;
    if (row < Q) {
      if (c0v) st_ef(L0 + row, v.x, pol);
      if (c1v) st_ef(L1 + row, v.y, pol);
    }
  }
}

// -U(p, j) = (-L11^-1) A(p, j) in C layout (2 DMMA)
template <int NT>
__device__ __forceinline__ void neg_u(const double* T, const double* Xd, int p, int j, int lane,
                                      double& u0, double& u1) {
  const double2 xa = *reinterpret_cast<const double2*>(Xd + 2 * lane);
  const double* a = T + (j * NT + p) * 64;
  const int q = lane & 3, r = lane >> 2;
  u0 = u1 = 0.0;
  mma_acc(u0, u1, xa.x, a[tpos(q, r)]);
  mma_acc(u0, u1, xa.y, a[tpos(4 + q, r)]);
}

// U(p, j) (C layout, negated) to the packed U stream: rows 8p + r, columns 8j + 2q (+1)
__device__ __forceinline__ void store_u(double* Upe, int Q, int p, int j, int lane, double u0,
                                        double u1, uint64_t pol) {
  const int r = lane >> 2, c = 8 * j + 2 * (lane & 3), row = 8 * p + r;
  if (c < Q) st_ef(Upe + ou(c, Q) + row, -u0, pol);
  if (c + 1 < Q) st_ef(Upe + ou(c + 1, Q) + row, -u1, pol);
}

#ifdef MH_LU_TRACE
// phase timestamps of CTA 0's second block (steady state), printed at its end
__device__ long long g_lu_trace[64][8][6];
#define LU_TR(k, pp)                                                                  \
  if (blockIdx.x == 0 && e == gridDim.x && lane == 0 && (pp) < 64)                     \
    g_lu_trace[pp][w][k] = clock64() - tr0;
#else
#define LU_TR(k, pp)
#endif

// The next block's A into the tiles whose last use in this block is done:
// tile row m and tile column m (min(ti, tj) = m) are free once panel m's
// trailing update and stores have passed a CTA barrier.  Asynchronous 8-byte
// copies (cp.async, no registers held), pads zero-filled; a half-tile per
// instruction (lane l: row 4 h + l / 8, column l % 8), so each warp
// instruction reads four 64-byte row segments.
template <int NT, int W>
__device__ __forceinline__ void fetch_free_tiles(double* T, const double* An, int Q, int m, int wk,
                                                 int lane, uint64_t pol) {
  const int rr = lane >> 3, cc = lane & 7;
  const unsigned tbase = (unsigned)__cvta_generic_to_shared(T);
  // half-tile k: tile (m, m + k / 2) for k < 2 (NT - m), then (m + 1 + (k' / 2), m)
  for (int k = wk; k < 4 * (NT - m) - 2; k += W) {
    const bool rowpart = k < 2 * (NT - m);
    const int kk = rowpart ? k : k - 2 * (NT - m);
    const int h = kk & 1, t = kk >> 1;
    const int ti = rowpart ? m : m + 1 + t, tj = rowpart ? m + t : m;
    const int row = 8 * ti + 4 * h + rr, col = 8 * tj + cc;
    const unsigned nb = (row < Q && col < Q) ? 8u : 0u;
    const unsigned dst = tbase + 8u * (unsigned)((tj * NT + ti) * 64 + tpos(4 * h + rr, cc));
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2, %3;"
                 ::"r"(dst), "l"(nb ? An + row * Q + col : An), "r"(nb), "l"(pol) : "memory");
  }
}

template <int NT>
__global__ void __launch_bounds__(CtaLu<NT>::kW * 32, CtaLu<NT>::kMinBlocks)
    lu_cta_kernel(LuArgs g) {
  using S = CtaLu<NT>;
  constexpr int W = S::kW;
  constexpr int NW = S::kWorkers;
  constexpr int KU = (NT - 1 + W - 1) / W;  // row tiles per warp in a column phase
  extern __shared__ __align__(16) double lu_smem[];
  double* T = lu_smem;
  double* X2 = T + S::kTileDoubles;  // two -L11^-1 buffers (panel parity)
  double* Ud = X2 + 128;             // U11^-1 of the fast path (swizzled tile)
  int* prow = reinterpret_cast<int*>(Ud + 64);
  int* psw = prow + 8 * NT;  // 8 exchanges of the current panel
  int* swapped = psw + 8;
  int* mode_s = swapped + 1;  // 0: diagonal block factored (fast), 1: whole panel factored
  int* fail_s = mode_s + 1;   // the L21 check of the fast path failed
  unsigned* amh_s = reinterpret_cast<unsigned*>(fail_s + 1);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = lane >> 2, q = lane & 3;
  const int Q = g.Q;
  const int np = (Q + 7) / 8;  // panels (<= NT)
  const uint64_t pol = pol_evict_first();
  // |l| bound of the fast path: far above the rounding of L21 = A21 U11^-1
  constexpr double kLmax = 1.0 - 1.0 / 1024.0;

  // the first block's A (later blocks arrive tile by tile while the previous
  // one is factored); padding rows / columns are zero-filled and stay zero
  // through every update, exchange and store of the kernel
  if (blockIdx.x < g.nblocks)
    for (int m = 0; m < NT; ++m)
      fetch_free_tiles<NT, W>(T, g.A + (int64_t)blockIdx.x * Q * Q, Q, m, w, lane, pol);
  if (threadIdx.x == 0) *fail_s = 0;

  for (int64_t e = blockIdx.x; e < g.nblocks; e += gridDim.x) {
#ifdef MH_LU_TRACE
    const long long tr0 = clock64();
#endif
    const double* __restrict__ Ae = g.A + e * (int64_t)Q * Q;
    double* Lpe = g.Lp + e * g.ldL;
    double* Upe = g.Up + e * g.ldL;
    const double* An = g.A + (e + gridDim.x) * (int64_t)Q * Q;  // the next block
    const bool has_next = e + gridDim.x < g.nblocks;
    if (threadIdx.x == 0) {
      *swapped = 0;
      *amh_s = 0u;
    }
    for (int i = threadIdx.x; i < 8 * NT; i += W * 32) prow[i] = i;
    asm volatile("cp.async.wait_all;" ::: "memory");
    LU_TR(0, 0)
    __syncthreads();
    // max|A| (singularity test) while panel 0's diagonal block is factored:
    // warp 0 over tile column 0 first, the other warps over the rest
    double dmin = DBL_MAX;             // warp 0: min |U_jj| (per lane)
    double pv_l = 1.0, rcp_l = 1.0;    // warp 0: the pending panel's U_jj, 1/U_jj (lane jj)
    double orig[8];                    // warp 0: the pending diagonal block's rows
    {
      unsigned amh = 0;
      const int i0 = w == 0 ? lane : 32 * NT + 32 * (w - 1) + lane;
      const int i1 = w == 0 ? 32 * NT : 32 * NT * NT;
      for (int i = i0; i < i1; i += w == 0 ? 32 : 32 * (W - 1)) {
        const double2 v = reinterpret_cast<const double2*>(T)[i];
        amh = max(amh, max(hiabs(v.x), hiabs(v.y)));
      }
      amh = __reduce_max_sync(kFull, amh);
      if (lane == 0) atomicMax(amh_s, amh);
    }
    if (w == 0) {
      const bool fast = diag_fast<NT>(T, X2, Ud, psw, g, e, 0, min(8, Q), lane, pv_l, rcp_l, orig);
      if (!fast) factor_panel_pivot<NT>(T, X2, psw, swapped, g, e, 0, lane, dmin);
      if (lane == 0) *mode_s = fast ? 0 : 1;
      if (!fast && lane == 0) atomicAdd(&g_lu_fallbacks[0], 1ull);
    }
    LU_TR(1, 0)
    __syncthreads();

    for (int p = 0; p < np; ++p) {
      const double* Xd = X2 + 64 * (p & 1);
      const int c0 = 8 * p, ncol = min(8, Q - c0);
      const bool more = p + 1 < np;
      int mode = *mode_s;
      if (mode == 0) {
        // ---- L21 = A21 U11^-1 (2 DMMA per tile, with the |l| check) and, when
        // it passes, column p+1's update -- the originals kept for a fallback
        double2 oc[KU], on[KU];
        bool ok = true;
        {
          const double ub0 = Ud[tpos(q, r)], ub1 = Ud[tpos(4 + q, r)];
#pragma unroll
          for (int k = 0; k < KU; ++k) {
            const int i = p + 1 + w + k * W;
            if (i < NT) {
              double* Lt = tile_at<NT>(T, i, p);
              const double a0 = Lt[tpos(r, q)], a1 = Lt[tpos(r, 4 + q)];
              double2* C = reinterpret_cast<double2*>(Lt + tpos(r, 2 * q));
              oc[k] = *C;
              double2 l = make_double2(0.0, 0.0);
              mma_acc(l.x, l.y, a0, ub0);
              mma_acc(l.x, l.y, a1, ub1);
              ok &= fabs(l.x) <= kLmax && fabs(l.y) <= kLmax;
              *C = l;
            }
          }
        }
        if (more) {
          double u0, u1;
          neg_u<NT>(T, Xd, p, p + 1, lane, u0, u1);
          if (w == 0) store_u(Upe, Q, p, p + 1, lane, u0, u1, pol);
          const double b0 = bfrag_c(u0, u1, 0, lane), b1 = bfrag_c(u0, u1, 1, lane);
          __syncwarp();
#pragma unroll
          for (int k = 0; k < KU; ++k) {
            const int i = p + 1 + w + k * W;
            if (i < NT) {
              const double* Lt = tile_at<NT>(T, i, p);
              double2* C = reinterpret_cast<double2*>(tile_at<NT>(T, i, p + 1) + tpos(r, 2 * q));
              on[k] = *C;
              double2 c = on[k];
              mma_acc(c.x, c.y, Lt[tpos(r, q)], b0);
              mma_acc(c.x, c.y, Lt[tpos(r, 4 + q)], b1);
              *C = c;
            }
          }
        }
        if (!__all_sync(kFull, ok) && lane == 0) atomicOr(fail_s, 1);
        __syncwarp();
        __syncthreads();  // B1 (fast)
        if (*fail_s) {
          // a row below the diagonal block would win the pivot search: restore
          // and factor the whole panel with it (then the mode-1 path below)
#pragma unroll
          for (int k = 0; k < KU; ++k) {
            const int i = p + 1 + w + k * W;
            if (i < NT) {
              *reinterpret_cast<double2*>(tile_at<NT>(T, i, p) + tpos(r, 2 * q)) = oc[k];
              if (more) *reinterpret_cast<double2*>(tile_at<NT>(T, i, p + 1) + tpos(r, 2 * q)) = on[k];
            }
          }
          if (w == 0 && lane < 8) {
            double* d = tile_at<NT>(T, p, p);
#pragma unroll
            for (int cp = 0; cp < 4; ++cp)
              *reinterpret_cast<double2*>(d + tpos(lane, 2 * cp)) = make_double2(orig[2 * cp], orig[2 * cp + 1]);
          }
          __syncthreads();
          if (w == 0) factor_panel_pivot<NT>(T, X2 + 64 * (p & 1), psw, swapped, g, e, p, lane, dmin);
          if (threadIdx.x == 0) {
            *fail_s = 0;
            atomicAdd(&g_lu_fallbacks[1], 1ull);
          }
          __syncthreads();
          mode = 1;
        } else if (w == 0) {  // the fast panel is final
          dmin = fmin(dmin, fabs(pv_l));
        }
      }
      if (mode == 1) {
        // ---- W_p: the panel's row exchanges outside it (rare)
        if (*swapped) {
          for (int c = 8 * (p + 1) + threadIdx.x; c < 8 * NT; c += W * 32) {
            for (int jj = 0; jj < ncol; ++jj) {
              const int pr = psw[jj];
              if (pr == jj) continue;
              const int ra = c0 + jj, rb = c0 + pr;
              double* x = tile_at<NT>(T, ra >> 3, c >> 3) + tpos(ra & 7, c & 7);
              double* y = tile_at<NT>(T, rb >> 3, c >> 3) + tpos(rb & 7, c & 7);
              const double t = *x;
              *x = *y;
              *y = t;
            }
          }
          for (int j = threadIdx.x; j < c0; j += W * 32) {
            for (int jj = 0; jj < ncol; ++jj) {
              const int pr = psw[jj];
              if (pr == jj) continue;
              double* x = Lpe + ol(j, Q) + (c0 + jj - j - 1);
              double* y = Lpe + ol(j, Q) + (c0 + pr - j - 1);
              const double t = *x;
              *x = *y;
              *y = t;
            }
          }
          if (threadIdx.x == 0) {
            for (int jj = 0; jj < ncol; ++jj) {
              const int pr = psw[jj];
              if (pr == jj) continue;
              const int t = prow[c0 + jj];
              prow[c0 + jj] = prow[c0 + pr];
              prow[c0 + pr] = t;
            }
          }
          __syncthreads();
          if (threadIdx.x == 0) *swapped = 0;
        }
        // ---- U_p: column p+1, row tiles split over all warps (loads first)
        if (more && (w == 0 || p + 1 + w < NT)) {
          double2 cc[KU];
          double la[KU][2];
#pragma unroll
          for (int k = 0; k < KU; ++k) {
            const int i = p + 1 + w + k * W;
            if (i < NT) {
              const double* L = tile_at<NT>(T, i, p);
              la[k][0] = L[tpos(r, q)];
              la[k][1] = L[tpos(r, 4 + q)];
              cc[k] = *reinterpret_cast<const double2*>(tile_at<NT>(T, i, p + 1) + tpos(r, 2 * q));
            }
          }
          double u0, u1;
          neg_u<NT>(T, Xd, p, p + 1, lane, u0, u1);
          const double b0 = bfrag_c(u0, u1, 0, lane), b1 = bfrag_c(u0, u1, 1, lane);
#pragma unroll
          for (int k = 0; k < KU; ++k) {
            const int i = p + 1 + w + k * W;
            if (i < NT) {
              mma_acc(cc[k].x, cc[k].y, la[k][0], b0);
              mma_acc(cc[k].x, cc[k].y, la[k][1], b1);
              *reinterpret_cast<double2*>(tile_at<NT>(T, i, p + 1) + tpos(r, 2 * q)) = cc[k];
            }
          }
          if (w == 0) store_u(Upe, Q, p, p + 1, lane, u0, u1, pol);
        }
        __syncthreads();  // B1 (exchanging panel)
      }
      LU_TR(3, p + 1)
      // ---- concurrently: F_{p+1} (warp 0) | stores and copies (mover) |
      //      U(p, j >= p+2) and the trailing update (workers)
      if (w == 0) {
        if (more) {
          const bool fast = diag_fast<NT>(T, X2 + 64 * ((p + 1) & 1), Ud, psw, g, e, p + 1,
                                          min(8, Q - c0 - 8), lane, pv_l, rcp_l, orig);
          if (!fast)
            factor_panel_pivot<NT>(T, X2 + 64 * ((p + 1) & 1), psw, swapped, g, e, p + 1, lane, dmin);
          if (lane == 0) *mode_s = fast ? 0 : 1;
          if (!fast && lane == 0) atomicAdd(&g_lu_fallbacks[0], 1ull);
        }
      } else if (w == S::kMover) {
        // panel p's L and diagonal-block U to their streams; the next block's
        // tiles of row / column p - 1 (free since the last barrier)
        store_panel<NT>(T, Lpe, Upe, Q, p, 0, 1, lane, pol);
        if (p > 0 && has_next) fetch_free_tiles<NT, 1>(T, An, Q, p - 1, 0, lane, pol);
      } else {
        const int wk = w - 1 - (S::kMover >= 0 && w > S::kMover ? 1 : 0);
        if (p + 2 < NT) {
          // -U(p, j), j >= p+2, in place (and U to its stream)
          for (int j = p + 2 + wk; j < NT; j += NW) {
            double u0, u1;
            neg_u<NT>(T, Xd, p, j, lane, u0, u1);
            store_u(Upe, Q, p, j, lane, u0, u1, pol);
            *reinterpret_cast<double2*>(tile_at<NT>(T, p, j) + tpos(r, 2 * q)) = make_double2(u0, u1);
          }
          asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
          // C(i, j) += L(i, p) (-U(p, j)): units of a strip of two tile columns
          // (their -U B fragments held in registers) times a chunk of row
          // tiles, walked two rows at a time with all loads first
          const int nr = NT - 1 - p, ncl = NT - 2 - p;
          const int ns = (ncl + 1) / 2;
          const int nch = min(nr, (2 * NW + ns - 1) / ns);
          const int cr = (nr + nch - 1) / nch;
          // u / ns as a multiply-high (exact for the small u here; ns = 1 needs the 33rd bit)
          const unsigned long long nsm = (0x100000000ull + (unsigned)ns - 1) / (unsigned)ns;
          const int oa0 = tpos(r, q), oa1 = tpos(r, 4 + q), oc = tpos(r, 2 * q);
          const int ob0 = tpos(q, r), ob1 = tpos(4 + q, r);
          for (int u = wk; u < ns * nch; u += NW) {
            const int ch = (int)(((unsigned long long)u * nsm) >> 32), sj = u - ch * ns;
            const int j0 = p + 2 + 2 * sj;
            const bool two = j0 + 1 < NT;
            const double* U0 = T + (j0 * NT + p) * 64;
            const double* U1 = two ? U0 + NT * 64 : U0;
            const double b00 = U0[ob0], b01 = U0[ob1], b10 = U1[ob0], b11 = U1[ob1];
            const int ib = p + 1 + ch * cr, ie = min(NT, ib + cr);
            const double* Lt = T + (p * NT + ib) * 64;
            double* C0 = T + (j0 * NT + ib) * 64;
            double* C1 = two ? C0 + NT * 64 : C0;  // every address stays inside the tiles
            for (int i = ib; i < ie; i += 2, Lt += 128, C0 += 128, C1 += 128) {
              const int d2 = i + 1 < ie ? 64 : 0;
              const double a00 = Lt[oa0], a01 = Lt[oa1];
              const double a10 = Lt[d2 + oa0], a11 = Lt[d2 + oa1];
              double2 c00 = *reinterpret_cast<const double2*>(C0 + oc);
              double2 c01 = *reinterpret_cast<const double2*>(C1 + oc);
              double2 c10 = *reinterpret_cast<const double2*>(C0 + d2 + oc);
              double2 c11 = *reinterpret_cast<const double2*>(C1 + d2 + oc);
              mma_acc(c00.x, c00.y, a00, b00);
              mma_acc(c01.x, c01.y, a00, b10);
              mma_acc(c10.x, c10.y, a10, b00);
              mma_acc(c11.x, c11.y, a10, b10);
              mma_acc(c00.x, c00.y, a01, b01);
              mma_acc(c01.x, c01.y, a01, b11);
              mma_acc(c10.x, c10.y, a11, b01);
              mma_acc(c11.x, c11.y, a11, b11);
              // duplicates (one column / one row left) store before the real tile
              *reinterpret_cast<double2*>(C1 + d2 + oc) = c11;
              *reinterpret_cast<double2*>(C0 + d2 + oc) = c10;
              *reinterpret_cast<double2*>(C1 + oc) = c01;
              *reinterpret_cast<double2*>(C0 + oc) = c00;
            }
          }
        }
        if (S::kMover < 0) {  // no mover warp: the workers store and copy
          store_panel<NT>(T, Lpe, Upe, Q, p, wk, NW, lane, pol);
          if (p > 0 && has_next) fetch_free_tiles<NT, NW>(T, An, Q, p - 1, wk, lane, pol);
        }
      }
      LU_TR(5, p + 1)
      __syncthreads();  // B2
    }
    LU_TR(0, 63)
    for (int64_t i = (int64_t)Q * (Q - 1) / 2 + threadIdx.x; i < g.ldL; i += W * 32) {
      Lpe[i] = 0.0;
      Upe[i] = 0.0;
    }
    for (int i = threadIdx.x; i < Q; i += W * 32) g.perm[e * Q + i] = prow[i];
    if (w == 0) {
      for (int o = 16; o; o >>= 1) dmin = fmin(dmin, __shfl_xor_sync(kFull, dmin, o));
      const int sing = singular_of(Ae, Q * Q, *amh_s, dmin, lane);
      if (lane == 0) g.stat[e] = sing;
    }
    __syncthreads();
    if (has_next)
      for (int m = np - 2; m < NT; ++m) fetch_free_tiles<NT, W>(T, An, Q, m, w, lane, pol);
#ifdef MH_LU_TRACE
    if (blockIdx.x == 0 && e == gridDim.x && threadIdx.x == 0) {
      __threadfence_block();
      for (int pp = 0; pp < 64; ++pp)
        for (int ww = 0; ww < W; ++ww) {
          const long long* t = g_lu_trace[pp][ww];
          if (t[0] | t[1] | t[2] | t[3] | t[4] | t[5])
            printf("TR p%d w%d %lld %lld %lld %lld %lld %lld\n", pp, ww, t[0], t[1], t[2], t[3], t[4], t[5]);
        }
    }
#endif
  }
}

template <int NT>
int launch_nt(mh_system* s, const LuArgs& g, cudaEvent_t start) {
  using S = CtaLu<NT>;
  const size_t smem = S::smem_bytes();
  MH_CHECK_CUDA(cudaFuncSetAttribute(lu_cta_kernel<NT>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  MH_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lu_cta_kernel<NT>,
                                                              S::kW * 32, smem));
  per_sm = std::max(per_sm, 1);
  const int64_t grid = std::min<int64_t>(g.nblocks, (int64_t)per_sm * s->num_sms);
  static const bool verbose = getenv("MEHDG_LU_VERBOSE") != nullptr;
  if (verbose) {
    unsigned long long fb[2] = {0, 0};
    cudaStreamSynchronize(s->stream);
    cudaMemcpyFromSymbol(fb, g_lu_fallbacks, sizeof(fb));
    fprintf(stderr, "lu_cta NT=%d warps=%d smem=%zu ctas/SM=%d grid=%lld fallbacks so far: diag %llu, L21 %llu\n",
            NT, S::kW, smem, per_sm, (long long)grid, fb[0], fb[1]);
  }
  if (start) MH_CHECK_CUDA(cudaEventRecord(start, s->stream));
  lu_cta_kernel<NT><<<(unsigned)grid, S::kW * 32, smem, s->stream>>>(g);
  MH_CHECK_CUDA(cudaGetLastError());
  return MH_OK;
}

}  // namespace

// Q in 33..168 (NT = ceil(Q / 8) tiles; 227 KB of shared memory at NT = 21)
bool lu_cta_supported(int Q) { return Q > 32 && Q <= 168; }

int launch_lu_cta(mh_system* s, const LuArgs& g, cudaEvent_t start) {
  const int nt = (g.Q + 7) / 8;
#define MH_NT(N) \
  if (nt <= N) return launch_nt<N>(s, g, start);
  MH_NT(6) MH_NT(8) MH_NT(10) MH_NT(11) MH_NT(12) MH_NT(14) MH_NT(16) MH_NT(18) MH_NT(21)
#undef MH_NT
  set_error("Q > 168 is not supported by the CTA-resident batched LU");
  return MH_E_UNSUPPORTED;
}

}  // namespace mh
