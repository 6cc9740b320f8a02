// Batched fp64 LU with partial pivoting, one warp per block, DMMA updates.
//
// Replaces _factorize_local's dense branch (schur_solver.py:105-111):
// scipy.linalg.lu_factor (LAPACK getrf, partial pivoting, first index on ties)
// and the singularity test min|diag U| <= 1e-13 max|A|.  Same outputs as the
// other LU kernels (lu.cu): the packed L / U streams the element kernel reads,
// diag(U), 1/U_jj, LAPACK pivots, composed row permutation, status.
//
// Left-looking by panels of 8 columns.  The panel lives in registers as NT
// tiles of 8 rows in the C-fragment layout of mma.m8n8k4.f64 (lane = 4 r + q
// holds rows 8t + r, columns 2q, 2q + 1), so every update with an earlier
// panel kb is two DMMA per tile:
//   1. gather the panel's columns of A by position (row permutation prow in
//      shared memory; A is read exactly once);
//   2. for kb < jb (unrolled, so tile kb is a static register):
//        -U_kb   = (-L11(kb)^-1) T_kb        (2 DMMA)
//        T_t    += L(rows of t, kb) (-U_kb)  (2 DMMA per tile t > kb)
//      -U_kb goes to the packed U stream.  L(., kb) and -L11(kb)^-1 come from
//      the warp's scratch slot, stored once per panel in A-fragment order (one
//      16-byte load per lane per tile); the slot is reused block after block,
//      so it stays in L2 while the A / L / U streams pass through (evict-first);
//   3. the rows >= c0 move through shared memory to a row layout relative to
//      the panel (lane l, register a <-> row c0 + l + 32 a, so the pivot row of
//      column jj is always lane jj of register 0) and the panel is factored in
//      registers: idamax = per-lane max, then max of the |a| bit pattern and
//      min of the position over the warp (three REDUX; first index on ties),
//      reciprocal scaling (division below DBL_MIN, as dgetf2), rank-1 updates;
//      a row exchange (rare) goes out of line through shared memory and also
//      exchanges the stored L rows and prow;
//   4. L, the diagonal-block U, diag(U) and 1/U_jj are stored, and the panel's
//      L tiles plus the inverse of its unit-lower diagonal block go to scratch.
// Persistent grid: warp w walks blocks w, w + W, ... (W = resident warps).

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdlib>

#include "lu_tile_common.cuh"

namespace mh {
namespace {

constexpr int kTileWarps = 4;

template <int NT>
struct TileShape {
  static constexpr int R = (NT + 3) / 4;       // rows per lane in row layout
  static constexpr int LDP = 32 * R + 4;       // column stride (2 LDP = 8 mod 16: conflict-free)
  // -L11(kb)^-1 tiles live in shared memory when they fit next to the panel
  static constexpr bool kLinvSmem = NT <= 21;
  static constexpr int kWarpDoubles = 8 * LDP + 64 + (kLinvSmem ? NT * 64 : 0);
  static constexpr int kWarpInts = 32 * R;           // prow
  static constexpr int kSlotDoubles = NT * (NT + 1) / 2 * 64;
  static constexpr int kMinBlocks = NT <= 16 ? 3 : 2;
  static constexpr size_t smem_bytes() {
    return (size_t)kTileWarps * (kWarpDoubles * sizeof(double) + kWarpInts * sizeof(int));
  }
};

// Row exchange k <-> p (positions c0 + jj, c0 + prel) of the panel held in Pw
// (relative rows), prow, the stored L stream (columns < c0) and the scratch
// L tiles of the earlier panels.  Out of line: it is rare.
__device__ __noinline__ void exchange_rows(double* Pw, int ldp, int* prow, double* Lpe,
                                           double* slot, int Q, int nt, int jb, int jj,
                                           int prel, int lane) {
  const int c0 = 8 * jb, k = c0 + jj, p = c0 + prel;
  if (lane < 8) {
    double* col = Pw + lane * ldp;
    const double t = col[jj];
    col[jj] = col[prel];
    col[prel] = t;
  }
  if (lane == 0) {
    const int t = prow[k];
    prow[k] = prow[p];
    prow[p] = t;
  }
  for (int j = lane; j < c0; j += 32) {
    double* ck = Lpe + off_lower(j, Q) + (k - j - 1);
    double* cp = Lpe + off_lower(j, Q) + (p - j - 1);
    const double t = *ck;
    *ck = *cp;
    *cp = t;
  }
  for (int idx = lane; idx < 4 * jb; idx += 32) {
    const int kb = idx >> 2, qq = idx & 3;
    double2* sk = reinterpret_cast<double2*>(slot + tri(kb, k >> 3, nt) * 64) + 4 * (k & 7) + qq;
    double2* sp = reinterpret_cast<double2*>(slot + tri(kb, p >> 3, nt) * 64) + 4 * (p & 7) + qq;
    const double2 t = *sk;
    *sk = *sp;
    *sp = t;
  }
  __syncwarp();
}

// Factor the 8-column panel held in Pw (column-major, rows relative to the
// panel's first row c0 = 8 jb) by one warp, in a register row layout (lane l,
// register a <-> relative row l + 32 a), and store L, the diagonal block's U,
// piv / udiag / dinv.  The factored panel is left in Pw.  `tiles` holds the L
// tiles of the earlier panels (A-fragment order) that a row exchange must
// also exchange.
template <int R, int LDP>
__device__ __forceinline__ void factor_panel(double* Pw, int* prow, double* Lpe, double* Upe,
                                             double* tiles, int nt, const LuArgs& g, int64_t e,
                                             int jb, int lane, uint64_t pol, double& dmin) {
  const int Q = g.Q, c0 = 8 * jb;
  const int ncol = min(8, Q - c0), nrel = Q - c0;
  bool valid[R];
#pragma unroll
  for (int a = 0; a < R; ++a) valid[a] = lane + 32 * a < nrel;
  double P[8][R];
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int a = 0; a < R; ++a) P[c][a] = Pw[c * LDP + lane + 32 * a];
  __syncwarp();
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    if (jj >= ncol) break;
    // Fast path: idamax takes the first row of maximum |a|, so the diagonal stays
    // the pivot exactly when no row below it is strictly larger -- one broadcast of
    // the diagonal, one compare per element, one vote; its reciprocal is already
    // on its way while the vote resolves.  Otherwise the exact search below.
    double pv = __shfl_sync(kFull, P[jj][0], jj);
    int prel = jj;
    double rcp = __drcp_rn(pv);
    bool larger = false;
    {
      const double apd = fabs(pv);
#pragma unroll
      for (int a = 0; a < R; ++a)
        if ((a > 0 || lane > jj) && valid[a] && fabs(P[jj][a]) > apd) larger = true;
    }
    if (__any_sync(kFull, larger)) {
      // idamax over relative rows jj..nrel-1 (first index on ties): per-lane best,
      // then the warp max of (hi word + 1, lo word) of |a| and the first position
      double bv = 0.0, babs = -1.0;
      int bpos = INT_MAX;
#pragma unroll
      for (int a = 0; a < R; ++a) {
        const double x = P[jj][a], ax = fabs(x);
        if ((a > 0 || lane >= jj) && valid[a] && ax > babs) {
          babs = ax;
          bv = x;
          bpos = lane + 32 * a;
        }
      }
      const uint64_t bits = (uint64_t)__double_as_longlong(babs);
      const unsigned khi = babs < 0.0 ? 0u : (unsigned)(bits >> 32) + 1u;
      const unsigned mhi = __reduce_max_sync(kFull, khi);
      const unsigned klo = khi == mhi ? (unsigned)bits : 0u;
      const unsigned mlo = __reduce_max_sync(kFull, klo);
      prel = (int)__reduce_min_sync(
          kFull, (unsigned)((khi == mhi && (unsigned)bits == mlo) ? bpos : INT_MAX));
      pv = __shfl_sync(kFull, bv, prel & 31);
      if (prel != jj && pv != 0.0) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
#pragma unroll
          for (int a = 0; a < R; ++a) Pw[c * LDP + lane + 32 * a] = P[c][a];
        __syncwarp();
        exchange_rows(Pw, LDP, prow, Lpe, tiles, Q, nt, jb, jj, prel, lane);
#pragma unroll
        for (int c = 0; c < 8; ++c)
#pragma unroll
          for (int a = 0; a < R; ++a) P[c][a] = Pw[c * LDP + lane + 32 * a];
        __syncwarp();
      }
      rcp = __drcp_rn(pv);
    }
    if (pv != 0.0) {
      if (fabs(pv) >= DBL_MIN) {
#pragma unroll
        for (int a = 0; a < R; ++a)
          if (lane + 32 * a > jj) P[jj][a] *= rcp;
      } else {
#pragma unroll
        for (int a = 0; a < R; ++a)
          if (lane + 32 * a > jj) P[jj][a] = slow_div(P[jj][a], pv);
      }
    }
#pragma unroll
    for (int c = jj + 1; c < 8; ++c) {
      const double u = __shfl_sync(kFull, P[c][0], jj);
#pragma unroll
      for (int a = 0; a < R; ++a)
        if (lane + 32 * a > jj) P[c][a] = fma(-P[jj][a], u, P[c][a]);
    }
    if (lane == 0) {
      const int k = c0 + jj;
      g.piv[e * Q + k] = c0 + prel;
      g.udiag[e * Q + k] = pv;
      g.dinv[e * Q + k] = rcp;
    }
    const double apv = fabs(pv);
    dmin = apv < dmin ? apv : dmin;
  }
  // ---- 4. store L (below the diagonal) and the diagonal block's U
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if (c >= ncol) break;
    const int j = c0 + c;
    double* lcol = Lpe + (ol32(j, Q) - c - 1);  // + rel
#pragma unroll
    for (int a = 0; a < R; ++a) {
      const int rel = lane + 32 * a;
      if (rel > c && rel < nrel) st_first(lcol + rel, P[c][a], pol);
    }
    if (lane < c) st_first(Upe + ou32(j, Q) + c0 + lane, P[c][0], pol);
  }
#pragma unroll
  for (int c = 0; c < 8; ++c)
#pragma unroll
    for (int a = 0; a < R; ++a) Pw[c * LDP + lane + 32 * a] = P[c][a];
  __syncwarp();
}

template <int NT>
__global__ void __launch_bounds__(kTileWarps * 32, TileShape<NT>::kMinBlocks)
    lu_tile_kernel(LuArgs g, double* __restrict__ scr, int scr_pol, int a_pol,
                   const int64_t* __restrict__ list, const int* __restrict__ list_count) {
  using S = TileShape<NT>;
  constexpr int R = S::R, LDP = S::LDP;
  extern __shared__ double smem_tile[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = lane >> 2, q = lane & 3;
  double* Pw = smem_tile + w * S::kWarpDoubles;  // 8 columns x LDP relative rows
  double* stg = Pw + 8 * LDP;                     // 8 x 8 inverse staging
  double* Ls = stg + 64;                          // -L11^-1 tiles (kLinvSmem)
  int* prow = reinterpret_cast<int*>(smem_tile + kTileWarps * S::kWarpDoubles) + w * S::kWarpInts;
  const int Q = g.Q;
  const int npanel = (Q + 7) / 8;
  const int64_t wid = (int64_t)blockIdx.x * kTileWarps + w;
  double* slot = scr + wid * S::kSlotDoubles;
  const uint64_t pol = policy_evict_first();
  const uint64_t spol = make_policy(scr_pol), apol = make_policy(a_pol ? 2 : 0);

  // with a list (the blocks the pipelined kernel handed back, lu_pipe.cu) the
  // grid walks list[0 .. *list_count)
  const int64_t nwork = list ? (int64_t)*list_count : g.nblocks;
  for (int64_t it = wid; it < nwork; it += (int64_t)gridDim.x * kTileWarps) {
    const int64_t e = list ? list[it] : it;
    const double* __restrict__ Ae = g.A + e * (int64_t)Q * Q;
    double* Lpe = g.Lp + e * g.ldL;
    double* Upe = g.Up + e * g.ldL;
    for (int i = lane; i < 32 * R; i += 32) prow[i] = i;
    __syncwarp();
    unsigned amh = 0;  // max over the block of the high word of |a_ij|
    double dmin = DBL_MAX;

    for (int jb = 0; jb < npanel; ++jb) {
      const int c0 = 8 * jb;
      const int ncol = min(8, Q - c0);
      const int nrel = Q - c0;  // rows at or below the panel's first row
      const int ca = c0 + 2 * q;
      const bool v0 = ca < Q, v1 = ca + 1 < Q;
      // ---- 1. gather (C-fragment layout)
      double T[NT][2];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int pos = 8 * t + r;
        const bool vr = pos < Q;
        const double* src = Ae + prow[vr ? pos : 0] * Q + ca;
        T[t][0] = (vr && v0) ? ld_a(src, apol) : 0.0;
        T[t][1] = (vr && v1) ? ld_a(src + 1, apol) : 0.0;
        amh = max(amh, max(hi_abs(T[t][0]), hi_abs(T[t][1])));
      }
      // ---- 2. left-looking updates with the earlier panels (DMMA)
      {
        double* U0 = Upe + ou32(v0 ? ca : 0, Q) + r;
        double* U1 = Upe + ou32(v1 ? ca + 1 : 0, Q) + r;
#pragma unroll
        for (int kb = 0; kb < NT - 1; ++kb) {
          if (kb >= jb) break;
          // the L tiles' loads go out first and overlap the -U_kb chain
          double2 lf[NT];
#pragma unroll
          for (int t = kb + 1; t < NT; ++t) {
            if (8 * t >= Q) break;  // padding tiles (NT rounded up)
            lf[t] = ld_v2(slot + tri(kb, t, NT) * 64 + 2 * lane, spol);
          }
          const double2 li = S::kLinvSmem
                                 ? *reinterpret_cast<const double2*>(Ls + kb * 64 + 2 * lane)
                                 : ld_v2(slot + tri(kb, kb, NT) * 64 + 2 * lane, spol);
          double u0 = 0.0, u1 = 0.0;  // -U_kb (C layout)
          dmma_acc(u0, u1, li.x, bfrag(T[kb][0], T[kb][1], 0, lane));
          dmma_acc(u0, u1, li.y, bfrag(T[kb][0], T[kb][1], 1, lane));
          const double ub0 = bfrag(u0, u1, 0, lane), ub1 = bfrag(u0, u1, 1, lane);
#pragma unroll
          for (int t = kb + 1; t < NT; ++t) {
            if (8 * t >= Q) break;
            dmma_acc(T[t][0], T[t][1], lf[t].x, ub0);
            dmma_acc(T[t][0], T[t][1], lf[t].y, ub1);
          }
          if (v0) st_first(U0 + 8 * kb, -u0, pol);
          if (v1) st_first(U1 + 8 * kb, -u1, pol);
        }
      }
      // ---- 3. rows >= c0 to the relative row layout through shared memory
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        if (t >= jb) {
          Pw[(2 * q) * LDP + 8 * (t - jb) + r] = T[t][0];
          Pw[(2 * q + 1) * LDP + 8 * (t - jb) + r] = T[t][1];
        }
      }
      __syncwarp();
      factor_panel<R, LDP>(Pw, prow, Lpe, Upe, slot, NT, g, e, jb, lane, pol, dmin);
      if (jb + 1 < npanel) {
        // L tiles (rows of tile t > jb) and -L11^-1 to scratch, A-fragment order
        for (int t = jb + 1; t < NT; ++t) {
          const int rel = 8 * (t - jb) + r;
          const bool vr = rel < nrel;
          double2 o;
          o.x = vr ? Pw[q * LDP + rel] : 0.0;
          o.y = vr ? Pw[(4 + q) * LDP + rel] : 0.0;
          st_v2(slot + tri(jb, t, NT) * 64 + 2 * lane, o, spol);
        }
        if (S::kLinvSmem) {
          neg_linv<LDP>(Pw, Ls + jb * 64, lane);
        } else {
          neg_linv<LDP>(Pw, stg, lane);
          __syncwarp();
          st_v2(slot + tri(jb, jb, NT) * 64 + 2 * lane,
                *reinterpret_cast<const double2*>(stg + 2 * lane), spol);
        }
      }
      __syncwarp();
    }
    for (int64_t i = (int64_t)Q * (Q - 1) / 2 + lane; i < g.ldL; i += 32) {
      Lpe[i] = 0.0;
      Upe[i] = 0.0;
    }
    for (int i = lane; i < Q; i += 32) g.perm[e * Q + i] = prow[i];
    const int sing = singular_test(Ae, Q * Q, __reduce_max_sync(kFull, amh), dmin, lane);
    if (lane == 0) g.stat[e] = sing;
    __syncwarp();
  }
}

template <int NT>
int launch_nt(mh_system* s, const LuArgs& g, cudaEvent_t start, const int64_t* list,
              const int* list_count, int64_t nwork) {
  using S = TileShape<NT>;
  const size_t smem = S::smem_bytes();
  MH_CHECK_CUDA(cudaFuncSetAttribute(lu_tile_kernel<NT>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  MH_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lu_tile_kernel<NT>,
                                                              kTileWarps * 32, smem));
  per_sm = std::max(per_sm, 1);
  // resident CTAs per SM: 3 (12 warps) measured best at c2 / c3 -- more warps
  // hide more latency but their scratch slots crowd L2 (MEHDG_LU_CTAS overrides)
  per_sm = std::max(1, std::min(per_sm, s->knobs.lu_ctas));
  const int scr_pol = s->knobs.lu_scr_pol, a_pol = s->knobs.lu_a_pol;
  const int64_t need = (nwork + kTileWarps - 1) / kTileWarps;
  const int64_t grid = std::min<int64_t>(need, (int64_t)per_sm * s->num_sms);
  MH_CHECK(s->lu_scr.ensure((size_t)grid * kTileWarps * S::kSlotDoubles));
  if (start) MH_CHECK_CUDA(cudaEventRecord(start, s->stream));
  lu_tile_kernel<NT><<<(unsigned)grid, kTileWarps * 32, smem, s->stream>>>(g, s->lu_scr.p, scr_pol, a_pol,
                                                                             list, list_count);
  MH_CHECK_CUDA(cudaGetLastError());
  return MH_OK;
}

}  // namespace

// Q in 33..256: NT = ceil(Q / 8) tiles, instantiated for the BASELINE shapes
// (Q = 84, 91, 165, 220 -> NT = 11, 12, 21, 28) and a few sizes between.
// `list` / `list_count` (device) / `nwork` (host copy of the count): factor only
// the listed blocks; nullptr / nullptr / -1: all of them.
int launch_lu_tile(mh_system* s, const LuArgs& g, cudaEvent_t start, const int64_t* list,
                   const int* list_count, int64_t nwork) {
  if (nwork < 0) nwork = g.nblocks;
  const int nt = (g.Q + 7) / 8;
#define MH_NT(N) \
  if (nt <= N) return launch_nt<N>(s, g, start, list, list_count, nwork);
  MH_NT(6) MH_NT(8) MH_NT(10) MH_NT(11) MH_NT(12) MH_NT(14) MH_NT(16) MH_NT(18) MH_NT(21)
  MH_NT(24) MH_NT(28) MH_NT(32)
#undef MH_NT
  set_error("Q > 256 is not supported by the batched LU");
  return MH_E_UNSUPPORTED;
}

}  // namespace mh
