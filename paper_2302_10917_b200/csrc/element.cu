// Fused per-macro element kernel: one warp per macro, persistent warps fed
// by a TMA bulk-copy stream (stream.cuh).
//
// Replaces the macro_task of apply_schur (schur_solver.py:271-277),
// macro_rhs of condense (:244-246) and the reconstruct_interior task
// (:426-429).  Per macro e, with lane l owning rows i = l + 32 r:
//   gather   ue = uhat through the face table (zeros on Dirichlet slots)
//   step 1   x  = P (B ue)        B = op.B, streamed as op.B^T rows (nc x Q)
//   step 2   y  = U^-1 L^-1 x     column-oriented substitution with warp
//                                 shuffles; L and U are streamed as packed
//                                 column segments (forward: L columns
//                                 0..Q-2, backward: U columns Q-1..1)
//   step 3   v  = C y             op.C rows, 32-row transpose-reduce
//   write    V[e*nc + c]          the macro's slot segment; the face kernel
//                                 subtracts it in left-then-right order, so
//                                 there are no atomics and the result is
//                                 deterministic.
// Modes: kApply (above), kRhs (x = P R_u, writes v), kRecon
// (x = P (R_u - B ue), writes y = u_e).
//
// HBM traffic per macro = 8 (nc Q [B] + Q(Q-1) [L,U] + nc Q [C]) + small
// vectors.  When op.C = op.B^T (the BASELINE operator) the C segment is the
// same memory as the B segment; it is fetched with an L2 evict_last policy
// on its first read so the second read is served from L2.
//
// The kernel is issue-bound once the stream keeps HBM busy, so the loops
// are written for instruction count: rows / columns are consumed in groups
// of four behind one ring-window check, and a group that does not wrap
// around the ring end is read with immediate-offset shared loads.

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "mh_internal.h"
#include "stream.cuh"

// the kMb instantiations leave the macro loop body after step 1 (`continue`): the
// steps behind it are unreachable there by design
#pragma nv_diag_suppress 128

namespace mh {
namespace {

// Consumer warps (macros in flight) per CTA, plus one producer warp; 12 / kWPB
// CTAs per SM.  3 + 1 warps at 4 CTAs/SM (12 consumers, 4 producers per SM)
// measured 5.52 TB/s at c2 against 5.32 for 4 + 1 at 3 CTAs/SM (same box);
// 2 + 1 at 6 CTAs/SM (96 registers) 4.75.
#ifndef MH_ELEM_WPB
#define MH_ELEM_WPB 3
#endif
#ifndef MH_ELEM_MINB
#define MH_ELEM_MINB (12 / MH_ELEM_WPB)
#endif
#ifndef MH_ELEM_G
#define MH_ELEM_G 8  // L / U columns per ring-window check in the substitutions (4 when 8 Q does not fit)
#endif
#ifndef MH_ELEM_GR
#define MH_ELEM_GR 8  // op.B^T / op.C rows per ring-window check in steps 1 and 3 (when 8 Q <= 800)
#endif
#ifndef MH_ELEM_RING
#define MH_ELEM_RING 2048
#endif
constexpr int kWPB = MH_ELEM_WPB;
constexpr int kThreads = (kWPB + 1) * 32;

struct ElemArgs {
  const int32_t* elem_ufac;
  const double* uhat;
  const double* uhalo;  // received halo segments (trace index >= F)
  const double* Bt;     // N x ldB   (op.B^T rows, nc x Q)
  const double* Cm;     // N x ldB   (op.C rows,   nc x Q)
  const double* Lp;     // N x ldL   packed strict lower, columns 0..Q-2
  const double* Up;     // N x ldL   packed strict upper, columns Q-1..1
  const double* dinv;
  const int32_t* perm;
  const double* Ru;
  double* out;
  int64_t N, F, ldB, ldL;
  int64_t e_lo;  // macros [e_lo, N) are processed
  int Q, nc, t, nfe;
  int c_is_bt;
  int bpol, lpol;  // L2 policies of the op.B^T first read and of the L / U streams
  const int* skip;  // a stopped speculative GMRES step: return at once
};

// 8 per-lane partial sums -> the full sum of partial (lane >> 2) & 7, held by
// the 4 lanes with that value of bits 2..4 (3 transpose stages + 2 reductions:
// 9 shuffles per 8 sums, 8 live registers instead of 32)
__device__ __forceinline__ double transpose_reduce8(double (&p)[8], int lane) {
#pragma unroll
  for (int w = 4, bit = 16; w >= 1; w >>= 1, bit >>= 1) {
    const bool upper = (lane & bit) != 0;
#pragma unroll
    for (int q = 0; q < w; ++q) {
      const double send = upper ? p[q] : p[q + w];
      const double keep = upper ? p[q + w] : p[q];
      p[q] = keep + __shfl_xor_sync(kFull, send, bit);
    }
  }
  double v = p[0];
  v += __shfl_xor_sync(kFull, v, 2);
  v += __shfl_xor_sync(kFull, v, 1);
  return v;
}

template <int RING>
__device__ __forceinline__ bool no_wrap(uint32_t lo, uint32_t span) {
  return rmod<RING>(lo) + span <= (uint32_t)RING;
}

// x_i += sum over NR rows c of op.B^T[c][perm_i] * ue_c, rows at stream p, p+Q, ...
template <int R, int NR, int RING, bool WRAP, bool PERM>
__device__ __forceinline__ void gemv_rows(double (&acc)[R], const double* ring, uint32_t p, int Q,
                                          const double* su, const int (&pr)[R], int lane) {
#pragma unroll
  for (int u = 0; u < NR; ++u) {
    const double uc = su[u];
    const double* cb = ring + rmod<RING>(p);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = PERM ? pr[r] : lane + 32 * r;
      const double b = WRAP ? ring[rmod<RING>(p + (uint32_t)i)] : cb[i];
      if (lane + 32 * r < Q) acc[r] = fma(b, uc, acc[r]);
    }
    p += Q;
  }
}

// forward substitution over NC packed L columns j0.. (JB = j0 / 32 is a
// compile-time constant once the caller's block loop is unrolled)
template <int R, int NC, int RING, bool WRAP>
__device__ __forceinline__ void fwd_cols(double (&y)[R], const double* ring, uint32_t p, int JB,
                                         int j0, int Q, int lane) {
  const int jj0 = j0 & 31;
#pragma unroll
  for (int u = 0; u < NC; ++u) {
    const int j = j0 + u;
    const uint32_t q0 = p - (uint32_t)(j + 1);  // stream position of "row 0"
    const double yj = __shfl_sync(kFull, y[JB], jj0 + u);
    const double* cb = ring + rmod<RING>(q0);
#pragma unroll
    for (int r = JB; r < R; ++r) {
      const int i = lane + 32 * r;
      const double l = WRAP ? ring[rmod<RING>(q0 + (uint32_t)i)] : cb[i];
      if (r > JB || lane > jj0 + u) y[r] = fma(-l, yj, y[r]);
    }
    p += (uint32_t)(Q - 1 - j);
  }
}

// back substitution over NC packed U columns j0, j0-1, .. (descending)
template <int R, int NC, int RING, bool WRAP>
__device__ __forceinline__ void bwd_cols(double (&y)[R], const double (&dr)[R],
                                         const double* ring, uint32_t p, int JB, int j0,
                                         int lane) {
  const int jj0 = j0 & 31;
#pragma unroll
  for (int u = 0; u < NC; ++u) {
    const int j = j0 - u;
    if (lane == jj0 - u) y[JB] *= dr[JB];
    const double yj = __shfl_sync(kFull, y[JB], jj0 - u);
    const double* cb = ring + rmod<RING>(p);
#pragma unroll
    for (int r = 0; r <= JB; ++r) {
      const int i = lane + 32 * r;
      const double uv = WRAP ? ring[rmod<RING>(p + (uint32_t)i)] : cb[i];
      if (r < JB || lane < jj0 - u) y[r] = fma(-uv, yj, y[r]);
    }
    p += (uint32_t)j;
  }
}

// partial dot product of one op.C row with y
template <int R, int RING, bool WRAP>
__device__ __forceinline__ double dot_row(const double (&y)[R], const double* ring, uint32_t p,
                                          int Q, int lane) {
  double acc = 0.0;
  const double* cb = ring + rmod<RING>(p);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = lane + 32 * r;
    const double c = WRAP ? ring[rmod<RING>(p + (uint32_t)i)] : cb[i];
    if (i < Q) acc = fma(c, y[r], acc);
  }
  return acc;
}

template <int R, int MODE, int RING, int CH>
__global__ void __launch_bounds__(kThreads, MH_ELEM_MINB)
element_kernel(ElemArgs a) {
  if (a.skip && *a.skip) return;
  constexpr int S = RING / CH;
  using PipeT = Pipe<RING, CH, kWPB>;
  using ConsT = Consumer<RING, CH>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ Segment segs[4];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int Q = a.Q, nc = a.nc, t = a.t;
  const int nchB = (int)(a.ldB / CH), nchL = (int)(a.ldL / CH);
  double* rings = reinterpret_cast<double*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(rings + (size_t)kWPB * RING);
  uint64_t* empty = full + kWPB * S;
  double* su_all = reinterpret_cast<double*>(empty + kWPB * S);
  const int nseg = MODE == kMb ? 1 : (MODE != kRhs ? 1 : 0) + 2 + (MODE != kRecon ? 1 : 0);
  (void)t;
  if (threadIdx.x == 0) {
    int n = 0;
    if (MODE != kRhs) segs[n++] = Segment{a.Bt, a.ldB, nchB, (MODE == kApply && a.c_is_bt) ? a.bpol : 0};
    if (MODE != kMb) {
      segs[n++] = Segment{a.Lp, a.ldL, nchL, a.lpol};
      segs[n++] = Segment{a.Up, a.ldL, nchL, a.lpol};
      if (MODE != kRecon) segs[n++] = Segment{a.Cm, a.ldB, nchB, 0};
    }
    for (int i = 0; i < 2 * kWPB * S; ++i) mbar_init(&full[i], 1);  // full + empty
    fence_mbar_init();
  }
  __syncthreads();  // the only CTA-wide barrier
  const int64_t W = (int64_t)gridDim.x * kWPB;
  if (w == kWPB) {  // producer warp
    if (lane == 0)
      PipeT::produce(rings, full, empty, segs, nseg, a.e_lo + (int64_t)blockIdx.x * kWPB, W, a.N,
                     kWPB);
    return;
  }
  const double* ring = rings + (size_t)w * RING;
  double* su = su_all + (size_t)w * ((nc + 3) & ~3);
  ConsT cs;
  cs.full = full + w * S;
  cs.empty = empty + w * S;
  const uint32_t offL = (MODE != kRhs) ? (uint32_t)a.ldB : 0u;
  const uint32_t offU = offL + (uint32_t)a.ldL;
  const uint32_t offC = offU + (uint32_t)a.ldL;
  const uint32_t E = MODE == kMb ? (uint32_t)a.ldB : offC + ((MODE != kRecon) ? (uint32_t)a.ldB : 0u);

  // Software pipeline over a warp's macros: the small per-macro vectors of
  // the NEXT macro (perm, 1/U_jj, face table, gathered uhat) are loaded while
  // this one is processed, so their latency never sits at the start of a macro.
  constexpr int RC = 8;  // gathered slot values per lane (nc <= 256)
  int pr_n[R];
  double dr_n[R];
  int32_t ef_n[kMaxSlots];
  double g_n[RC];
  auto load_meta = [&](int64_t en) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = lane + 32 * r;
      pr_n[r] = (MODE != kMb && i < Q) ? __ldg(a.perm + en * Q + i) : i;
      dr_n[r] = (MODE != kMb && i < Q) ? __ldg(a.dinv + en * Q + i) : 0.0;
    }
#pragma unroll
#pragma unroll
    for (int k = 0; k < kMaxSlots; ++k)
      ef_n[k] = k < a.nfe ? __ldg(a.elem_ufac + en * a.nfe + k) : -1;
  };
  auto gather_next = [&]() {
#pragma unroll
    for (int q = 0; q < RC; ++q) {
      const int c = lane + 32 * q;
      double v = 0.0;
      if (c < nc) {
        const int k = c / t, s = c - k * t;
        int f = ef_n[0];
#pragma unroll
        for (int kk = 1; kk < kMaxSlots; ++kk) f = (k == kk) ? ef_n[kk] : f;
        if (f >= 0)
          v = f < a.F ? __ldg(a.uhat + (int64_t)f * t + s)
                      : __ldg(a.uhalo + (int64_t)(f - a.F) * t + s);
      }
      g_n[q] = v;
    }
  };
  const int64_t e_first = a.e_lo + (int64_t)blockIdx.x * kWPB + w;
  if (e_first < a.N) {
    load_meta(e_first);
    if (MODE != kRhs) gather_next();
  }

  uint32_t base = 0;
  for (int64_t e = e_first; e < a.N; e += W, base += E) {
    int pr[R];
    double dr[R];
    bool ident = true;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = lane + 32 * r;
      pr[r] = pr_n[r];
      dr[r] = dr_n[r];
      ident = ident && pr[r] == i;
    }
    if (MODE != kRhs) {
#pragma unroll
      for (int q = 0; q < RC; ++q)
        if (lane + 32 * q < nc) su[lane + 32 * q] = g_n[q];
    }
    const int64_t en = e + W;
    if (en < a.N) load_meta(en);  // lands while this macro is processed
    const bool has_perm = !__all_sync(kFull, ident);
    double y[R];
    if (MODE == kRhs) {
#pragma unroll
      for (int r = 0; r < R; ++r) y[r] = (lane + 32 * r < Q) ? __ldg(a.Ru + e * Q + pr[r]) : 0.0;
    } else {
      __syncwarp();
      double acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = 0.0;
      uint32_t p = base;
      int c = 0;
      constexpr int GR = (MH_ELEM_GR > 4 && MH_ELEM_GR * 32 * R <= (RING / CH - 1) * CH)
                             ? MH_ELEM_GR : 4;  // rows per ring-window check
      // 8-row groups only while they span at most ~half the ring slack (c2, c3;
      // at Q = 165 most 8-row groups would wrap the ring end)
      const bool rows8 = 8 * Q <= 800;
      for (; rows8 && c + GR <= nc; c += GR, p += (uint32_t)(GR * Q)) {  // step 1: x = B ue
        cs.window(p, p + (uint32_t)(GR * Q), lane);
        if (!has_perm && no_wrap<RING>(p, (uint32_t)(GR * Q) + 32u * R)) {
          gemv_rows<R, GR, RING, false, false>(acc, ring, p, Q, su + c, pr, lane);
        } else {
          gemv_rows<R, GR, RING, true, true>(acc, ring, p, Q, su + c, pr, lane);
        }
      }
      for (; c + 4 <= nc; c += 4, p += 4u * (uint32_t)Q) {
        cs.window(p, p + 4u * Q, lane);
        gemv_rows<R, 4, RING, true, true>(acc, ring, p, Q, su + c, pr, lane);
      }
      for (; c < nc; ++c, p += (uint32_t)Q) {
        cs.window(p, p + Q, lane);
        gemv_rows<R, 1, RING, true, true>(acc, ring, p, Q, su + c, pr, lane);
      }
      __syncwarp();  // su is rewritten for the next macro
      if (en < a.N) gather_next();  // its face table arrived during step 1
      if (MODE == kMb) {  // explicit element Schur: the rows were S_e^T's, Q = nc
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int i = lane + 32 * r;
          if (i < Q) a.out[e * Q + i] = acc[r];
        }
        continue;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (MODE == kApply) y[r] = acc[r];
        else y[r] = (lane + 32 * r < Q) ? __ldg(a.Ru + e * Q + pr[r]) - acc[r] : 0.0;
      }
    }

    // step 2a: unit-lower forward substitution over packed L columns 0..Q-2
    {
      uint32_t p = base + offL;
#pragma unroll
      for (int jb = 0; jb < R; ++jb) {
        const int jend = min(jb * 32 + 32, Q - 1);
        int j0 = jb * 32;
        constexpr int G = (MH_ELEM_G > 4 && MH_ELEM_G * 32 * R <= (RING / CH - 1) * CH) ? MH_ELEM_G : 4;
        for (; j0 + G <= jend; j0 += G) {
          const uint32_t span = (uint32_t)(G * (Q - 1 - j0) - G * (G - 1) / 2);
          cs.window(p, p + span, lane);
          if (no_wrap<RING>(p - (uint32_t)(j0 + 1), span + (uint32_t)(j0 + 1) + 32u * R + 8u)) {
            fwd_cols<R, G, RING, false>(y, ring, p, jb, j0, Q, lane);
            p += span;
          } else {
#pragma unroll 1
            for (int u = 0; u < G; ++u) {  // rare: the group wraps around the ring end
              fwd_cols<R, 1, RING, true>(y, ring, p, jb, j0 + u, Q, lane);
              p += (uint32_t)(Q - 1 - (j0 + u));
            }
          }
        }
        for (; j0 < jend; ++j0) {
          const uint32_t span = (uint32_t)(Q - 1 - j0);
          cs.window(p, p + span, lane);
          fwd_cols<R, 1, RING, true>(y, ring, p, jb, j0, Q, lane);
          p += span;
        }
      }
    }
    // step 2b: upper back substitution over packed U columns Q-1 .. 0 (column
    // 0 has no strictly-upper entries, only the diagonal)
    {
      uint32_t p = base + offU;
#pragma unroll
      for (int jb = R - 1; jb >= 0; --jb) {
        int j0 = min(jb * 32 + 31, Q - 1);
        constexpr int G = (MH_ELEM_G > 4 && MH_ELEM_G * 32 * R <= (RING / CH - 1) * CH) ? MH_ELEM_G : 4;
        for (; j0 - (G - 1) >= jb * 32; j0 -= G) {
          const uint32_t span = (uint32_t)(G * j0 - G * (G - 1) / 2);
          cs.window(p, p + span, lane);
          if (no_wrap<RING>(p, span + 32u * R + 8u)) {
            bwd_cols<R, G, RING, false>(y, dr, ring, p, jb, j0, lane);
            p += span;
          } else {
#pragma unroll 1
            for (int u = 0; u < G; ++u) {
              bwd_cols<R, 1, RING, true>(y, dr, ring, p, jb, j0 - u, lane);
              p += (uint32_t)(j0 - u);
            }
          }
        }
        for (; j0 >= jb * 32; --j0) {
          cs.window(p, p + j0, lane);
          bwd_cols<R, 1, RING, true>(y, dr, ring, p, jb, j0, lane);
          p += (uint32_t)j0;
        }
      }
    }

    if (MODE == kRecon) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = lane + 32 * r;
        if (i < Q) a.out[e * Q + i] = y[r];
      }
      continue;
    }

    // step 3: v_c = sum_i C[c][i] y_i, 8 rows per transpose-reduce
    uint32_t p = base + offC;
    for (int c0 = 0; c0 < nc; c0 += 8) {
      double pp[8];
      const int nrow = min(8, nc - c0);
      constexpr bool G8 = MH_ELEM_GR >= 8 && 8 * 32 * R <= (RING / CH - 1) * CH;
      if (G8 && nrow == 8 && 8 * Q <= 800) {  // one ring-window check for the 8 rows
        cs.window(p, p + 8u * Q, lane);
        if (no_wrap<RING>(p, 8u * Q + 32u * R)) {
#pragma unroll
          for (int u = 0; u < 8; ++u) pp[u] = dot_row<R, RING, false>(y, ring, p + u * Q, Q, lane);
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u) pp[u] = dot_row<R, RING, true>(y, ring, p + u * Q, Q, lane);
        }
        p += 8u * Q;
      } else
#pragma unroll
      for (int q0 = 0; q0 < 8; q0 += 4) {
        if (q0 + 4 <= nrow) {
          cs.window(p, p + 4u * Q, lane);
          if (no_wrap<RING>(p, 4u * Q + 32u * R)) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
              pp[q0 + u] = dot_row<R, RING, false>(y, ring, p + u * Q, Q, lane);
          } else {
#pragma unroll
            for (int u = 0; u < 4; ++u)
              pp[q0 + u] = dot_row<R, RING, true>(y, ring, p + u * Q, Q, lane);
          }
          p += 4u * Q;
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (q0 + u < nrow) {
              cs.window(p, p + Q, lane);
              pp[q0 + u] = dot_row<R, RING, true>(y, ring, p, Q, lane);
              p += Q;
            } else {
              pp[q0 + u] = 0.0;
            }
          }
        }
      }
      const double v = transpose_reduce8(pp, lane);
      const int row = (lane >> 2) & 7;
      if ((lane & 3) == 0 && row < nrow) a.out[e * nc + c0 + row] = v;
    }
  }
}

template <int RING, int CH>
size_t smem_bytes(int nc) {
  return (size_t)kWPB * RING * sizeof(double) + (size_t)2 * kWPB * (RING / CH) * sizeof(uint64_t) +
         (size_t)kWPB * ((nc + 3) & ~3) * sizeof(double);
}

template <int R, int MODE, int RING, int CH>
int launch_rc(mh_system* s, const ElemArgs& a, cudaStream_t st) {
  static_assert(kStreamChunk % CH == 0, "HBM padding must be a multiple of the ring chunk");
  const size_t smem = smem_bytes<RING, CH>(s->nc);
  auto kern = element_kernel<R, MODE, RING, CH>;
  // attribute + occupancy are host-side driver calls (microseconds): once per
  // instantiation and shared-memory size, not per apply (GMRES launches an
  // apply per Arnoldi step right after a host round trip)
  // the max-dynamic-smem attribute is per function and process-wide: a
  // process-wide cache keyed by (device, kernel, smem), the attribute only ever
  // raised (a launch with less smem stays valid), under a mutex
  int per_sm = launch_occupancy(s->device, reinterpret_cast<const void*>(kern), kThreads, smem);
  if (per_sm < 0) return MH_E_CUDA;
  if (per_sm < 1) per_sm = 1;
  if (s->knobs.elem_ctas > 0) per_sm = std::max(1, std::min(per_sm, s->knobs.elem_ctas));
  int64_t grid = (int64_t)s->num_sms * per_sm;
  const int64_t need = (a.N - a.e_lo + kWPB - 1) / kWPB;
  if (grid > need) grid = need;
  kern<<<(unsigned)grid, kThreads, smem, st>>>(a);
  MH_CHECK_CUDA(cudaGetLastError());
  return MH_OK;
}

template <int R, int MODE>
int launch_rm(mh_system* s, const ElemArgs& a, cudaStream_t st) {
  // 16 KB rings of four 4 KB chunks, 12 consumer warps per SM.  Measured
  // alternatives at c2: 8 KB rings of 2 KB chunks at 16 consumers/SM -13%,
  // 12 KB rings of three 4 KB chunks -1.5%, 2 KB / 1 KB chunks (MEHDG_ELEM_CH)
  // -22% / -57%.
  const int ch = s->knobs.elem_ch;
  if (ch == 256) return launch_rc<R, MODE, MH_ELEM_RING, 256>(s, a, st);
  if (ch == 128) return launch_rc<R, MODE, MH_ELEM_RING, 128>(s, a, st);
  return launch_rc<R, MODE, MH_ELEM_RING, 512>(s, a, st);
}

#include "element_split.cuh"

// v = S_e ue through the same stream pipeline: one segment (S_e^T, nc rows of nc)
int launch_mb(mh_system* s, const double* uhat, double* out, cudaStream_t st) {
  ElemArgs a{};
  a.elem_ufac = s->elem_ufac.p;
  a.uhat = uhat;
  a.uhalo = s->halo_u.p;
  a.Bt = s->S.p;
  a.out = out;
  a.N = s->N;
  a.e_lo = 0;
  a.F = s->F;
  a.ldB = s->ldS;
  a.ldL = kStreamChunk;
  a.Q = s->nc;
  a.nc = s->nc;
  a.t = s->t;
  a.nfe = s->nfe;
  a.skip = s->skip;
  switch ((s->nc + 31) / 32) {
    case 1: return launch_rc<1, kMb, MH_ELEM_RING, 512>(s, a, st);
    case 2: return launch_rc<2, kMb, MH_ELEM_RING, 512>(s, a, st);
    case 3: return launch_rc<3, kMb, MH_ELEM_RING, 512>(s, a, st);
    case 4: return launch_rc<4, kMb, MH_ELEM_RING, 512>(s, a, st);
    case 5: return launch_rc<5, kMb, MH_ELEM_RING, 512>(s, a, st);
    case 6: return launch_rc<6, kMb, MH_ELEM_RING, 512>(s, a, st);
    case 7: return launch_rc<7, kMb, MH_ELEM_RING, 512>(s, a, st);
    case 8: return launch_rc<8, kMb, MH_ELEM_RING, 512>(s, a, st);
  }
  set_error("element kernel: nc > 256 unsupported");
  return MH_E_UNSUPPORTED;
}

template <int MODE>
int launch_mode(mh_system* s, const double* uhat, double* out, cudaStream_t st, int64_t e_lo,
                int64_t e_hi) {
  if (e_hi <= e_lo) return MH_OK;
  ElemArgs a;
  a.elem_ufac = s->elem_ufac.p;
  a.uhat = uhat;
  a.uhalo = s->halo_u.p;
  a.Bt = s->Bt.p;
  a.Cm = s->c_is_bt ? s->Bt.p : s->Cm.p;
  a.Lp = s->Lp.p;
  a.Up = s->Up.p;
  a.dinv = s->dinv.p;
  a.perm = s->perm.p;
  a.Ru = s->Ru.p;
  a.out = out;
  a.N = e_hi;
  a.e_lo = e_lo;
  a.F = s->F;
  a.ldB = s->ldB;
  a.ldL = s->ldL;
  a.Q = s->Q;
  a.nc = s->nc;
  a.t = s->t;
  a.nfe = s->nfe;
  a.c_is_bt = s->c_is_bt ? 1 : 0;
  a.bpol = s->knobs.elem_bpol;
  a.lpol = s->knobs.elem_lpol;
  a.skip = MODE == kApply ? s->skip : nullptr;
  // apply mode with op.C = op.B^T and three or more row groups: the macro split
  // over its row groups, few macros in flight (MEHDG_ELEM_SPLIT)
  if (MODE == kApply && s->knobs.elem_split && s->c_is_bt && s->Q > 64) return launch_split(s, a, st);
  switch ((s->Q + 31) / 32) {
    case 1: return launch_rm<1, MODE>(s, a, st);
    case 2: return launch_rm<2, MODE>(s, a, st);
    case 3: return launch_rm<3, MODE>(s, a, st);
    case 4: return launch_rm<4, MODE>(s, a, st);
    case 5: return launch_rm<5, MODE>(s, a, st);
    case 6: return launch_rm<6, MODE>(s, a, st);
    case 7: return launch_rm<7, MODE>(s, a, st);
    case 8: return launch_rm<8, MODE>(s, a, st);
  }
  set_error("element kernel: Q > 256 unsupported");
  return MH_E_UNSUPPORTED;
}

}  // namespace

int launch_element_range(mh_system* s, int mode, const double* uhat, double* out,
                         cudaStream_t st, int64_t e_lo, int64_t e_hi) {
  if (s->Q > 256 || s->nc > 256) {
    set_error("element kernel: Q and nc must be <= 256");
    return MH_E_UNSUPPORTED;
  }
  e_lo = std::max<int64_t>(e_lo, 0);
  e_hi = std::min<int64_t>(e_hi, s->N);
  switch (mode) {
    case kApply: return launch_mode<kApply>(s, uhat, out, st, e_lo, e_hi);
    case kRhs: return launch_mode<kRhs>(s, uhat, out, st, e_lo, e_hi);
    case kRecon: return launch_mode<kRecon>(s, uhat, out, st, e_lo, e_hi);
  }
  set_error("bad element mode");
  return MH_E_ARG;
}

int launch_element_mb_stream(mh_system* s, const double* uhat, double* out) {
  if (s->N == 0) return MH_OK;
  return launch_mb(s, uhat, out, s->stream);
}

int launch_element(mh_system* s, int mode, const double* uhat, double* out) {
  return launch_element_range(s, mode, uhat, out, s->stream, 0, s->N);
}

}  // namespace mh
