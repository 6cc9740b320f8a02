// Explicit element Schur complements (matrix-based mode "mb").
//
// Replaces assemble_schur_explicit's macro_task (schur_solver.py:392-398):
//     Y = A^-1 B[:, mask]   (lu_solve with nc right-hand sides)
//     S_e = C[mask] Y
// and the "mb" operator S @ v of solve (schur_solver.py:513-515).  S_e is
// formed for all nc slots (Dirichlet rows/columns are masked by the caller)
// and stored transposed, St[c][c'] = (C A^-1 B)[c'][c], so that the apply
// kernel reads it with coalesced loads.  The apply streams N*nc^2 doubles
// per call instead of N*(Q^2 + 2 nc Q): 7.8x fewer bytes at BASELINE c2.
//
// form_dmma_kernel: the two triangular solves with nc right-hand sides and the
// C Y product as dense 8 x 8 tile contractions on the fp64 tensor cores
// (mma.m8n8k4.f64, SASS DMMA.8x8x4).  One CTA per (macro, group of up to 8 tile
// columns of right-hand sides); a warp owns ONE tile column, X = P B[:, 8
// columns], held in registers as ceil(Q / 8) C fragments, and runs the blocked
// right-looking substitutions
//     Y_k = L_kk^-1 X_k;  X_i -= L_ik Y_k (i > k)      (forward)
//     Y_k = U_kk^-1 X_k;  X_i -= U_ik Y_k (i < k)      (backward)
// with the inverses of the 8 x 8 diagonal blocks (formed once per CTA, 8 lanes
// per block) and the off-diagonal tiles of -L, then of -U, staged by the whole
// CTA from the packed streams (coalesced column reads) into shared memory in
// A-fragment order -- each inner step is two conflict-free shared loads and two
// DMMA.  S^T tile (c, c') = sum_k C(c', k) Y_k is accumulated over the row
// tiles with C's rows as A fragments.

#include "mh_internal.h"

namespace mh {
namespace {

constexpr int kMbWarps = 4;

__host__ __device__ __forceinline__ int64_t off_lower(int j, int Q) {
  return (int64_t)j * (Q - 1) - (int64_t)j * (j - 1) / 2;
}
__host__ __device__ __forceinline__ int64_t off_upper(int j, int Q) {
  return (int64_t)Q * (Q - 1) / 2 - (int64_t)j * (j + 1) / 2;
}

struct FormArgs {
  const double* Bt;   // N x ldB  (op.B^T rows: Bt[c*Q + i] = B[i][c])
  const double* Cm;   // N x ldB  (op.C rows:   Cm[c*Q + i] = C[c][i])
  const double* Lp;
  const double* Up;
  const double* dinv;
  const int32_t* perm;
  double* St;         // N x ldS, block e: St[c * nc + c'] = (C A^-1 B)[c'][c]
  int64_t N, ldB, ldL, ldS;
  int Q, nc;
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// B fragment (4 x 8) of k-step kk of an 8 x 8 tile held as a C fragment: B[k][n]
// = T[4 kk + k][n]; lane (k = lane & 3, n = lane >> 2) takes it from the lane
// holding T's row 4 kk + k, column pair n / 2.
__device__ __forceinline__ double bfrag_of_c(double x0, double x1, int kk, int lane) {
  const int src = 4 * (4 * kk + (lane & 3)) + (lane >> 3);
  const double v0 = __shfl_sync(kFull, x0, src);
  const double v1 = __shfl_sync(kFull, x1, src);
  return ((lane >> 2) & 1) ? v1 : v0;
}

constexpr int kFormGroup = 8;  // S^T row tiles accumulated per pass over Y

// Tile columns are staged in NCH chunks (one, or two when all of -L does not fit
// the shared-memory budget): chunk c holds the block columns [NT c / NCH, NT (c+1) / NCH).
template <int NT>
struct FormCfg {
  static constexpr int NCH = NT > 28 ? 2 : 1;
  static constexpr int k0(int c) { return NT * c / NCH; }
  // tiles of L's block columns [a, b): sum over k of (NT - 1 - k)
  static constexpr int ltiles(int a, int b) { return (b - a) * (NT - 1) - (b * (b - 1) / 2 - a * (a - 1) / 2); }
  // tiles of U's block columns [a, b): sum over k of k
  static constexpr int utiles(int a, int b) { return b * (b - 1) / 2 - a * (a - 1) / 2; }
  static constexpr int max_tiles() {
    int m = 1;
    for (int c = 0; c < NCH; ++c) {
      const int l = ltiles(k0(c), k0(c + 1)), u = utiles(k0(c), k0(c + 1));
      m = l > m ? l : m;
      m = u > m ? u : m;
    }
    return m;
  }
  static constexpr size_t smem_bytes() { return (size_t)(max_tiles() + 2 * NT) * 64 * sizeof(double); }
};

// The substitution steps as template recursions over the block index, so every
// X[..] index is a compile-time constant (the tile column stays in registers).
struct FormCtx {
  const double* tiles;  // the staged chunk: tile t at t * 64, [k-step][lane]
  const double* Ce;
  const double* inv;
  int Q, nc, nt, lane, r, q;
};

// forward steps KB in [KB, K1) on a chunk staged from block column K0
template <int NT, int K0, int KB, int K1>
__device__ __forceinline__ void form_fwd(double (&X)[NT][2], const FormCtx& c) {
  if constexpr (KB < K1) {
    if (KB < c.nt) {
      const double b0 = bfrag_of_c(X[KB][0], X[KB][1], 0, c.lane);
      const double b1 = bfrag_of_c(X[KB][0], X[KB][1], 1, c.lane);
      double y0 = 0.0, y1 = 0.0;
      dmma(y0, y1, c.inv[(KB * 2 + 0) * 32 + c.lane], b0);
      dmma(y0, y1, c.inv[(KB * 2 + 1) * 32 + c.lane], b1);
      X[KB][0] = y0;
      X[KB][1] = y1;
      if (KB + 1 < c.nt) {
        const double yb0 = bfrag_of_c(y0, y1, 0, c.lane), yb1 = bfrag_of_c(y0, y1, 1, c.lane);
        const double* tl = c.tiles + (FormCfg<NT>::ltiles(K0, KB) - KB - 1) * 64 + c.lane;  // + it * 64
#pragma unroll
        for (int it = KB + 1; it < NT; ++it) {
          if (it < c.nt) {
            dmma(X[it][0], X[it][1], tl[it * 64], yb0);
            dmma(X[it][0], X[it][1], tl[it * 64 + 32], yb1);
          }
        }
      }
    }
    form_fwd<NT, K0, KB + 1, K1>(X, c);
  }
}

// backward steps KB down to K0 on a chunk staged from block column K0
template <int NT, int K0, int KB>
__device__ __forceinline__ void form_bwd(double (&X)[NT][2], const FormCtx& c) {
  if constexpr (KB >= K0) {
    if (KB < c.nt) {
      const double b0 = bfrag_of_c(X[KB][0], X[KB][1], 0, c.lane);
      const double b1 = bfrag_of_c(X[KB][0], X[KB][1], 1, c.lane);
      double y0 = 0.0, y1 = 0.0;
      dmma(y0, y1, c.inv[((NT + KB) * 2 + 0) * 32 + c.lane], b0);
      dmma(y0, y1, c.inv[((NT + KB) * 2 + 1) * 32 + c.lane], b1);
      X[KB][0] = y0;
      X[KB][1] = y1;
      if (KB > 0) {
        const double yb0 = bfrag_of_c(y0, y1, 0, c.lane), yb1 = bfrag_of_c(y0, y1, 1, c.lane);
        const double* tl = c.tiles + FormCfg<NT>::utiles(K0, KB) * 64 + c.lane;  // + it * 64
#pragma unroll
        for (int it = 0; it < KB; ++it) {
          dmma(X[it][0], X[it][1], tl[it * 64], yb0);
          dmma(X[it][0], X[it][1], tl[it * 64 + 32], yb1);
        }
      }
    }
    form_bwd<NT, K0, KB - 1>(X, c);
  }
}

// C's A fragments of row-tile step KB for the kFormGroup output tiles from g0
template <int NT>
__device__ __forceinline__ void form_cy_load(double (&a)[kFormGroup][2], int KB, int g0,
                                             const FormCtx& c) {
  const int i0 = 8 * KB + c.q, i1 = i0 + 4;
#pragma unroll
  for (int g = 0; g < kFormGroup; ++g) {
    const int cp = 8 * (g0 + g) + c.r;
    a[g][0] = (KB < c.nt && cp < c.nc && i0 < c.Q) ? __ldg(c.Ce + (size_t)cp * c.Q + i0) : 0.0;
    a[g][1] = (KB < c.nt && cp < c.nc && i1 < c.Q) ? __ldg(c.Ce + (size_t)cp * c.Q + i1) : 0.0;
  }
}

// acc(g) += C(tile g0 + g, k) Y_k over the row tiles k; the next step's C
// fragments are loaded before this step's DMMAs
template <int NT>
__device__ __forceinline__ void form_cy(const double (&X)[NT][2], double (&acc)[kFormGroup][2],
                                        int g0, const FormCtx& c) {
  // (two CTAs per SM for NT <= 12: 128 registers, no room for the second buffer)
  constexpr bool kAhead = NT > 12;
  double a[kAhead ? 2 : 1][kFormGroup][2];
  if (kAhead) form_cy_load<NT>(a[0], 0, g0, c);
#pragma unroll
  for (int KB = 0; KB < NT; ++KB) {
    if (!kAhead) form_cy_load<NT>(a[0], KB, g0, c);
    else if (KB + 1 < NT) form_cy_load<NT>(a[(KB + 1) & 1], KB + 1, g0, c);
    if (KB < c.nt) {
      const double yb0 = bfrag_of_c(X[KB][0], X[KB][1], 0, c.lane);
      const double yb1 = bfrag_of_c(X[KB][0], X[KB][1], 1, c.lane);
#pragma unroll
      for (int g = 0; g < kFormGroup; ++g) {
        dmma(acc[g][0], acc[g][1], a[kAhead ? (KB & 1) : 0][g][0], yb0);
        dmma(acc[g][0], acc[g][1], a[kAhead ? (KB & 1) : 0][g][1], yb1);
      }
    }
  }
}

// Stage -L's block columns [K0, K1) (tiles below the diagonal block, rows up to
// 8 NT, zero beyond Q) in A-fragment order: a warp per matrix column, lanes over
// its rows (the packed column is contiguous in global memory).
template <int NT, int K0, int K1>
__device__ __forceinline__ void stage_lower(double* tiles, const double* Le, int Q, int w, int W,
                                            int lane) {
  for (int j = 8 * K0 + w; j < 8 * K1; j += W) {
    const int kb = j >> 3, cj = j & 7;
    double* tc = tiles + (FormCfg<NT>::ltiles(K0, kb) - kb - 1) * 64 + (cj >> 2) * 32 + (cj & 3);
    const double* col = Le + off_lower(j, Q) - (j + 1);
    // all of the column's loads first, then the stores (the loads of a plain loop
    // wait for one another behind the shared-memory stores)
    constexpr int NI = (8 * NT + 31) / 32;
    double v[NI];
#pragma unroll
    for (int k = 0; k < NI; ++k) {
      const int i = 8 * (kb + 1) + lane + 32 * k;
      v[k] = (i < Q && j < Q) ? -__ldg(col + i) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < NI; ++k) {
      const int i = 8 * (kb + 1) + lane + 32 * k;
      if (i < 8 * NT) tc[(i >> 3) * 64 + (i & 7) * 4] = v[k];
    }
  }
}

// the same for -U's block columns [K0, K1): tiles above the diagonal block
template <int NT, int K0, int K1>
__device__ __forceinline__ void stage_upper(double* tiles, const double* Ue, int Q, int w, int W,
                                            int lane) {
  for (int j = 8 * K0 + w; j < 8 * K1; j += W) {
    const int kb = j >> 3, cj = j & 7;
    double* tc = tiles + FormCfg<NT>::utiles(K0, kb) * 64 + (cj >> 2) * 32 + (cj & 3);
    const double* col = Ue + off_upper(j, Q);
    constexpr int NI = (8 * NT + 31) / 32;
    double v[NI];
#pragma unroll
    for (int k = 0; k < NI; ++k) {
      const int i = lane + 32 * k;
      v[k] = (i < 8 * kb && j < Q) ? -__ldg(col + i) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < NI; ++k) {
      const int i = lane + 32 * k;
      if (i < 8 * kb) tc[(i >> 3) * 64 + (i & 7) * 4] = v[k];
    }
  }
}

template <int NT, int C>
__device__ __forceinline__ void form_fwd_chunks(double (&X)[NT][2], FormCtx& ctx, double* tiles,
                                                const double* Le, int w, int W, bool active) {
  using Cfg = FormCfg<NT>;
  if constexpr (C < Cfg::NCH) {
    constexpr int K0 = Cfg::k0(C), K1 = Cfg::k0(C + 1);
    stage_lower<NT, K0, K1>(tiles, Le, ctx.Q, w, W, ctx.lane);
    __syncthreads();
    if (active) form_fwd<NT, K0, K0, K1>(X, ctx);
    __syncthreads();
    form_fwd_chunks<NT, C + 1>(X, ctx, tiles, Le, w, W, active);
  }
}

template <int NT, int C>
__device__ __forceinline__ void form_bwd_chunks(double (&X)[NT][2], FormCtx& ctx, double* tiles,
                                                const double* Ue, int w, int W, bool active) {
  using Cfg = FormCfg<NT>;
  if constexpr (C >= 0) {
    constexpr int K0 = Cfg::k0(C), K1 = Cfg::k0(C + 1);
    stage_upper<NT, K0, K1>(tiles, Ue, ctx.Q, w, W, ctx.lane);
    __syncthreads();
    if (active) form_bwd<NT, K0, K1 - 1>(X, ctx);
    __syncthreads();
    form_bwd_chunks<NT, C - 1>(X, ctx, tiles, Ue, w, W, active);
  }
}

template <int NT>
__global__ void __launch_bounds__(256, NT <= 12 ? 2 : 1) form_dmma_kernel(FormArgs a) {
  extern __shared__ __align__(16) double form_smem[];
  double* inv = form_smem;              // [L | U][block][k-step][lane]: A fragments
  double* tiles = inv + 2 * NT * 64;    // the staged chunk of -L / -U tiles
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
  const int r = lane >> 2, q = lane & 3;
  const int64_t e = blockIdx.x;
  const int Q = a.Q, nc = a.nc;
  const int nt = (Q + 7) >> 3, nct = (nc + 7) >> 3;
  const double* __restrict__ Bte = a.Bt + e * a.ldB;
  const double* __restrict__ Ce = a.Cm + e * a.ldB;
  const double* __restrict__ Le = a.Lp + e * a.ldL;
  const double* __restrict__ Ue = a.Up + e * a.ldL;
  const int32_t* __restrict__ pe = a.perm + e * Q;
  const double* __restrict__ de = a.dinv + e * Q;
  double* __restrict__ Se = a.St + e * a.ldS;

  // ---- the inverses of the diagonal blocks: 8 lanes per block, one column each
  for (int kb = w * 4 + (lane >> 3); kb < nt; kb += 4 * W) {
    const int col = lane & 7, d0 = 8 * kb;
    double x[8];
    // L_kk^-1 (unit lower): column col by forward substitution
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      double sacc = 0.0;
#pragma unroll
      for (int m = 0; m < rr; ++m) {
        const int i = d0 + rr, j = d0 + m;
        const double l = i < Q ? __ldg(Le + off_lower(j, Q) + (i - j - 1)) : 0.0;
        sacc = fma(-l, x[m], sacc);
      }
      x[rr] = rr < col ? 0.0 : (rr == col ? 1.0 : sacc);
      inv[(kb * 2 + (col >> 2)) * 32 + rr * 4 + (col & 3)] = x[rr];
    }
    // U_kk^-1: column col by back substitution (the diagonal as 1 / U_jj)
#pragma unroll
    for (int i = 7; i >= 0; --i) {
      double sacc = i == col ? 1.0 : 0.0;
#pragma unroll
      for (int m = i + 1; m < 8; ++m) {
        const int j = d0 + m;
        const double u = j < Q ? __ldg(Ue + off_upper(j, Q) + d0 + i) : 0.0;
        sacc = fma(-u, x[m], sacc);
      }
      const double di = d0 + i < Q ? __ldg(de + d0 + i) : 1.0;
      x[i] = i > col ? 0.0 : sacc * di;
      inv[((NT + kb) * 2 + (col >> 2)) * 32 + i * 4 + (col & 3)] = x[i];
    }
  }

  FormCtx ctx{tiles, Ce, inv, Q, nc, nt, lane, r, q};
  const int ct = blockIdx.y * W + w;  // this warp's tile column of right-hand sides
  const bool active = ct < nct;
  const int c0 = 8 * ct + 2 * q;  // this lane's column pair (c0, c0 + 1)
  double X[NT][2];
  // X = P B[:, tile] as C fragments: rows 8 it + r
#pragma unroll
  for (int it = 0; it < NT; ++it) {
    const int i = 8 * it + r;
    X[it][0] = X[it][1] = 0.0;
    if (active && it < nt && i < Q) {
      const int pi = __ldg(pe + i);
      if (c0 < nc) X[it][0] = __ldg(Bte + (size_t)c0 * Q + pi);
      if (c0 + 1 < nc) X[it][1] = __ldg(Bte + (size_t)(c0 + 1) * Q + pi);
    }
  }
  form_fwd_chunks<NT, 0>(X, ctx, tiles, Le, w, W, active);                      // unit lower
  form_bwd_chunks<NT, FormCfg<NT>::NCH - 1>(X, ctx, tiles, Ue, w, W, active);   // upper
  if (!active) return;
  // ---- S^T tiles: (c' tile g, this column tile) = sum_k C(c', k) Y_k
  for (int g0 = 0; g0 < nct; g0 += kFormGroup) {
    double acc[kFormGroup][2];
#pragma unroll
    for (int g = 0; g < kFormGroup; ++g) acc[g][0] = acc[g][1] = 0.0;
    form_cy<NT>(X, acc, g0, ctx);
#pragma unroll
    for (int g = 0; g < kFormGroup; ++g) {
      const int cp = 8 * (g0 + g) + r;
      if (cp < nc) {
        if (c0 < nc) Se[(size_t)c0 * nc + cp] = acc[g][0];
        if (c0 + 1 < nc) Se[(size_t)(c0 + 1) * nc + cp] = acc[g][1];
      }
    }
  }
}

struct MbArgs {
  const int32_t* elem_ufac;
  const double* uhat;
  const double* uhalo;
  const double* St;
  double* V;
  int64_t N, F, ldS;
  int nc, t, nfe;
};

// v = S_e ue per macro, a warp per macro with plain global loads (lanes over
// output slots c', loop over input slots c).  The default apply streams S_e
// through the element kernel's TMA ring instead (element.cu, mode kMb); this
// kernel remains as its cross-check (MEHDG_MB_STREAM=0).
__global__ void __launch_bounds__(kMbWarps * 32) mb_apply_kernel(MbArgs a) {
  extern __shared__ double su_all[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * kMbWarps + w;
  if (e >= a.N) return;
  const int nc = a.nc, t = a.t;
  double* su = su_all + (size_t)w * nc;
  const int32_t* ef = a.elem_ufac + e * a.nfe;
  for (int c = lane; c < nc; c += 32) {
    const int k = c / t, s = c - k * t;
    const int f = __ldg(ef + k);
    su[c] = f < 0 ? 0.0
            : (f < a.F ? __ldg(a.uhat + (int64_t)f * t + s)
                       : __ldg(a.uhalo + (int64_t)(f - a.F) * t + s));
  }
  __syncwarp();
  const double* Se = a.St + e * a.ldS;
  // two 32-slot output groups per pass (nc <= 64 in one pass) for load-level parallelism
  for (int cp0 = 0; cp0 < nc; cp0 += 64) {
    const int cpa = cp0 + lane, cpb = cp0 + 32 + lane;
    const bool va = cpa < nc, vb = cpb < nc;
    double acca = 0.0, accb = 0.0;
#pragma unroll 8
    for (int c = 0; c < nc; ++c) {
      const double uc = su[c];
      const double* col = Se + (size_t)c * nc;
      if (va) acca = fma(__ldg(col + cpa), uc, acca);
      if (vb) accb = fma(__ldg(col + cpb), uc, accb);
    }
    if (va) a.V[e * nc + cpa] = acca;
    if (vb) a.V[e * nc + cpb] = accb;
  }
}

template <int NT>
int launch_form(mh_system* s, const FormArgs& a) {
  const int nct = (a.nc + 7) / 8;
  const int rounds = (nct + 7) / 8;
  const int W = (nct + rounds - 1) / rounds;  // warps: column tiles spread evenly over the CTAs
  const size_t smem = FormCfg<NT>::smem_bytes();
  if (launch_occupancy(s->device, reinterpret_cast<const void*>(form_dmma_kernel<NT>), 32 * W, smem) < 1) {
    set_error("element Schur: the form kernel does not fit this device");
    return MH_E_UNSUPPORTED;
  }
  form_dmma_kernel<NT><<<dim3((unsigned)s->N, (unsigned)rounds), 32 * W, smem, s->stream>>>(a);
  MH_CHECK_CUDA(cudaGetLastError());
  return MH_OK;
}

}  // namespace

int launch_element_schur(mh_system* s) {
  if (s->N == 0) return MH_OK;
  FormArgs a;
  a.Bt = s->Bt.p;
  a.Cm = s->c_is_bt ? s->Bt.p : s->Cm.p;
  a.Lp = s->Lp.p;
  a.Up = s->Up.p;
  a.dinv = s->dinv.p;
  a.perm = s->perm.p;
  a.St = s->S.p;
  a.N = s->N;
  a.ldB = s->ldB;
  a.ldL = s->ldL;
  a.ldS = s->ldS;
  a.Q = s->Q;
  a.nc = s->nc;
  const int nt = (s->Q + 7) / 8;
#define MH_FORM(N_) \
  if (nt <= N_) return launch_form<N_>(s, a);
  MH_FORM(4) MH_FORM(8) MH_FORM(12) MH_FORM(16) MH_FORM(21) MH_FORM(24) MH_FORM(28) MH_FORM(32)
#undef MH_FORM
  set_error("element Schur: Q > 256 unsupported");
  return MH_E_UNSUPPORTED;
}

int launch_element_mb(mh_system* s, const double* u) {
  if (s->N == 0) return MH_OK;
  if (s->knobs.mb_stream) return launch_element_mb_stream(s, u, s->V.p);
  MbArgs a;
  a.elem_ufac = s->elem_ufac.p;
  a.uhat = u;
  a.uhalo = s->halo_u.p;
  a.St = s->S.p;
  a.V = s->V.p;
  a.N = s->N;
  a.F = s->F;
  a.ldS = s->ldS;
  a.nc = s->nc;
  a.t = s->t;
  a.nfe = s->nfe;
  const unsigned grid = (unsigned)((s->N + kMbWarps - 1) / kMbWarps);
  const size_t smem = (size_t)kMbWarps * s->nc * sizeof(double);
  mb_apply_kernel<<<grid, kMbWarps * 32, smem, s->stream>>>(a);
  MH_CHECK_CUDA(cudaGetLastError());
  return MH_OK;
}

}  // namespace mh
