// Fused per-macro element kernel: one warp per macro-element.
//
// Replaces the macro_task of apply_schur (schur_solver.py:271-277),
// macro_rhs of condense (:244-246) and the reconstruct_interior task
// (:426-429).  Per macro e, with lane l owning rows i = l + 32 r:
//   gather   ue = uhat through the face table (zeros on Dirichlet slots)
//   step 1   x  = P (B ue)        B = op.B, streamed as op.B^T rows (nc x Q)
//   step 2   y  = U^-1 L^-1 x     column-oriented substitution, warp shuffles
//   step 3   v  = C y             op.C rows, 32-row transpose-reduce
//   write    V[e*nc + c]          the macro's slot segment; the face kernel
//                                 subtracts it in left-then-right order, so
//                                 there are no atomics and results are
//                                 deterministic.
// Modes: kApply (above), kRhs (x = P R_u, writes v), kRecon
// (x = P (R_u - B ue), writes y = u_e).
// All block data is streamed exactly once per launch with
// ld.global.nc.L1::no_allocate; only op.C is read a second time (when
// op.C = op.B^T the step-3 read hits the L2 lines step 1 brought in, which
// are loaded with an evict_last policy).

#include "mh_internal.h"

namespace mh {
namespace {

constexpr int kElemWarps = 4;  // warps (macros) per CTA

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// streaming read: no L1 allocation, L2 evict-first
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(p), "l"(policy_evict_first()));
  return v;
}
// read that will be repeated by this warp shortly: keep in L2
__device__ __forceinline__ double ld_keep(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(v) : "l"(p), "l"(policy_evict_last()));
  return v;
}

struct ElemArgs {
  const int32_t* elem_ufac;
  const double* uhat;
  const double* uhalo;  // received halo segments (trace index >= F)
  const double* Bt;
  const double* Cm;
  const double* LU;
  const double* dinv;
  const int32_t* perm;
  const double* Ru;
  double* out;
  int64_t N, F;
  int Q, nc, t, nfe;
  int c_is_bt;
};

// Unit-lower forward substitution, column-oriented: at step j the lane that
// owns row j broadcasts y_j and every row i > j does y_i -= L_ij y_j.
template <int R>
__device__ __forceinline__ void forward_unit_lower(double (&y)[R], const double* __restrict__ LUe,
                                                   int Q, int lane) {
#pragma unroll
  for (int jb = 0; jb < R; ++jb) {
#pragma unroll 4
    for (int jj = 0; jj < 32; ++jj) {
      const int j = jb * 32 + jj;
      if (j < Q - 1) {
        const double yj = __shfl_sync(kFull, y[jb], jj);
        const double* col = LUe + (size_t)j * Q;
#pragma unroll
        for (int r = jb; r < R; ++r) {
          const int i = lane + 32 * r;
          if (i > j && i < Q) y[r] = fma(-ld_stream(col + i), yj, y[r]);
        }
      }
    }
  }
}

// Upper back substitution with the stored reciprocal diagonal.
template <int R>
__device__ __forceinline__ void backward_upper(double (&y)[R], const double* __restrict__ LUe,
                                               const double (&dr)[R], int Q, int lane) {
#pragma unroll
  for (int jb = R - 1; jb >= 0; --jb) {
#pragma unroll 4
    for (int jj = 31; jj >= 0; --jj) {
      const int j = jb * 32 + jj;
      if (j < Q) {
        if (lane == jj) y[jb] *= dr[jb];
        const double yj = __shfl_sync(kFull, y[jb], jj);
        const double* col = LUe + (size_t)j * Q;
#pragma unroll
        for (int r = 0; r <= jb; ++r) {
          const int i = lane + 32 * r;
          if (i < j) y[r] = fma(-ld_stream(col + i), yj, y[r]);
        }
      }
    }
  }
}

// 32 per-lane partial sums -> lane l holds the full sum of partial l
// (butterfly transpose-reduce: 31 shuffles for 32 sums).
__device__ __forceinline__ double transpose_reduce32(double (&p)[32], int lane) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const bool upper = (lane & w) != 0;
#pragma unroll
    for (int q = 0; q < w; ++q) {
      const double send = upper ? p[q] : p[q + w];
      const double keep = upper ? p[q + w] : p[q];
      p[q] = keep + __shfl_xor_sync(kFull, send, w);
    }
  }
  return p[0];
}

template <int R, int MODE>
__global__ void __launch_bounds__(kElemWarps * 32)
element_kernel(ElemArgs a) {
  extern __shared__ double s_u[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * kElemWarps + w;
  if (e >= a.N) return;  // warp-uniform; no CTA-wide barriers below
  const int Q = a.Q, nc = a.nc, t = a.t;
  const size_t QQ = (size_t)Q * Q;
  const size_t CQ = (size_t)nc * Q;

  int pr[R];
  double dr[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = lane + 32 * r;
    pr[r] = i < Q ? __ldg(a.perm + e * Q + i) : 0;
    dr[r] = i < Q ? __ldg(a.dinv + e * Q + i) : 0.0;
  }

  double y[R];
  if (MODE == kRhs) {
#pragma unroll
    for (int r = 0; r < R; ++r) y[r] = (lane + 32 * r < Q) ? __ldg(a.Ru + e * Q + pr[r]) : 0.0;
  } else {
    double* su = s_u + w * nc;
    const int32_t* ef = a.elem_ufac + e * a.nfe;
    for (int c = lane; c < nc; c += 32) {
      const int k = c / t, s = c - k * t;
      const int f = __ldg(ef + k);
      su[c] = f < 0 ? 0.0
              : (f < a.F ? __ldg(a.uhat + (int64_t)f * t + s)
                         : __ldg(a.uhalo + (int64_t)(f - a.F) * t + s));
    }
    __syncwarp();
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    const double* Bte = a.Bt + e * CQ;
#pragma unroll 4
    for (int c = 0; c < nc; ++c) {
      const double uc = su[c];
      const double* row = Bte + (size_t)c * Q;
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (lane + 32 * r < Q) {
          const double b = (MODE == kApply && a.c_is_bt) ? ld_keep(row + pr[r]) : ld_stream(row + pr[r]);
          acc[r] = fma(b, uc, acc[r]);
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (MODE == kApply) y[r] = acc[r];
      else y[r] = (lane + 32 * r < Q) ? __ldg(a.Ru + e * Q + pr[r]) - acc[r] : 0.0;
    }
  }

  const double* LUe = a.LU + e * QQ;
  forward_unit_lower<R>(y, LUe, Q, lane);
  backward_upper<R>(y, LUe, dr, Q, lane);

  if (MODE == kRecon) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = lane + 32 * r;
      if (i < Q) a.out[e * Q + i] = y[r];
    }
    return;
  }

  // step 3: v_c = sum_i C[c][i] y_i
  const double* Ce = a.Cm + e * CQ;
  for (int c0 = 0; c0 < nc; c0 += 32) {
    double pp[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      double acc = 0.0;
      const int c = c0 + q;
      if (c < nc) {
        const double* row = Ce + (size_t)c * Q;
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (lane + 32 * r < Q) acc = fma(ld_stream(row + lane + 32 * r), y[r], acc);
      }
      pp[q] = acc;
    }
    const double v = transpose_reduce32(pp, lane);
    if (c0 + lane < nc) a.out[e * nc + c0 + lane] = v;
  }
}

template <int MODE>
int launch_mode(mh_system* s, const double* uhat, double* out) {
  ElemArgs a;
  a.elem_ufac = s->elem_ufac.p;
  a.uhat = uhat;
  a.uhalo = s->halo_u.p;
  a.Bt = s->Bt.p;
  a.Cm = s->c_is_bt ? s->Bt.p : s->Cm.p;
  a.LU = s->LU.p;
  a.dinv = s->dinv.p;
  a.perm = s->perm.p;
  a.Ru = s->Ru.p;
  a.out = out;
  a.N = s->N;
  a.F = s->F;
  a.Q = s->Q;
  a.nc = s->nc;
  a.t = s->t;
  a.nfe = s->nfe;
  a.c_is_bt = s->c_is_bt ? 1 : 0;
  if (s->N == 0) return MH_OK;
  const unsigned grid = (unsigned)((s->N + kElemWarps - 1) / kElemWarps);
  const size_t smem = (size_t)kElemWarps * s->nc * sizeof(double);
  const int R = (s->Q + 31) / 32;
  switch (R) {
#define MH_ELEM_CASE(RR)                                                              \
  case RR:                                                                            \
    element_kernel<RR, MODE><<<grid, kElemWarps * 32, smem, s->stream>>>(a);          \
    break;
    MH_ELEM_CASE(1)
    MH_ELEM_CASE(2)
    MH_ELEM_CASE(3)
    MH_ELEM_CASE(4)
    MH_ELEM_CASE(5)
    MH_ELEM_CASE(6)
    MH_ELEM_CASE(7)
    MH_ELEM_CASE(8)
#undef MH_ELEM_CASE
    default:
      set_error("element kernel: Q > 256 unsupported");
      return MH_E_UNSUPPORTED;
  }
  MH_CHECK_CUDA(cudaGetLastError());
  return MH_OK;
}

}  // namespace

int launch_element(mh_system* s, int mode, const double* uhat, double* out) {
  if ((size_t)s->nc * sizeof(double) * kElemWarps > 48 * 1024) {
    set_error("element kernel: nc too large");
    return MH_E_UNSUPPORTED;
  }
  switch (mode) {
    case kApply: return launch_mode<kApply>(s, uhat, out);
    case kRhs: return launch_mode<kRhs>(s, uhat, out);
    case kRecon: return launch_mode<kRecon>(s, uhat, out);
  }
  set_error("bad element mode");
  return MH_E_ARG;
}

}  // namespace mh
