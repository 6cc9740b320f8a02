// Face kernels: one warp per unknown face.
//
//   face_factor_kernel  _factorize_face (schur_solver.py:130-147):
//                       Cholesky of -D ("chol-neg"), then of D ("chol-pos"),
//                       then LU with partial pivoting ("lu"); singular if
//                       min|diag U| < 1e-13 max|D| -> SingularFaceBlock.
//   face_reduce_kernel  step 4 of apply_schur (schur_solver.py:284-290):
//                       w_f = D_f uhat_f - v_left - v_right (that order), or
//                       the reduced RHS f_f = R_hat_f - v_left - v_right
//                       (schur_solver.py:247-253); optionally fused with
//                       the D^-1 preconditioner (the GMRES M(A v) step).
//   precond_kernel      apply_preconditioner (schur_solver.py:296-305):
//                       z_f = D_f^-1 w_f.
//
// The factor kernel turns the accepted factorisation (sign * L L^T, or
// P D = L U) into the explicit inverse D_f^-1 (t right-hand sides solved by
// the lanes of the warp), so the preconditioner is a GEMV with independent,
// coalesced loads instead of a chain of 2t dependent substitution steps.
// Face data layout: D and D^-1 column-major (t x t).

#include <algorithm>
#include <cfloat>

#include "mh_internal.h"
#include "stream.cuh"

namespace mh {
namespace {

constexpr int kFaceWarps = 4;

struct FaceArgs {
  const double* D;
  const double* Rhat;
  const int32_t* vslot;
  const double* V;
  const double* uhat;
  double* out;
  const double* Dinv;
  int64_t F;
  int64_t ldF;  // per-face stride of D / D^-1 (t^2 rounded up to 16 bytes)
  int t;
  const int* skip;  // a stopped speculative GMRES step: return at once
};

// z <- M z for the column-major t x t matrix M (rows lane + 32 r); the input
// vector is staged in the warp's shared buffer sw
template <int RT>
__device__ __forceinline__ void warp_gemv(double (&z)[RT], const double* __restrict__ M, int t,
                                          double* sw, int lane) {
#pragma unroll
  for (int r = 0; r < RT; ++r)
    if (lane + 32 * r < t) sw[lane + 32 * r] = z[r];
  __syncwarp();
#pragma unroll
  for (int r = 0; r < RT; ++r) z[r] = 0.0;
#pragma unroll 8
  for (int s = 0; s < t; ++s) {  // sum over s ascending
    const double ws = sw[s];
#pragma unroll
    for (int r = 0; r < RT; ++r) {
      const int i = lane + 32 * r;
      if (i < t) z[r] = fma(__ldg(M + (size_t)s * t + i), ws, z[r]);
    }
  }
  __syncwarp();
}

template <int RT, bool RHS, bool PRE>
__global__ void __launch_bounds__(kFaceWarps * 32) face_reduce_kernel(FaceArgs a) {
  if (a.skip && *a.skip) return;
  extern __shared__ double s_buf[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t f = (int64_t)blockIdx.x * kFaceWarps + w;
  if (f >= a.F) return;
  const int t = a.t;
  double* sw = s_buf + w * t;
  double z[RT];
#pragma unroll
  for (int r = 0; r < RT; ++r) {
    const int i = lane + 32 * r;
    z[r] = i < t ? __ldg((RHS ? a.Rhat : a.uhat) + f * t + i) : 0.0;
  }
  const int sl = __ldg(a.vslot + 2 * f), sr = __ldg(a.vslot + 2 * f + 1);
  if (PRE && !RHS) {
    // M(A u)_f = D_f^-1 (D_f u_f - v_L - v_R) = u_f - D_f^-1 (v_L + v_R): the
    // same operator reading only D_f^-1 (one t x t block per face, not two)
    double q[RT];
#pragma unroll
    for (int r = 0; r < RT; ++r) {
      const int i = lane + 32 * r;
      q[r] = 0.0;
      if (i < t) {
        if (sl >= 0) q[r] = __ldg(a.V + (int64_t)sl * t + i);
        if (sr >= 0) q[r] += __ldg(a.V + (int64_t)sr * t + i);
      }
    }
    warp_gemv<RT>(q, a.Dinv + f * a.ldF, t, sw, lane);
#pragma unroll
    for (int r = 0; r < RT; ++r) {
      const int i = lane + 32 * r;
      if (i < t) a.out[f * t + i] = z[r] - q[r];
    }
    return;
  }
  if (!RHS) warp_gemv<RT>(z, a.D + f * a.ldF, t, sw, lane);  // D_f uhat_f
#pragma unroll
  for (int r = 0; r < RT; ++r) {
    const int i = lane + 32 * r;
    if (i < t) {
      if (sl >= 0) z[r] -= __ldg(a.V + (int64_t)sl * t + i);  // left first
      if (sr >= 0) z[r] -= __ldg(a.V + (int64_t)sr * t + i);  // then right
    }
  }
  if (PRE) warp_gemv<RT>(z, a.Dinv + f * a.ldF, t, sw, lane);
#pragma unroll
  for (int r = 0; r < RT; ++r) {
    const int i = lane + 32 * r;
    if (i < t) a.out[f * t + i] = z[r];
  }
}

// Faces with t > 32 (c4 t = 55, c5 t = 45), the apply and the fused M(A u):
// each warp owns one face at a time and pulls its t x t block (16-24 KB,
// contiguous, 16-byte aligned with the padded face stride) into shared memory
// with one cp.async.bulk (TMA) while it loads the face's vectors; the GEMV then
// reads the block from shared memory in the same order (columns ascending) as
// warp_gemv, so the results are bitwise those of face_reduce_kernel.  A CTA
// holds as many warps (blocks in flight) as ~200 KB of shared memory allows.
template <int RT, bool PRE>
__global__ void __launch_bounds__(8 * 32) face_bulk_kernel(FaceArgs a) {
  if (a.skip && *a.skip) return;
  extern __shared__ __align__(128) double s_bulk[];
  __shared__ uint64_t mbar[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int t = a.t;
  const int64_t ldF = a.ldF;
  double* buf = s_bulk + (size_t)w * (ldF + 128);
  double* sw = buf + ldF;
  const uint32_t bytes = (uint32_t)(ldF * sizeof(double));
  const double* Mbase = PRE ? a.Dinv : a.D;
  if (lane == 0) {
    mbar_init(&mbar[w], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const uint64_t pol = l2_policy_evict_first();
  uint32_t phase = 0;
  for (int64_t f = (int64_t)blockIdx.x * nw + w; f < a.F; f += (int64_t)gridDim.x * nw) {
    if (lane == 0) {
      fence_proxy_async_smem();  // the previous face's reads before the copy's writes
      mbar_expect_tx(&mbar[w], bytes);
      bulk_g2s(buf, Mbase + f * ldF, bytes, &mbar[w], pol);
    }
    double z[RT], q[RT];
    const int sl = __ldg(a.vslot + 2 * f), sr = __ldg(a.vslot + 2 * f + 1);
#pragma unroll
    for (int r = 0; r < RT; ++r) {
      const int i = lane + 32 * r;
      z[r] = i < t ? __ldg(a.uhat + f * t + i) : 0.0;
      q[r] = 0.0;
      if (PRE && i < t) {  // q = v_L + v_R (left first)
        if (sl >= 0) q[r] = __ldg(a.V + (int64_t)sl * t + i);
        if (sr >= 0) q[r] += __ldg(a.V + (int64_t)sr * t + i);
      }
    }
    // the GEMV input: D^-1 applies to q (fused preconditioner), D to uhat_f
#pragma unroll
    for (int r = 0; r < RT; ++r) {
      const int i = lane + 32 * r;
      if (i < t) sw[i] = PRE ? q[r] : z[r];
    }
    __syncwarp();
    while (!mbar_try_wait(&mbar[w], phase)) {
    }
    phase ^= 1;
    double y[RT];
#pragma unroll
    for (int r = 0; r < RT; ++r) y[r] = 0.0;
#pragma unroll 8
    for (int s2 = 0; s2 < t; ++s2) {  // sum over columns ascending, as warp_gemv
      const double ws = sw[s2];
#pragma unroll
      for (int r = 0; r < RT; ++r) {
        const int i = lane + 32 * r;
        if (i < t) y[r] = fma(buf[(size_t)s2 * t + i], ws, y[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < RT; ++r) {
      const int i = lane + 32 * r;
      if (i < t) {
        double o;
        if (PRE) {
          o = z[r] - y[r];  // u_f - D_f^-1 (v_L + v_R)
        } else {
          o = y[r];
          if (sl >= 0) o -= __ldg(a.V + (int64_t)sl * t + i);  // left first
          if (sr >= 0) o -= __ldg(a.V + (int64_t)sr * t + i);  // then right
        }
        a.out[f * t + i] = o;
      }
    }
    __syncwarp();
  }
}

// Small faces (t <= G): a group of G lanes (G = 16: two faces per warp) per
// face, lane g owning row g; every column load of the GEMVs is issued up
// front (static unroll over TMAX = G columns) for memory-level parallelism.
template <int G, bool RHS, bool PRE>
__global__ void __launch_bounds__(kFaceWarps * 32) face_small_kernel(FaceArgs a) {
  if (a.skip && *a.skip) return;
  __shared__ double s_u[kFaceWarps * 32];
  constexpr int FPB = kFaceWarps * 32 / G;  // faces per CTA
  const int tid = threadIdx.x, g = tid % G, grp = tid / G;
  const int64_t f = (int64_t)blockIdx.x * FPB + grp;
  const bool valid_face = f < a.F;
  const int t = a.t;
  const bool row = valid_face && g < t;
  double* su = s_u + grp * G;
  double z = row ? __ldg((RHS ? a.Rhat : a.uhat) + f * t + g) : 0.0;
  const unsigned mask = G == 32 ? kFull : (0xffffu << (tid & 16));
  if (PRE && !RHS) {  // u_f - D_f^-1 (v_L + v_R), see face_reduce_kernel
    double q = 0.0;
    if (row) {
      const int sl = __ldg(a.vslot + 2 * f), sr = __ldg(a.vslot + 2 * f + 1);
      if (sl >= 0) q = __ldg(a.V + (int64_t)sl * t + g);
      if (sr >= 0) q += __ldg(a.V + (int64_t)sr * t + g);
    }
    su[g] = q;
    __syncwarp(mask);
    const double* Mi = a.Dinv + (valid_face ? f : 0) * a.ldF;
    double acc = 0.0;
#pragma unroll
    for (int s = 0; s < G; ++s)
      if (s < t && row) acc = fma(__ldg(Mi + (size_t)s * t + g), su[s], acc);
    if (row) a.out[f * t + g] = z - acc;
    return;
  }
  if (!RHS) {
    su[g] = z;
    __syncwarp(mask);
    const double* Df = a.D + (valid_face ? f : 0) * a.ldF;
    double acc = 0.0;
#pragma unroll
    for (int s = 0; s < G; ++s)
      if (s < t && row) acc = fma(__ldg(Df + (size_t)s * t + g), su[s], acc);
    z = acc;
    __syncwarp(mask);
  }
  if (row) {
    const int sl = __ldg(a.vslot + 2 * f), sr = __ldg(a.vslot + 2 * f + 1);
    if (sl >= 0) z -= __ldg(a.V + (int64_t)sl * t + g);  // left first
    if (sr >= 0) z -= __ldg(a.V + (int64_t)sr * t + g);  // then right
  }
  if (PRE) {
    su[g] = z;
    __syncwarp(mask);
    const double* Mi = a.Dinv + (valid_face ? f : 0) * a.ldF;
    double acc = 0.0;
#pragma unroll
    for (int s = 0; s < G; ++s)
      if (s < t && row) acc = fma(__ldg(Mi + (size_t)s * t + g), su[s], acc);
    z = acc;
  }
  if (row) a.out[f * t + g] = z;
}

template <int RT>
__global__ void __launch_bounds__(kFaceWarps * 32) precond_kernel(FaceArgs a) {
  if (a.skip && *a.skip) return;
  extern __shared__ double s_buf[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t f = (int64_t)blockIdx.x * kFaceWarps + w;
  if (f >= a.F) return;
  const int t = a.t;
  double z[RT];
#pragma unroll
  for (int r = 0; r < RT; ++r) {
    const int i = lane + 32 * r;
    z[r] = i < t ? __ldg(a.uhat + f * t + i) : 0.0;
  }
  warp_gemv<RT>(z, a.Dinv + f * a.ldF, t, s_buf + w * t, lane);
#pragma unroll
  for (int r = 0; r < RT; ++r) {
    const int i = lane + 32 * r;
    if (i < t) a.out[f * t + i] = z[r];
  }
}

// ---- factorisation -------------------------------------------------------

// Cholesky of the column-major t x t matrix S in place (lower). Returns false
// on a non-positive (or NaN) pivot, like LAPACK potrf.
__device__ bool warp_cholesky(double* S, int t, int lane) {
  for (int j = 0; j < t; ++j) {
    double* cj = S + (size_t)j * t;
    const double d = cj[j];
    if (!(d > 0.0)) return false;
    const double ljj = sqrt(d);
    const double r = 1.0 / ljj;
    __syncwarp();
    for (int i = j + 1 + lane; i < t; i += 32) cj[i] *= r;
    if (lane == 0) cj[j] = ljj;
    __syncwarp();
    for (int k = j + 1; k < t; ++k) {
      double* ck = S + (size_t)k * t;
      const double lkj = cj[k];
      for (int i = k + lane; i < t; i += 32) ck[i] = fma(-cj[i], lkj, ck[i]);
    }
    __syncwarp();
  }
  return true;
}

// LU with partial pivoting of the column-major t x t matrix S (dgetf2 rules).
__device__ void warp_lu(double* S, int t, int lane, int* perm) {
  for (int i = lane; i < t; i += 32) perm[i] = i;
  __syncwarp();
  for (int k = 0; k < t; ++k) {
    double* ck = S + (size_t)k * t;
    double best = -1.0;
    int bi = k;
    for (int i = k + lane; i < t; i += 32) {
      const double v = fabs(ck[i]);
      if (v > best) { best = v; bi = i; }
    }
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(kFull, best, o);
      const int oi = __shfl_xor_sync(kFull, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    const int p = bi;
    const double pv = ck[p];
    __syncwarp();
    if (lane == 0) {
      const int tmp = perm[k];
      perm[k] = perm[p];
      perm[p] = tmp;
    }
    if (pv != 0.0) {
      if (p != k)
        for (int j = lane; j < t; j += 32) {
          double* c = S + (size_t)j * t;
          const double x = c[k];
          c[k] = c[p];
          c[p] = x;
        }
      __syncwarp();
      if (fabs(pv) >= DBL_MIN) {
        const double r = 1.0 / pv;
        for (int i = k + 1 + lane; i < t; i += 32) ck[i] *= r;
      } else {
        for (int i = k + 1 + lane; i < t; i += 32) ck[i] /= pv;
      }
    }
    __syncwarp();
    for (int j = k + 1; j < t; ++j) {
      double* c = S + (size_t)j * t;
      const double akj = c[k];
      for (int i = k + 1 + lane; i < t; i += 32) c[i] = fma(-ck[i], akj, c[i]);
    }
    __syncwarp();
  }
}

// Column j of D^-1 for each lane j (< t, in chunks of 32): solve with the
// factor in S.  chol: sign * (L L^T)^-1 e_j;  lu: U^-1 L^-1 P e_j.
__device__ void warp_inverse(const double* S, const int* pm, int t, bool chol, double sign,
                             double* scratch, double* out, int lane) {
  for (int j0 = 0; j0 < t; j0 += 32) {
    const int j = j0 + lane;
    const bool act = j < t;
    double* x = scratch + lane;  // x[i * 32]: this lane's column
    if (act) {
      for (int i = 0; i < t; ++i) x[i * 32] = chol ? (i == j ? 1.0 : 0.0) : (pm[i] == j ? 1.0 : 0.0);
      // forward: L y = b (L lower; unit diagonal for LU)
      for (int k = 0; k < t; ++k) {
        double yk = x[k * 32];
        if (chol) {
          yk /= S[(size_t)k * t + k];
          x[k * 32] = yk;
        }
        for (int i = k + 1; i < t; ++i) x[i * 32] = fma(-S[(size_t)k * t + i], yk, x[i * 32]);
      }
      // backward: L^T x = y (chol) or U x = y (lu), column-oriented
      for (int k = t - 1; k >= 0; --k) {
        const double xk = x[k * 32] / S[(size_t)k * t + k];
        x[k * 32] = xk;
        for (int i = 0; i < k; ++i) {
          const double uik = chol ? S[(size_t)i * t + k] : S[(size_t)k * t + i];
          x[i * 32] = fma(-uik, xk, x[i * 32]);
        }
      }
      for (int i = 0; i < t; ++i) out[(size_t)j * t + i] = sign * x[i * 32];
    }
    __syncwarp();
  }
}

__global__ void face_factor_kernel(const double* __restrict__ Drm, double* __restrict__ Dcm,
                                   double* __restrict__ Dinv, int8_t* __restrict__ Fkind,
                                   int64_t F, int t, int wpb, int64_t ldF) {
  extern __shared__ double s_fac[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t f = (int64_t)blockIdx.x * wpb + w;
  if (f >= F) return;
  const size_t TT = (size_t)t * t;
  double* S = s_fac + (size_t)w * (TT + 64 + 32 * (size_t)t);
  int* pm = reinterpret_cast<int*>(S + TT);
  double* scratch = S + TT + 64;
  const double* Df = Drm + f * TT;
  double dmax = 0.0;
  for (size_t idx = lane; idx < TT; idx += 32) {  // row-major in -> column-major copy
    const int i = (int)(idx / t), j = (int)(idx - (size_t)i * t);
    const double v = __ldg(Df + idx);
    Dcm[f * ldF + (size_t)j * t + i] = v;
    dmax = fmax(dmax, fabs(v));
  }
  for (int o = 16; o; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(kFull, dmax, o));

  int kind = MH_FACE_SINGULAR;
  double sign = 1.0;
  for (int attempt = 0; attempt < 2 && kind == MH_FACE_SINGULAR; ++attempt) {
    sign = attempt == 0 ? -1.0 : 1.0;
    for (size_t idx = lane; idx < TT; idx += 32) {
      const int i = (int)(idx / t), j = (int)(idx - (size_t)i * t);
      S[(size_t)j * t + i] = sign * __ldg(Df + idx);
    }
    __syncwarp();
    if (warp_cholesky(S, t, lane)) kind = attempt == 0 ? MH_FACE_CHOL_NEG : MH_FACE_CHOL_POS;
    __syncwarp();
  }
  if (kind == MH_FACE_SINGULAR) {
    sign = 1.0;
    for (size_t idx = lane; idx < TT; idx += 32) {
      const int i = (int)(idx / t), j = (int)(idx - (size_t)i * t);
      S[(size_t)j * t + i] = __ldg(Df + idx);
    }
    __syncwarp();
    warp_lu(S, t, lane, pm);
    double dmin = DBL_MAX;
    for (int i = lane; i < t; i += 32) dmin = fmin(dmin, fabs(S[(size_t)i * t + i]));
    for (int o = 16; o; o >>= 1) dmin = fmin(dmin, __shfl_xor_sync(kFull, dmin, o));
    kind = (dmin < 1e-13 * fmax(dmax, 1e-300)) ? MH_FACE_SINGULAR : MH_FACE_LU;
  }
  __syncwarp();
  if (kind != MH_FACE_SINGULAR)
    warp_inverse(S, pm, t, kind != MH_FACE_LU, sign, scratch, Dinv + f * ldF, lane);
  if (lane == 0) Fkind[f] = (int8_t)kind;
}

__global__ void transpose_batched_kernel(const double* __restrict__ in, double* __restrict__ out,
                                         int rows, int cols, int64_t ostride) {
  // in: batch x rows x cols (row-major) -> out: batch x cols x rows
  __shared__ double tile[32][33];
  const int64_t b = blockIdx.z;
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  const double* ib = in + b * (size_t)rows * cols;
  double* ob = out + b * ostride;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int r = r0 + k, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[k][threadIdx.x] = ib[(size_t)r * cols + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int c = c0 + k, r = r0 + threadIdx.x;
    if (r < rows && c < cols) ob[(size_t)c * rows + r] = tile[threadIdx.x][k];
  }
}

FaceArgs make_args(mh_system* s, const double* in, double* out) {
  FaceArgs a;
  a.D = s->D.p;
  a.Rhat = s->Rhat.p;
  a.vslot = s->face_vslot.p;
  a.V = s->V.p;
  a.uhat = in;
  a.out = out;
  a.Dinv = s->Dinv.p;
  a.ldF = s->ldF;
  a.skip = s->skip;
  a.F = s->F;
  a.t = s->t;
  return a;
}

}  // namespace

int launch_transpose_batched(cudaStream_t st, const double* in, double* out, int64_t batch,
                             int rows, int cols, int64_t ostride) {
  if (batch == 0) return MH_OK;
  if (ostride < 0) ostride = (int64_t)rows * cols;
  dim3 grid((cols + 31) / 32, (rows + 31) / 32, 1);
  dim3 block(32, 8);
  for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
    const int64_t nb = batch - b0 < 65535 ? batch - b0 : 65535;
    grid.z = (unsigned)nb;
    transpose_batched_kernel<<<grid, block, 0, st>>>(in + b0 * (size_t)rows * cols,
                                                     out + b0 * ostride, rows, cols, ostride);
    MH_CHECK_CUDA(cudaGetLastError());
  }
  return MH_OK;
}

int launch_face_factor(mh_system* s, const double* Drm) {
  if (s->F == 0) return MH_OK;
  const int t = s->t;
  const size_t per = ((size_t)t * t + 64 + 32 * (size_t)t) * sizeof(double);
  int wpb = (int)((48 * 1024) / per);
  if (wpb < 1) wpb = 1;
  if (wpb > 8) wpb = 8;
  size_t smem = per * wpb;
  if (smem > 48 * 1024) {
    if (smem > (size_t)s->max_smem_optin) {
      set_error("face block too large for the face factor kernel");
      return MH_E_UNSUPPORTED;
    }
    MH_CHECK_CUDA(cudaFuncSetAttribute(face_factor_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  const unsigned grid = (unsigned)((s->F + wpb - 1) / wpb);
  face_factor_kernel<<<grid, wpb * 32, smem, s->stream>>>(Drm, s->D.p, s->Dinv.p, s->Fkind.p,
                                                          s->F, t, wpb, s->ldF);
  MH_CHECK_CUDA(cudaGetLastError());
  return MH_OK;
}

template <int G>
int launch_small(mh_system* s, const FaceArgs& a, int rhs_mode, int pre) {
  constexpr int FPB = kFaceWarps * 32 / G;
  const unsigned grid = (unsigned)((s->F + FPB - 1) / FPB);
  if (rhs_mode) {
    if (pre) face_small_kernel<G, true, true><<<grid, kFaceWarps * 32, 0, s->stream>>>(a);
    else face_small_kernel<G, true, false><<<grid, kFaceWarps * 32, 0, s->stream>>>(a);
  } else {
    if (pre) face_small_kernel<G, false, true><<<grid, kFaceWarps * 32, 0, s->stream>>>(a);
    else face_small_kernel<G, false, false><<<grid, kFaceWarps * 32, 0, s->stream>>>(a);
  }
  MH_CHECK_CUDA(cudaGetLastError());
  return MH_OK;
}

int launch_face_reduce(mh_system* s, const double* uhat, double* w, int rhs_mode, int pre) {
  if (s->F == 0) return MH_OK;
  FaceArgs a = make_args(s, uhat, w);
  if (s->t <= 16) return launch_small<16>(s, a, rhs_mode, pre);
  if (s->t <= 32) return launch_small<32>(s, a, rhs_mode, pre);
  if (!rhs_mode && s->knobs.face_bulk) {
    const size_t per = (size_t)(s->ldF + 128) * sizeof(double);
    const int nw = (int)std::max<size_t>(1, std::min<size_t>(8, (size_t)(200 * 1024) / per));
    const size_t smem = per * nw;
    const int RTb = (s->t + 31) / 32;
    const void* fn = nullptr;
    if (RTb == 2) fn = pre ? (const void*)face_bulk_kernel<2, true> : (const void*)face_bulk_kernel<2, false>;
    else if (RTb == 3) fn = pre ? (const void*)face_bulk_kernel<3, true> : (const void*)face_bulk_kernel<3, false>;
    else if (RTb == 4) fn = pre ? (const void*)face_bulk_kernel<4, true> : (const void*)face_bulk_kernel<4, false>;
    if (fn) {
      const int per_sm = launch_occupancy(s->device, fn, nw * 32, smem);
      if (per_sm < 0) return MH_E_CUDA;
      const int64_t need = (s->F + nw - 1) / nw;
      const unsigned grid = (unsigned)std::min<int64_t>(need, (int64_t)std::max(1, per_sm) * s->num_sms);
      void* args[] = {(void*)&a};
      MH_CHECK_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(nw * 32), args, smem, s->stream));
      return MH_OK;
    }
  }
  const unsigned grid = (unsigned)((s->F + kFaceWarps - 1) / kFaceWarps);
  const size_t smem = (size_t)kFaceWarps * s->t * sizeof(double);
  const int RT = (s->t + 31) / 32;
#define MH_FACE_LAUNCH(RR, RHS, PRE) \
  face_reduce_kernel<RR, RHS, PRE><<<grid, kFaceWarps * 32, smem, s->stream>>>(a)
#define MH_FACE_SWITCH(RR)                                   \
  if (RT == RR) {                                            \
    if (rhs_mode) {                                          \
      if (pre) MH_FACE_LAUNCH(RR, true, true);               \
      else MH_FACE_LAUNCH(RR, true, false);                  \
    } else {                                                 \
      if (pre) MH_FACE_LAUNCH(RR, false, true);              \
      else MH_FACE_LAUNCH(RR, false, false);                 \
    }                                                        \
  }
  MH_FACE_SWITCH(1) else MH_FACE_SWITCH(2) else MH_FACE_SWITCH(3) else MH_FACE_SWITCH(4) else {
    set_error("face kernels: t > 128 unsupported");
    return MH_E_UNSUPPORTED;
  }
#undef MH_FACE_SWITCH
#undef MH_FACE_LAUNCH
  MH_CHECK_CUDA(cudaGetLastError());
  return MH_OK;
}

int launch_precond(mh_system* s, const double* w, double* z) {
  if (s->F == 0) return MH_OK;
  FaceArgs a = make_args(s, w, z);
  const unsigned grid = (unsigned)((s->F + kFaceWarps - 1) / kFaceWarps);
  const size_t smem = (size_t)kFaceWarps * s->t * sizeof(double);
  const int RT = (s->t + 31) / 32;
  switch (RT) {
    case 1: precond_kernel<1><<<grid, kFaceWarps * 32, smem, s->stream>>>(a); break;
    case 2: precond_kernel<2><<<grid, kFaceWarps * 32, smem, s->stream>>>(a); break;
    case 3: precond_kernel<3><<<grid, kFaceWarps * 32, smem, s->stream>>>(a); break;
    case 4: precond_kernel<4><<<grid, kFaceWarps * 32, smem, s->stream>>>(a); break;
    default:
      set_error("face kernels: t > 128 unsupported");
      return MH_E_UNSUPPORTED;
  }
  MH_CHECK_CUDA(cudaGetLastError());
  return MH_OK;
}

}  // namespace mh
