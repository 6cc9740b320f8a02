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
// form_kernel: one CTA (2 warps) per macro; each lane owns one right-hand
// side (column c of B), kept in shared memory, and runs the column-oriented
// forward / back substitution over the packed factors (L1-resident
// broadcast loads), then the C Y product.

#include "mh_internal.h"

namespace mh {
namespace {

constexpr int kFormWarps = 2;
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
  double* St;         // N x nc x nc
  int64_t N, ldB, ldL;
  int Q, nc;
};

__global__ void __launch_bounds__(kFormWarps * 32) form_kernel(FormArgs a) {
  extern __shared__ double ys_all[];  // per warp: Q x 32
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e = blockIdx.x;
  const int Q = a.Q, nc = a.nc;
  double* ys = ys_all + (size_t)w * Q * 32;
  const double* Bte = a.Bt + e * a.ldB;
  const double* Ce = a.Cm + e * a.ldB;
  const double* Le = a.Lp + e * a.ldL;
  const double* Ue = a.Up + e * a.ldL;
  const int32_t* pe = a.perm + e * Q;
  const double* de = a.dinv + e * Q;
  for (int c0 = w * 32; c0 < nc; c0 += kFormWarps * 32) {
    const int c = c0 + lane;
    const bool valid = c < nc;
    // x = P B[:, c]
    for (int i = 0; i < Q; ++i) ys[i * 32 + lane] = valid ? __ldg(Bte + (size_t)c * Q + __ldg(pe + i)) : 0.0;
    // forward: unit lower, column-oriented
    for (int k = 0; k < Q - 1; ++k) {
      const double yk = ys[k * 32 + lane];
      const double* col = Le + off_lower(k, Q) - (k + 1);
      for (int i = k + 1; i < Q; ++i) ys[i * 32 + lane] = fma(-__ldg(col + i), yk, ys[i * 32 + lane]);
    }
    // backward: upper with reciprocal diagonal
    for (int k = Q - 1; k >= 0; --k) {
      const double yk = ys[k * 32 + lane] * __ldg(de + k);
      ys[k * 32 + lane] = yk;
      const double* col = Ue + off_upper(k, Q);
      for (int i = 0; i < k; ++i) ys[i * 32 + lane] = fma(-__ldg(col + i), yk, ys[i * 32 + lane]);
    }
    // St[c][c'] = sum_i C[c'][i] y_i
    if (valid)
      for (int cp = 0; cp < nc; ++cp) {
        const double* crow = Ce + (size_t)cp * Q;
        double acc = 0.0;
        for (int i = 0; i < Q; ++i) acc = fma(__ldg(crow + i), ys[i * 32 + lane], acc);
        a.St[(e * nc + c) * (int64_t)nc + cp] = acc;
      }
    __syncwarp();
  }
}

struct MbArgs {
  const int32_t* elem_ufac;
  const double* uhat;
  const double* uhalo;
  const double* St;
  double* V;
  int64_t N, F;
  int nc, t, nfe;
};

// v = S_e ue per macro (lanes over output slots c', loop over input slots c)
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
  const double* Se = a.St + e * (int64_t)nc * nc;
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
  a.Q = s->Q;
  a.nc = s->nc;
  const size_t smem = (size_t)kFormWarps * s->Q * 32 * sizeof(double);
  if (smem > (size_t)s->max_smem_optin) {
    set_error("element Schur: Q too large for the form kernel");
    return MH_E_UNSUPPORTED;
  }
  MH_CHECK_CUDA(cudaFuncSetAttribute(form_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  form_kernel<<<(unsigned)s->N, kFormWarps * 32, smem, s->stream>>>(a);
  MH_CHECK_CUDA(cudaGetLastError());
  return MH_OK;
}

int launch_element_mb(mh_system* s, const double* u) {
  if (s->N == 0) return MH_OK;
  MbArgs a;
  a.elem_ufac = s->elem_ufac.p;
  a.uhat = u;
  a.uhalo = s->halo_u.p;
  a.St = s->S.p;
  a.V = s->V.p;
  a.N = s->N;
  a.F = s->F;
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
