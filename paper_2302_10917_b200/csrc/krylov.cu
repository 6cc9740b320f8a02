// Device GMRES: restarted, left-preconditioned, modified Gram-Schmidt with
// Givens rotations -- the control flow of the reference gmres
// (schur_solver.py:308-385) with all vector work on the device.
//
// Vector kernels use a fixed 512-chunk partition and a fixed-order final
// sum (last-block-done ticket), so every dot product is deterministic and
// independent of the GPU model.  One MGS step is one kernel:
//     w -= H[i-1,k] V[i-1]   (coefficient read from device memory)
//     H[i,k] = V[i] . w
// so an Arnoldi step costs k+2 small launches and ONE device->host copy of
// the new Hessenberg column; the Givens rotations, the residual estimate
// and the cycle-end triangular solve run on the host in double, exactly
// as the reference does them in numpy.

#include <cmath>
#include <cstdlib>
#include <vector>

#include "mh_internal.h"

namespace mh {

struct Krylov {
  int64_t n = 0;
  int restart = 0;
  DBuf<double> V, w, tmp, tmp2, part, hcol, ydev, scal;
  DBuf<unsigned> ticket;
  double* h_host = nullptr;  // pinned
  bool persistent = false;   // a system's workspace, reused across solves
  // CUDA graphs of the Arnoldi step's MGS block, one per basis size k (captured
  // on first use, replayed afterwards; they bake in the buffer addresses above)
  std::vector<cudaGraphExec_t> mgs;
  cudaStream_t gs = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  void drop_graphs() {
    for (cudaGraphExec_t& g : mgs)
      if (g) cudaGraphExecDestroy(g);
    mgs.clear();
  }
  int alloc(int64_t n_, int restart_) {
    if (n_ == n && restart_ == restart && V.p) return MH_OK;
    drop_graphs();
    n = n_;
    restart = restart_;
    MH_CHECK(V.alloc((size_t)(restart + 1) * (size_t)n));
    MH_CHECK(w.alloc((size_t)n));
    MH_CHECK(tmp.alloc((size_t)n));
    MH_CHECK(tmp2.alloc((size_t)n));
    MH_CHECK(part.alloc(kDotBlocks));
    MH_CHECK(hcol.alloc((size_t)restart + 2));
    MH_CHECK(ydev.alloc((size_t)restart + 1));
    MH_CHECK(scal.alloc(4));
    MH_CHECK(ticket.alloc(1));
    MH_CHECK_CUDA(cudaMemset(ticket.p, 0, sizeof(unsigned)));
    if (h_host) cudaFreeHost(h_host);
    MH_CHECK_CUDA(cudaMallocHost(&h_host, sizeof(double) * (restart + 4)));
    return MH_OK;
  }
  ~Krylov() {
    drop_graphs();
    if (gs) cudaStreamDestroy(gs);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_out) cudaEventDestroy(ev_out);
    V.release(); w.release(); tmp.release(); tmp2.release(); part.release();
    hcol.release(); ydev.release(); scal.release(); ticket.release();
    if (h_host) cudaFreeHost(h_host);
  }
};

void free_krylov(Krylov* k) { delete k; }

namespace {

__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kDotThreads / 32; ++i) r += red[i];
  return r;  // valid on thread 0
}

// Fused MGS step.  mode 0: plain dot(x, y); mode 1: w -= c*Vp then dot(Vi, w);
// mode 2: w -= c*Vp then dot(w, w) and out <- sqrt.  Result to *out (device).
__global__ void __launch_bounds__(kDotThreads)
dot_kernel(int64_t n, double* __restrict__ w, const double* __restrict__ Vp,
           const double* __restrict__ coef, const double* __restrict__ Vi, int mode,
           bool take_sqrt, double* __restrict__ part, unsigned* __restrict__ ticket,
           double* __restrict__ out) {
  __shared__ double red[kDotThreads / 32];
  __shared__ bool last;
  const int64_t b = blockIdx.x;
  const int64_t lo = n * b / kDotBlocks, hi = n * (b + 1) / kDotBlocks;
  const double c = (mode != 0 && coef) ? *coef : 0.0;
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += kDotThreads) {
    double wi = w[i];
    if (mode != 0 && coef) {
      wi = __dsub_rn(wi, __dmul_rn(c, Vp[i]));  // numpy: wv -= H*V (two roundings)
      w[i] = wi;
    }
    const double yi = (mode == 2) ? wi : Vi[i];
    acc = fma(wi, yi, acc);
  }
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) {
    part[b] = s;
    __threadfence();
    const unsigned tk = atomicAdd(ticket, 1u);
    last = (tk == kDotBlocks - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // fixed-order final reduction of the 512 partials
  double v = 0.0;
  for (int i = threadIdx.x; i < kDotBlocks; i += kDotThreads) v += ((volatile double*)part)[i];
  const double tot = block_sum(v, red);
  if (threadIdx.x == 0) {
    *out = (mode == 2 && take_sqrt) ? sqrt(tot) : tot;
    *ticket = 0u;
  }
}

// The whole MGS block of Arnoldi step k in ONE CTA for short vectors (n <=
// kSmallMgsN): the k + 2 dependent reductions are block reductions instead of
// k + 2 grid launches (launch latency bounds them at this size).  Same
// arithmetic per element as dot_kernel (w -= h V in two roundings, fma dots);
// each thread owns the same indices in every pass, so the in-place updates
// need no synchronisation beyond the reductions.
constexpr int kSmallMgsThreads = 1024;
constexpr int64_t kSmallMgsN = 1 << 16;

__device__ __forceinline__ double block_sum_bcast(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double r = lane < kSmallMgsThreads / 32 ? red[lane] : 0.0;
    for (int o = 16; o; o >>= 1) r += __shfl_xor_sync(kFull, r, o);
    if (lane == 0) red[32] = r;
  }
  __syncthreads();
  const double r = red[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kSmallMgsThreads)
mgs_small_kernel(int64_t n, double* __restrict__ w, const double* __restrict__ V, int k,
                 double* __restrict__ hcol, double* __restrict__ vnext) {
  __shared__ double red[33];
  double c = 0.0;
  const double* Vp = nullptr;
  for (int i = 0; i <= k + 1; ++i) {
    const double* Vi = V + (size_t)i * n;  // i = k + 1: the norm of w
    double acc = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += kSmallMgsThreads) {
      double wj = w[j];
      if (i > 0) {
        wj = __dsub_rn(wj, __dmul_rn(c, Vp[j]));
        w[j] = wj;
      }
      acc = fma(wj, i <= k ? Vi[j] : wj, acc);
    }
    double h = block_sum_bcast(acc, red);
    if (i == k + 1) h = sqrt(h);
    if (threadIdx.x == 0) hcol[i] = h;
    c = h;
    Vp = Vi;
  }
  if (!(c > 1e-300)) return;
  for (int64_t j = threadIdx.x; j < n; j += kSmallMgsThreads) vnext[j] = w[j] / c;
}

// V[k+1] = w / h if h > 1e-300 (else left zero: breakdown)
__global__ void normalize_kernel(int64_t n, const double* __restrict__ w,
                                 const double* __restrict__ h, double* __restrict__ out) {
  const double hv = *h;
  if (!(hv > 1e-300)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = w[i] / hv;
}

__global__ void scale_kernel(int64_t n, const double* __restrict__ x, double inv_div,
                             double* __restrict__ out) {
  // out = x / beta (division kept, like numpy r / beta)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[i] / inv_div;
}

__global__ void sub_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i] - b[i];
}

// x += V[:k]^T y
__global__ void update_x_kernel(int64_t n, int k, const double* __restrict__ V,
                                const double* __restrict__ y, double* __restrict__ x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < k; ++j) acc = fma(V[(size_t)j * n + i], y[j], acc);
    x[i] = x[i] + acc;
  }
}

constexpr int kVecGrid = 1184;  // 8 x 148
constexpr int kVecThreads = 256;

struct OpFn {
  int (*fn)(void*, const double*, double*) = nullptr;
  void* ctx = nullptr;
  int operator()(const double* in, double* out) const {
    int s = fn(ctx, in, out);
    if (s != MH_OK && s != MH_E_CUDA && s != MH_E_UNSUPPORTED && s != MH_E_STATE) {
      set_error("operator callback failed");
      return MH_E_CALLBACK;
    }
    return s;
  }
};

// Dot product (and fused MGS update).  With a multi-GPU system the local
// sum is all-gathered and added in rank order, identically on every rank.
thread_local mh_system* g_comm_sys = nullptr;  // bound for the duration of one solve

int dot_dev(cudaStream_t st, Krylov* K, int64_t n, double* w, const double* Vp,
            const double* coef, const double* Vi, int mode, double* out) {
  const bool multi = g_comm_sys && (g_comm_sys->nranks > 1 || g_comm_sys->nccl);
  dot_kernel<<<kDotBlocks, kDotThreads, 0, st>>>(n, w, Vp, coef, Vi, mode, !multi, K->part.p,
                                                  K->ticket.p, multi ? K->scal.p + 3 : out);
  MH_CHECK_CUDA(cudaGetLastError());
  if (multi) MH_CHECK(allreduce_scalar(g_comm_sys, K->scal.p + 3, out, mode == 2));
  return MH_OK;
}

int read_scalars(cudaStream_t st, Krylov* K, const double* dev, int count) {
  MH_CHECK_CUDA(cudaMemcpyAsync(K->h_host, dev, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
  MH_CHECK_CUDA(cudaStreamSynchronize(st));
  return MH_OK;
}

// z = M(A v): fused op if given, else apply then precond.
int apply_MA(const OpFn& A, const OpFn& M, const OpFn& MA, const double* v, double* z,
             double* scratch) {
  if (MA.fn) return MA(v, z);
  if (!M.fn) return A(v, z);
  MH_CHECK(A(v, scratch));
  return M(scratch, z);
}

int gmres_core(cudaStream_t st, Krylov* K, int64_t n, const OpFn& A, const OpFn& M,
               const OpFn& MA, double tol, int restart, int maxiter, const double* rhs,
               double* x, int* iterations, int* converged, double* hist_host, int hist_cap,
               int* hist_len);

// The MGS block of Arnoldi step k: H[0..k, k] and H[k+1, k] = ||w||, V[k+1] = w / H[k+1, k],
// and the new Hessenberg column copied to the pinned host buffer.
int enqueue_mgs(cudaStream_t st, Krylov* K, int64_t n, int k) {
  double* V = K->V.p;
  const bool multi = g_comm_sys && (g_comm_sys->nranks > 1 || g_comm_sys->nccl);
  const char* sv = getenv("MEHDG_MGS_SMALL");
  if (!multi && n <= kSmallMgsN && !(sv && sv[0] == '0')) {
    mgs_small_kernel<<<1, kSmallMgsThreads, 0, st>>>(n, K->w.p, V, k, K->hcol.p,
                                                     V + (size_t)(k + 1) * n);
    MH_CHECK_CUDA(cudaGetLastError());
    MH_CHECK_CUDA(cudaMemcpyAsync(K->h_host, K->hcol.p, sizeof(double) * (k + 2),
                                  cudaMemcpyDeviceToHost, st));
    return MH_OK;
  }
  for (int i = 0; i <= k; ++i) {
    const double* Vi = V + (size_t)i * n;
    const double* Vp = i > 0 ? V + (size_t)(i - 1) * n : nullptr;
    const double* coef = i > 0 ? K->hcol.p + (i - 1) : nullptr;
    MH_CHECK(dot_dev(st, K, n, K->w.p, Vp, coef, Vi, 1, K->hcol.p + i));
  }
  MH_CHECK(dot_dev(st, K, n, K->w.p, V + (size_t)k * n, K->hcol.p + k, nullptr, 2,
                   K->hcol.p + k + 1));
  normalize_kernel<<<dim3(1184), dim3(256), 0, st>>>(n, K->w.p, K->hcol.p + k + 1,
                                                     V + (size_t)(k + 1) * n);
  MH_CHECK_CUDA(cudaGetLastError());
  MH_CHECK_CUDA(cudaMemcpyAsync(K->h_host, K->hcol.p, sizeof(double) * (k + 2),
                                cudaMemcpyDeviceToHost, st));
  return MH_OK;
}

// Replays (capturing on first use) the graph of step k on a private stream
// ordered after `st`; returns with the Hessenberg column in K->h_host.  The
// k + 3 launches of a step then cost one graph launch: same kernels, same
// arguments, bitwise the same results.
int run_mgs(cudaStream_t st, Krylov* K, int64_t n, int k) {
  if (!K->gs) {
    MH_CHECK_CUDA(cudaStreamCreateWithFlags(&K->gs, cudaStreamNonBlocking));
    MH_CHECK_CUDA(cudaEventCreateWithFlags(&K->ev_in, cudaEventDisableTiming));
    MH_CHECK_CUDA(cudaEventCreateWithFlags(&K->ev_out, cudaEventDisableTiming));
  }
  if ((int)K->mgs.size() < K->restart) K->mgs.resize((size_t)K->restart, nullptr);
  if (!K->mgs[k]) {
    cudaGraph_t g = nullptr;
    MH_CHECK_CUDA(cudaStreamBeginCapture(K->gs, cudaStreamCaptureModeThreadLocal));
    const int st_enq = enqueue_mgs(K->gs, K, n, k);
    const cudaError_t ce = cudaStreamEndCapture(K->gs, &g);
    MH_CHECK(st_enq);
    MH_CHECK_CUDA(ce);
    MH_CHECK_CUDA(cudaGraphInstantiate(&K->mgs[k], g, 0));
    cudaGraphDestroy(g);
  }
  MH_CHECK_CUDA(cudaEventRecord(K->ev_in, st));
  MH_CHECK_CUDA(cudaStreamWaitEvent(K->gs, K->ev_in, 0));
  MH_CHECK_CUDA(cudaGraphLaunch(K->mgs[k], K->gs));
  MH_CHECK_CUDA(cudaEventRecord(K->ev_out, K->gs));
  MH_CHECK_CUDA(cudaStreamWaitEvent(st, K->ev_out, 0));
  MH_CHECK_CUDA(cudaEventSynchronize(K->ev_out));
  return MH_OK;
}

struct CommScope {  // binds the communicator of a system to the dot products
  explicit CommScope(mh_system* s) { g_comm_sys = s; }
  ~CommScope() { g_comm_sys = nullptr; }
};

int gmres_core(cudaStream_t st, Krylov* K, int64_t n, const OpFn& A, const OpFn& M,
               const OpFn& MA, double tol, int restart, int maxiter, const double* rhs,
               double* x, int* iterations, int* converged, double* hist_host, int hist_cap,
               int* hist_len) {
  std::vector<double> history;
  MH_CHECK_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, st));
  // bnorm = ||M b||
  const double* mb = rhs;
  if (M.fn) {
    MH_CHECK(M(rhs, K->tmp.p));
    mb = K->tmp.p;
  }
  MH_CHECK(dot_dev(st, K, n, const_cast<double*>(mb), nullptr, nullptr, nullptr, 2, K->scal.p));
  MH_CHECK(read_scalars(st, K, K->scal.p, 1));
  const double bnorm = K->h_host[0];
  int it = 0;
  bool conv = false;
  auto finish = [&](void) {
    if (iterations) *iterations = it;
    if (converged) *converged = conv ? 1 : 0;
    if (hist_len) *hist_len = (int)history.size();
    if (hist_host)
      for (int i = 0; i < (int)history.size() && i < hist_cap; ++i) hist_host[i] = history[i];
  };
  if (bnorm == 0.0) {
    history.push_back(0.0);
    conv = true;
    finish();
    return MH_OK;
  }
  const int m = restart;
  const char* gv = getenv("MEHDG_GMRES_GRAPHS");
  const bool use_graphs = K->persistent &&
                          !(g_comm_sys && (g_comm_sys->nranks > 1 || g_comm_sys->nccl)) &&
                          !(gv && gv[0] == '0');
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), y(m);
  auto Hat = [&](int i, int k) -> double& { return H[(size_t)i * m + k]; };
  double* V = K->V.p;
  const dim3 vg(kVecGrid), vb(kVecThreads);
  while (it < maxiter && !conv) {
    // r = M(b - A x)
    MH_CHECK(A(x, K->tmp.p));
    sub_kernel<<<vg, vb, 0, st>>>(n, rhs, K->tmp.p, K->tmp2.p);
    MH_CHECK_CUDA(cudaGetLastError());
    double* r = K->tmp2.p;
    if (M.fn) {
      MH_CHECK(M(K->tmp2.p, K->w.p));
      r = K->w.p;
    }
    MH_CHECK(dot_dev(st, K, n, r, nullptr, nullptr, nullptr, 2, K->scal.p));
    MH_CHECK(read_scalars(st, K, K->scal.p, 1));
    const double beta = K->h_host[0];
    if (history.empty()) history.push_back(beta);
    if (beta / bnorm <= tol) {
      conv = true;
      break;
    }
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(cs.begin(), cs.end(), 0.0);
    std::fill(sn.begin(), sn.end(), 0.0);
    std::fill(g.begin(), g.end(), 0.0);
    scale_kernel<<<vg, vb, 0, st>>>(n, r, beta, V);
    MH_CHECK_CUDA(cudaGetLastError());
    g[0] = beta;
    int k_used = 0;
    bool breakdown = false;
    for (int k = 0; k < m; ++k) {
      double* Vk = V + (size_t)k * n;
      MH_CHECK(apply_MA(A, M, MA, Vk, K->w.p, K->tmp.p));
      // MGS: H[i,k] = V[i].w ; w -= H[i,k] V[i]   (fused one step behind), as one
      // CUDA graph per k on a single device (the multi-rank dots go through NCCL)
      if (use_graphs) {
        MH_CHECK(run_mgs(st, K, n, k));
      } else {
        MH_CHECK(enqueue_mgs(st, K, n, k));
        MH_CHECK_CUDA(cudaStreamSynchronize(st));
      }
      for (int i = 0; i <= k + 1; ++i) Hat(i, k) = K->h_host[i];
      if (!(Hat(k + 1, k) > 1e-300)) breakdown = true;
      for (int i = 0; i < k; ++i) {
        const double tt = cs[i] * Hat(i, k) + sn[i] * Hat(i + 1, k);
        Hat(i + 1, k) = -sn[i] * Hat(i, k) + cs[i] * Hat(i + 1, k);
        Hat(i, k) = tt;
      }
      const double denom = std::hypot(Hat(k, k), Hat(k + 1, k));
      if (denom == 0.0) {
        k_used = k + 1;
        breakdown = true;
        break;
      }
      cs[k] = Hat(k, k) / denom;
      sn[k] = Hat(k + 1, k) / denom;
      Hat(k, k) = denom;
      Hat(k + 1, k) = 0.0;
      g[k + 1] = -sn[k] * g[k];
      g[k] = cs[k] * g[k];
      it += 1;
      const double res = std::fabs(g[k + 1]);
      history.push_back(res);
      k_used = k + 1;
      if (res / bnorm <= tol) {
        conv = true;
        break;
      }
      if (breakdown || it >= maxiter) break;
    }
    if (k_used > 0) {
      // y = solve_triangular(H[:k,:k], g[:k]) (upper, column-oriented like dtrsv)
      for (int j = 0; j < k_used; ++j) y[j] = g[j];
      for (int j = k_used - 1; j >= 0; --j) {
        y[j] = y[j] / Hat(j, j);
        for (int i = 0; i < j; ++i) y[i] -= y[j] * Hat(i, j);
      }
      for (int j = 0; j < k_used; ++j) K->h_host[j] = y[j];
      MH_CHECK_CUDA(cudaMemcpyAsync(K->ydev.p, K->h_host, sizeof(double) * k_used,
                                    cudaMemcpyHostToDevice, st));
      update_x_kernel<<<vg, vb, 0, st>>>(n, k_used, V, K->ydev.p, x);
      MH_CHECK_CUDA(cudaGetLastError());
      MH_CHECK_CUDA(cudaStreamSynchronize(st));  // h_host reused below
    }
    if (breakdown && !conv) break;  // invariant Krylov subspace
  }
  if (!conv) {  // one true-residual recheck (schur_solver.py:382-384)
    MH_CHECK(A(x, K->tmp.p));
    sub_kernel<<<vg, vb, 0, st>>>(n, rhs, K->tmp.p, K->tmp2.p);
    MH_CHECK_CUDA(cudaGetLastError());
    double* r = K->tmp2.p;
    if (M.fn) {
      MH_CHECK(M(K->tmp2.p, K->w.p));
      r = K->w.p;
    }
    MH_CHECK(dot_dev(st, K, n, r, nullptr, nullptr, nullptr, 2, K->scal.p));
    MH_CHECK(read_scalars(st, K, K->scal.p, 1));
    conv = K->h_host[0] / bnorm <= tol;
  }
  finish();
  return MH_OK;
}

// ---- system operators ------------------------------------------------------
int sys_apply(void* ctx, const double* in, double* out) { return mh_apply((mh_system*)ctx, in, out); }
int sys_apply_mb(void* ctx, const double* in, double* out) {
  return mh_apply_mb((mh_system*)ctx, in, out);
}
int sys_precond(void* ctx, const double* in, double* out) {
  return mh_precond((mh_system*)ctx, in, out);
}
int sys_apply_precond(void* ctx, const double* in, double* out) {
  return mh_apply_precond((mh_system*)ctx, in, out);
}

}  // namespace
}  // namespace mh

using namespace mh;

extern "C" int mh_dot(void* stream, int64_t n, const double* x, const double* y, double* out) {
  if (n < 0 || (n > 0 && (!x || !y)) || !out) {
    set_error("mh_dot: bad arguments");
    return MH_E_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  Krylov K;
  MH_CHECK(K.part.alloc(kDotBlocks));
  MH_CHECK(K.ticket.alloc(1));
  MH_CHECK(K.scal.alloc(1));
  MH_CHECK_CUDA(cudaMemsetAsync(K.ticket.p, 0, sizeof(unsigned), st));
  dot_kernel<<<kDotBlocks, kDotThreads, 0, st>>>(n, const_cast<double*>(x), nullptr, nullptr, y, 0,
                                                  true, K.part.p, K.ticket.p, K.scal.p);
  MH_CHECK_CUDA(cudaGetLastError());
  MH_CHECK_CUDA(cudaMemcpyAsync(out, K.scal.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  MH_CHECK_CUDA(cudaStreamSynchronize(st));
  return MH_OK;
}

static int check_gmres_args(double tol, int restart, int maxiter) {
  if (!(tol > 0.0 && tol < 1.0)) {
    set_error("tolerance must lie in (0, 1)");
    return MH_E_ARG;
  }
  if (restart < 1 || maxiter < 0) {
    set_error("restart must be >= 1 and maxiter >= 0");
    return MH_E_ARG;
  }
  return MH_OK;
}

extern "C" int mh_gmres(mh_system* s, double tol, int restart, int maxiter, int use_precond,
                        int mode, const double* rhs, double* x, int* iterations, int* converged,
                        double* hist_host, int hist_cap, int* hist_len) {
  if (!s || !rhs || !x) {
    set_error("mh_gmres: null argument");
    return MH_E_ARG;
  }
  MH_CHECK(check_gmres_args(tol, restart, maxiter));
  if (!s->factored) {
    set_error("mh_gmres before mh_factorize");
    return MH_E_STATE;
  }
  if (mode == 1 && !s->have_mb) {
    set_error("mode mb requires mh_form_element_schur");
    return MH_E_STATE;
  }
  MH_CHECK_CUDA(cudaSetDevice(s->device));
  if (!s->kry) {
    s->kry = new Krylov();
    s->kry->persistent = true;
  }
  const int64_t n = s->F * (int64_t)s->t;
  MH_CHECK(s->kry->alloc(n, restart));
  OpFn A, M, MA;
  A.fn = mode == 1 ? sys_apply_mb : sys_apply;
  A.ctx = s;
  if (use_precond) {
    M.fn = sys_precond;
    M.ctx = s;
    if (mode == 0) {
      MA.fn = sys_apply_precond;
      MA.ctx = s;
    }
  }
  CommScope scope(s);
  return gmres_core(s->stream, s->kry, n, A, M, MA, tol, restart, maxiter, rhs, x, iterations,
                    converged, hist_host, hist_cap, hist_len);
}

extern "C" int mh_gmres_op(int device, void* stream, int64_t n, mh_op_fn apply, void* apply_ctx,
                           mh_op_fn precond, void* precond_ctx, double tol, int restart,
                           int maxiter, const double* rhs, double* x, int* iterations,
                           int* converged, double* hist_host, int hist_cap, int* hist_len) {
  if (!apply || n < 0 || (n > 0 && (!rhs || !x))) {
    set_error("mh_gmres_op: bad arguments");
    return MH_E_ARG;
  }
  MH_CHECK(check_gmres_args(tol, restart, maxiter));
  MH_CHECK_CUDA(cudaSetDevice(device));
  Krylov K;
  MH_CHECK(K.alloc(n, restart));
  OpFn A, M, MA;
  A.fn = apply;
  A.ctx = apply_ctx;
  if (precond) {
    M.fn = precond;
    M.ctx = precond_ctx;
  }
  return gmres_core((cudaStream_t)stream, &K, n, A, M, MA, tol, restart, maxiter, rhs, x,
                    iterations, converged, hist_host, hist_cap, hist_len);
}
