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

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <vector>

#include "mh_internal.h"

namespace mh {

constexpr int kDotPartsMax = 2048;  // partials of a dot product (one warp each)
constexpr int kDotWarps = 8;        // warps per block of the grid dot kernel

// The number of partials of an n-vector dot product: a power of two near n / 64
// in [32, 2048] (a few elements per lane: each reduction phase is one memory
// round trip) -- a function of n alone, so every kernel (and rank count) that
// reduces the same vector uses the same partition.
__host__ __device__ inline int dot_parts(int64_t n) {
  int p = 32;
  while (p < kDotPartsMax && (int64_t)p * 2 * 64 <= n) p *= 2;
  return p;
}

// The Givens state of a pipelined solve (device pointers and the solve's
// constants, themselves in device memory so that a captured graph stays valid
// from solve to solve): par = {bnorm, tol, maxiter}.
struct GivensDev {
  double* H;
  double* cs;
  double* sn;
  double* g;
  double* hist;
  int* ctl;
  const double* par;
  int m;
};

struct Krylov {
  int64_t n = 0;
  int restart = 0;
  DBuf<double> V, w, tmp, tmp2, part, hcol, ydev, scal;
  DBuf<unsigned> ticket, bar;  // bar: the MGS kernel's grid barrier (count, generation)
  int num_sms = 148;
  double* h_host = nullptr;  // pinned
  // device Arnoldi pipeline (pipelined solves): the Hessenberg matrix, the
  // rotations, g, the per-step residual estimates and the control block
  DBuf<double> Hd, csd, snd, gd, histd;
  DBuf<double> cgs;          // CGS2: partials (2 x (restart+2) x dot_parts) and sums
  DBuf<int> ctl;             // GmresCtl
  DBuf<double> gpar;         // {bnorm, tol, maxiter} of the running solve
  DBuf<GivensDev> gvd;       // the device copy of the Givens state (fused MGS tail)
  int* ctl_host = nullptr;   // pinned: two slots of kCtlInts, then 4 doubles (the solve constants)
  const int* skip = nullptr; // &ctl->stop while a pipelined cycle runs
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
    MH_CHECK(part.alloc(2 * kDotPartsMax));
    MH_CHECK(hcol.alloc((size_t)restart + 2));
    MH_CHECK(bar.alloc(2));
    MH_CHECK_CUDA(cudaMemset(bar.p, 0, 2 * sizeof(unsigned)));
    {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    MH_CHECK(ydev.alloc((size_t)restart + 1));
    MH_CHECK(scal.alloc(4));
    MH_CHECK(ticket.alloc(1));
    MH_CHECK_CUDA(cudaMemset(ticket.p, 0, sizeof(unsigned)));
    if (h_host) cudaFreeHost(h_host);
    MH_CHECK_CUDA(cudaMallocHost(&h_host, sizeof(double) * ((size_t)(restart + 1) * restart + 4 * restart + 8)));
    MH_CHECK(Hd.alloc((size_t)(restart + 1) * restart));
    MH_CHECK(csd.alloc((size_t)restart));
    MH_CHECK(snd.alloc((size_t)restart));
    MH_CHECK(gd.alloc((size_t)restart + 1));
    MH_CHECK(histd.alloc((size_t)restart));
    MH_CHECK(ctl.alloc(8));
    MH_CHECK(gpar.alloc(4));
    MH_CHECK(gvd.alloc(1));
    {
      GivensDev gh{Hd.p, csd.p, snd.p, gd.p, histd.p, ctl.p, gpar.p, restart};
      MH_CHECK_CUDA(cudaMemcpy(gvd.p, &gh, sizeof(gh), cudaMemcpyHostToDevice));
    }
    MH_CHECK(cgs.alloc((size_t)(restart + 2) * kDotPartsMax + 4 * ((size_t)restart + 2)));
    if (!ctl_host) MH_CHECK_CUDA(cudaMallocHost(&ctl_host, sizeof(int) * 16 + sizeof(double) * 4));
    return MH_OK;
  }
  ~Krylov() {
    drop_graphs();
    if (gs) cudaStreamDestroy(gs);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_out) cudaEventDestroy(ev_out);
    V.release(); w.release(); tmp.release(); tmp2.release(); part.release();
    hcol.release(); ydev.release(); scal.release(); ticket.release(); bar.release();
    Hd.release(); csd.release(); snd.release(); gd.release(); histd.release(); ctl.release();
    cgs.release(); gpar.release(); gvd.release();
    if (h_host) cudaFreeHost(h_host);
    if (ctl_host) cudaFreeHost(ctl_host);
  }
};

void free_krylov(Krylov* k) { delete k; }

namespace {

// ---- deterministic dot products --------------------------------------
// A dot product is the fixed-order sum of P = dot_parts(n) partials; partial b
// covers [n b / P, n (b+1) / P) and is computed by ONE warp (lane l
// accumulates elements lo + l, lo + l + 32, ... with fma, then a fixed xor
// tree).  The final sum: lane l adds partials l, l + 32, ... in order, then the
// same xor tree.  The grid kernel (a warp per partial, last-block-done final
// sum) and the one-CTA MGS kernel (each warp several partials) therefore give
// bitwise the same value -- as do 1 and N ranks (rank partials all-gathered and
// added in rank order).

__device__ __forceinline__ double warp_xor_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// partial b of (w - c Vp) . y, updating w in place when coef is given
// (mode 1: y = Vi; mode 2: y = w itself)
__device__ __forceinline__ double dot_partial(int64_t n, int P, int b, double* __restrict__ w,
                                              const double* __restrict__ Vp, double c, bool upd,
                                              const double* __restrict__ Vi, int mode, int lane) {
  const int64_t lo = n * b / P, hi = n * (b + 1) / P;
  double acc = 0.0;
  // batches of 8 elements per lane: all loads of a batch first (w may alias
  // nothing, but the compiler cannot move loads above the previous stores)
  for (int64_t i0 = lo + lane; i0 < hi; i0 += 32 * 8) {
    double wv[8], pv[8], yv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = i0 + 32 * u;
      const bool ok = i < hi;
      wv[u] = ok ? w[i] : 0.0;
      pv[u] = (ok && upd) ? Vp[i] : 0.0;
      yv[u] = (ok && mode != 2) ? Vi[i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = i0 + 32 * u;
      if (i < hi) {
        double wi = wv[u];
        if (upd) {
          wi = __dsub_rn(wi, __dmul_rn(c, pv[u]));  // numpy: wv -= H*V (two roundings)
          w[i] = wi;
        }
        acc = fma(wi, mode == 2 ? wi : yv[u], acc);
      }
    }
  }
  return warp_xor_sum(acc);
}

// the fixed-order sum of the P partials (one warp).  The partials were
// published before a fence + barrier / ticket: L2-coherent loads (ld.cg, no
// stale L1 line), issued together rather than one volatile load at a time
__device__ __forceinline__ double parts_sum(const double* part, int P, int lane) {
  // all of a lane's partials (<= kDotPartsMax / 32) in flight at once, then the
  // fixed-order sum: one memory round trip instead of one per load
  constexpr int kMax = kDotPartsMax / 32;
  double x[kMax];
#pragma unroll
  for (int u = 0; u < kMax; ++u) x[u] = (lane + 32 * u < P) ? __ldcg(part + lane + 32 * u) : 0.0;
  double v = 0.0;
#pragma unroll
  for (int u = 0; u < kMax; ++u)
    if (lane + 32 * u < P) v += x[u];
  return warp_xor_sum(v);
}

// The same total by a whole 8-warp CTA: warp g sums the g-th eighth of the
// partials (lane l adds its partials l, l + 32, ... in order, then the xor tree),
// the eight group sums are added in order.  At most 8 loads per lane, one memory
// round trip; every thread returns the total.  THE dot-product value of the
// single-rank kernels (dot_kernel, mgs_kernel, mgs_reg_kernel all end here).
// sg: 8 doubles of shared memory, free again after the caller's next barrier.
__device__ __forceinline__ double parts_sum_cta(const double* part, int P, double* sg, int lane,
                                                int wp) {
  constexpr int kMax = kDotPartsMax / 8 / 32;
  const int per = P >> 3;  // P is a power of two >= 32
  const double* pg = part + wp * per;
  double x[kMax];
#pragma unroll
  for (int u = 0; u < kMax; ++u) x[u] = (lane + 32 * u < per) ? __ldcg(pg + lane + 32 * u) : 0.0;
  double v = 0.0;
#pragma unroll
  for (int u = 0; u < kMax; ++u)
    if (lane + 32 * u < per) v += x[u];
  v = warp_xor_sum(v);
  if (lane == 0) sg[wp] = v;
  __syncthreads();
  double t = sg[0];
#pragma unroll
  for (int g = 1; g < 8; ++g) t += sg[g];
  return t;
}

// Fused MGS step.  mode 0: plain dot(x, y); mode 1: w -= c*Vp then dot(Vi, w);
// mode 2: w -= c*Vp then dot(w, w) and out <- sqrt.  Result to *out (device).
// A set *skip (a stopped speculative GMRES step) makes it a no-op.
__global__ void __launch_bounds__(kDotWarps * 32)
dot_kernel(int64_t n, double* __restrict__ w, const double* __restrict__ Vp,
           const double* __restrict__ coef, const double* __restrict__ Vi, int mode,
           bool take_sqrt, double* __restrict__ part, unsigned* __restrict__ ticket,
           double* __restrict__ out, const int* __restrict__ skip) {
  if (skip && *skip) return;
  __shared__ bool last;
  __shared__ double sg[8];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int b = blockIdx.x * kDotWarps + wp;
  const int P = gridDim.x * kDotWarps;
  const bool upd = mode != 0 && coef;
  const double c = upd ? *coef : 0.0;
  const double s = dot_partial(n, P, b, w, Vp, c, upd, Vi, mode, lane);
  if (lane == 0) part[b] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned tk = atomicAdd(ticket, 1u);
    last = (tk == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const double tot = parts_sum_cta(part, P, sg, lane, wp);
  if (threadIdx.x == 0) {
    *out = (mode == 2 && take_sqrt) ? sqrt(tot) : tot;
    *ticket = 0u;
  }
}

// The whole MGS block of Arnoldi step k in ONE launch: the k + 2 dependent
// reductions (H[0..k, k] and ||w||), each followed by a grid-wide barrier,
// then V[k+1] = w / ||w||.  Warp gw computes partials gw, gw + (all warps),
// ... exactly as dot_kernel's warps do, every block then sums the same
// partials in the same order (double-buffered, so one barrier per reduction):
// the results are bitwise those of k + 2 dot_kernel launches.  8-warp CTAs
// (MEHDG_MGS_CTAS per SM at most), launched cooperatively (all resident).
constexpr int kMgsThreads = 256;


// Control block of a pipelined GMRES cycle (device ints)
enum GmresCtl { kStop = 0, kKUsed = 1, kIt = 2, kConv = 3, kBreak = 4, kSteps = 5 };
constexpr int kCtlInts = 8;
constexpr int kMaxRestartSmem = 1024;  // restart lengths the device Givens supports

// Step k's Givens update, one warp, the reference's arithmetic
// (schur_solver.py:351-375): the new Hessenberg column, the previous rotations,
// the new rotation, g, the residual estimate and the stopping rules.  Once a
// cycle stops (converged, breakdown, maxiter) every later step of it is a no-op
// -- the host enqueues steps ahead without waiting for each one.
// sh / sc / ss: kMaxRestartSmem (+2) doubles of shared memory each.
__device__ __forceinline__ void givens_step(const double* hcol, const GivensDev& G, int k,
                                            double* sh, double* sc, double* ss, int lane) {
  if (G.ctl[kStop]) return;
  const int m = G.m;
  const double bnorm = G.par[0], tol = G.par[1];
  const int maxiter = (int)G.par[2];
  for (int i = lane; i <= k + 1; i += 32) sh[i] = __ldcg(hcol + i);
  for (int i = lane; i < k; i += 32) {
    sc[i] = G.cs[i];
    ss[i] = G.sn[i];
  }
  __syncwarp();
  if (lane == 0) {
    const bool breakdown = !(sh[k + 1] > 1e-300);
    for (int i = 0; i < k; ++i) {
      const double tt = sc[i] * sh[i] + ss[i] * sh[i + 1];
      sh[i + 1] = -ss[i] * sh[i] + sc[i] * sh[i + 1];
      sh[i] = tt;
    }
    const double denom = hypot(sh[k], sh[k + 1]);
    if (denom == 0.0) {
      G.ctl[kKUsed] = k + 1;
      G.ctl[kBreak] = 1;
      G.ctl[kStop] = 1;
    } else {
      const double c = sh[k] / denom, sgn = sh[k + 1] / denom;
      G.cs[k] = c;
      G.sn[k] = sgn;
      sh[k] = denom;
      sh[k + 1] = 0.0;
      const double gk = G.g[k];
      G.g[k + 1] = -sgn * gk;
      G.g[k] = c * gk;
      const int it = ++G.ctl[kIt];
      const double res = fabs(G.g[k + 1]);
      G.hist[G.ctl[kSteps]++] = res;
      G.ctl[kKUsed] = k + 1;
      if (res / bnorm <= tol) {
        G.ctl[kConv] = 1;
        G.ctl[kStop] = 1;
      } else if (breakdown || it >= maxiter) {
        G.ctl[kBreak] = breakdown ? 1 : 0;
        G.ctl[kStop] = 1;
      }
    }
  }
  __syncwarp();
  for (int i = lane; i <= k + 1; i += 32) G.H[(size_t)i * m + k] = sh[i];
}

// Grid-wide barrier of a cooperative launch on ONE monotonic counter: barrier b
// of a launch is passed once the counter reaches base + (b + 1) G, base being
// the counter's value when the launch started (a multiple of G: read by every
// CTA before its own first arrival, when at most G - 1 others have arrived,
// and rounded down).  One fire-and-forget increment and one polled line per
// barrier -- no second atomic by the last arriver.  The counter is zeroed at
// the start of every solve; all launches of a solve use the same grid.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();  // this CTA's partials before its arrival
    atomicAdd(count, 1u);
    while ((int)(ld_acquire_u32(count) - target) < 0) {
    }
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned barrier_base(const unsigned* count, unsigned* sbase) {
  if (threadIdx.x == 0) {
    const unsigned v = ld_acquire_u32(count);
    *sbase = v - v % gridDim.x;
  }
  __syncthreads();
  return *sbase;
}

__global__ void __launch_bounds__(kMgsThreads)
mgs_kernel(int64_t n, double* __restrict__ w, const double* __restrict__ V, int k,
           double* __restrict__ hcol, double* __restrict__ vnext, double* __restrict__ part2,
           unsigned* __restrict__ bar, const int* __restrict__ skip, const GivensDev* gv) {
  if (skip && *skip) return;
  __shared__ double sg[8];
  __shared__ unsigned sbase;
  __shared__ double gsh[kMaxRestartSmem + 2], gsc[kMaxRestartSmem], gss[kMaxRestartSmem];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int WB = kMgsThreads / 32;
  const int gw = blockIdx.x * WB + wp, nw = gridDim.x * WB;
  const int P = dot_parts(n);
  const unsigned base = gridDim.x > 1 ? barrier_base(bar, &sbase) : 0u;
  double c = 0.0;
  const double* Vp = nullptr;
  for (int i = 0; i <= k + 1; ++i) {
    const double* Vi = V + (size_t)i * n;  // i = k + 1: the norm of w
    const int mode = i <= k ? 1 : 2;
    double* part = part2 + (i & 1) * kDotPartsMax;
    for (int b = gw; b < P; b += nw) {
      const double pv = dot_partial(n, P, b, w, Vp, c, i > 0, Vi, mode, lane);
      if (lane == 0) part[b] = pv;
    }
    if (gridDim.x > 1) grid_barrier(bar, base + (unsigned)(i + 1) * gridDim.x);
    else __syncthreads();
    double h = parts_sum_cta(part, P, sg, lane, wp);
    if (i == k + 1) h = sqrt(h);
    if (blockIdx.x == 0 && threadIdx.x == 0) hcol[i] = h;
    c = h;
    Vp = Vi;
  }
  if (gv && blockIdx.x == 0 && wp == 0) {
    __syncwarp();
    givens_step(hcol, *gv, k, gsh, gsc, gss, lane);
  }
  if (!(c > 1e-300)) return;
  for (int64_t j = blockIdx.x * (int64_t)kMgsThreads + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * kMgsThreads)
    vnext[j] = w[j] / c;
}

// The same MGS block with w and the previous basis vector held in registers
// (a warp per partial, at most E elements per lane): each reduction reads one
// basis vector from memory -- the next one is loaded BEFORE the barrier of the
// current reduction, so its latency hides behind the barrier -- and nothing is
// written until V[k+1] = w / ||w||.  Per element the operations and their
// order are dot_partial's, so the results are bitwise those of mgs_kernel /
// dot_kernel.
template <int E>
__global__ void __launch_bounds__(kMgsThreads, E <= 12 ? 2 : 1)
mgs_reg_kernel(int64_t n, const double* __restrict__ w, const double* __restrict__ V, int k,
               double* __restrict__ hcol, double* __restrict__ vnext,
               double* __restrict__ part2, unsigned* __restrict__ bar,
               const int* __restrict__ skip, const GivensDev* gv) {
  if (skip && *skip) return;
  __shared__ double sg[8];
  __shared__ unsigned sbase;
  __shared__ double gsh[kMaxRestartSmem + 2], gsc[kMaxRestartSmem], gss[kMaxRestartSmem];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int b = blockIdx.x * (kMgsThreads / 32) + wp;
  const int P = dot_parts(n);
  const int64_t lo = b < P ? n * b / P : 0, hi = b < P ? n * (b + 1) / P : 0;
  const int cnt = (int)(hi - lo) - lane;  // element e of this lane is valid when 32 e < cnt
  const unsigned base = barrier_base(bar, &sbase);
  const double* vcur = V + lo + lane;
  double wr[E], vp[E], yv[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    wr[e] = 32 * e < cnt ? w[lo + lane + 32 * e] : 0.0;
    yv[e] = 32 * e < cnt ? vcur[32 * e] : 0.0;  // V_0
    vp[e] = 0.0;
  }
  double c = 0.0;
  for (int i = 0; i <= k + 1; ++i) {
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (32 * e < cnt) {
        double wi = wr[e];
        if (i > 0) wi = __dsub_rn(wi, __dmul_rn(c, vp[e]));
        wr[e] = wi;
        acc = fma(wi, i <= k ? yv[e] : wi, acc);
      }
      vp[e] = yv[e];
    }
    if (i + 1 <= k) {  // the next basis vector, in flight across the barrier
      vcur += n;
#pragma unroll
      for (int e = 0; e < E; ++e) yv[e] = 32 * e < cnt ? vcur[32 * e] : 0.0;
    }
    acc = warp_xor_sum(acc);
    double* part = part2 + (i & 1) * kDotPartsMax;
    if (lane == 0 && b < P) part[b] = acc;
    grid_barrier(bar, base + (unsigned)(i + 1) * gridDim.x);
    double h = parts_sum_cta(part, P, sg, lane, wp);
    if (i == k + 1) h = sqrt(h);
    if (blockIdx.x == 0 && threadIdx.x == 0) hcol[i] = h;
    c = h;
  }
  if (gv && blockIdx.x == 0 && wp == 0) {
    __syncwarp();
    givens_step(hcol, *gv, k, gsh, gsc, gss, lane);
  }
  if (!(c > 1e-300)) return;
  double* vn = vnext + lo + lane;
#pragma unroll
  for (int e = 0; e < E; ++e)
    if (32 * e < cnt) vn[32 * e] = wr[e] / c;
}

// ---- the multi-rank Arnoldi step: classical Gram-Schmidt twice (CGS2) --
// MGS needs k + 2 dependent reductions per step, i.e. k + 2 collectives on a
// multi-rank system; CGS2 needs two: h = V^T w (one batched reduction of k + 2
// values, the last being ||w||^2), w -= V h, then h2 = V^T w and ||w||^2 again,
// w -= V h2; H[0..k, k] = h + h2 and ||w_final||^2 = ||w||^2 - ||h2||^2.  Each
// batched reduction uses the dot partition (dot_parts(n) warp partials, fixed
// order), the rank sums are all-gathered and added in rank order: every rank
// holds identical values.  Within the solve tolerance of MGS, not bitwise.
__global__ void __launch_bounds__(kDotWarps * 32)
multidot_kernel(int64_t n, const double* __restrict__ V, int m, const double* __restrict__ w,
                double* __restrict__ part, unsigned* __restrict__ ticket,
                double* __restrict__ out, const int* __restrict__ skip) {
  if (skip && *skip) return;
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int b = blockIdx.x * kDotWarps + wp;
  const int P = gridDim.x * kDotWarps;
  const int64_t lo = n * b / P, hi = n * (b + 1) / P;
  for (int i = 0; i <= m; ++i) {  // i < m: V_i . w; i == m: w . w
    const double* y = i < m ? V + (size_t)i * n : w;
    double acc = 0.0;
#pragma unroll 4
    for (int64_t j = lo + lane; j < hi; j += 32) acc = fma(w[j], y[j], acc);
    acc = warp_xor_sum(acc);
    if (lane == 0) part[(size_t)i * P + b] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned tk = atomicAdd(ticket, 1u);
    last = (tk == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int i = wp; i <= m; i += kDotWarps) {
    const double tot = parts_sum(part + (size_t)i * P, P, lane);
    if (lane == 0) out[i] = tot;
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

// w -= sum_i h[i] V_i (i ascending)
__global__ void cgs_update_kernel(int64_t n, const double* __restrict__ V, int m,
                                  const double* __restrict__ h, double* __restrict__ w,
                                  const int* __restrict__ skip) {
  if (skip && *skip) return;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    double x = w[j];
    for (int i = 0; i < m; ++i) x = __dsub_rn(x, __dmul_rn(h[i], V[(size_t)i * n + j]));
    w[j] = x;
  }
}

// H[0..k, k] = h + h2; H[k+1, k] = sqrt(||w||^2 - ||h2||^2)
__global__ void cgs_finalize_kernel(const double* __restrict__ h, const double* __restrict__ h2,
                                    int k, double* __restrict__ hcol, const int* __restrict__ skip) {
  if (skip && *skip) return;
  if (threadIdx.x != 0) return;
  double q = 0.0;
  for (int i = 0; i <= k; ++i) {
    hcol[i] = h[i] + h2[i];
    q = fma(h2[i], h2[i], q);
  }
  hcol[k + 1] = sqrt(fmax(h2[k + 1] - q, 0.0));
}

// V[k+1] = w / h if h > 1e-300 (else left zero: breakdown)
__global__ void normalize_kernel(int64_t n, const double* __restrict__ w,
                                 const double* __restrict__ h, double* __restrict__ out,
                                 const int* __restrict__ skip) {
  if (skip && *skip) return;
  const double hv = *h;
  if (!(hv > 1e-300)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = w[i] / hv;
}

// Step k's Givens update as its own launch (multi-rank CGS2 steps and the
// MGS block as separate launches; the one-launch MGS block does it in its tail)
__global__ void givens_kernel(const double* __restrict__ hcol, GivensDev G, int k) {
  __shared__ double sh[kMaxRestartSmem + 2], sc[kMaxRestartSmem], ss[kMaxRestartSmem];
  givens_step(hcol, G, k, sh, sc, ss, threadIdx.x);
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

// the Krylov knobs also serve operator-only solves (mh_gmres_op, no system):
// read once per process
const Knobs& proc_knobs() {
  static const Knobs k = [] {
    Knobs x;
    x.read();
    return x;
  }();
  return k;
}

int dot_dev(cudaStream_t st, Krylov* K, int64_t n, double* w, const double* Vp,
            const double* coef, const double* Vi, int mode, double* out) {
  const bool multi = g_comm_sys && (g_comm_sys->nranks > 1 || g_comm_sys->nccl);
  dot_kernel<<<dot_parts(n) / kDotWarps, kDotWarps * 32, 0, st>>>(
      n, w, Vp, coef, Vi, mode, !multi, K->part.p, K->ticket.p, multi ? K->scal.p + 3 : out,
      K->skip);
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
// True when the MGS block of a step is ONE launch (which can then run the
// step's Givens update in its tail).
bool mgs_one_launch() {
  const bool multi = g_comm_sys && (g_comm_sys->nranks > 1 || g_comm_sys->nccl);
  return !multi && proc_knobs().mgs_small;
}

int enqueue_mgs(cudaStream_t st, Krylov* K, int64_t n, int k, bool copy_host = true,
                bool fuse_givens = false) {
  double* V = K->V.p;
  const bool multi = g_comm_sys && (g_comm_sys->nranks > 1 || g_comm_sys->nccl);
  if (!multi && proc_knobs().mgs_small) {
    // one launch for the whole block: a warp per partial with w in registers
    // when every partial fits E elements per lane and the grid, else memory
    const int P = dot_parts(n);
    const int64_t per_lane = (n / P + 1 + 31) / 32;
    const int wpb = kMgsThreads / 32;
    const void* fn = (const void*)mgs_kernel;
    int G = std::max(1, std::min(K->num_sms * proc_knobs().mgs_ctas, P / wpb));
    if (proc_knobs().mgs_reg && per_lane <= 16) {
      const void* fr = per_lane <= 4 ? (const void*)mgs_reg_kernel<4>
                       : per_lane <= 8 ? (const void*)mgs_reg_kernel<8>
                       : per_lane <= 10 ? (const void*)mgs_reg_kernel<10>
                       : per_lane <= 12 ? (const void*)mgs_reg_kernel<12>
                                        : (const void*)mgs_reg_kernel<16>;
      int dev = 0;
      MH_CHECK_CUDA(cudaGetDevice(&dev));
      const int per_sm = launch_occupancy(dev, fr, kMgsThreads, 0);
      if (per_sm > 0 && P / wpb <= per_sm * K->num_sms) {  // all CTAs co-resident
        G = P / wpb;
        fn = fr;
      }
    }
    double* vnext = V + (size_t)(k + 1) * n;
    const GivensDev* gv = fuse_givens ? K->gvd.p : nullptr;
    void* args[] = {(void*)&n, (void*)&K->w.p, (void*)&V, (void*)&k, (void*)&K->hcol.p,
                    (void*)&vnext, (void*)&K->part.p, (void*)&K->bar.p, (void*)&K->skip,
                    (void*)&gv};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(kMgsThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = G > 1 ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MH_CHECK_CUDA(cudaLaunchKernelExC(&cfg, fn, args));
    if (copy_host)
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
                                                     V + (size_t)(k + 1) * n, K->skip);
  MH_CHECK_CUDA(cudaGetLastError());
  if (copy_host)
    MH_CHECK_CUDA(cudaMemcpyAsync(K->h_host, K->hcol.p, sizeof(double) * (k + 2),
                                  cudaMemcpyDeviceToHost, st));
  return MH_OK;
}

// The multi-rank Arnoldi step (CGS2, two collectives): H[0..k+1, k] to hcol,
// V[k+1] = w / H[k+1, k].
int enqueue_cgs2(cudaStream_t st, Krylov* K, int64_t n, int k) {
  double* V = K->V.p;
  const int m = k + 1;
  const int P = dot_parts(n);
  double* part = K->cgs.p;
  double* loc = part + (size_t)(K->restart + 2) * kDotPartsMax;
  double* hA = loc + (K->restart + 2);
  double* hB = hA + (K->restart + 2);
  const dim3 vg(kVecGrid), vb(kVecThreads);
  for (int pass = 0; pass < 2; ++pass) {
    double* h = pass == 0 ? hA : hB;
    multidot_kernel<<<P / kDotWarps, kDotWarps * 32, 0, st>>>(n, V, m, K->w.p, part, K->ticket.p,
                                                            loc, K->skip);
    MH_CHECK_CUDA(cudaGetLastError());
    MH_CHECK(allreduce_vec(g_comm_sys, loc, m + 1, h));  // one collective
    cgs_update_kernel<<<vg, vb, 0, st>>>(n, V, m, h, K->w.p, K->skip);
    MH_CHECK_CUDA(cudaGetLastError());
  }
  cgs_finalize_kernel<<<1, 32, 0, st>>>(hA, hB, k, K->hcol.p, K->skip);
  MH_CHECK_CUDA(cudaGetLastError());
  normalize_kernel<<<vg, vb, 0, st>>>(n, K->w.p, K->hcol.p + k + 1, V + (size_t)(k + 1) * n,
                                      K->skip);
  MH_CHECK_CUDA(cudaGetLastError());
  return MH_OK;
}

// Replays (capturing on first use, on a private stream) the graph of step k's
// MGS block in order on `st`; asynchronous.  The
// k + 3 launches of a step then cost one graph launch: same kernels, same
// arguments, bitwise the same results.  Pipelined solves only (the graph
// leaves the Hessenberg column on the device for givens_kernel).
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
    const int st_enq = enqueue_mgs(K->gs, K, n, k, false, true);
    const cudaError_t ce = cudaStreamEndCapture(K->gs, &g);
    MH_CHECK(st_enq);
    MH_CHECK_CUDA(ce);
    MH_CHECK_CUDA(cudaGraphInstantiate(&K->mgs[k], g, 0));
    cudaGraphDestroy(g);
  }
  MH_CHECK_CUDA(cudaGraphLaunch(K->mgs[k], st));  // captured on gs, launched in order on st
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
  MH_CHECK_CUDA(cudaMemsetAsync(K->bar.p, 0, 2 * sizeof(unsigned), st));
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
      // MGS: H[i,k] = V[i].w ; w -= H[i,k] V[i]   (fused one step behind)
      MH_CHECK(enqueue_mgs(st, K, n, k));
      MH_CHECK_CUDA(cudaStreamSynchronize(st));
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

// The same solve for operators that run on the device (a system's apply /
// preconditioner): the Arnoldi steps are enqueued ahead -- chunks of kAhead,
// the host reading the control block of the previous chunk while the next one
// runs -- and the Givens rotations run on the device (givens_kernel), so no
// host round trip sits between two steps.  Steps enqueued after the cycle
// stopped are no-ops (the element / face / dot kernels read the stop flag).
// The restart-cycle logic, the triangular solve for y (host, double) and the
// final true-residual recheck are gmres_core's.
constexpr int kAhead = 2;

int gmres_pipelined(mh_system* s, cudaStream_t st, Krylov* K, int64_t n, const OpFn& A,
                    const OpFn& M, const OpFn& MA, double tol, int restart, int maxiter,
                    const double* rhs, double* x, int* iterations, int* converged,
                    double* hist_host, int hist_cap, int* hist_len) {
  std::vector<double> history;
  MH_CHECK_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, st));
  MH_CHECK_CUDA(cudaMemsetAsync(K->bar.p, 0, 2 * sizeof(unsigned), st));
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
  const bool multi = g_comm_sys && (g_comm_sys->nranks > 1 || g_comm_sys->nccl);
  const bool use_graphs = !multi && proc_knobs().gmres_graphs;
  const bool fused = mgs_one_launch();  // the Givens update in the MGS launch's tail
  const GivensDev gvh{K->Hd.p, K->csd.p, K->snd.p, K->gd.p, K->histd.p, K->ctl.p, K->gpar.p, m};
  {
    double* par = reinterpret_cast<double*>(K->ctl_host + 16);  // pinned, written once per solve
    par[0] = bnorm;
    par[1] = tol;
    par[2] = (double)maxiter;
    MH_CHECK_CUDA(cudaMemcpyAsync(K->gpar.p, par, 3 * sizeof(double), cudaMemcpyHostToDevice, st));
  }
  std::vector<double> H((size_t)(m + 1) * m), g(m + 1), y(m), hist(m);
  auto Hat = [&](int i, int k) -> double& { return H[(size_t)i * m + k]; };
  double* V = K->V.p;
  const dim3 vg(kVecGrid), vb(kVecThreads);
  cudaEvent_t ev[2] = {nullptr, nullptr};
  for (auto& e : ev) MH_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  struct Guard {  // clear the stop flag's users and the events on every exit
    mh_system* s;
    Krylov* K;
    cudaEvent_t* ev;
    ~Guard() {
      s->skip = nullptr;
      K->skip = nullptr;
      for (int i = 0; i < 2; ++i) cudaEventDestroy(ev[i]);
    }
  } guard{s, K, ev};
  // MEHDG_GMRES_TRACE: CUDA events around each step's apply / MGS / Givens,
  // the summed times printed to stderr (design measurements only)
  struct Trace {
    bool on = getenv("MEHDG_GMRES_TRACE") != nullptr;
    std::vector<std::pair<int, cudaEvent_t>> ev;
    void mark(cudaStream_t st, int tag) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, st);
      ev.emplace_back(tag, e);
    }
    ~Trace() {
      if (!on) return;
      cudaDeviceSynchronize();
      double t[4] = {0, 0, 0, 0};
      for (size_t i = 1; i < ev.size(); ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second);
        t[ev[i - 1].second ? ev[i - 1].first : 0] += ms;
      }
      fprintf(stderr, "gmres trace: apply %.3f ms, mgs %.3f ms, givens %.3f ms, gaps %.3f ms (%zu marks)\n",
              t[0], t[1], t[2], t[3], ev.size());
      for (auto& pr : ev) cudaEventDestroy(pr.second);
    }
  } tr;
  bool x_zero = true;
  while (it < maxiter && !conv) {
    // r = M(b - A x), beta (host: the cycle's start and stop tests); with x = 0
    // (the first cycle) A x = 0 exactly and r = M b, already formed for bnorm
    double* r;
    if (x_zero) {
      r = M.fn ? K->tmp.p : const_cast<double*>(rhs);
    } else {
      MH_CHECK(A(x, K->tmp.p));
      sub_kernel<<<vg, vb, 0, st>>>(n, rhs, K->tmp.p, K->tmp2.p);
      MH_CHECK_CUDA(cudaGetLastError());
      r = K->tmp2.p;
      if (M.fn) {
        MH_CHECK(M(K->tmp2.p, K->w.p));
        r = K->w.p;
      }
    }
    double beta = bnorm;  // x = 0: r = M b, whose norm is bnorm (the same reduction)
    if (!x_zero) {
      MH_CHECK(dot_dev(st, K, n, r, nullptr, nullptr, nullptr, 2, K->scal.p));
      MH_CHECK(read_scalars(st, K, K->scal.p, 1));
      beta = K->h_host[0];
    }
    if (history.empty()) history.push_back(beta);
    if (beta / bnorm <= tol) {
      conv = true;
      break;
    }
    // the cycle's device state: H = cs = sn = g = 0, g[0] = beta, control block
    MH_CHECK_CUDA(cudaMemsetAsync(K->Hd.p, 0, sizeof(double) * (size_t)(m + 1) * m, st));
    MH_CHECK_CUDA(cudaMemsetAsync(K->csd.p, 0, sizeof(double) * m, st));
    MH_CHECK_CUDA(cudaMemsetAsync(K->snd.p, 0, sizeof(double) * m, st));
    MH_CHECK_CUDA(cudaMemsetAsync(K->gd.p, 0, sizeof(double) * (m + 1), st));
    K->h_host[0] = beta;
    MH_CHECK_CUDA(cudaMemcpyAsync(K->gd.p, K->h_host, sizeof(double), cudaMemcpyHostToDevice, st));
    int* ch = K->ctl_host;
    for (int i = 0; i < kCtlInts; ++i) ch[i] = 0;
    ch[kIt] = it;
    MH_CHECK_CUDA(cudaMemcpyAsync(K->ctl.p, ch, sizeof(int) * kCtlInts, cudaMemcpyHostToDevice, st));
    scale_kernel<<<vg, vb, 0, st>>>(n, r, beta, V);
    MH_CHECK_CUDA(cudaGetLastError());
    // no host wait here: h_host[0] and ch[0..8) are next written by the host after
    // the cycle's final synchronize, and the chunk read-backs into ch are ordered
    // after the upload on the stream
    K->skip = K->ctl.p + kStop;
    s->skip = K->skip;
    int k = 0, chunk = 0;
    bool stopped = false;
    while (k < m && !stopped) {
      const int k1 = std::min(m, k + kAhead);
      for (; k < k1; ++k) {
        double* Vk = V + (size_t)k * n;
        if (tr.on) tr.mark(st, 0);
        MH_CHECK(apply_MA(A, M, MA, Vk, K->w.p, K->tmp.p));
        if (tr.on) tr.mark(st, 1);
        if (multi) MH_CHECK(enqueue_cgs2(st, K, n, k));  // two collectives per step
        else if (use_graphs) MH_CHECK(run_mgs(st, K, n, k));
        else MH_CHECK(enqueue_mgs(st, K, n, k, false, fused));
        if (tr.on) tr.mark(st, 2);
        if (!fused) {
          givens_kernel<<<1, 32, 0, st>>>(K->hcol.p, gvh, k);
          MH_CHECK_CUDA(cudaGetLastError());
        }
        if (tr.on) tr.mark(st, 3);
      }
      const int slot = chunk & 1;
      MH_CHECK_CUDA(cudaMemcpyAsync(ch + 8 * slot, K->ctl.p, sizeof(int) * kCtlInts,
                                    cudaMemcpyDeviceToHost, st));
      MH_CHECK_CUDA(cudaEventRecord(ev[slot], st));
      if (chunk > 0) {  // the previous chunk's control block, while this one runs
        MH_CHECK_CUDA(cudaEventSynchronize(ev[slot ^ 1]));
        stopped = ch[8 * (slot ^ 1) + kStop] != 0;
      }
      ++chunk;
    }
    MH_CHECK_CUDA(cudaStreamSynchronize(st));
    s->skip = nullptr;
    K->skip = nullptr;
    // the cycle's outcome to the host
    MH_CHECK_CUDA(cudaMemcpy(ch, K->ctl.p, sizeof(int) * kCtlInts, cudaMemcpyDeviceToHost));
    const int k_used = ch[kKUsed], steps = ch[kSteps];
    it = ch[kIt];
    conv = ch[kConv] != 0;
    const bool breakdown = ch[kBreak] != 0;
    if (steps > 0) {
      MH_CHECK_CUDA(cudaMemcpy(hist.data(), K->histd.p, sizeof(double) * steps, cudaMemcpyDeviceToHost));
      history.insert(history.end(), hist.begin(), hist.begin() + steps);
    }
    if (k_used > 0) {
      MH_CHECK_CUDA(cudaMemcpy(H.data(), K->Hd.p, sizeof(double) * (size_t)(m + 1) * m,
                               cudaMemcpyDeviceToHost));
      MH_CHECK_CUDA(cudaMemcpy(g.data(), K->gd.p, sizeof(double) * (m + 1), cudaMemcpyDeviceToHost));
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
      x_zero = false;
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
  MH_CHECK(K.part.alloc(kDotPartsMax));
  MH_CHECK(K.ticket.alloc(1));
  MH_CHECK(K.scal.alloc(1));
  MH_CHECK_CUDA(cudaMemsetAsync(K.ticket.p, 0, sizeof(unsigned), st));
  dot_kernel<<<dot_parts(n) / kDotWarps, kDotWarps * 32, 0, st>>>(
      n, const_cast<double*>(x), nullptr, nullptr, y, 0, true, K.part.p, K.ticket.p, K.scal.p,
      nullptr);
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
  if (restart > kMaxRestartSmem)  // beyond the device Givens' staging: the host loop
    return gmres_core(s->stream, s->kry, n, A, M, MA, tol, restart, maxiter, rhs, x, iterations,
                      converged, hist_host, hist_cap, hist_len);
  return gmres_pipelined(s, s->stream, s->kry, n, A, M, MA, tol, restart, maxiter, rhs, x,
                         iterations, converged, hist_host, hist_cap, hist_len);
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
