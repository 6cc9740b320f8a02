// Batched fp64 LU, one CTA per block: panels pipelined over update warps, the
// panel-to-panel chain on dedicated factor warps, L tiles in shared memory,
// DMMA updates.
//
// Replaces _factorize_local's dense branch (schur_solver.py:105-111) like the
// other LU kernels; same outputs (packed L / U streams, diag(U), 1/U_jj, LAPACK
// pivots, row permutation, status), bitwise the tile kernel's (lu_tile.cu): every
// element sees the same sequence of operations, only who runs them and where L
// lives changes.
//
// Left-looking by panels of 8 columns, as lu_tile.cu.  What the measurements on
// B200 say (tools/lat_probe.cu, the MH_PIPE_TRACE build): one warp issues a
// dependent-free DFMA only every ~10 cycles and a DMMA.8x8x4 every ~27, so a
// panel factored by ONE warp costs ~7-10k cycles and everything else waits for
// it.  Hence the split:
//  * update warps (4 .. W-1) own panels round-robin.  A panel lives in its warp's
//    registers (NT tiles in the DMMA C-fragment layout).  The warp gathers the
//    panel's columns of A and applies the earlier panels kb as they are
//    published: -U_kb = (-L11(kb)^-1) T_kb, T_t += L(t, kb) (-U_kb), the A
//    fragments coming from shared memory with one 16-byte load per lane (the
//    tile kernel reads them from a per-warp scratch slot in L2 / HBM).  After
//    the newest panel it hands the diagonal tile over first, then the rows
//    below (staged in the panel's own, not yet published, tile column).
//  * factor warp 0 factors the 8 x 8 diagonal tile in the C-fragment layout
//    (two elements per lane; per column one pivot shuffle, the reciprocal, one
//    shuffle of the scaled column, two FMAs), publishes U11, the reciprocals and
//    -L11^-1;
//  * factor warps 0..3 then run the rows below the diagonal block, one or two
//    rows per lane, through the row form of the same elimination,
//        x_c <- x_c - sum_{m < c} l_m U_mc  (m ascending),  l_c = x_c / U_cc,
//    write the panel's L tiles in A-fragment order and publish the panel.
//
// Pivoting: the diagonal is kept as pivot and LAPACK's rule is checked on the
// same intermediate values — idamax takes the first row of maximum |a|, so the
// diagonal stays exactly when no row below is strictly larger.  A block that
// needs a row exchange is handed back (its index is appended to a list) and
// factored by lu_tile_kernel, which does the exchanges; the BASELINE blocks
// (A + Q I) never do.
//
// Shared memory: NT (NT - 1) / 2 tiles of 512 bytes plus 256 bytes of staging pad
// per panel, NT inverse diagonal blocks (Q = 91: 41 KB; Q = 165: 119 KB;
// Q = 220: 216 KB, one CTA per SM).

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "lu_tile_common.cuh"
#include "stream.cuh"

namespace mh {
namespace {

constexpr int kNF = 4;  // factor warps (warps 0..3: one per SM sub-partition)

template <int NT>
struct PipeShape {
  static constexpr int R = (NT + 3) / 4;    // 32-row groups of a full-height panel
  static constexpr int AA = (R + kNF - 1) / kNF;  // row groups per factor warp (1 or 2)
  // tile column kb: tiles (kb + 1 .. NT - 1, kb), then 32 doubles of staging pad
  static constexpr int col_base(int kb) { return kb * ((NT - 1) * 64 + 32) - 32 * kb * (kb - 1); }
  static constexpr int kTileDoubles = NT * ((NT - 1) * 64 + 32) - 32 * NT * (NT - 1);
  static constexpr int kInvDoubles = NT * 64;      // -L11^-1 per panel
  static constexpr int kDiagDoubles = 2 * 96;      // two diagonal-block slots: 8 x 8, rc, mode
  static constexpr int kBars = 4 * NT;             // pub, staged, dstaged, ddone
  static constexpr int kCtlInts = 16;
  static constexpr size_t smem_bytes() {
    return (size_t)(kTileDoubles + kInvDoubles + kDiagDoubles + 64 + kBars) * sizeof(double) +
           kCtlInts * sizeof(int);
  }
};

#ifdef MH_PIPE_TRACE
// phase stamps (clock64) of the panels of CTA 0's second block
__device__ long long g_pipe_trace[64 * 8];
#define MH_TR(slot) \
  if (tracing && lane == 0) g_pipe_trace[jb * 8 + (slot)] = clock64();
#else
#define MH_TR(slot)
#endif

// control words in shared memory
enum { kBail = 1, kAmh = 2 /* 2 slots */, kDmin = 4 /* 2 slots x 2 ints */ };

// experiments: MH_PIPE_NOFENCE drops the explicit fences before the barrier
// arrivals (mbarrier.arrive is a release at CTA scope), MH_PIPE_POLL polls with
// test_wait instead of the suspending try_wait
#ifdef MH_PIPE_NOFENCE
#define MH_FENCE()
#else
#define MH_FENCE() __threadfence_block()
#endif
__device__ __forceinline__ void pipe_wait(uint64_t* bar, uint32_t phase) {
#ifdef MH_PIPE_POLL
  while (!mbar_test_wait(bar, phase)) {
  }
#else
  while (!mbar_try_wait(bar, phase)) {
  }
#endif
}

__device__ __forceinline__ void bar_factor_warps() {
  asm volatile("bar.sync 1, %0;" ::"n"(kNF * 32) : "memory");
}

template <int NT, int W, int MINB>
__global__ void __launch_bounds__(W * 32, MINB)
    lu_pipe_kernel(LuArgs g, int a_pol, int* __restrict__ fb_count, int64_t* __restrict__ fb_list) {
  using S = PipeShape<NT>;
  constexpr int AA = S::AA;
  constexpr int NU = W - kNF;
  extern __shared__ double smem_pipe[];
  double* Lt = smem_pipe;
  double* invs = Lt + S::kTileDoubles;
  double* dslots = invs + S::kInvDoubles;
  double* stg = dslots + S::kDiagDoubles;  // spare 8 x 8
  // mbarriers, each completed once per block (so the phase a waiter tests is the
  // CTA's block count modulo 2)
  uint64_t* pub = reinterpret_cast<uint64_t*>(stg + 64);  // panel's tiles + inverse published
  uint64_t* staged = pub + NT;      // rows below the diagonal block are staged
  uint64_t* dstaged = staged + NT;  // the diagonal tile is staged
  uint64_t* ddone = dstaged + NT;   // the diagonal block is factored
  int* ctl = reinterpret_cast<int*>(ddone + NT);
  volatile int* vctl = ctl;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = lane >> 2, q = lane & 3;
  const int Q = g.Q;
  const int npanel = (Q + 7) / 8;
  const uint64_t pol = policy_evict_first();
  const uint64_t apol = make_policy(a_pol ? 2 : 0);

  if (threadIdx.x == 0) {
    for (int k = 0; k < NT; ++k) {
      mbar_init(&pub[k], kNF);
      mbar_init(&staged[k], 1);
      mbar_init(&dstaged[k], 1);
      mbar_init(&ddone[k], 1);
    }
    fence_mbar_init();
    ctl[kBail] = 0;
    ctl[kAmh] = ctl[kAmh + 1] = 0;
    *reinterpret_cast<unsigned long long*>(ctl + kDmin) = ~0ull;
    *reinterpret_cast<unsigned long long*>(ctl + kDmin + 2) = ~0ull;
  }
  __syncthreads();

  int it = 0;  // blocks this CTA has started
  for (int64_t e = blockIdx.x; e < g.nblocks; e += gridDim.x, ++it) {
    const double* __restrict__ Ae = g.A + e * (int64_t)Q * Q;
    double* Lpe = g.Lp + e * g.ldL;
    double* Upe = g.Up + e * g.ldL;
    const uint32_t phase = it & 1;
    unsigned amh = 0;          // max over the warp's panels of the high word of |a_ij|
    double dmin = DBL_MAX;
#ifdef MH_PIPE_TRACE
    const bool tracing = blockIdx.x == 0 && it == 1;
#endif
    // A block that was handed back (row exchanges) keeps its barrier protocol —
    // every barrier completes exactly once per block — but skips the work; tiles
    // read in between may be stale, which only feeds results nobody keeps.

    if (w >= kNF) {
      // ================= update warp: panels u, u + NU, ...
      for (int jb = w - kNF; jb < npanel; jb += NU) {
        MH_TR(0)
        const bool dead = vctl[kBail] == it + 1;
        const int c0 = 8 * jb;
        const int ca = c0 + 2 * q;
        const bool v0 = ca < Q, v1 = ca + 1 < Q;
        // ---- 1. the panel's columns of A (C-fragment layout)
        double T[NT][2];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int pos = 8 * t + r;
          const bool vr = pos < Q && !dead;
          const double* src = Ae + (vr ? pos : 0) * Q + ca;
          T[t][0] = (vr && v0) ? ld_a(src, apol) : 0.0;
          T[t][1] = (vr && v1) ? ld_a(src + 1, apol) : 0.0;
          amh = max(amh, max(hi_abs(T[t][0]), hi_abs(T[t][1])));
        }
        // ---- 2. updates with the earlier panels as they are published
        {
          double* U0 = Upe + ou32(v0 ? ca : 0, Q) + r;
          double* U1 = Upe + ou32(v1 ? ca + 1 : 0, Q) + r;
#pragma unroll
          for (int kb = 0; kb < NT - 1; ++kb) {
            if (kb >= jb) break;
            pipe_wait(&pub[kb], phase);
            MH_TR(1)
            if (dead) continue;
            const double2* tl = reinterpret_cast<const double2*>(Lt + S::col_base(kb)) + lane;
            const double2 li = *(reinterpret_cast<const double2*>(invs + kb * 64) + lane);
            double u0 = 0.0, u1 = 0.0;  // -U_kb (C layout)
            dmma_acc(u0, u1, li.x, bfrag(T[kb][0], T[kb][1], 0, lane));
            dmma_acc(u0, u1, li.y, bfrag(T[kb][0], T[kb][1], 1, lane));
            const double ub0 = bfrag(u0, u1, 0, lane), ub1 = bfrag(u0, u1, 1, lane);
#pragma unroll
            for (int t = kb + 1; t < NT; ++t) {
              if (8 * t >= Q) break;  // padding tiles (NT rounded up)
              const double2 lf = tl[(t - kb - 1) * 32];
              dmma_acc(T[t][0], T[t][1], lf.x, ub0);
              dmma_acc(T[t][0], T[t][1], lf.y, ub1);
              if (t == kb + 1 && kb + 1 == jb) {
                // the diagonal tile is complete: hand it to factor warp 0 first
                double* ds = dslots + (jb & 1) * 96;
                ds[(2 * q) * 8 + r] = T[t][0];
                ds[(2 * q + 1) * 8 + r] = T[t][1];
                MH_FENCE();
                __syncwarp();
                if (lane == 0) mbar_arrive(&dstaged[jb]);
                MH_TR(2)
              }
            }
            if (v0) st_first(U0 + 8 * kb, -u0, pol);
            if (v1) st_first(U1 + 8 * kb, -u1, pol);
          }
        }
        if (jb == 0 || dead) {  // no update ran: the diagonal tile is A's (or nobody's)
          double* ds = dslots + (jb & 1) * 96;
          ds[(2 * q) * 8 + r] = T[0][0];
          ds[(2 * q + 1) * 8 + r] = T[0][1];
          MH_FENCE();
          __syncwarp();
          if (lane == 0) mbar_arrive(&dstaged[jb]);
          MH_TR(2)
        }
        // ---- 3. rows below the diagonal block to the row layout (column-major,
        //         stride ld = 4 mod 8: conflict-free both ways), staged in the
        //         panel's own tile column
        double* col = Lt + S::col_base(jb);
        const int ld = 8 * (NT - 1 - jb) + 4;
#pragma unroll
        for (int t = 1; t < NT; ++t) {
          if (t > jb) {
            col[(2 * q) * ld + 8 * (t - jb - 1) + r] = T[t][0];
            col[(2 * q + 1) * ld + 8 * (t - jb - 1) + r] = T[t][1];
          }
        }
        MH_FENCE();
        __syncwarp();
        if (lane == 0) mbar_arrive(&staged[jb]);
        MH_TR(3)
      }
    } else {
      // ================= factor warps 0 .. 3
      for (int jb = 0; jb < npanel; ++jb) {
        const bool dead = vctl[kBail] == it + 1;
        const int c0 = 8 * jb;
        const int ncol = min(8, Q - c0);
        const int nrel = Q - c0 - 8;  // rows below the diagonal block
        double* ds = dslots + (jb & 1) * 96;
        double* col = Lt + S::col_base(jb);
        const int ld = 8 * (NT - 1 - jb) + 4;
        bool ok = true;
        double x0 = 0.0, x1 = 0.0;  // warp 0: the diagonal tile (C layout)
        double rc[8];
        int mode[8];
        if (w == 0) {
          // ---- the diagonal block: the chain's serial part
          pipe_wait(&dstaged[jb], phase);
          if (!dead) {
            x0 = ds[(2 * q) * 8 + r];
            x1 = ds[(2 * q + 1) * 8 + r];
            __syncwarp();
            ok = factor_diag_tile(x0, x1, rc, mode, ncol, lane, dmin);
            ds[(2 * q) * 8 + r] = x0;
            ds[(2 * q + 1) * 8 + r] = x1;
            if (lane < 8) {
              double rv = rc[0];
              int mv = mode[0];
#pragma unroll
              for (int j = 1; j < 8; ++j) {
                rv = lane == j ? rc[j] : rv;
                mv = lane == j ? mode[j] : mv;
              }
              ds[64 + lane] = rv;
              ds[72 + lane] = (double)mv;
            }
            __syncwarp();
            if (jb + 1 < npanel) neg_linv<8>(ds, invs + jb * 64, lane);
          }
          MH_FENCE();
          __syncwarp();
          if (lane == 0) mbar_arrive(&ddone[jb]);
          MH_TR(4)
        }
        // ---- the rows below: every factor warp its row groups a = w, w + 4
        pipe_wait(&staged[jb], phase);
        pipe_wait(&ddone[jb], phase);
        double P[8][AA];
        double D[8][8];  // U on and above the diagonal: D[c][m], m <= c
        if (!dead) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
#pragma unroll
            for (int m = 0; m <= c; m += 2) {
              const double2 v = *reinterpret_cast<const double2*>(ds + c * 8 + m);
              D[c][m] = v.x;
              if (m + 1 < 8) D[c][m + 1] = v.y;
            }
            if (w != 0) {
              rc[c] = ds[64 + c];
              mode[c] = (int)ds[72 + c];
            }
          }
#pragma unroll
          for (int c = 0; c < 8; ++c)
#pragma unroll
            for (int a = 0; a < AA; ++a) {
              const int rel = lane + 32 * (w + kNF * a);
              P[c][a] = rel < nrel ? col[c * ld + rel] : 0.0;
            }
        }
        // the tiles go where the staged rows are: everyone loads before anyone writes
        // (unconditional: the factor warps may see the hand-back flag at different panels)
        bar_factor_warps();
        if (!dead) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
#pragma unroll
            for (int m = 0; m < c; ++m)
#pragma unroll
              for (int a = 0; a < AA; ++a) P[c][a] = fma(-P[m][a], D[c][m], P[c][a]);
#pragma unroll
            for (int a = 0; a < AA; ++a) {
              double x = P[c][a];
              if (fabs(x) > fabs(D[c][c])) ok = false;
              if (mode[c] == 1) x *= rc[c];
              else if (mode[c] == 2) x = slow_div(x, D[c][c]);
              P[c][a] = x;
            }
          }
          ok = __all_sync(kFull, ok);
          if (!ok && lane == 0) vctl[kBail] = it + 1;
          // ---- the panel's L tiles to shared memory (A-fragment order)
          if (jb + 1 < npanel) {
#pragma unroll
            for (int a = 0; a < AA; ++a) {
              const int rel = lane + 32 * (w + kNF * a);
              if (rel < 8 * (NT - 1 - jb)) {
                double2* dst = reinterpret_cast<double2*>(col + (rel >> 3) * 64) + 4 * (rel & 7);
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) dst[qq] = make_double2(P[qq][a], P[4 + qq][a]);
              }
            }
          }
        }
        MH_FENCE();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pub[jb]);  // release: the tiles are visible to the waiters
        MH_TR(5)
        if (dead) continue;
        // ---- the packed streams, off the panel-to-panel chain
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (c >= ncol) break;
          const int j = c0 + c;
          double* lcol = Lpe + (ol32(j, Q) - c - 1) + 8;  // + rel (row c0 + 8 + rel)
#pragma unroll
          for (int a = 0; a < AA; ++a) {
            const int rel = lane + 32 * (w + kNF * a);
            if (rel < nrel) st_first(lcol + rel, P[c][a], pol);
          }
        }
        if (w == 0) {
          // the diagonal block: lane (i, q) holds row i, columns 2q and 2q + 1
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = 2 * q + h, j = c0 + c;
            const double v = h ? x1 : x0;
            if (c < ncol && r < ncol) {
              if (r > c) st_first(Lpe + (ol32(j, Q) - c - 1) + r, v, pol);
              else if (r < c) st_first(Upe + ou32(j, Q) + c0 + r, v, pol);
              else {
                double rv = rc[0];
#pragma unroll
                for (int jj = 1; jj < 8; ++jj) rv = c == jj ? rc[jj] : rv;
                g.piv[e * Q + j] = j;
                g.udiag[e * Q + j] = v;
                g.dinv[e * Q + j] = rv;
              }
            }
          }
        }
      }
    }

    // ---- the block's status: max |a| and min |u_jj| over the warps
    const int slot = it & 1;
    amh = __reduce_max_sync(kFull, amh);
    if (lane == 0) {
      atomicMax(reinterpret_cast<unsigned*>(ctl + kAmh + slot), amh);
      atomicMin(reinterpret_cast<unsigned long long*>(ctl + kDmin + 2 * slot),
                (unsigned long long)__double_as_longlong(dmin));
    }
    __syncthreads();  // every warp is done with the block's tiles
    const bool bailed = vctl[kBail] == it + 1;
    if (!bailed) {
      for (int64_t i = (int64_t)Q * (Q - 1) / 2 + threadIdx.x; i < g.ldL; i += W * 32) {
        Lpe[i] = 0.0;
        Upe[i] = 0.0;
      }
      for (int i = threadIdx.x; i < Q; i += W * 32) g.perm[e * Q + i] = i;
    }
    if (w == W - 1) {
      if (bailed) {
        if (lane == 0) fb_list[atomicAdd(fb_count, 1)] = e;
      } else {
        const unsigned a = (unsigned)vctl[kAmh + slot];
        const double d = __longlong_as_double(
            (long long)*reinterpret_cast<volatile unsigned long long*>(ctl + kDmin + 2 * slot));
        const int sing = singular_test(Ae, Q * Q, a, d, lane);
        if (lane == 0) g.stat[e] = sing;
      }
      __syncwarp();
      if (lane == 0) {  // the slot is used again two blocks on, past the next barrier
        ctl[kAmh + slot] = 0;
        *reinterpret_cast<unsigned long long*>(ctl + kDmin + 2 * slot) = ~0ull;
      }
    }
  }
}

template <int NT, int W>
int launch_pipe(mh_system* s, const LuArgs& g, cudaEvent_t start) {
  using S = PipeShape<NT>;
  constexpr size_t smem = S::smem_bytes();
  // resident CTAs the kernel is compiled for: what shared memory allows, within
  // 128 registers per thread at 16 warps per SM
  constexpr int kBySmem = (int)((227 * 1024) / (smem + 1024));
  constexpr int kByRegs = 16 / W < 1 ? 1 : 16 / W;
  constexpr int MINB = kBySmem < 1 ? 1 : (kBySmem > kByRegs ? kByRegs : kBySmem);
  auto kern = lu_pipe_kernel<NT, W, MINB>;
  if (smem > (size_t)s->max_smem_optin) {
    set_error("pipelined LU: block does not fit shared memory");
    return MH_E_UNSUPPORTED;
  }
  MH_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  MH_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W * 32, smem));
  per_sm = std::max(per_sm, 1);
  if (s->knobs.lu_pipe_ctas > 0) per_sm = std::min(per_sm, s->knobs.lu_pipe_ctas);
  const int64_t grid = std::min<int64_t>(g.nblocks, (int64_t)per_sm * s->num_sms);
  MH_CHECK(s->lu_fb.ensure((size_t)g.nblocks + 1));
  int64_t* fb = s->lu_fb.p;
  int* fb_count = reinterpret_cast<int*>(fb);  // word 0: the count; the list follows
  if (start) MH_CHECK_CUDA(cudaEventRecord(start, s->stream));
  MH_CHECK_CUDA(cudaMemsetAsync(fb, 0, sizeof(int64_t), s->stream));
  kern<<<(unsigned)grid, W * 32, smem, s->stream>>>(g, s->knobs.lu_a_pol, fb_count, fb + 1);
  MH_CHECK_CUDA(cudaGetLastError());
  // blocks that need row exchanges go through the tile kernel
  int nfb = 0;
  MH_CHECK_CUDA(cudaMemcpyAsync(&nfb, fb_count, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
  MH_CHECK_CUDA(cudaStreamSynchronize(s->stream));
  s->lu_fallback_blocks = nfb;
#ifdef MH_PIPE_TRACE
  {
    static long long tr[64 * 8];
    cudaMemcpyFromSymbol(tr, g_pipe_trace, sizeof(tr));
    fprintf(stderr, "pipe trace NT=%d W=%d: panel start lastpub diag-staged staged | diag-done published\n", NT, W);
    for (int jb = 0; jb < (g.Q + 7) / 8; ++jb)
      fprintf(stderr, "%2d %8lld %8lld %8lld %8lld | %8lld %8lld\n", jb, tr[jb * 8] - tr[0],
              tr[jb * 8 + 1] - tr[0], tr[jb * 8 + 2] - tr[0], tr[jb * 8 + 3] - tr[0],
              tr[jb * 8 + 4] - tr[0], tr[jb * 8 + 5] - tr[0]);
  }
#endif
  if (nfb > 0) MH_CHECK(launch_lu_tile(s, g, nullptr, fb + 1, fb_count, nfb));
  return MH_OK;
}

template <int NT>
int launch_pipe_w(mh_system* s, const LuArgs& g, cudaEvent_t start) {
  // warps per block: the four factor warps plus four update warps (255 registers
  // at one CTA per SM); eight update warps (MEHDG_LU_PIPE_W=12) spill and measured
  // slower at every BASELINE shape
  int W = 8;
  if (s->knobs.lu_pipe_w > 0) W = s->knobs.lu_pipe_w;
  if (W <= 8) return launch_pipe<NT, 8>(s, g, start);
  return launch_pipe<NT, 12>(s, g, start);
}

}  // namespace

// Q in 33..224 (NT = ceil(Q / 8) <= 28 tile rows fit shared memory)
bool lu_pipe_supported(int Q) { return Q > 32 && (Q + 7) / 8 <= 28; }

int launch_lu_pipe(mh_system* s, const LuArgs& g, cudaEvent_t start) {
  const int nt = (g.Q + 7) / 8;
#define MH_NT(N) \
  if (nt <= N) return launch_pipe_w<N>(s, g, start);
  MH_NT(6) MH_NT(8) MH_NT(11) MH_NT(12) MH_NT(16) MH_NT(21) MH_NT(24) MH_NT(28)
#undef MH_NT
  set_error("pipelined LU: Q > 224 unsupported");
  return MH_E_UNSUPPORTED;
}

}  // namespace mh
