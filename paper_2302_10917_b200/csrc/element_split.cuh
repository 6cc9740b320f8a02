// Element kernel, apply mode, one macro per CTA: the macro's rows are split over
// G consumer warps (warp g owns rows 32 g .. 32 g + 31), fed by one shared TMA
// ring (stream.cuh) that a producer warp keeps full.  Included by element.cu.
//
// Why: with one warp per macro (element_kernel) 12 macros per SM are in flight,
// and when op.C = op.B^T (one array, read in step 1 and again in step 3) their
// B blocks — 12 x 148 x 8 nc Q bytes: 133 MB at c3, 422 MB at c5, 687 MB at c4 —
// do not stay in L2 between the two reads: the kernel moves 1.3-1.5x its
// algorithmic bytes.  Here 2-6 macros per SM are in flight (c5: 70-105 MB).
//
// Per macro (same arithmetic as element_kernel; y is bitwise the same, v differs
// in the order of the final sums):
//   step 1   x_i = sum_c B^T[c][perm_i] ue_c        every warp its 32 rows
//   step 2a  forward substitution by 32-column blocks: the owner warp of block
//            jb solves its 32 x 32 triangle with shuffles, publishes the 32 values
//            through shared memory (mbarrier xf[jb]); the warps below apply the
//            block's columns to their rows
//   step 2b  back substitution the same way, blocks descending (xb[jb])
//   step 3   v_c = sum_i C[c][i] y_i: per-warp partial sums (8 rows per
//            transpose-reduce) to shared memory, summed over the warps in order
// A warp always asks the ring for the range it needs next BEFORE it waits for
// another warp's values, so every chunk it does not need is handed back as soon
// as it has landed and the producer never waits on an idle warp.

template <int G, int RING, int CH>
struct SplitShape {
  static constexpr int S = RING / CH;
  static constexpr int kThreadsS = (G + 1) * 32;
  static size_t smem_bytes(int nc) {
    const int ncp = (nc + 3) & ~3;
    return (size_t)RING * sizeof(double) + (size_t)(2 * S + 2 * G) * sizeof(uint64_t) +
           (size_t)(2 * ncp + 2 * 32 * G + G * ncp) * sizeof(double);
  }
};

#ifdef MH_SPLIT_TRACE
// clock64 stamps of CTA 0's third macro, per consumer warp: start, step 1 done,
// forward done, backward done, step 3 done, macro done
__device__ long long g_split_trace[8 * 8];
#define MH_ST(slot) \
  if (blockIdx.x == 0 && it == 2 && lane == 0) g_split_trace[g * 8 + (slot)] = clock64();
#else
#define MH_ST(slot)
#endif

template <int G>
__device__ __forceinline__ void bar_consumers() {
  asm volatile("bar.sync 1, %0;" ::"n"(G * 32) : "memory");
}

template <int G, int RING, int CH>
__global__ void __launch_bounds__((G + 1) * 32) element_split_kernel(ElemArgs a) {
  if (a.skip && *a.skip) return;
  constexpr int S = RING / CH;
  static_assert((RING & (RING - 1)) == 0, "ring size must be a power of two");
  using PipeT = Pipe<RING, CH, 1>;
  using ConsT = Consumer<RING, CH>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ Segment segs[4];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int Q = a.Q, nc = a.nc, t = a.t;
  const int ncp = (nc + 3) & ~3;
  const int nchB = (int)(a.ldB / CH), nchL = (int)(a.ldL / CH);
  double* ring = reinterpret_cast<double*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + RING);
  uint64_t* empty = full + S;
  uint64_t* xf = empty + S;  // forward block jb published
  uint64_t* xb = xf + G;     // backward block jb published
  double* su_all = reinterpret_cast<double*>(xb + G);  // gathered uhat, two buffers
  double* yf = su_all + 2 * ncp;                        // published forward values
  double* yb = yf + 32 * G;                             // published backward values
  double* part = yb + 32 * G;                           // step 3 partial sums [G][ncp]
  if (threadIdx.x == 0) {
    segs[0] = Segment{a.Bt, a.ldB, nchB, a.c_is_bt ? a.bpol : 0};
    segs[1] = Segment{a.Lp, a.ldL, nchL, a.lpol};
    segs[2] = Segment{a.Up, a.ldL, nchL, a.lpol};
    segs[3] = Segment{a.Cm, a.ldB, nchB, 0};
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], G);
    }
    for (int i = 0; i < 2 * G; ++i) mbar_init(&xf[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t W = gridDim.x;
  const int64_t e_first = a.e_lo + blockIdx.x;
  if (g == G) {  // producer warp
    if (lane == 0) PipeT::produce(ring, full, empty, segs, 4, e_first, W, a.N, 1);
    return;
  }
  ConsT cs;
  cs.full = full;
  cs.empty = empty;
  const uint32_t offL = (uint32_t)a.ldB;
  const uint32_t offU = offL + (uint32_t)a.ldL;
  const uint32_t offC = offU + (uint32_t)a.ldL;
  const uint32_t E = offC + (uint32_t)a.ldB;
  const int i = 32 * g + lane;  // this lane's row
  const bool valid = i < Q;
  const int tid = threadIdx.x;  // among the consumers: 0 .. 32 G - 1
  constexpr int KG = (256 + 32 * G - 1) / (32 * G);  // gathered slot values per lane

  // the next macro's small vectors are loaded while this one is processed
  int pr_n = i;
  double dr_n = 0.0;
  int32_t ef_n[kMaxSlots];
  double g_n[KG];
  auto load_meta = [&](int64_t en) {
    pr_n = valid ? __ldg(a.perm + en * Q + i) : i;
    dr_n = valid ? __ldg(a.dinv + en * Q + i) : 0.0;
#pragma unroll
    for (int k = 0; k < kMaxSlots; ++k)
      ef_n[k] = k < a.nfe ? __ldg(a.elem_ufac + en * a.nfe + k) : -1;
  };
  auto gather_next = [&]() {
#pragma unroll
    for (int qq = 0; qq < KG; ++qq) {
      const int c = tid + 32 * G * qq;
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
      g_n[qq] = v;
    }
  };
  auto store_su = [&](double* su) {
#pragma unroll
    for (int qq = 0; qq < KG; ++qq) {
      const int c = tid + 32 * G * qq;
      if (c < nc) su[c] = g_n[qq];
    }
  };
  if (e_first < a.N) {
    load_meta(e_first);
    gather_next();
    store_su(su_all);
  }
  bar_consumers<G>();

  uint32_t base = 0;
  int it = 0;
  for (int64_t e = e_first; e < a.N; e += W, base += E, ++it) {
    const uint32_t phase = it & 1;
    const double* su = su_all + (it & 1) * ncp;
    const int pr = pr_n;
    const double dr = dr_n;
    const int64_t en = e + W;
    if (en < a.N) load_meta(en);  // lands while this macro is processed
    MH_ST(0)
    // ---- step 1: x = P (B ue), 8 rows of op.B^T per ring-window check
    double y = 0.0;
    {
      uint32_t p = base;
      int c = 0;
      for (; c + 8 <= nc; c += 8, p += 8u * (uint32_t)Q) {
        cs.window(p, p + 8u * (uint32_t)Q, lane);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double b = ring[rmod<RING>(p + (uint32_t)(u * Q + pr))];
          if (valid) y = fma(b, su[c + u], y);
        }
      }
      for (; c < nc; ++c, p += (uint32_t)Q) {
        cs.window(p, p + (uint32_t)Q, lane);
        const double b = ring[rmod<RING>(p + (uint32_t)pr)];
        if (valid) y = fma(b, su[c], y);
      }
    }
    MH_ST(1)
    if (en < a.N) gather_next();  // its face table arrived during step 1

    // ---- step 2a: unit-lower forward substitution, packed L columns 0 .. Q-2
    {
      uint32_t p = base + offL;
#pragma unroll
      for (int jb = 0; jb < G; ++jb) {
        const int jbeg = 32 * jb, jend = min(jbeg + 32, Q - 1);
        if (jbeg >= jend) break;
        const int ncols = jend - jbeg;
        // doubles of the block's columns: sum over j of (Q - 1 - j)
        const uint32_t blk = (uint32_t)(ncols * (Q - 1 - jbeg) - ncols * (ncols - 1) / 2);
        if (g < jb) {  // rows above the block: nothing to do
          p += blk;
          continue;
        }
        if (g > jb) {  // ask for the first columns, then wait for the owner's values
          cs.window(p, p + (uint32_t)(min(8, ncols) * (Q - 1 - jbeg)), lane);
          while (!mbar_try_wait(&xf[jb], phase)) {
          }
        }
        for (int j0 = jbeg; j0 < jend; j0 += 8) {
          const int n8 = min(8, jend - j0);
          const uint32_t span = (uint32_t)(n8 * (Q - 1 - j0) - n8 * (n8 - 1) / 2);
          cs.window(p, p + span, lane);
          if (g == jb) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              if (u < n8) {
                const int j = j0 + u;
                const double yj = __shfl_sync(kFull, y, j & 31);
                const double l = ring[rmod<RING>(p - (uint32_t)(j + 1) + (uint32_t)i)];
                if (valid && lane > (j & 31)) y = fma(-l, yj, y);
                p += (uint32_t)(Q - 1 - j);
              }
            }
          } else {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              if (u < n8) {
                const int j = j0 + u;
                const double yj = yf[j];
                const double l = ring[rmod<RING>(p - (uint32_t)(j + 1) + (uint32_t)i)];
                if (valid) y = fma(-l, yj, y);
                p += (uint32_t)(Q - 1 - j);
              }
            }
          }
        }
        if (g == jb) {
          yf[i] = y;
          __threadfence_block();
          __syncwarp();
          if (lane == 0) mbar_arrive(&xf[jb]);
        }
      }
      // the owner of a block without L columns (the last row group when Q - 1 is
      // a multiple of 32) still completes its barrier: nobody waits for it
#pragma unroll
      for (int jb = 0; jb < G; ++jb)
        if (g == jb && 32 * jb >= Q - 1 && lane == 0) mbar_arrive(&xf[jb]);
    }
    MH_ST(2)
    // ---- step 2b: upper back substitution, packed U columns Q-1 .. 0
    {
      uint32_t p = base + offU;
#pragma unroll
      for (int jb = G - 1; jb >= 0; --jb) {
        const int jlo = 32 * jb, jhi = min(jlo + 31, Q - 1);
        if (jlo > jhi) continue;  // no rows in this group
        const int ncols = jhi - jlo + 1;
        // doubles of the block's columns: sum over j of j
        const uint32_t blk = (uint32_t)(ncols * jhi - ncols * (ncols - 1) / 2);
        if (g > jb) {  // rows below the block: nothing to do
          p += blk;
          continue;
        }
        if (g < jb) {
          cs.window(p, p + (uint32_t)(min(8, ncols) * jhi), lane);
          while (!mbar_try_wait(&xb[jb], phase)) {
          }
        }
        for (int j0 = jhi; j0 >= jlo; j0 -= 8) {
          const int n8 = min(8, j0 - jlo + 1);
          const uint32_t span = (uint32_t)(n8 * j0 - n8 * (n8 - 1) / 2);
          cs.window(p, p + span, lane);
          if (g == jb) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              if (u < n8) {
                const int j = j0 - u;
                if (lane == (j & 31)) y *= dr;
                const double yj = __shfl_sync(kFull, y, j & 31);
                const double uv = ring[rmod<RING>(p + (uint32_t)i)];
                if (lane < (j & 31)) y = fma(-uv, yj, y);
                p += (uint32_t)j;
              }
            }
          } else {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              if (u < n8) {
                const int j = j0 - u;
                const double yj = yb[j];
                const double uv = ring[rmod<RING>(p + (uint32_t)i)];
                y = fma(-uv, yj, y);
                p += (uint32_t)j;
              }
            }
          }
        }
        if (g == jb) {
          yb[i] = y;
          __threadfence_block();
          __syncwarp();
          if (lane == 0) mbar_arrive(&xb[jb]);
        }
      }
#pragma unroll
      for (int jb = 0; jb < G; ++jb)
        if (g == jb && 32 * jb > Q - 1 && lane == 0) mbar_arrive(&xb[jb]);
    }

    MH_ST(3)
    // ---- step 3: v_c = sum_i C[c][i] y_i: this warp's 32 rows, 8 rows of op.C
    //      per transpose-reduce
    {
      uint32_t p = base + offC;
      for (int c0 = 0; c0 < nc; c0 += 8) {
        const int nrow = min(8, nc - c0);
        cs.window(p, p + (uint32_t)(nrow * Q), lane);
        double pp[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double cv = ring[rmod<RING>(p + (uint32_t)(u * Q + i))];
          pp[u] = (valid && u < nrow) ? cv * y : 0.0;
        }
        p += (uint32_t)(nrow * Q);
        const double v = transpose_reduce8(pp, lane);
        const int row = (lane >> 2) & 7;
        if ((lane & 3) == 0 && row < nrow) part[g * ncp + c0 + row] = v;
      }
    }
    MH_ST(4)
    bar_consumers<G>();  // every warp's partial sums are in
    for (int c = tid; c < nc; c += 32 * G) {
      double v = part[c];
#pragma unroll
      for (int gg = 1; gg < G; ++gg) v += part[gg * ncp + c];
      a.out[e * nc + c] = v;
    }
    if (en < a.N) store_su(su_all + ((it + 1) & 1) * ncp);
    bar_consumers<G>();  // part / su / yf / yb may be reused
    MH_ST(5)
  }
}

#ifdef MH_SPLIT_TRACE
#define MH_SPLIT_DUMP(G_, R_, P_)                                                               \
  {                                                                                             \
    static int dumped = 0;                                                                      \
    if (dumped++ == 3) {                                                                        \
      cudaStreamSynchronize(st);                                                                \
      long long tr[64];                                                                         \
      cudaMemcpyFromSymbol(tr, g_split_trace, sizeof(tr));                                      \
      fprintf(stderr, "split trace G=%d RING=%d CTAs/SM=%d: warp | step1 fwd bwd step3 end\n", \
              G_, R_, P_);                                                                      \
      for (int w = 0; w < G_; ++w)                                                              \
        fprintf(stderr, "%d | %lld %lld %lld %lld %lld\n", w, tr[w * 8 + 1] - tr[w * 8],       \
                tr[w * 8 + 2] - tr[w * 8], tr[w * 8 + 3] - tr[w * 8], tr[w * 8 + 4] - tr[w * 8], \
                tr[w * 8 + 5] - tr[w * 8]);                                                     \
    }                                                                                           \
  }
#else
#define MH_SPLIT_DUMP(G_, R_, P_)
#endif

template <int G>
int launch_split_g(mh_system* s, const ElemArgs& a, cudaStream_t st) {
  // ring: the warps that wait for a block's values hold the ring at the block's
  // first column while its owner reads through the last one: a 32-column block
  // (at most 32 (Q - 1) - 496 doubles) plus chunk rounding, as a power of two
  constexpr int CH = 512;
  const int need = 32 * (s->Q - 1) - 496 + 3 * CH;
  const int64_t work = a.N - a.e_lo;
#define MH_SPLIT(RING_)                                                                         \
  if (need <= RING_) {                                                                          \
    using Sh = SplitShape<G, RING_, CH>;                                                        \
    auto kern = element_split_kernel<G, RING_, CH>;                                             \
    const size_t smem = Sh::smem_bytes(s->nc);                                                  \
    int per_sm = launch_occupancy(s->device, reinterpret_cast<const void*>(kern),               \
                                  Sh::kThreadsS, smem);                                         \
    if (per_sm < 0) return MH_E_CUDA;                                                           \
    if (per_sm < 1) per_sm = 1;                                                                 \
    /* macros in flight: their B blocks (8 nc Q bytes each) are to stay in L2 */              \
    const int cap = s->knobs.elem_split_ctas > 0                                                \
                        ? s->knobs.elem_split_ctas                                              \
                        : (int)(100e6 / ((double)s->num_sms * 8.0 * s->nc * s->Q));             \
    per_sm = std::max(1, std::min(per_sm, cap));                                                \
    const int64_t grid = std::min<int64_t>(work, (int64_t)s->num_sms * per_sm);                 \
    kern<<<(unsigned)grid, Sh::kThreadsS, smem, st>>>(a);                                        \
    MH_CHECK_CUDA(cudaGetLastError());                                                          \
    MH_SPLIT_DUMP(G, RING_, per_sm)                                                             \
    return MH_OK;                                                                               \
  }
  MH_SPLIT(4096) MH_SPLIT(8192) MH_SPLIT(16384)
#undef MH_SPLIT
  set_error("split element kernel: ring too small");
  return MH_E_UNSUPPORTED;
}

// apply mode with the macro split over its row groups (3 <= ceil(Q / 32) <= 8)
int launch_split(mh_system* s, const ElemArgs& a, cudaStream_t st) {
  switch ((s->Q + 31) / 32) {
    case 3: return launch_split_g<3>(s, a, st);
    case 4: return launch_split_g<4>(s, a, st);
    case 5: return launch_split_g<5>(s, a, st);
    case 6: return launch_split_g<6>(s, a, st);
    case 7: return launch_split_g<7>(s, a, st);
    case 8: return launch_split_g<8>(s, a, st);
  }
  set_error("split element kernel: 64 < Q <= 256");
  return MH_E_UNSUPPORTED;
}
