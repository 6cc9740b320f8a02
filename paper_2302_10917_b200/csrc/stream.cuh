// Per-warp TMA bulk-copy stream: a warp consumes a long sequence of
// contiguous HBM segments through a shared-memory ring that its lane 0
// keeps full with cp.async.bulk (the 1-D TMA engine) and mbarrier
// completion.  Memory-level parallelism therefore does not depend on
// registers or on the compiler hoisting loads: up to S chunks of CH
// doubles are in flight per warp at all times.
//
// Stream positions are 32-bit (doubles).  The stream of a warp is the
// concatenation, over the macros it owns (e = e0, e0 + W, e0 + 2W, ...),
// of up to 4 per-macro segments (e.g. op.B^T | L | U | op.C), each padded
// in HBM to whole chunks, so chunk c of the stream is one bulk copy into
// ring slot c % S.
//
// Consumer protocol (warp-uniform): before reading stream positions
// [a, b) call `window(a, b)`; it is a single compare on the fast path.  On
// the slow path it releases every chunk ending at or before `a`, refills
// the ring and waits for the chunks covering [.., b).  b - a must not
// exceed (S - 1) * CH.
#pragma once

#include <stdint.h>

namespace mh {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Per-macro segment of the stream.  Every segment is padded to a multiple
// of the chunk size CH in HBM, so each chunk is exactly one bulk copy.
struct Segment {
  const double* base;  // segment of macro e starts at base + e * stride
  int64_t stride;      // doubles between consecutive macros (multiple of CH)
  int nch;             // chunks in the segment
  int keep;            // 1: L2 evict_last (re-read soon), 0: evict_first
};

// Ring state of one warp, kept in shared memory so that the out-of-line
// slow path does not force the consumer's registers onto the stack.
struct RingState {
  Segment seg[4];
  double* ring;
  uint64_t* bar;
  int64_t pe;          // producer cursor: macro of the next chunk
  int64_t W;           // macro stride between a warp's macros
  uint64_t pol_first, pol_last;
  uint32_t nchunks;    // chunks in this warp's stream
  uint32_t issued;     // chunks issued
  uint32_t waited;     // chunks landed
  int ps, pq;          // producer cursor: segment, chunk within segment
  int nseg;
};

template <int RING, int CH>
struct Ring {
  static constexpr int S = RING / CH;
  static constexpr uint32_t M = RING - 1;
  static_assert((RING & (RING - 1)) == 0, "ring must be a power of two");
  static_assert(RING % CH == 0 && S >= 2, "ring must hold >= 2 chunks");

  static __device__ void init(RingState* st, int lane, double* ring, uint64_t* bar,
                              const Segment* seg, int nseg, int64_t e0, int64_t W,
                              int64_t nmacro) {
    if (lane == 0) {
      int per = 0;
      for (int s = 0; s < nseg; ++s) {
        st->seg[s] = seg[s];
        per += seg[s].nch;
      }
      st->ring = ring;
      st->bar = bar;
      st->pe = e0;
      st->W = W;
      st->pol_first = l2_policy_evict_first();
      st->pol_last = l2_policy_evict_last();
      const int64_t mine = e0 < nmacro ? (nmacro - e0 + W - 1) / W : 0;
      st->nchunks = (uint32_t)(mine * per);
      st->issued = st->waited = 0;
      st->ps = 0;
      st->pq = 0;
      st->nseg = nseg;
      while (st->seg[st->ps].nch == 0) ++st->ps;  // skip empty leading segments
      for (int i = 0; i < S; ++i) mbar_init(&bar[i], 1);
      fence_mbar_init();
    }
    __syncwarp();
  }

  // lane 0: issue the next chunk (one 8*CH-byte bulk copy)
  static __device__ __forceinline__ void issue_next(RingState* st, uint32_t c) {
    const int slot = (int)(c % S);
    const Segment& sg = st->seg[st->ps];
    mbar_expect_tx(&st->bar[slot], CH * 8u);
    bulk_g2s(st->ring + slot * CH, sg.base + st->pe * sg.stride + (int64_t)st->pq * CH, CH * 8u,
             &st->bar[slot], sg.keep ? st->pol_last : st->pol_first);
    if (++st->pq == sg.nch) {
      st->pq = 0;
      do {
        if (++st->ps == st->nseg) {
          st->ps = 0;
          st->pe += st->W;
        }
      } while (st->seg[st->ps].nch == 0);
    }
  }

  // Slow path of the consumer's window check: release [.., a), refill,
  // wait for [.., b).  Returns the new ready end (stream position up to
  // which data has landed).
  static __device__ __noinline__ uint32_t slow(RingState* st, uint32_t a, uint32_t b, int lane) {
    uint32_t limit = a / CH + S;
    const uint32_t nchunks = st->nchunks;
    if (limit > nchunks) limit = nchunks;
    const uint32_t issued = st->issued;
    uint32_t waited = st->waited;
    __syncwarp();  // every lane is done with the slots being refilled
    if (lane == 0 && issued < limit) {
      fence_proxy_async_smem();
      for (uint32_t c = issued; c < limit; ++c) issue_next(st, c);
      st->issued = limit;
    }
    while (waited * CH < b) {
      const int slot = (int)(waited % S);
      const uint32_t parity = (waited / S) & 1u;
      while (!mbar_try_wait(&st->bar[slot], parity)) {
      }
      ++waited;
    }
    __syncwarp();
    if (lane == 0) st->waited = waited;
    return waited * CH;
  }
};

}  // namespace mh
