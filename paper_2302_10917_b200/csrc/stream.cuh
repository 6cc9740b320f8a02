// Per-warp TMA bulk-copy stream: a consumer warp reads a long sequence of
// contiguous HBM segments through a shared-memory ring that a producer warp
// of the same CTA keeps full with cp.async.bulk (the 1-D TMA engine) and
// mbarrier completion.  Memory-level parallelism therefore does not depend
// on registers or on the compiler hoisting loads: up to S chunks of CH
// doubles are in flight per consumer at all times, and the consumer's own
// issue slots are spent on arithmetic.
//
// Stream positions are 32-bit (doubles).  The stream of a warp is the
// concatenation, over the macros it owns (e = e0, e0 + W, e0 + 2W, ...),
// of up to 4 per-macro segments (e.g. op.B^T | L | U | op.C), each padded
// in HBM to whole chunks, so chunk c of the stream is one bulk copy into
// ring slot c % S.
//
// Consumer protocol (warp-uniform): before reading stream positions
// [a, b) call `window(a, b)`; it is a single compare on the fast path.  On
// the slow path it releases every chunk ending at or before `a` (empty
// barrier arrive) and waits for the chunks covering [.., b) (full barrier
// wait).  b - a must not exceed (S - 1) * CH.
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
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last_half() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, 0.5;" : "=l"(p));
  return p;
}
// segment policy: 0 evict_first, 1 evict_last, 2 normal, 3 evict_last on half the lines
__device__ __forceinline__ uint64_t l2_policy(int keep) {
  return keep == 1 ? l2_policy_evict_last()
         : keep == 2 ? l2_policy_evict_normal()
         : keep == 3 ? l2_policy_evict_last_half() : l2_policy_evict_first();
}

__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ring offset of a stream position (RING need not be a power of two)
template <int RING>
__device__ __forceinline__ uint32_t rmod(uint32_t x) {
  return (RING & (RING - 1)) == 0 ? (x & (RING - 1)) : (x % RING);
}

// Per-macro segment of the stream.  Every segment is padded to a multiple
// of the chunk size CH in HBM, so each chunk is exactly one bulk copy.
struct Segment {
  const double* base;  // segment of macro e starts at base + e * stride
  int64_t stride;      // doubles between consecutive macros (multiple of CH)
  int nch;             // chunks in the segment
  int keep;            // L2 policy: 0 evict_first, 1 evict_last (re-read soon), 2 normal, 3 half evict_last
};

// Warp-specialised ring pipeline: a producer warp of the CTA owns the
// streams of the CTA's consumer warps.  Per consumer ring of S slots:
//   full[slot]   producer arrive.expect_tx + bulk copy complete_tx; consumer waits
//   empty[slot]  consumer lane 0 arrives after the warp has read the slot;
//                producer waits before refilling it
template <int RING, int CH, int NCONS>
struct Pipe {
  static constexpr int S = RING / CH;
  static_assert(RING % CH == 0 && S >= 2, "ring must hold >= 2 chunks");

  // producer warp, lane 0: feed the NCONS consumer streams until done.  The
  // per-chunk path is a pointer bump: the segment table (shared memory) is
  // only consulted when a consumer's stream crosses into its next segment.
  static __device__ void produce(double* rings, uint64_t* full, uint64_t* empty,
                                 const Segment* seg, int nseg, int64_t warp0, int64_t W,
                                 int64_t nmacro, int ncons) {
    int per = 0;
    for (int s = 0; s < nseg; ++s) per += seg[s].nch;
    int first_seg = 0;
    while (first_seg < nseg && seg[first_seg].nch == 0) ++first_seg;
    const double* src[NCONS];
    uint64_t pol[NCONS];
    int64_t pe[NCONS];
    uint32_t issued[NCONS], nchunks[NCONS];
    int ps[NCONS], rem[NCONS];
#pragma unroll
    for (int w = 0; w < NCONS; ++w) {
      const int64_t e0 = warp0 + w;
      const int64_t mine = (w < ncons && e0 < nmacro) ? (nmacro - e0 + W - 1) / W : 0;
      pe[w] = e0;
      issued[w] = 0;
      nchunks[w] = (uint32_t)(mine * per);
      ps[w] = first_seg;
      if (first_seg < nseg) {
        src[w] = seg[first_seg].base + e0 * seg[first_seg].stride;
        rem[w] = seg[first_seg].nch;
        pol[w] = l2_policy(seg[first_seg].keep);
      }
    }
    // Round-robin over the consumer rings, one chunk per ring per round,
    // blocking (try_wait suspends in hardware) on the slot it needs next:
    // consumers drain at similar rates, so each ring keeps S-1 chunks of slack.
    for (;;) {
      bool any = false;
#pragma unroll
      for (int w = 0; w < NCONS; ++w) {
        const uint32_t c = issued[w];
        if (c >= nchunks[w]) continue;
        any = true;
        const uint32_t slot = c % S;
        if (c >= S)
          while (!mbar_try_wait(&empty[w * S + slot], ((c / S) - 1) & 1u)) {
          }
        mbar_expect_tx(&full[w * S + slot], CH * 8u);
        bulk_g2s(rings + (size_t)w * RING + slot * CH, src[w], CH * 8u, &full[w * S + slot],
                 pol[w]);
        src[w] += CH;
        issued[w] = c + 1;
        if (--rem[w] == 0) {
          do {
            if (++ps[w] == nseg) {
              ps[w] = 0;
              pe[w] += W;
            }
          } while (seg[ps[w]].nch == 0);
          const Segment& sg = seg[ps[w]];
          src[w] = sg.base + pe[w] * sg.stride;
          rem[w] = sg.nch;
          pol[w] = l2_policy(sg.keep);
        }
      }
      if (!any) break;
    }
  }
};

// Consumer side of one ring (all lanes, warp-uniform state in registers).
template <int RING, int CH>
struct Consumer {
  static constexpr int S = RING / CH;
  uint64_t* full;
  uint64_t* empty;
  uint32_t released = 0, waited = 0, ready_end = 0;

  // make stream positions [.., b) readable, releasing every chunk before a.
  // Chunks are retired strictly in order and only after their data has
  // landed: a chunk the consumer skipped (segment padding) is waited for
  // before its slot is handed back, so the full/empty barrier phases of a
  // slot can never run two uses apart.
  __device__ __forceinline__ void window(uint32_t a, uint32_t b, int lane) {
    if (b <= ready_end) return;
    const uint32_t rel = a / CH;
    if (rel > released) {
      __syncwarp();  // the whole warp is done with those slots
      while (released < rel) {
        if (waited <= released) {
          while (!mbar_try_wait(&full[released % S], (released / S) & 1u)) {
          }
          waited = released + 1;
        }
        if (lane == 0) mbar_arrive(&empty[released % S]);
        ++released;
      }
    }
    while (waited * CH < b) {
      const uint32_t c = waited;
      while (!mbar_try_wait(&full[c % S], (c / S) & 1u)) {
      }
      ++waited;
    }
    ready_end = waited * CH;
  }
};

}  // namespace mh
