// Device-initiated expert-parallel exchange over NVLink (world > 1).
//
// Every layer owns one peer-visible exchange region (cudaMalloc + CUDA IPC, mapped by every rank):
//   recv[2]    expert layout, double-buffered by step parity  <- peers' pack kernels (dispatch)
//   gathered   [P][send rows] indexed by (source rank, slot)   <- peers' GEMM2 epilogues (combine; with
//              sequence migration a row goes to every destination rank that needs it)
//   rowmask    [recv rows] destination-rank bitmask of each expert row <- sources (with dispatch)
//   mig_*      sequence-migration tables / token metadata / returned dY, dw
//   dexp       expert layout                                   <- peers' uncondense-backward (combine bwd)
//   dsend      send layout                                     <- peers' dgrad1 epilogues (dispatch bwd)
//   cnt_inbox  [P][E] representative counts                    <- peers (count exchange)
//   flags      [phase][P] step sequence numbers               <- peers (release stores)
// Producers store rows straight into the destination rank's buffer; the last CTA of a producing kernel
// publishes `seq` to every peer's flag with a system-scope release; consumers wait with acquire loads.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "luffy_internal.h"
#include "xplan.h"

namespace luffy {

enum XPhase { XP_CNT = 0, XP_DISP = 1, XP_COMB = 2, XP_CBWD = 3, XP_DBWD = 4, XP_MIG = 5, XP_META = 6, XP_MIGB = 7,
              XP_RES = 8, XP_NUM = 9 };
constexpr int kMaxWorld = 64;

// Completion signal of one producing kernel.
struct XSignal {
  uint32_t* counter;        // local CTA-completion counter (reset by the last CTA)
  uint32_t* const* flag;    // [P] address of (phase, my rank) in each peer's flag array
  int P;
  const uint32_t* seqp;     // the step's sequence number (device word, luffy_layer::dseq)
};

// Row redirect for an epilogue.  mask == nullptr: expert-layout row r goes to rank rank_of[r], row
// slot_of[r] of that rank's buffer peer_base[rank]; rank_of[r] < 0 = padding (not sent).
// mask != nullptr: the row goes to every rank g set in mask[r], row rank_of[r] * stride + slot_of[r].
struct XRedirect {
  const int32_t* rank_of;
  const int32_t* slot_of;
  void* const* peer_base;
  const unsigned long long* mask;
  int64_t stride;
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Call by every thread of every CTA at the end of a producing kernel.
__device__ __forceinline__ void xsignal_done(const XSignal& s) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const uint32_t total = gridDim.x * gridDim.y * gridDim.z;
    const uint32_t prev = atomicAdd(s.counter, 1u);
    if (prev == total - 1) {
      *s.counter = 0u;
      __threadfence_system();
      const uint32_t seq = *s.seqp;
      for (int p = 0; p < s.P; ++p) st_release_sys(s.flag[p], seq);
    }
  }
}

XSignal make_signal(const luffy_layer* L, int phase);

// Bounded cross-rank wait.  A peer that stops publishing must not hang or kill this rank's context: after
// `timeout_ns` the waiter records (phase + 1, seq) in the layer's error word (device memory, mirrored into
// pinned host memory mapped into the device, so the host reads it without a synchronisation) and proceeds
// as if the flag had arrived (the data of that step is garbage; flags are left unchanged).  Every later wait of the layer
// sees the error word and returns at once, and the next luffy_* call on the layer returns LUFFY_E_STATE.
struct XErr {
  uint32_t* word;        // [2] device memory (L2): (phase + 1, seq) of the first timed-out wait, 0 = none
  uint32_t* host;        // [2] its mirror in mapped pinned host memory (read by the host without a sync;
                         //     written only on a timeout -- device-side polling never touches PCIe)
  uint64_t timeout_ns;
};

XErr make_xerr(const luffy_layer* L);

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}

// true when the flag reached seq, false on timeout or an earlier failure of the layer.
__device__ __forceinline__ bool xwait_flag(const uint32_t* flag, uint32_t seq, const XErr& e, int phase) {
  if (ld_acquire_sys(flag) >= seq) return true;
  if (ld_volatile_u32(e.word) != 0u) return false;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (uint32_t it = 1;; ++it) {
    __nanosleep(32);
    if (ld_acquire_sys(flag) >= seq) return true;
    if ((it & 255u) == 0u) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (ld_volatile_u32(e.word) != 0u) return false;
      if (t - t0 > e.timeout_ns) {
        if (atomicCAS(e.word, 0u, (uint32_t)phase + 1u) == 0u) {
          atomicExch(e.word + 1, seq);
          atomicExch_system(e.host + 1, seq);
          atomicExch_system(e.host, (uint32_t)phase + 1u);
        }
        __threadfence_system();
        return false;
      }
    }
  }
}

// Tile-level wait for dispatched rows (fused dispatch -> GEMM1): a consumer of rows [r0, r1) of local
// expert el waits only for the source ranks whose rows fall in that range (flags[q] >= seq, published by
// q's pack-and-push kernel), instead of a stream-wide wait for every rank.
struct XWaitRows {
  const uint32_t* flags;   // [P] this rank's XP_DISP flags (one per source rank)
  const uint32_t* seqp;    // the step's sequence number (device word)
  int P, E, El, me;
  const int32_t* cnt_all;  // [P][E] rows each source sends to each expert
  const int32_t* roff;     // [El+1] expert-layout offsets of the local experts
  XErr err;
};
__device__ __forceinline__ void xwait_rows(const XWaitRows& w, int el, int r0, int r1) {
  const int e = w.me * w.El + el;
  const uint32_t seq = *w.seqp;
  int base = w.roff[el];
  for (int q = 0; q < w.P; ++q) {
    const int n = w.cnt_all[q * w.E + e];
    if (n > 0 && base < r1 && base + n > r0) xwait_flag(w.flags + q, seq, w.err, XP_DISP);
    base += n;
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");  // peer-written rows -> TMA (async proxy) reads
}

}  // namespace luffy
