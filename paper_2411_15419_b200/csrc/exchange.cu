// Device-initiated dispatch over NVLink (world > 1): count exchange, layout plan and the fused
// pack-and-push of representative rows into the owning ranks' receive buffers (P:143 dispatch phase,
// only representatives).  No host synchronisation: every rank derives every layout from
// the all-to-all counts on the device.  See exchange.cuh for the buffers and the signalling protocol.
#include <cstdlib>

#include "common.cuh"
#include "exchange.cuh"
#include "tc_common.cuh"

namespace luffy {
namespace {

// Wait until every rank published `seq` for this phase (bounded: see xwait_flag).
__global__ void xwait_kernel(const uint32_t* __restrict__ flags, int P, const uint32_t* seqp, XErr err, int phase) {
  pdl_enter();
  const int p = threadIdx.x;
  if (p < P) xwait_flag(flags + p, *seqp, err, phase);
  __syncthreads();
}

// First launch of a step at world > 1 (luffy_route): the device step number every exchange of the step
// publishes and waits for.  Device-resident, so a step captured in a CUDA graph bumps it on every replay.
__global__ void xstep_kernel(uint32_t* dseq) {
  pdl_enter();
  if (threadIdx.x == 0) *dseq += 1u;
}

// Count exchange and layout plan in ONE single-CTA kernel: push my counts to every rank, publish XP_CNT,
// wait for every rank's counts, then derive the plan with the shared host/device xplan_body (xplan.h).
__global__ void xcnt_plan_kernel(const int32_t* __restrict__ nrep, int E, int me, int32_t* const* peer_cnt, int P,
                                 XSignal sig, const uint32_t* __restrict__ flags, const int32_t* __restrict__ inbox,
                                 int32_t* __restrict__ cnt_all, int32_t* __restrict__ roff, int32_t* __restrict__ dst_base,
                                 int32_t* __restrict__ src_soff, XErr err) {
  pdl_enter();
  for (int i = threadIdx.x; i < P * E; i += blockDim.x) {
    const int p = i / E, e = i % E;
    peer_cnt[p][(size_t)me * E + e] = nrep[e];
  }
  xsignal_done(sig);  // (single CTA: publishes XP_CNT to every rank)
  if (threadIdx.x < P) xwait_flag(flags + threadIdx.x, *sig.seqp, err, XP_CNT);
  __syncthreads();
  xplan_body(inbox, P, E, me, cnt_all, roff, dst_base, src_soff, threadIdx.x, blockDim.x);
}

// Per expert-layout row: the source rank and its send slot (for the combine and dispatch-backward
// epilogues); padding rows -> -1 and zeroed in the receive buffer and in dexp.
__global__ void __launch_bounds__(256) xplan_rows_kernel(const int32_t* __restrict__ cnt_all, const int32_t* __restrict__ roff,
                                                         const int32_t* __restrict__ src_soff, int P, int E, int me,
                                                         int d, int64_t max_rows, int32_t* __restrict__ rank_of,
                                                         int32_t* __restrict__ slot_of, bf16* __restrict__ recv,
                                                         bf16* __restrict__ dexp, int elem_bytes,
                                                         unsigned long long* __restrict__ rowmask) {
  pdl_enter();
  const int El = E / P;
  const int64_t rows = roff[El];
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += nthreads)
    if (!xplan_row(r, cnt_all, roff, src_soff, P, E, me, rank_of + r, slot_of + r))
      rowmask[r] = 0ull;  // padding rows are not combined anywhere
  // padding rows (the tail of each local expert segment) are zeroed in the receive buffer and in the
  // backward buffer: one warp per row, 16-byte coalesced stores
  const int lane = threadIdx.x & 31;
  const int64_t nw = nthreads >> 5;
  int64_t wgl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t rb = (size_t)d * elem_bytes;
  for (int el = 0; el < El; ++el) {
    const int e = me * El + el;
    int64_t used = 0;
    for (int q = 0; q < P; ++q) used += cnt_all[q * E + e];
    const int64_t p0 = roff[el] + used, p1 = roff[el + 1];
    for (int64_t r = p0 + wgl; r < p1; r += nw) {
      uint4* a = reinterpret_cast<uint4*>(reinterpret_cast<char*>(recv) + r * rb);
      uint4* b = reinterpret_cast<uint4*>(reinterpret_cast<char*>(dexp) + r * rb);
      for (size_t j = lane; j < rb / 16; j += 32) {
        a[j] = make_uint4(0, 0, 0, 0);
        b[j] = make_uint4(0, 0, 0, 0);
      }
    }
    wgl = (wgl + (p1 - p0)) % nw;  // spread the next segment's rows over other warps
  }
}

// Fused pack + dispatch: every representative row is copied from x straight into the owner's
// receive buffer (16-byte vector stores over NVLink), then XP_DISP is published.
template <typename T>
__global__ void __launch_bounds__(256) xpack_push_kernel(const T* __restrict__ x, const int32_t* __restrict__ perm,
                                                         const int32_t* __restrict__ soff, const int32_t* __restrict__ dst_base,
                                                         int E, int El, int d, void* const* peer_recv, XSignal sig,
                                                         const unsigned long long* __restrict__ dmask,
                                                         unsigned long long* const* peer_rowmask, int me) {
  pdl_enter();
  __shared__ int32_t soff_s[LUFFY_MAX_EXPERTS + 1];
  __shared__ int32_t base_s[LUFFY_MAX_EXPERTS];
  for (int i = threadIdx.x; i <= E; i += blockDim.x) {
    soff_s[i] = soff[i];
    if (i < E) base_s[i] = dst_base[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t rows = soff_s[E];
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < rows; s += nw) {
    const int t = perm[s];
    if (t < 0) continue;
    const int e = find_group(soff_s, E, s);
    const int p = e / El;
    const int64_t drow = (int64_t)base_s[e] + (s - soff_s[e]);
    T* dst = static_cast<T*>(peer_recv[p]) + drow * d;
    // where the expert output of this row must be combined: home (me) or the destinations of the
    // sequences that use it (sequence migration)
    if (lane == 0) peer_rowmask[p][drow] = dmask ? dmask[s] : (1ull << me);
    const T* src = x + (size_t)t * d;
    for (int c = lane * 8; c < d; c += 256) {
      if constexpr (sizeof(T) == 2) {
        *reinterpret_cast<uint4*>(dst + c) = *reinterpret_cast<const uint4*>(src + c);
      } else {
        *reinterpret_cast<float4*>(dst + c) = *reinterpret_cast<const float4*>(src + c);
        *reinterpret_cast<float4*>(dst + c + 4) = *reinterpret_cast<const float4*>(src + c + 4);
      }
    }
  }
  xsignal_done(sig);
}

// The same fused pack + dispatch through the TMA engine: every representative row streams through a ring of
// shared-memory row buffers -- bulk load of x[t] (mbarrier completion), then one bulk store of the whole row
// into its owner's receive buffer (a peer's memory over NVLink, or this GPU's) -- so each row crosses NVLink
// as one large transfer issued by one thread instead of 16-byte stores from a warp.  Rows are processed in
// batches of `stages` (all loads of a batch first, then the stores as the loads land).
template <typename T>
__global__ void __launch_bounds__(32) xpack_push_tma_kernel(const T* __restrict__ x, const int32_t* __restrict__ perm,
                                                            const int32_t* __restrict__ soff,
                                                            const int32_t* __restrict__ dst_base, int E, int El, int d,
                                                            void* const* peer_recv, XSignal sig,
                                                            const unsigned long long* __restrict__ dmask,
                                                            unsigned long long* const* peer_rowmask, int me, int stages) {
  pdl_enter();
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ int32_t soff_s[LUFFY_MAX_EXPERTS + 1];
  __shared__ int32_t base_s[LUFFY_MAX_EXPERTS];
  __shared__ __align__(8) uint64_t bar[32];
  const int lane = threadIdx.x;
  for (int i = lane; i <= E; i += 32) {
    soff_s[i] = soff[i];
    if (i < E) base_s[i] = dst_base[i];
  }
  const uint32_t rb = (uint32_t)(d * sizeof(T));
  if (lane == 0) {
    for (int j = 0; j < stages; ++j) tc::mbar_init(&bar[j], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (lane == 0) {
    const int64_t rows = soff_s[E];
    uint32_t phase = 0;  // bit j: parity of stage j's next completion (a stage skipped for padding keeps it)
    for (int64_t b0 = blockIdx.x; b0 < rows; b0 += (int64_t)gridDim.x * stages) {
      tc::bulk_wait_read();  // the previous batch's stores have read the ring
      int tj[32];
      for (int j = 0; j < stages; ++j) {
        const int64_t s = b0 + (int64_t)j * gridDim.x;
        tj[j] = s < rows ? perm[s] : -1;
        if (tj[j] >= 0) {
          tc::mbar_expect_tx(&bar[j], rb);
          tc::bulk_load(ring + (size_t)j * rb, x + (size_t)tj[j] * d, rb, &bar[j]);
        }
      }
      for (int j = 0; j < stages; ++j) {
        if (tj[j] < 0) continue;
        const int64_t s = b0 + (int64_t)j * gridDim.x;
        const int e = find_group(soff_s, E, s);
        const int p = e / El;
        const int64_t drow = (int64_t)base_s[e] + (s - soff_s[e]);
        peer_rowmask[p][drow] = dmask ? dmask[s] : (1ull << me);
        tc::mbar_wait(&bar[j], (phase >> j) & 1u);
        phase ^= 1u << j;
        tc::bulk_store(static_cast<T*>(peer_recv[p]) + drow * d, ring + (size_t)j * rb, rb);
        tc::bulk_commit();
      }
    }
    tc::bulk_wait_all();                                   // the rows have been written ...
    asm volatile("fence.proxy.async.global;" ::: "memory");  // ... and are ordered before the release below
  }
  __syncwarp();
  xsignal_done(sig);
}

inline int grid_warps(int64_t warps) {
  int64_t b = (warps + 7) / 8;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 8));
}

}  // namespace

int launch_xwait(const luffy_layer* L, int phase, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  launch_pdl(xwait_kernel, 1, 64, 0, st, L->x_flags + phase * L->P, L->P, (const uint32_t*)L->dseq, make_xerr(L), phase);
  LUFFY_LAUNCHED();
  return 0;
}

int launch_xstep(const luffy_layer* L, void* s) {
  launch_pdl(xstep_kernel, 1, 32, 0, static_cast<cudaStream_t>(s), L->dseq);
  LUFFY_LAUNCHED();
  return 0;
}

XErr make_xerr(const luffy_layer* L) {
  XErr e;
  e.word = L->x_errw;
  e.host = L->x_err_d;
  e.timeout_ns = L->x_timeout_ns;
  return e;
}

XSignal make_signal(const luffy_layer* L, int phase) {
  XSignal sg;
  sg.counter = L->x_counters + phase;
  sg.flag = L->x_flagptr + phase * L->P;
  sg.P = L->P;
  sg.seqp = L->dseq;
  return sg;
}

// Dispatch at world > 1: [counts + wait + plan] -> [row plan | fused pack/push] -> wait for every rank's rows.
int launch_xdispatch(luffy_layer* L, const void* x, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  const int par = L->seq & 1;
  launch_pdl(xcnt_plan_kernel, 1, 256, 0, st, L->nrep, L->E, L->rank, L->x_peer_cnt, L->P, make_signal(L, XP_CNT),
                                      L->x_flags + XP_CNT * L->P, L->x_cnt_inbox, L->cnt_all, L->roff, L->x_dst_base,
                                      L->x_src_soff, make_xerr(L));
  LUFFY_LAUNCHED();
  launch_pdl(xplan_rows_kernel, 148, 256, 0, st, L->cnt_all, L->roff, L->x_src_soff, L->P, L->E, L->rank, L->d, L->recv_max,
                                         L->x_rank_of, L->x_slot_of, static_cast<bf16*>(L->x_recv[par]),
                                         static_cast<bf16*>(L->x_dexp), L->dtype == LUFFY_BF16 ? 2 : 4, L->x_rowmask);
  LUFFY_LAUNCHED();
  // LUFFY_PUSH_TMA=1 selects the bulk-copy push.  Measured at C2, N=2 (CUPTI, warm): 36.1 us (240 GB/s over
  // NVLink) against 23.7 us (365 GB/s) for the warp-store push, which therefore stays the default.
  static const bool tma_push = [] {
    const char* v = std::getenv("LUFFY_PUSH_TMA");
    return v && v[0] == '1';
  }();
  if (tma_push) {
    const size_t rb = (size_t)L->d * (L->dtype == LUFFY_BF16 ? 2 : 4);
    const int stages = (int)std::max<size_t>(2, std::min<size_t>(16, (96 * 1024) / rb));
    const int smem = (int)(stages * rb);
    const int grid = 2 * device_sms();
    if (L->dtype == LUFFY_BF16) {
      LUFFY_CUDA_TRY(smem_optin((const void*)xpack_push_tma_kernel<bf16>, smem));
      launch_pdl(xpack_push_tma_kernel<bf16>, grid, 32, smem, st, static_cast<const bf16*>(x), (const int32_t*)L->perm,
                 (const int32_t*)L->soff, (const int32_t*)L->x_dst_base, L->E, L->El, L->d, L->x_peer_recv + par * L->P,
                 make_signal(L, XP_DISP), (const unsigned long long*)(L->mig ? L->dmask : nullptr), L->x_peer_rowmask,
                 L->rank, stages);
    } else {
      LUFFY_CUDA_TRY(smem_optin((const void*)xpack_push_tma_kernel<float>, smem));
      launch_pdl(xpack_push_tma_kernel<float>, grid, 32, smem, st, static_cast<const float*>(x), (const int32_t*)L->perm,
                 (const int32_t*)L->soff, (const int32_t*)L->x_dst_base, L->E, L->El, L->d, L->x_peer_recv + par * L->P,
                 make_signal(L, XP_DISP), (const unsigned long long*)(L->mig ? L->dmask : nullptr), L->x_peer_rowmask,
                 L->rank, stages);
    }
    LUFFY_LAUNCHED();
    if (L->dtype == LUFFY_BF16) return 0;
    return launch_xwait(L, XP_DISP, s);
  }
  const int blocks = grid_warps(L->Rpad_max);
  if (L->dtype == LUFFY_BF16)
    launch_pdl(xpack_push_kernel<bf16>, blocks, 256, 0, st, static_cast<const bf16*>(x), L->perm, L->soff, L->x_dst_base, L->E,
                                                    L->El, L->d, L->x_peer_recv + par * L->P, make_signal(L, XP_DISP),
                                                    L->mig ? L->dmask : nullptr, L->x_peer_rowmask, L->rank);
  else
    launch_pdl(xpack_push_kernel<float>, blocks, 256, 0, st, static_cast<const float*>(x), L->perm, L->soff, L->x_dst_base, L->E,
                                                     L->El, L->d, L->x_peer_recv + par * L->P, make_signal(L, XP_DISP),
                                                     L->mig ? L->dmask : nullptr, L->x_peer_rowmask, L->rank);
  LUFFY_LAUNCHED();
  // bf16: the expert FFN's GEMM1 waits per tile for the source ranks of its rows (fused dispatch, exchange.cuh
  // XWaitRows); the fp32 SIMT path waits here for every rank
  if (L->dtype == LUFFY_BF16) return 0;
  return launch_xwait(L, XP_DISP, s);
}

}  // namespace luffy
