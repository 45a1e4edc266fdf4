// Sequence migration on the device (world > 1): SURVEY §8a row 15 (K9) and the migration-aware combine
// of row 7.  The paper migrates a whole sequence in the combine phase to the GPU chosen by Alg. 1
// (P:264-299), pulling its expert outputs there instead of back to its home GPU.
//
//  K9 (seq_rows):   rows_at[s][j] = number of DISTINCT representative rows (send slots) used by the copies
//                   of sequence s whose expert lives on rank j (reading R16: condensed copies are rebuilt
//                   from their representative's row, so a row is pulled once per destination) -- pushed to
//                   every rank so that every rank runs the same deterministic planner (no controller).
//  set_migration:   dmask[slot] = set of destination ranks of the sequences whose copies use the slot;
//                   the dispatch ships dmask with each row, and the GEMM2 epilogue stores the expert output
//                   row into every destination's gathered buffer (row index (home rank, slot)).
//  meta push:       (home rank, home token, slots, gate weights) of every token go to its destination,
//                   which runs the uncondense for the tokens of the sequences it hosts.
//  backward:        the destination returns dY and d(gate weight) of each token to its home rank, where the
//                   atomic-free condensed backward runs unchanged.
#include "common.cuh"
#include "exchange.cuh"

namespace luffy {
namespace {

__device__ __forceinline__ int seq_of(const int32_t* seq_start, int S, int t) {
  int lo = 0, hi = S;  // seq_start[lo] <= t < seq_start[lo+1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (seq_start[mid] <= t) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void zero_u32_kernel(uint32_t* __restrict__ p, int64_t n) {
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = 0u;
}

// distinct slots per sequence: bit (s, pos[t, j]) for every copy of every token t of sequence s
__global__ void seq_bits_kernel(const int32_t* __restrict__ pos, const int32_t* __restrict__ seq_start, int S, int T, int k,
                                int words, uint32_t* __restrict__ bits) {
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)T * k; i += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / k);
    const int s = seq_of(seq_start, S, t);
    const int u = pos[i];
    atomicOr(bits + (int64_t)s * words + (u >> 5), 1u << (u & 31));
  }
}

// rows_at[s][j] = popcount of the bits of sequence s inside rank j's slot range; pushed to every rank.
__global__ void seq_rows_push_kernel(const uint32_t* __restrict__ bits, const int32_t* __restrict__ soff, int S, int P,
                                     int El, int words, int me, int Smax, int32_t* const* peer_mig, XSignal sig) {
  pdl_enter();
  for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < S * P; i += gridDim.x * (blockDim.x >> 5)) {
    const int s = i / P, j = i % P;
    const int w0 = soff[j * El] >> 5, w1 = soff[(j + 1) * El] >> 5;
    int c = 0;
    for (int w = w0 + (threadIdx.x & 31); w < w1; w += 32) c += __popc(bits[(int64_t)s * words + w]);
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0)
      for (int p = 0; p < P; ++p) peer_mig[p][((int64_t)me * Smax + s) * P + j] = c;
  }
  xsignal_done(sig);
}

__global__ void zero_u64_kernel(unsigned long long* __restrict__ p, int64_t n) {
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = 0ull;
}

__global__ void slot_dmask_kernel(const int32_t* __restrict__ pos, const int32_t* __restrict__ seq_start,
                                  const int32_t* __restrict__ seq_dest, int S, int T, int k,
                                  unsigned long long* __restrict__ dmask) {
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)T * k; i += (int64_t)gridDim.x * blockDim.x) {
    const int s = seq_of(seq_start, S, (int)(i / k));
    atomicOr(dmask + pos[i], 1ull << seq_dest[s]);
  }
}

// (home rank, home token, slots, weights) of every token to the rank hosting its sequence.
__global__ void mig_meta_push_kernel(const int32_t* __restrict__ pos, const float* __restrict__ w,
                                     const int32_t* __restrict__ seq_start, const int32_t* __restrict__ seq_dest,
                                     const int32_t* __restrict__ out_start, int S, int T, int k, int me,
                                     int32_t* const* peer_meta, float* const* peer_meta_w, XSignal sig) {
  pdl_enter();
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
    const int s = seq_of(seq_start, S, t);
    const int g = seq_dest[s];
    const int64_t i = out_start[s] + (t - seq_start[s]);
    int32_t* m = peer_meta[g] + i * (2 + k);
    m[0] = me;
    m[1] = t;
    for (int j = 0; j < k; ++j) {
      m[2 + j] = pos[(int64_t)t * k + j];
      peer_meta_w[g][i * k + j] = w[(int64_t)t * k + j];
    }
  }
  xsignal_done(sig);
}

// y[i] = sum_j w[i, j] * gathered[(home_i, slot_ij)] for the tokens this rank hosts (P:405 at the
// destination of the migrated sequence).
template <typename T>
__global__ void __launch_bounds__(256) uncondense_mig_kernel(const T* __restrict__ gathered, const int32_t* __restrict__ meta,
                                                             const float* __restrict__ meta_w, int64_t n_out, int k, int d,
                                                             int64_t Rpad, const T* __restrict__ res, T* __restrict__ y) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_out; i += nw) {
    const int32_t* m = meta + i * (2 + k);
    const int64_t h = m[0];
    for (int c = lane * 8; c < d; c += 256) {
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (res != nullptr) load8(res + i * d + c, acc);  // residual row pushed from the home rank
      for (int j = 0; j < k; ++j) {
        const float wj = meta_w[i * k + j];
        float v[8];
        load8(gathered + (h * Rpad + m[2 + j]) * d + c, v);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = fmaf(wj, v[q], acc[q]);
      }
      store8(y + i * d + c, acc);
    }
  }
}

// Residual rows of a block y = x + MoE(x): x of every token to the rank hosting its sequence (row order of
// the hosted tokens: home rank, sequence, token).
template <typename T>
__global__ void __launch_bounds__(256) res_push_kernel(const T* __restrict__ x, const int32_t* __restrict__ seq_start,
                                                       const int32_t* __restrict__ seq_dest,
                                                       const int32_t* __restrict__ out_start, int S, int T_, int d,
                                                       void* const* peer_res, XSignal sig) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < T_; t += (gridDim.x * blockDim.x) >> 5) {
    const int s = seq_of(seq_start, S, t);
    const int64_t i = out_start[s] + (t - seq_start[s]);
    T* dst = static_cast<T*>(peer_res[seq_dest[s]]) + i * d;
    for (int c = lane * 8; c < d; c += 256) {
      if constexpr (sizeof(T) == 2) {
        *reinterpret_cast<uint4*>(dst + c) = *reinterpret_cast<const uint4*>(x + (int64_t)t * d + c);
      } else {
        *reinterpret_cast<float4*>(dst + c) = *reinterpret_cast<const float4*>(x + (int64_t)t * d + c);
        *reinterpret_cast<float4*>(dst + c + 4) = *reinterpret_cast<const float4*>(x + (int64_t)t * d + c + 4);
      }
    }
  }
  xsignal_done(sig);
}

// Backward at the destination: d(gate weight) and dY of every hosted token back to its home rank.
template <typename T>
__global__ void __launch_bounds__(256) mig_bwd_push_kernel(const T* __restrict__ dy, const T* __restrict__ gathered,
                                                           const int32_t* __restrict__ meta, int64_t n_out, int k, int d,
                                                           int64_t Rpad, void* const* peer_dy_in, float* const* peer_dw_in,
                                                           XSignal sig) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_out; i += nw) {
    const int32_t* m = meta + i * (2 + k);
    const int h = m[0];
    const int64_t t = m[1];
    T* dst = static_cast<T*>(peer_dy_in[h]) + t * d;
    for (int c = lane * 8; c < d; c += 256) {
      if constexpr (sizeof(T) == 2) {
        *reinterpret_cast<uint4*>(dst + c) = *reinterpret_cast<const uint4*>(dy + i * d + c);
      } else {
        *reinterpret_cast<float4*>(dst + c) = *reinterpret_cast<const float4*>(dy + i * d + c);
        *reinterpret_cast<float4*>(dst + c + 4) = *reinterpret_cast<const float4*>(dy + i * d + c + 4);
      }
    }
    for (int j = 0; j < k; ++j) {
      const T* o = gathered + ((int64_t)h * Rpad + m[2 + j]) * d;
      float s = 0.f;
      for (int c = lane * 8; c < d; c += 256) {
        float a[8], b[8];
        load8(dy + i * d + c, a);
        load8(o + c, b);
#pragma unroll
        for (int q = 0; q < 8; ++q) s = fmaf(a[q], b[q], s);
      }
      s = warp_sum(s);
      if (lane == 0) peer_dw_in[h][t * k + j] = s;
    }
  }
  xsignal_done(sig);
}

inline int blocks_for(int64_t n, int per) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + per - 1) / per, 148 * 8)); }

}  // namespace

int launch_seq_rows(luffy_layer* L, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  const int words = (int)(L->Rpad_max / 32);
  launch_pdl(zero_u32_kernel, blocks_for((int64_t)L->S * words, 256), 256, 0, st, L->seq_bits, (int64_t)L->S * words);
  LUFFY_LAUNCHED();
  launch_pdl(seq_bits_kernel, blocks_for((int64_t)L->T * L->k, 256), 256, 0, st, L->pos, L->seq_start, L->S, L->T, L->k, words,
                                                                         L->seq_bits);
  LUFFY_LAUNCHED();
  launch_pdl(seq_rows_push_kernel, blocks_for((int64_t)L->S * L->P, 8), 256, 0, st, L->seq_bits, L->soff, L->S, L->P, L->El, words,
                                                                             L->rank, L->Smax, L->x_peer_mig,
                                                                             make_signal(L, XP_MIG));
  LUFFY_LAUNCHED();
  return launch_xwait(L, XP_MIG, s);
}

int launch_set_migration(luffy_layer* L, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  launch_pdl(zero_u64_kernel, blocks_for(L->Rpad_max, 256), 256, 0, st, L->dmask, L->Rpad_max);
  LUFFY_LAUNCHED();
  launch_pdl(slot_dmask_kernel, blocks_for((int64_t)L->T * L->k, 256), 256, 0, st, L->pos, L->seq_start, L->seq_dest_l, L->S, L->T,
                                                                           L->k, L->dmask);
  LUFFY_LAUNCHED();
  return 0;
}

int launch_mig_meta_push(luffy_layer* L, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  launch_pdl(mig_meta_push_kernel, blocks_for(L->T, 256), 256, 0, st, L->pos, L->w, L->seq_start, L->seq_dest_l, L->out_start, L->S,
                                                              L->T, L->k, L->rank, L->x_peer_meta, L->x_peer_meta_w,
                                                              make_signal(L, XP_META));
  LUFFY_LAUNCHED();
  return 0;
}

int launch_uncondense_mig(const luffy_layer* L, const void* x_res, void* y, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  const void* res = nullptr;
  if (x_res) {  // residual block: push this rank's x rows to the hosts of their sequences, then wait
    const int bp = blocks_for(L->T, 8);
    if (L->dtype == LUFFY_BF16)
      launch_pdl(res_push_kernel<bf16>, bp, 256, 0, st, static_cast<const bf16*>(x_res), L->seq_start, L->seq_dest_l,
                 L->out_start, L->S, L->T, L->d, L->x_peer_res, make_signal(L, XP_RES));
    else
      launch_pdl(res_push_kernel<float>, bp, 256, 0, st, static_cast<const float*>(x_res), L->seq_start, L->seq_dest_l,
                 L->out_start, L->S, L->T, L->d, L->x_peer_res, make_signal(L, XP_RES));
    LUFFY_LAUNCHED();
    LUFFY_CUDA_TRY(launch_xwait(L, XP_RES, s));
    res = L->x_res;
  }
  const int b = blocks_for(L->n_out, 8);
  if (L->dtype == LUFFY_BF16)
    launch_pdl(uncondense_mig_kernel<bf16>, b, 256, 0, st, static_cast<const bf16*>(L->x_gathered), L->x_meta, L->x_meta_w,
                                                   L->n_out, L->k, L->d, L->Rpad_max, static_cast<const bf16*>(res),
                                                   static_cast<bf16*>(y));
  else
    launch_pdl(uncondense_mig_kernel<float>, b, 256, 0, st, static_cast<const float*>(L->x_gathered), L->x_meta, L->x_meta_w,
                                                    L->n_out, L->k, L->d, L->Rpad_max, static_cast<const float*>(res),
                                                    static_cast<float*>(y));
  LUFFY_LAUNCHED();
  return 0;
}

int launch_mig_bwd_push(const luffy_layer* L, const void* dy, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  const int b = blocks_for(L->n_out, 8);
  if (L->dtype == LUFFY_BF16)
    launch_pdl(mig_bwd_push_kernel<bf16>, b, 256, 0, st, static_cast<const bf16*>(dy), static_cast<const bf16*>(L->x_gathered),
                                                 L->x_meta, L->n_out, L->k, L->d, L->Rpad_max, L->x_peer_dy_in,
                                                 L->x_peer_dw_in, make_signal(L, XP_MIGB));
  else
    launch_pdl(mig_bwd_push_kernel<float>, b, 256, 0, st, static_cast<const float*>(dy), static_cast<const float*>(L->x_gathered),
                                                  L->x_meta, L->n_out, L->k, L->d, L->Rpad_max, L->x_peer_dy_in,
                                                  L->x_peer_dw_in, make_signal(L, XP_MIGB));
  LUFFY_LAUNCHED();
  return launch_xwait(L, XP_MIGB, s);
}

}  // namespace luffy
