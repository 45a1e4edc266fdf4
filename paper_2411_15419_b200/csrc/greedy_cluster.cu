// Representative selection per expert group on a thread-block CLUSTER (DSMEM), the fast path of the
// exact parallel-rounds greedy (condense.cu has the algorithm statement).
//
// Groups are independent (only tokens of the same expert are compared), so each group gets its
// own cluster of CS CTAs and no grid-wide barrier is needed.  Every CTA owns a slice of the group's
// rows and keeps REPLICAS of the group-wide state in its shared memory: the alive bitset, the winner
// bitset, the priority keys and the 1-hop maxima.  A value computed for an owned row is broadcast to
// the replicas of all CTAs through distributed shared memory, so the neighbour maxima are gathered from
// local shared memory.  Phases are separated by cluster barriers:
//   A  residual degree -> key (broadcast); count alive rows
//   B  m1 = max key over the alive closed neighbourhood (broadcast)
//   C  m2 = max m1 over the alive closed neighbourhood; winner iff m2 == key (broadcast bit)
//   D  winners and their alive neighbours leave (rep = winner; alive bit cleared in every replica)
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace luffy {
namespace {

constexpr int GC_THREADS = 1024;

template <int CS>
__global__ void __launch_bounds__(GC_THREADS, 1) greedy_cluster_kernel(const int32_t* __restrict__ goff,
                                                                      const int32_t* __restrict__ gcnt,
                                                                      const int64_t* __restrict__ adjoff,
                                                                      const uint32_t* __restrict__ adj,
                                                                      int32_t* __restrict__ rep_local,
                                                                      uint32_t* __restrict__ ctrl, int nmax,
                                                                      int max_rounds, int cache_words) {
  pdl_enter();
  extern __shared__ __align__(16) uint8_t gsm[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int e = blockIdx.x / CS;
  const int g0 = goff[e];
  const int n = gcnt[e];
  const int W = (goff[e + 1] - g0) >> 5;
  unsigned long long* key = reinterpret_cast<unsigned long long*>(gsm);
  unsigned long long* m1 = key + nmax;
  uint32_t* alive = reinterpret_cast<uint32_t*>(m1 + nmax);
  uint32_t* win = alive + (nmax >> 5);
  uint32_t* cnt = win + (nmax >> 5);  // [2] alive counters (by round parity)
  uint32_t* rowc = cnt + 4;            // cache of this CTA's own adjacency rows (read-only for the whole kernel)
  const uint32_t* A = adj + (n > 0 ? adjoff[e] : 0);
  // owned rows [r0, r1)
  const int R = ((n + CS - 1) / CS + 31) / 32 * 32;
  const int r0 = min(n, rank * R), r1 = min(n, r0 + R);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;

  for (int w = threadIdx.x; w < W; w += blockDim.x) {
    const int valid = n - w * 32;
    alive[w] = valid >= 32 ? 0xffffffffu : (valid <= 0 ? 0u : ((1u << valid) - 1u));
    win[w] = 0u;
  }
  if (threadIdx.x < 2) cnt[threadIdx.x] = 0u;
  const int ncached = W > 0 ? min(r1 - r0, cache_words / W) : 0;
  for (int64_t i = threadIdx.x; i < (int64_t)ncached * W; i += blockDim.x) rowc[i] = A[(int64_t)r0 * W + i];
  auto ROW = [&](int r) -> const uint32_t* { return r - r0 < ncached ? rowc + (r - r0) * W : A + (int64_t)r * W; };
  for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) rep_local[g0 + r] = -1;
  if (rank == CS - 1)  // padding rows of the group's row space: never representatives
    for (int r = n + threadIdx.x; r < W * 32; r += blockDim.x) rep_local[g0 + r] = -1;
  cluster.sync();

  int round = 0;
  for (;; ++round) {
    if (round >= max_rounds) break;
    // ---- A: degree -> key, broadcast; count alive
    for (int w = threadIdx.x; w < W; w += blockDim.x) win[w] = 0u;
    for (int r = r0 + wid; r < r1; r += nwarp) {
      if (!((alive[r >> 5] >> (r & 31)) & 1u)) continue;
      const uint32_t* row = ROW(r);
      int deg = 0;
      for (int w = lane; w < W; w += 32) deg += __popc(row[w] & alive[w]);
      deg = __reduce_add_sync(0xffffffffu, deg);
      const unsigned long long k = ((unsigned long long)deg << 32) | (unsigned long long)(0xffffffffu - (uint32_t)r);
      if (lane < CS) *cluster.map_shared_rank(key + r, lane) = k;
      if (lane == 0) atomicAdd(cnt + (round & 1), 1u);
    }
    cluster.sync();
    uint32_t left = 0;
    for (int j = 0; j < CS; ++j) left += *cluster.map_shared_rank(cnt + (round & 1), j);
    if (left == 0u) break;
    // ---- B: m1 = max key over the alive closed neighbourhood (local replicas; set bits only)
    for (int r = r0 + wid; r < r1; r += nwarp) {
      if (!((alive[r >> 5] >> (r & 31)) & 1u)) continue;
      const uint32_t* row = ROW(r);
      unsigned long long m = key[r];
      for (int w = lane; w < W; w += 32) {
        uint32_t bits = row[w] & alive[w];
        while (bits) {
          const unsigned long long v = key[w * 32 + __ffs(bits) - 1];
          bits &= bits - 1u;
          m = v > m ? v : m;
        }
      }
      m = warp_max_u64(m);
      if (lane < CS) *cluster.map_shared_rank(m1 + r, lane) = m;
    }
    cluster.sync();
    // ---- C: winner iff max m1 over the alive closed neighbourhood equals key[r].  Every alive neighbour j
    // has m1[j] >= key[r] (r is in j's neighbourhood), so r wins iff m1[r] == key[r] and no alive neighbour
    // has m1[j] != key[r]: most rows lose without a scan and a scan stops at the first violation.
    for (int r = r0 + wid; r < r1; r += nwarp) {
      if (!((alive[r >> 5] >> (r & 31)) & 1u)) continue;
      const unsigned long long kr = key[r];
      if (m1[r] != kr) continue;
      const uint32_t* row = ROW(r);
      bool lose = false;
      for (int wb = 0; wb < W; wb += 32) {
        const int w = wb + lane;
        if (w < W) {
          uint32_t bits = row[w] & alive[w];
          while (bits && !lose) {
            lose = m1[w * 32 + __ffs(bits) - 1] != kr;
            bits &= bits - 1u;
          }
        }
        if (__any_sync(0xffffffffu, lose)) {
          lose = true;
          break;
        }
      }
      if (!lose && lane < CS) atomicOr(cluster.map_shared_rank(win + (r >> 5), lane), 1u << (r & 31));
    }
    cluster.sync();
    // ---- D: claims (a non-winner has at most one winner neighbour: winners are >= 3 hops apart)
    if (threadIdx.x == 0) cnt[(round + 1) & 1] = 0u;
    for (int r = r0 + wid; r < r1; r += nwarp) {
      if (!((alive[r >> 5] >> (r & 31)) & 1u)) continue;
      int owner = -1;
      if ((win[r >> 5] >> (r & 31)) & 1u) {
        owner = r;
      } else {
        const uint32_t* row = ROW(r);
        int found = 0x7fffffff;
        for (int w = lane; w < W; w += 32) {
          const uint32_t bits = row[w] & win[w];
          if (bits) found = min(found, w * 32 + __ffs(bits) - 1);
        }
        found = __reduce_min_sync(0xffffffffu, found);
        if (found != 0x7fffffff) owner = found;
      }
      if (owner >= 0) {
        if (lane == 0) rep_local[g0 + r] = g0 + owner;
        if (lane < CS) atomicAnd(cluster.map_shared_rank(alive + (r >> 5), lane), ~(1u << (r & 31)));
      }
    }
    cluster.sync();
  }
  if (rank == 0 && threadIdx.x == 0) atomicMax(ctrl + 2, (uint32_t)round);
  cluster.sync();  // no CTA may exit while a peer can still read its shared memory (the counters above)
}

template <int CS>
int launch_cluster(luffy_layer* L, int nmax, size_t smem, int cache_words, cudaStream_t st) {
  auto kern = greedy_cluster_kernel<CS>;
  LUFFY_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (CS > 8) LUFFY_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(L->E * CS);
  cfg.blockDim = dim3(GC_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  LUFFY_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, (const int32_t*)L->goff, (const int32_t*)L->gcnt,
                                    (const int64_t*)L->adjoff, (const uint32_t*)L->adj, L->rep_local, L->ctrl, nmax,
                                    kGreedyMaxRounds, cache_words));
  LUFFY_LAUNCHED();
  return 0;
}

}  // namespace

// Returns 0 on success, -1 if the cluster path does not apply (group capacity beyond shared memory).
int launch_greedy_cluster(luffy_layer* L, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  const int nmax = (int)round_up(std::min<int64_t>(L->Tmax, L->Cpad_max), 128);  // a group holds <= T copies
  const size_t state = (size_t)nmax * 16 + (size_t)(nmax / 32) * 8 + 16;
  if (state > 200 * 1024) return -1;
  const size_t cache_bytes = std::min<size_t>(224 * 1024 - state, 96 * 1024) / 16 * 16;  // own-row cache
  const size_t smem = state + cache_bytes;
  const int cache_words = (int)(cache_bytes / 4);
  LUFFY_CUDA_TRY(cudaMemsetAsync(L->ctrl, 0, sizeof(uint32_t) * 64, st));
  static int cs = 0;  // cluster size: 16 (non-portable) when the device accepts it, else 8
  if (cs == 0) {
    cs = 16;
    cudaFuncSetAttribute(greedy_cluster_kernel<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(greedy_cluster_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(GC_THREADS);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 16;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, greedy_cluster_kernel<16>, &cfg) != cudaSuccess || nclusters < 1) cs = 8;
    cudaGetLastError();
  }
  return cs == 16 ? launch_cluster<16>(L, nmax, smem, cache_words, st) : launch_cluster<8>(L, nmax, smem, cache_words, st);
}

}  // namespace luffy
