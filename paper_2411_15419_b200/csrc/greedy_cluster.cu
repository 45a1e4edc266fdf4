// Representative selection per expert group on a thread-block CLUSTER (DSMEM), the fast path of the
// exact parallel-rounds greedy (condense.cu has the algorithm statement).
//
// Groups are independent (only tokens of the same expert are compared), so each group gets its
// own cluster of CS CTAs (several groups per cluster, scheduled by cost, when fewer clusters fit than
// groups) and no grid-wide barrier is needed.  Every CTA owns a slice of the group's rows (whole 32-row
// words) and keeps REPLICAS of the group-wide state in its shared memory: the alive bitset, the winner
// bitset, the priority keys and the 1-hop maxima.  A phase writes only the CTA's own slice; after the
// cluster barrier every CTA copies the other slices through distributed shared memory (coalesced
// loads), so the neighbour maxima are read from local shared memory.  Phases:
//   A  residual degree -> key (broadcast); count alive rows
//   B  m1 = max key over the alive closed neighbourhood (broadcast)
//   C  m2 = max m1 over the alive closed neighbourhood; winner iff m2 == key (broadcast bit)
//   D  winners and their alive neighbours leave (rep = winner; alive bit cleared in every replica)
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace luffy {
namespace {

constexpr int GC_THREADS = 1024;

// Priority keys (residual degree, -index) packed into one integer (degree in the high half, so integer order
// is the greedy's order, R8); the cluster kernel uses 32-bit keys (groups < 65536 rows): one-word
// shared-memory traffic and compares.
template <typename KT>
__device__ __forceinline__ KT make_key(int deg, int r) {
  constexpr int S = sizeof(KT) * 4;
  constexpr KT M = (KT(1) << S) - 1;
  return (KT(deg) << S) | (M - KT(r));
}
template <typename KT>
__device__ __forceinline__ int key_deg(KT key) { return (int)(key >> (sizeof(KT) * 4)); }
__device__ __forceinline__ uint32_t warp_max_key(uint32_t v) { return __reduce_max_sync(0xffffffffu, v); }
__device__ __forceinline__ unsigned long long warp_max_key(unsigned long long v) { return warp_max_u64(v); }

template <int CS, typename KT>
__global__ void __launch_bounds__(GC_THREADS, 1) greedy_cluster_kernel(const int32_t* __restrict__ goff,
                                                                      const int32_t* __restrict__ gcnt,
                                                                      const int64_t* __restrict__ adjoff,
                                                                      const uint32_t* __restrict__ adj,
                                                                      int32_t* __restrict__ rep_local,
                                                                      uint32_t* __restrict__ ctrl, int nmax,
                                                                      int max_rounds, int cache_words, int E,
                                                                      int32_t* __restrict__ gnrep,
                                                                      int32_t* __restrict__ mrank,
                                                                      int32_t* __restrict__ mcnt_row,
                                                                      const uint32_t* __restrict__ gdone) {
  pdl_defer();
  // With the tensor-core Gram in front (gdone != nullptr) a group starts as soon as ITS pair tiles are in
  // (per-group counters, below) instead of waiting for the whole Gram grid: clusters take the SMs the Gram's
  // last partial wave leaves idle.  The grouping outputs read here were complete before the Gram released
  // its dependents (it waited for them first).
  if (gdone == nullptr) pdl_enter();
  else pdl_launch_only();
  extern __shared__ __align__(16) uint8_t gsm[];
  __shared__ int order_s[LUFFY_MAX_EXPERTS];
  __shared__ int list_s[LUFFY_MAX_EXPERTS];
  __shared__ int nlist_s, largest_s, nrep_s;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int cid = blockIdx.x / CS, ncl = gridDim.x / CS;
  // Groups -> clusters (fewer clusters than groups can be co-resident): longest-processing-time
  // assignment by cost n^2 (a round scans n rows of n/32 words), computed identically in every CTA:
  // rank by (cost desc, group asc), then each group to the least-loaded cluster (lowest index on ties).
  for (int i = threadIdx.x; i < E; i += blockDim.x) {
    const long long ci = (long long)gcnt[i] * gcnt[i];
    int rk = 0;
    for (int j = 0; j < E; ++j) {
      const long long cj = (long long)gcnt[j] * gcnt[j];
      rk += (cj > ci) || (cj == ci && j < i);
    }
    order_s[rk] = i;
  }
  __syncthreads();
  if (threadIdx.x == 0 && E <= ncl) {  // a cluster per group: LPT puts the r-th costliest on cluster r
    nlist_s = cid < E ? 1 : 0;
    if (cid < E) list_s[0] = order_s[cid];
    largest_s = order_s[0];
  } else if (threadIdx.x == 0) {
    long long load[32];
    for (int c = 0; c < ncl; ++c) load[c] = 0;
    int k = 0;
    for (int r = 0; r < E; ++r) {
      const int g = order_s[r];
      int best = 0;
      for (int c = 1; c < ncl; ++c)
        if (load[c] < load[best]) best = c;
      load[best] += (long long)gcnt[g] * gcnt[g] + 1;
      if (best == cid) list_s[k++] = g;
    }
    nlist_s = k;
    largest_s = order_s[0];
  }
  __syncthreads();
  int round = 0, max_round = 0;
  for (int gi = 0; gi < nlist_s; ++gi) {
  const int e = list_s[gi];
  const int g0 = goff[e];
  const int n = gcnt[e];
  const int W = (goff[e + 1] - g0) >> 5;
  if (gdone != nullptr) {  // this group's adjacency complete: 2 arrivals per pair tile
    if (threadIdx.x == 0) {
      const int nt = (W * 32 / 128 + 1) / 2;
      const uint32_t need = (uint32_t)(nt * (nt + 1));
      uint32_t got;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(got) : "l"(gdone + e) : "memory");
        if (got >= need) break;
        __nanosleep(100);
      }
    }
    __syncthreads();
  }
  KT* key = reinterpret_cast<KT*>(gsm);
  KT* m1 = key + nmax;
  uint32_t* alive = reinterpret_cast<uint32_t*>(m1 + nmax);
  uint32_t* win = alive + (nmax >> 5);
  uint32_t* cnt = win + (nmax >> 5);  // [2] alive counters (by round parity)
  uint32_t* rowc = cnt + 4;            // cache of this CTA's own adjacency rows (read-only for the whole kernel)
  const uint32_t* A = adj + (n > 0 ? adjoff[e] : 0);
  // owned rows [r0, r1)
  const int R = ((n + CS - 1) / CS + 31) / 32 * 32;
  const int r0 = min(n, rank * R), r1 = min(n, r0 + R);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  // phase timeline of the largest group (debug export LUFFY_DBG_GREEDY_TIMES): rank 0, thread 0
  const bool stamp = rank == 0 && threadIdx.x == 0 && e == largest_s;
  int nst = 0;
  auto STAMP = [&]() {
    if (stamp && nst < 28) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ctrl[8 + 2 * nst] = (uint32_t)t;
      ctrl[9 + 2 * nst] = (uint32_t)(t >> 32);
      ctrl[3] = (uint32_t)++nst;
    }
  };
  STAMP();
  // finer stamps (compute end, cluster barrier end) with LUFFY_GREEDY_FINE=1 builds only
#ifdef LUFFY_GREEDY_FINE
  auto FSTAMP = [&]() { STAMP(); };
#else
  auto FSTAMP = [&]() {};
#endif

  for (int w = threadIdx.x; w < W; w += blockDim.x) {
    const int valid = n - w * 32;
    alive[w] = valid >= 32 ? 0xffffffffu : (valid <= 0 ? 0u : ((1u << valid) - 1u));
    win[w] = 0u;
  }
  if (threadIdx.x < 2) cnt[threadIdx.x] = 0u;
  const int ncached = W > 0 ? min(r1 - r0, cache_words / W) : 0;
  {  // own rows -> shared memory, 16-byte vectors (row blocks start at multiples of 32 rows x W % 4 == 0 words)
    const uint4* src = reinterpret_cast<const uint4*>(A + (int64_t)r0 * W);
    uint4* dst = reinterpret_cast<uint4*>(rowc);
    const int nv = ncached * W / 4;
#pragma unroll 4
    for (int i = threadIdx.x; i < nv; i += blockDim.x) dst[i] = src[i];
  }
  // word w of adjacency row r: a shared-memory load for the cached rows (all of them at the usual group
  // sizes), a global load otherwise -- two explicit address spaces instead of one generic pointer
  auto RW = [&](int r, int w) -> uint32_t {
    return r - r0 < ncached ? rowc[(r - r0) * W + w] : __ldg(A + (int64_t)r * W + w);
  };
  for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) rep_local[g0 + r] = -1;
  if (rank == CS - 1)  // padding rows of the group's row space: never representatives
    for (int r = n + threadIdx.x; r < W * 32; r += blockDim.x) rep_local[g0 + r] = -1;
  __syncthreads();  // replicas and the row cache are read by every warp of the CTA
  STAMP();  // replicas initialised, own rows cached
  // Replica exchange: in every phase a CTA writes only its OWN slice (rows [r0, r1) of key / m1, words
  // [r0/32, (r0+R)/32) of win / alive; R is a multiple of 32) in its shared memory; after the cluster
  // barrier every CTA copies the other slices from their shared memory with coalesced DSMEM loads.
  auto gather_rows = [&](KT* arr) {
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
      const int j = r / R;
      if (j != rank) arr[r] = *cluster.map_shared_rank(arr + r, j);
    }
  };
  auto gather_words = [&](uint32_t* arr) {
    for (int w = threadIdx.x; w < W; w += blockDim.x) {
      const int j = (w * 32) / R;
      if (j != rank && j < CS) arr[w] = *cluster.map_shared_rank(arr + w, j);
    }
  };
  const int w0 = r0 >> 5, w1 = min(W, (rank * R + R) >> 5);  // owned words

  for (round = 0;; ++round) {
    if (round >= max_rounds) break;
    // alive rows left (identical in every replica): every warp counts, so the exit is uniform
    int left = 0;
    for (int w = lane; w < W; w += 32) left += __popc(alive[w]);
    if (__reduce_add_sync(0xffffffffu, left) == 0) break;
    // ---- A: residual degree -> key (own rows)
    FSTAMP();
    for (int w = w0 + threadIdx.x; w < w1; w += blockDim.x) win[w] = 0u;
    // one thread per row: W independent word loads and popcounts per thread, no cross-lane reduction
    for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
      if (!((alive[r >> 5] >> (r & 31)) & 1u)) continue;
      int deg = 0;
      for (int w = 0; w < W; ++w) deg += __popc(RW(r, w) & alive[w]);
      key[r] = make_key<KT>(deg, r);
    }
    FSTAMP();
    cluster.sync();
    FSTAMP();
    gather_rows(key);
    __syncthreads();
    STAMP();
    // ---- B: m1 = max key over the alive closed neighbourhood (own rows; set bits only)
    for (int r = r0 + wid; r < r1; r += nwarp) {
      if (!((alive[r >> 5] >> (r & 31)) & 1u)) continue;
      KT m = key[r];
      if (key_deg(m) == 0) {  // no alive neighbour: m1 = own key, no scan
        if (lane == 0) m1[r] = m;
        continue;
      }
      for (int w = lane; w < W; w += 32) {
        uint32_t bits = RW(r, w) & alive[w];
        while (bits) {
          const KT v = key[w * 32 + __ffs(bits) - 1];
          bits &= bits - 1u;
          m = v > m ? v : m;
        }
      }
      m = warp_max_key(m);
      if (lane == 0) m1[r] = m;
    }
    FSTAMP();
    cluster.sync();
    FSTAMP();
    gather_rows(m1);
    __syncthreads();
    STAMP();
    // ---- C: winner iff max m1 over the alive closed neighbourhood equals key[r].  Every alive neighbour j
    // has m1[j] >= key[r] (r is in j's neighbourhood), so r wins iff m1[r] == key[r] and no alive neighbour
    // has m1[j] != key[r]: most rows lose without a scan and a scan stops at the first violation.
    for (int r = r0 + wid; r < r1; r += nwarp) {
      if (!((alive[r >> 5] >> (r & 31)) & 1u)) continue;
      const KT kr = key[r];
      if (m1[r] != kr) continue;
      if (key_deg(kr) == 0) {  // isolated among the alive rows: wins without a scan
        if (lane == 0) atomicOr(win + (r >> 5), 1u << (r & 31));
        continue;
      }
      bool lose = false;
      for (int wb = 0; wb < W; wb += 32) {
        const int w = wb + lane;
        if (w < W) {
          uint32_t bits = RW(r, w) & alive[w];
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
      if (!lose && lane == 0) atomicOr(win + (r >> 5), 1u << (r & 31));
    }
    FSTAMP();
    cluster.sync();
    FSTAMP();
    gather_words(win);
    __syncthreads();
    STAMP();
    // ---- D0: member lists of this slice's winners, for the layout: a winner claims itself and its alive
    // neighbours (the alive replica still holds the state before this phase's claims), so its members in
    // token order are the set bits of (row & alive) | self -- each member's rank in that list and the
    // list's length are written here, which makes the layout's member placement a direct store
    for (int r = r0 + wid; r < r1; r += nwarp) {
      if (!((win[r >> 5] >> (r & 31)) & 1u)) continue;
      if (key_deg(key[r]) == 0) {  // a winner without alive neighbours is its own only member
        if (lane == 0) {
          mrank[g0 + r] = 0;
          mcnt_row[g0 + r] = 1;
        }
        continue;
      }
      int base = 0;
      for (int w0 = 0; w0 < W; w0 += 32) {
        const int w = w0 + lane;
        uint32_t m = w < W ? (RW(r, w) & alive[w]) : 0u;
        if (w == (r >> 5)) m |= 1u << (r & 31);
        const int cnt = __popc(m);
        int inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += u;
        }
        int k = base + inc - cnt;
        while (m) {
          const int b = __ffs(m) - 1;
          m &= m - 1u;
          mrank[g0 + 32 * w + b] = k++;
        }
        base += __shfl_sync(0xffffffffu, inc, 31);
      }
      if (lane == 0) mcnt_row[g0 + r] = base;
    }
    __syncthreads();  // the alive replica is read above before this CTA's own claims clear its words
    // ---- D: claims (a non-winner has at most one winner neighbour: winners are >= 3 hops apart)
    for (int r = r0 + wid; r < r1; r += nwarp) {
      if (!((alive[r >> 5] >> (r & 31)) & 1u)) continue;
      int owner = -1;
      if ((win[r >> 5] >> (r & 31)) & 1u) {
        owner = r;
      } else {
        int found = 0x7fffffff;
        for (int w = lane; w < W; w += 32) {
          const uint32_t bits = RW(r, w) & win[w];
          if (bits) found = min(found, w * 32 + __ffs(bits) - 1);
        }
        found = __reduce_min_sync(0xffffffffu, found);
        if (found != 0x7fffffff) owner = found;
      }
      if (owner >= 0 && lane == 0) {
        rep_local[g0 + r] = g0 + owner;
        atomicAnd(alive + (r >> 5), ~(1u << (r & 31)));
      }
    }
    FSTAMP();
    cluster.sync();
    FSTAMP();
    gather_words(alive);
    __syncthreads();
    STAMP();
  }
  max_round = max(max_round, round);
  cluster.sync();  // the replicas are reused by the next group, and no CTA may exit while a peer can still
                   // read its shared memory
  if (rank == 0) {  // publish the group's representative count (read by the layout for the send offsets)
    if (threadIdx.x == 0) nrep_s = 0;
    __syncthreads();
    int c = 0;
    for (int r = threadIdx.x; r < n; r += blockDim.x) c += rep_local[g0 + r] == g0 + r;
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0 && c) atomicAdd(&nrep_s, c);
    __syncthreads();
    if (threadIdx.x == 0) gnrep[e] = nrep_s;
    __syncthreads();
  }
  }
  if (rank == 0 && threadIdx.x == 0) atomicMax(ctrl + 2, (uint32_t)max_round);
}

template <int CS, typename KT>
int launch_cluster(luffy_layer* L, int nmax, size_t smem, int cache_words, int nclusters, cudaStream_t st) {
  auto kern = greedy_cluster_kernel<CS, KT>;
  LUFFY_CUDA_TRY(smem_optin((const void*)kern, (int)smem));
  if (CS > 8) LUFFY_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(std::min(L->E, std::max(1, std::min(nclusters, 32))) * CS);
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
                                    kGreedyMaxRounds, cache_words, L->E, L->gnrep, L->mrank, L->mcnt_row,
                                    (const uint32_t*)(L->gdone_live && pdl_enabled() ? L->gdone : nullptr)));
  LUFFY_LAUNCHED();
  return 0;
}

}  // namespace

// Returns 0 on success, -1 if the cluster path does not apply (group capacity beyond shared memory).
int launch_greedy_cluster(luffy_layer* L, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  const int nmax = (int)round_up(std::min<int64_t>(L->Tmax, L->Cpad_max), 128);  // a group holds <= T copies
  // 32-bit priority keys (make_key): the shared-memory budget below caps a group at 25600 rows < 65536
  const size_t state = (size_t)nmax * 8 + (size_t)(nmax / 32) * 8 + 16;
  if (state > 200 * 1024) return -1;
  const size_t cache_bytes = (224 * 1024 - state) / 16 * 16;  // own-row cache
  const size_t smem = state + cache_bytes;
  const int cache_words = (int)(cache_bytes / 4);
  // (the control block is zeroed by gather_norm_kernel, which precedes the Gram)
  // Cluster size: 16 CTAs when every group gets its own co-resident cluster, else 8 (twice as many clusters;
  // the groups are scheduled by cost onto them).  On B200 only 7 clusters of 16 (or of 12) and 15 of 8 fit.
  // the choice depends on (device, shared-memory size, E): cached per device under that key
  static const char tag = 0;
  int cs = 0, ncl = 0, packed = 0;
  const int64_t ckey = ((int64_t)smem << 16) | L->E;
  if (dev_cache_get(&tag, ckey, &packed)) {
    cs = packed >> 16;
    ncl = packed & 0xffff;
  } else {
    auto coresident = [&](auto kern, int size) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      smem_optin((const void*)kern, (int)smem);
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(size);
      cfg.blockDim = dim3(GC_THREADS);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = size;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) n = 0;
      cudaGetLastError();
      return n;
    };
    const int n16 = coresident(greedy_cluster_kernel<16, uint32_t>, 16);
    const int n12 = coresident(greedy_cluster_kernel<12, uint32_t>, 12);
    const int n8 = coresident(greedy_cluster_kernel<8, uint32_t>, 8);
    const char* force = std::getenv("LUFFY_GREEDY_CS");  // experiments: 16 / 12 / 8
    const int f = force ? std::atoi(force) : 0;
    if (f == 16 && n16 >= 1) { cs = 16; ncl = n16; }
    else if (f == 12 && n12 >= 1) { cs = 12; ncl = n12; }
    else if (f == 8 && n8 >= 1) { cs = 8; ncl = n8; }
    else if (n16 >= L->E) { cs = 16; ncl = n16; }  // every group on its own 16-CTA cluster
    else if (n8 >= 1) { cs = 8; ncl = n8; }         // more groups than clusters: twice as many clusters
    else { cs = 16; ncl = std::max(1, n16); }       // (measured: C2 44 us either way, C4 55 vs 69 us)
    if (std::getenv("LUFFY_VERBOSE"))
      std::fprintf(stderr, "[luffy] greedy clusters co-resident: %d x16, %d x12, %d x8 CTAs (smem %zu); using %d x %d\n",
                   n16, n12, n8, smem, ncl, cs);
    dev_cache_put(&tag, ckey, (cs << 16) | (ncl & 0xffff));
  }
  if (cs == 16) return launch_cluster<16, uint32_t>(L, nmax, smem, cache_words, ncl, st);
  if (cs == 12) return launch_cluster<12, uint32_t>(L, nmax, smem, cache_words, ncl, st);
  return launch_cluster<8, uint32_t>(L, nmax, smem, cache_words, ncl, st);
}

}  // namespace luffy
