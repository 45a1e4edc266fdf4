// Token condensation (token_to_token map P:405).
//
//  1. group_build: fast-similarity step 1 -- only copies routed to the same expert are compared.
//     Group e = copies (t, j) with idx[t, j] == e in ascending token order (R6), laid out in a padded
//     expert-major row space (segments of LUFFY_ROW_ALIGN rows).
//  2. gather_norm: the group rows (xg) and their fp64 norms.
//  3. gram: step 3 -- G = Xg Xg^T on upper-triangle tiles; the epilogue applies the threshold
//     (R4): edge(i, j) iff G_ij >= (2h - 1) |x_i| |x_j|, i != j, both norms > 0 (R7), and packs
//     the bits of (i, j) and (j, i) so the graph is symmetric by construction.  (bf16: tcgen05 kernel in
//     gram_tc.cu; fp32: the SIMT tile kernel below, exact fp32 FFMA.)
//  4. greedy: "keep the token with the highest degree ... condense its neighbouring tokens ... repeat"
//      with the dynamic residual degree and lowest-index ties (R8), computed EXACTLY by parallel
//     2-hop rounds: an alive node whose (degree, -index) is the strict maximum of its alive 2-hop ball
//     is selected together with all its alive neighbours; such winners are >= 3 hops apart, so their
//     claims are disjoint and commute with the sequential greedy.  One cooperative
//     kernel, grid-wide barriers between the phases of a round.
#include <cooperative_groups.h>

#include "common.cuh"

namespace luffy {
namespace {

// Grouping (fast-similarity step 1) in two launches over token chunks of GB_TCH tokens:
//  group_count_kernel   per chunk, copies per expert; the last CTA to finish (ticket) scans the chunk
//                       counts per expert into chunk prefixes and derives gcnt, goff (segments padded to
//                       kRowAlign), the adjacency word offsets and the greedy control block;
//  group_place_kernel   per chunk, the group row of every copy = goff[e] + chunk prefix + rank among the
//                       chunk's copies of e in token order (per-expert token bitmaps in shared memory), then
//                       one warp per token copies its row into each of its k group rows and writes the fp64
//                       norm -- x is read once per token.  Padding rows are zeroed.
constexpr int GB_TCH = 128;

__global__ void __launch_bounds__(GB_TCH) group_count_kernel(const int32_t* __restrict__ idx, int T, int k, int E,
                                                            int32_t* __restrict__ chunk, uint32_t* __restrict__ ticket,
                                                            int32_t* __restrict__ gcnt, int32_t* __restrict__ goff,
                                                            int64_t* __restrict__ adjoff, uint32_t* __restrict__ ctrl,
                                                            uint32_t* __restrict__ gdone) {
  pdl_enter();
  __shared__ int cnt[LUFFY_MAX_EXPERTS];
  __shared__ bool last;
  const int c = blockIdx.x, nch = gridDim.x;
  for (int e = threadIdx.x; e < E; e += blockDim.x) cnt[e] = 0;
  __syncthreads();
  const int t = c * GB_TCH + threadIdx.x;
  if (t < T)
    for (int j = 0; j < k; ++j) atomicAdd(&cnt[idx[(size_t)t * k + j]], 1);
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) chunk[(size_t)c * E + e] = cnt[e];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == (uint32_t)nch - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // last CTA: exclusive prefix over chunks per expert (in place), totals, padded offsets.  One warp per
  // expert scans its chunk column (lanes over chunks, all loads independent, warp shuffles for the sums).
  {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int e = wid; e < E; e += nw) {
      int carry = 0;
      for (int c0 = 0; c0 < nch; c0 += 32) {
        const int cc = c0 + lane;
        const int v = cc < nch ? __ldcg(chunk + (size_t)cc * E + e) : 0;
        int inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += u;
        }
        if (cc < nch) chunk[(size_t)cc * E + e] = carry + inc - v;
        carry += __shfl_sync(0xffffffffu, inc, 31);
      }
      if (lane == 0) {
        cnt[e] = carry;
        gcnt[e] = carry;
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 64; i += blockDim.x) ctrl[i] = 0u;  // greedy control block reset
  for (int i = threadIdx.x; i < E; i += blockDim.x) gdone[i] = 0u;  // Gram tiles finished per group
  __syncthreads();
  if (threadIdx.x == 0) {
    int o = 0;
    int64_t w = 0;
    for (int e = 0; e < E; ++e) {
      goff[e] = o;
      adjoff[e] = w;
      const int np = (cnt[e] + kRowAlign - 1) / kRowAlign * kRowAlign;
      o += np;
      w += (int64_t)np * np / 32;
    }
    goff[E] = o;
    adjoff[E] = w;
    *ticket = 0u;
  }
}

constexpr int GB_SUB = 4;  // placement CTAs per count chunk (GB_TCH / GB_SUB tokens each)

template <typename T>
__global__ void __launch_bounds__(256) group_place_kernel(const T* __restrict__ x, const int32_t* __restrict__ idx,
                                                          const float* __restrict__ w, int Tn, int k, int E, int d,
                                                          const int32_t* __restrict__ chunk, const int32_t* __restrict__ gcnt,
                                                          const int32_t* __restrict__ goff, int32_t* __restrict__ gtok,
                                                          float* __restrict__ gw, int32_t* __restrict__ gloc,
                                                          int32_t* __restrict__ gcopy, T* __restrict__ xg,
                                                          double* __restrict__ gnorm) {
  pdl_enter();
  constexpr int SUB = GB_TCH / GB_SUB;
  __shared__ uint32_t bits[LUFFY_MAX_EXPERTS][GB_TCH / 32];
  __shared__ int32_t base_s[LUFFY_MAX_EXPERTS];
  __shared__ int32_t rows_s[SUB][8];
  const int c = blockIdx.x / GB_SUB, sub = blockIdx.x % GB_SUB, ncta = gridDim.x;
  const int t0 = c * GB_TCH;
  const int nt = min(GB_TCH, Tn - t0);                 // tokens of the chunk
  const int s0 = min(sub * SUB, nt), ns = min(SUB, nt - s0);  // this CTA's tokens within the chunk (may be 0)
  for (int i = threadIdx.x; i < E * (GB_TCH / 32); i += blockDim.x) bits[i / (GB_TCH / 32)][i % (GB_TCH / 32)] = 0u;
  for (int e = threadIdx.x; e < E; e += blockDim.x) base_s[e] = goff[e] + chunk[(size_t)c * E + e];
  __syncthreads();
  for (int i = threadIdx.x; i < (s0 + ns) * k; i += blockDim.x) {  // bitmaps of the chunk's tokens up to ours
    const int tl = i / k;
    atomicOr(&bits[idx[(size_t)(t0 + tl) * k + i % k]][tl >> 5], 1u << (tl & 31));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ns * k; i += blockDim.x) {
    const int tl = s0 + i / k, j = i % k;
    const int t = t0 + tl;
    const int e = idx[(size_t)t * k + j];
    int rank = __popc(bits[e][tl >> 5] & ((1u << (tl & 31)) - 1u));
    for (int q = 0; q < (tl >> 5); ++q) rank += __popc(bits[e][q]);
    const int g = base_s[e] + rank;
    rows_s[tl - s0][j] = g;
    gtok[g] = t;
    gw[g] = w[(size_t)t * k + j];
    gloc[(size_t)t * k + j] = g;
    gcopy[g] = t * k + j;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int tl = wid; tl < ns; tl += nw) {  // one warp per token: its row into each of its k group rows
    const T* src = x + (size_t)(t0 + s0 + tl) * d;
    double ss = 0.0;
    for (int cb = 0; cb < d; cb += 4 * 256) {  // batches of 4 independent 16-byte loads per lane (bf16)
      uint4 u[4][sizeof(T) / 2];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int cc = cb + b * 256 + lane * 8;
        if (cc < d)
#pragma unroll
          for (int h = 0; h < (int)(sizeof(T) / 2); ++h) u[b][h] = reinterpret_cast<const uint4*>(src + cc)[h];
      }
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int cc = cb + b * 256 + lane * 8;
        if (cc >= d) break;
        for (int j = 0; j < k; ++j)
#pragma unroll
          for (int h = 0; h < (int)(sizeof(T) / 2); ++h)
            reinterpret_cast<uint4*>(xg + (size_t)rows_s[tl][j] * d + cc)[h] = u[b][h];
        float v[8];
        load8(reinterpret_cast<const T*>(&u[b][0]), v);
#pragma unroll
        for (int i = 0; i < 8; ++i) ss += (double)v[i] * (double)v[i];
      }
    }
    ss = warp_sum_d(ss);
    if (lane < k) gnorm[rows_s[tl][lane]] = sqrt(ss);
  }
  // padding rows of the group row space: zero rows, no token; spread over the CTAs
  for (int e = 0; e < E; ++e) {
    const int p0 = goff[e] + gcnt[e], p1 = goff[e + 1];
    for (int r = p0 + blockIdx.x * nw + wid; r < p1; r += ncta * nw) {
      for (int cc = lane * 8; cc < d; cc += 256) zero8(xg + (size_t)r * d + cc);
      if (lane == 0) {
        gtok[r] = -1;
        gw[r] = 0.f;
        gcopy[r] = -1;
        gnorm[r] = 0.0;
      }
    }
  }
}

// Decode a linear upper-triangle tile id into (group, I, J), J >= I, for tiles of `TS` rows.
__device__ __forceinline__ bool decode_tri_tile(int64_t id, const int32_t* goff_s, int E, int TS, int& e, int& I, int& J) {
  for (e = 0; e < E; ++e) {
    const int nt = (goff_s[e + 1] - goff_s[e]) / TS;
    const int64_t pairs = (int64_t)nt * (nt + 1) / 2;
    if (id < pairs) {
      // row I holds tiles J = I..nt-1; find I
      int i = 0;
      int64_t rem = id;
      while (rem >= nt - i) { rem -= nt - i; ++i; }
      I = i;
      J = i + (int)rem;
      return true;
    }
    id -= pairs;
  }
  return false;
}

// SIMT Gram + threshold + bit pack, fp32 FFMA (the fp32 path; also usable for bf16 inputs).
// 64x64 tiles, 256 threads, 4x4 outputs per thread, K staged through shared memory.
template <typename T>
__global__ void __launch_bounds__(256) gram_simt_kernel(const T* __restrict__ xg, const double* __restrict__ gnorm,
                                                        const int32_t* __restrict__ goff, const int32_t* __restrict__ gcnt,
                                                        const int64_t* __restrict__ adjoff, int E, int d, double c2h,
                                                        uint32_t* __restrict__ adj, float* __restrict__ gdump,
                                                        int64_t gdump_cap, unsigned long long* __restrict__ band) {
  pdl_enter();
  constexpr int TS = 64, BK = 32;
  __shared__ float As[BK][TS + 4];
  __shared__ float Bs[BK][TS + 4];
  __shared__ unsigned char edge[TS][TS + 4];
  __shared__ int32_t goff_s[LUFFY_MAX_EXPERTS + 1];
  for (int i = threadIdx.x; i <= E; i += blockDim.x) goff_s[i] = goff[i];
  __syncthreads();
  int e, I, J;
  if (!decode_tri_tile(blockIdx.x, goff_s, E, TS, e, I, J)) return;
  const int n = gcnt[e];
  const int npad = goff_s[e + 1] - goff_s[e];
  const int W = npad / 32;
  const T* A = xg + (size_t)(goff_s[e] + I * TS) * d;
  const T* B = xg + (size_t)(goff_s[e] + J * TS) * d;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < d; k0 += BK) {
    // load 64 rows x 32 k of A and B (transposed into [k][row])
    for (int i = threadIdx.x; i < TS * BK; i += blockDim.x) {
      const int r = i / BK, kk = i % BK;
      As[kk][r] = to_f(A[(size_t)r * d + k0 + kk]);
      Bs[kk][r] = to_f(B[(size_t)r * d + k0 + kk]);
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = As[kk][ty * 4 + i]; b[i] = Bs[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  int nband = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int li = I * TS + ty * 4 + i;
    const double ni = gnorm[goff_s[e] + li];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int lj = J * TS + tx * 4 + j;
      const double nj = gnorm[goff_s[e] + lj];
      const bool pair = li < n && lj < n && li != lj && ni > 0.0 && nj > 0.0;
      bool on = pair && (double)acc[i][j] >= c2h * ni * nj;
      edge[ty * 4 + i][tx * 4 + j] = on;
      if (band && pair && li < lj && fabs((double)acc[i][j] - c2h * ni * nj) <= 2e-5 * ni * nj) ++nband;
      if (gdump) {  // debug export of the accumulator (same layout as the tcgen05 Gram's)
        const int64_t o = adjoff[e] * 32 + (int64_t)li * npad + lj;
        if (o < gdump_cap) gdump[o] = acc[i][j];
      }
    }
  }
  if (band && nband) atomicAdd(band, (unsigned long long)nband);
  __syncthreads();
  uint32_t* base = adj + adjoff[e];
  const int t = threadIdx.x;
  if (I < J) {
    if (t < 128) {  // direct words: row I*64 + r, word J*2 + h
      const int r = t >> 1, h = t & 1;
      uint32_t word = 0;
      for (int b = 0; b < 32; ++b) word |= (uint32_t)edge[r][h * 32 + b] << b;
      base[(size_t)(I * TS + r) * W + J * 2 + h] = word;
    } else {        // transposed words: row J*64 + c, word I*2 + h
      const int c = (t - 128) >> 1, h = (t - 128) & 1;
      uint32_t word = 0;
      for (int b = 0; b < 32; ++b) word |= (uint32_t)edge[h * 32 + b][c] << b;
      base[(size_t)(J * TS + c) * W + I * 2 + h] = word;
    }
  } else if (t < 128) {  // diagonal tile: bit (r, c) = c > r ? edge[r][c] : c < r ? edge[c][r] : 0
    const int r = t >> 1, h = t & 1;
    uint32_t word = 0;
    for (int b = 0; b < 32; ++b) {
      const int c = h * 32 + b;
      const unsigned char v = c > r ? edge[r][c] : (c < r ? edge[c][r] : 0);
      word |= (uint32_t)v << b;
    }
    base[(size_t)(I * TS + r) * W + I * 2 + h] = word;
  }
}

// ---------------------------------------------------------------------------------------------------
// Greedy representative selection by exact parallel 2-hop rounds (cooperative launch).

__device__ __forceinline__ void stamp(uint32_t* ctrl) {
  // phase timeline for the debug export: block 0 records %globaltimer (ns) at every barrier
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const uint32_t i = ctrl[3];
    if (i < 28) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ctrl[8 + 2 * i] = (uint32_t)t;
      ctrl[9 + 2 * i] = (uint32_t)(t >> 32);
      ctrl[3] = i + 1;
    }
  }
}

__device__ __forceinline__ void grid_barrier(uint32_t* ctrl) {
  stamp(ctrl);
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile uint32_t* vgen = ctrl + 1;
    const uint32_t gen = *vgen;
    __threadfence();
    const uint32_t arrived = atomicAdd(ctrl, 1u);
    if (arrived == gridDim.x - 1) {
      atomicExch(ctrl, 0u);
      __threadfence();
      atomicAdd(ctrl + 1, 1u);
    } else {
      while (*vgen == gen) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

struct GreedyArgs {
  int E;
  const int32_t* goff;
  const int32_t* gcnt;
  const int64_t* adjoff;
  const uint32_t* adj;
  uint32_t* alive;
  uint32_t* win;
  unsigned long long* key;
  unsigned long long* m1;
  unsigned long long* m2;
  int32_t* rep_local;
  uint32_t* ctrl;
  int max_rounds;
};

__global__ void __launch_bounds__(256) greedy_kernel(GreedyArgs a) {
  pdl_enter();
  __shared__ int32_t goff_s[LUFFY_MAX_EXPERTS + 1];
  __shared__ int64_t adjoff_s[LUFFY_MAX_EXPERTS + 1];
  __shared__ int32_t gcnt_s[LUFFY_MAX_EXPERTS];
  const int E = a.E;
  for (int i = threadIdx.x; i <= E; i += blockDim.x) {
    goff_s[i] = a.goff[i];
    adjoff_s[i] = a.adjoff[i];
    if (i < E) gcnt_s[i] = a.gcnt[i];
  }
  __syncthreads();
  const int rows = goff_s[E];
  const int lane = threadIdx.x & 31;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int gwarp = (int)(gtid >> 5);
  const int nwarps = (int)(nthreads >> 5);

  for (int64_t wd = gtid; wd < rows / 32; wd += nthreads) {
    const int r0 = (int)wd * 32;
    const int g = find_group(goff_s, E, r0);
    const int valid = gcnt_s[g] - (r0 - goff_s[g]);
    a.alive[wd] = valid >= 32 ? 0xffffffffu : (valid <= 0 ? 0u : ((1u << valid) - 1u));
    a.win[wd] = 0u;
  }
  for (int64_t r = gtid; r < rows; r += nthreads) {
    a.rep_local[r] = -1;
    a.m1[r] = 0ull;
    a.m2[r] = 0ull;
  }
  grid_barrier(a.ctrl);

  // Two rows per warp (16 lanes per row).  The 1-hop and 2-hop maxima are PUSHED: every alive node
  // atomically max-es its value into its alive neighbours (no return value -> no load latency in the bit
  // walk; max is commutative, so the result equals the gather formulation).  3 barriers per round:
  //   A: residual degree -> key; push key into m1 (closed neighbourhood); count the alive nodes
  //   B: push m1 into m2
  //   C: winners (m2 == key) claim themselves and their alive neighbours (winners are >= 3 hops apart,
  //      so no node is claimed twice and no alive bit is read by one winner while another clears it)
  const int hl = lane & 15;
  const int half = lane >> 4;
  const int pairs = rows >> 1;
  int round = 0;
  for (;; ++round) {
    if (round >= a.max_rounds) break;
    // ---- phase A
    for (int p = gwarp; p < pairs; p += nwarps) {
      const int r = 2 * p + half;
      const uint32_t aw = __ldcg(a.alive + (r >> 5));
      if (!((aw >> ((2 * p) & 31)) & 3u)) continue;
      const bool me = (aw >> (r & 31)) & 1u;
      const int g = find_group(goff_s, E, r);
      const int rl = r - goff_s[g];
      const int W = (goff_s[g + 1] - goff_s[g]) >> 5;
      const uint32_t* row = a.adj + adjoff_s[g] + (int64_t)rl * W;
      const uint32_t* al = a.alive + (goff_s[g] >> 5);
      int deg = 0;
      if (me)
        for (int wd = hl; wd < W; wd += 16) deg += __popc(row[wd] & __ldcg(al + wd));
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) deg += __shfl_xor_sync(0xffffffffu, deg, o);
      if (me) {
        const unsigned long long key = ((unsigned long long)deg << 32) | (unsigned long long)(0xffffffffu - (uint32_t)rl);
        if (hl == 0) {
          a.key[r] = key;
          atomicMax(a.m1 + r, key);
          atomicAdd(a.ctrl + 64 + round, 1u);
        }
        unsigned long long* m1g = a.m1 + goff_s[g];
        for (int wd = hl; wd < W; wd += 16) {
          uint32_t bits = row[wd] & __ldcg(al + wd);
          while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            atomicMax(m1g + wd * 32 + b, key);
          }
        }
      }
    }
    grid_barrier(a.ctrl);
    if (__ldcg(a.ctrl + 64 + round) == 0u) break;
    // ---- phase B (warp-uniform control flow: both half-warps run every iteration; work is predicated)
    for (int p = gwarp; p < pairs; p += nwarps) {
      const int r = 2 * p + half;
      const uint32_t aw = __ldcg(a.alive + (r >> 5));
      if (!((aw >> ((2 * p) & 31)) & 3u)) continue;
      const bool me = (aw >> (r & 31)) & 1u;
      const int g = find_group(goff_s, E, r);
      const int rl = r - goff_s[g];
      const int W = (goff_s[g + 1] - goff_s[g]) >> 5;
      const uint32_t* row = a.adj + adjoff_s[g] + (int64_t)rl * W;
      const uint32_t* al = a.alive + (goff_s[g] >> 5);
      const unsigned long long v = me ? __ldcg(a.m1 + r) : 0ull;
      __syncwarp();
      if (me && hl == 0) {
        atomicMax(a.m2 + r, v);
        a.m1[r] = 0ull;  // reset for the next round (no more pushes into m1 this round)
      }
      if (me) {
        unsigned long long* m2g = a.m2 + goff_s[g];
        for (int wd = hl; wd < W; wd += 16) {
          uint32_t bits = row[wd] & __ldcg(al + wd);
          while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            atomicMax(m2g + wd * 32 + b, v);
          }
        }
      }
      __syncwarp();
    }
    grid_barrier(a.ctrl);
    // ---- phase C: winners claim
    for (int p = gwarp; p < pairs; p += nwarps) {
      const int r = 2 * p + half;
      const uint32_t aw = __ldcg(a.alive + (r >> 5));
      if (!((aw >> ((2 * p) & 31)) & 3u)) continue;
      const bool me = (aw >> (r & 31)) & 1u;
      const bool winner = me && __ldcg(a.m2 + r) == __ldcg(a.key + r);
      __syncwarp();
      if (me && hl == 0) a.m2[r] = 0ull;
      if (winner) {
        const int g = find_group(goff_s, E, r);
        const int rl = r - goff_s[g];
        const int W = (goff_s[g + 1] - goff_s[g]) >> 5;
        const uint32_t* row = a.adj + adjoff_s[g] + (int64_t)rl * W;
        uint32_t* al = a.alive + (goff_s[g] >> 5);
        if (hl == 0) {
          a.rep_local[r] = r;
          atomicAnd(a.alive + (r >> 5), ~(1u << (r & 31)));
        }
        for (int wd = hl; wd < W; wd += 16) {
          const uint32_t bits = row[wd] & __ldcg(al + wd);
          if (bits) {
            uint32_t bb = bits;
            while (bb) {
              const int b = __ffs(bb) - 1;
              bb &= bb - 1;
              a.rep_local[goff_s[g] + wd * 32 + b] = r;
            }
            atomicAnd(al + wd, ~bits);
          }
        }
      }
      __syncwarp();
    }
    grid_barrier(a.ctrl);
  }
  if (gtid == 0) a.ctrl[2] = (uint32_t)round;
}

// h > 1: no edges -- every copy represents itself.
__global__ void identity_rep_kernel(const int32_t* __restrict__ goff, const int32_t* __restrict__ gtok, int E,
                                    int32_t* __restrict__ rep_local, uint32_t* __restrict__ ctrl,
                                    const int32_t* __restrict__ gcnt, int32_t* __restrict__ gnrep,
                                    int32_t* __restrict__ mrank, int32_t* __restrict__ mcnt_row) {
  pdl_enter();
  const int rows = goff[E];
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    rep_local[r] = gtok[r] >= 0 ? (int32_t)r : -1;
    mrank[r] = 0;     // every copy is the only member of its own list
    mcnt_row[r] = 1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ctrl[2] = 0u;
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e < E; e += blockDim.x) gnrep[e] = gcnt[e];  // every copy represents itself
}

}  // namespace

int launch_group_build(luffy_layer* L, const void* x, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  if (L->k > 8) return (int)cudaErrorInvalidValue;
  const int nch = (L->T + GB_TCH - 1) / GB_TCH;
  launch_pdl(group_count_kernel, nch, GB_TCH, 0, st, (const int32_t*)L->idx, L->T, L->k, L->E, L->gchunk, L->gticket,
             L->gcnt, L->goff, L->adjoff, L->ctrl, L->gdone);
  LUFFY_LAUNCHED();
  if (L->dtype == LUFFY_BF16)
    launch_pdl(group_place_kernel<bf16>, nch * GB_SUB, 256, 0, st, static_cast<const bf16*>(x), (const int32_t*)L->idx,
               (const float*)L->w, L->T, L->k, L->E, L->d, (const int32_t*)L->gchunk, (const int32_t*)L->gcnt,
               (const int32_t*)L->goff, L->gtok, L->gw, L->gloc, L->gcopy, static_cast<bf16*>(L->xg), L->gnorm);
  else
    launch_pdl(group_place_kernel<float>, nch * GB_SUB, 256, 0, st, static_cast<const float*>(x), (const int32_t*)L->idx,
               (const float*)L->w, L->T, L->k, L->E, L->d, (const int32_t*)L->gchunk, (const int32_t*)L->gcnt,
               (const int32_t*)L->goff, L->gtok, L->gw, L->gloc, L->gcopy, static_cast<float*>(L->xg), L->gnorm);
  LUFFY_LAUNCHED();
  return 0;
}

int launch_identity_rep(luffy_layer* L, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  launch_pdl(identity_rep_kernel, 148, 256, 0, st, L->goff, L->gtok, L->E, L->rep_local, L->ctrl, L->gcnt, L->gnrep,
             L->mrank, L->mcnt_row);
  LUFFY_LAUNCHED();
  L->gnrep_valid = true;
  L->mrank_valid = true;
  return 0;
}

int launch_gram_simt(luffy_layer* L, float h, unsigned long long* band, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  const int64_t nt = L->Cpad_max / 64;
  const int64_t tiles = nt * (nt + 1) / 2;  // upper bound over any split of the rows into groups
  const double c2h = 2.0 * (double)h - 1.0;
  if (L->dtype == LUFFY_BF16)
    launch_pdl(gram_simt_kernel<bf16>, (unsigned)tiles, 256, 0, st, static_cast<const bf16*>(L->xg), L->gnorm, L->goff, L->gcnt,
                                                            L->adjoff, L->E, L->d, c2h, L->adj, L->dbg_gram,
                                                            (int64_t)L->dbg_gram_cap, band);
  else
    launch_pdl(gram_simt_kernel<float>, (unsigned)tiles, 256, 0, st, static_cast<const float*>(L->xg), L->gnorm, L->goff, L->gcnt,
                                                             L->adjoff, L->E, L->d, c2h, L->adj, L->dbg_gram,
                                                            (int64_t)L->dbg_gram_cap, band);
  LUFFY_LAUNCHED();
  return 0;
}

int launch_greedy_cluster(luffy_layer* L, void* s);

int launch_greedy(luffy_layer* L, void* s) {
  // fast path: one thread-block cluster per group with DSMEM replicas (greedy_cluster.cu)
  const int rc = launch_greedy_cluster(L, s);
  L->gnrep_valid = rc == 0;  // the cluster kernel publishes the per-group representative counts
  L->mrank_valid = rc == 0;  // ... and the member ranks / list lengths
  if (rc >= 0) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(s);
  LUFFY_CUDA_TRY(cudaMemsetAsync(L->ctrl, 0, sizeof(uint32_t) * (64 + kGreedyMaxRounds), st));
  int blocks = 0;
  if (!dev_cache_get((const void*)greedy_kernel, 0, &blocks)) {
    int per_sm = 0;
    LUFFY_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, greedy_kernel, 256, 0));
    blocks = std::max(1, std::min(per_sm, 8)) * device_sms();
    dev_cache_put((const void*)greedy_kernel, 0, blocks);
  }
  GreedyArgs a;
  a.E = L->E;
  a.goff = L->goff;
  a.gcnt = L->gcnt;
  a.adjoff = L->adjoff;
  a.adj = L->adj;
  a.alive = L->alive;
  a.win = L->win;
  a.key = reinterpret_cast<unsigned long long*>(L->key);
  a.m1 = reinterpret_cast<unsigned long long*>(L->m1);
  a.m2 = reinterpret_cast<unsigned long long*>(L->m2);
  a.rep_local = L->rep_local;
  a.ctrl = L->ctrl;
  a.max_rounds = kGreedyMaxRounds;
  void* args[] = {&a};
  LUFFY_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)greedy_kernel, dim3(blocks), dim3(256), args, 0, st));
  LUFFY_LAUNCHED();
  return 0;
}

}  // namespace luffy
