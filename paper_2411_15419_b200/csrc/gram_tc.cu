// Similarity Gram + threshold on tcgen05 (bf16 groups), "calculating similarity of rest token pairs
// ... easily parallelized" and P:378 (threshold graph).
//
// Per expert group e (rows xg[goff[e] .. goff[e+1]), zero padded to 128), only upper-triangle tiles
// (I <= J) of G = Xg Xg^T are computed, as 256x256 tiles on a CTA PAIR (cta_group::2, the leader issues
// M=256 N=256 MMAs): each CTA stages its 128 rows of the I block and its 128-row half of the J block
// (6-stage TMA ring, both operands K-major, SWIZZLE_128B) and owns a 128x256 fp32 accumulator in TMEM --
// half the staged bytes per flop of 128x128 single-CTA tiles, the limit of this kernel.  Half blocks past
// a group's padded end are computed on whatever rows follow and never written.  The epilogue decides
// each edge in fp64,
//     edge(i, j)  <=>  G_ij >= (2h - 1) |x_i| |x_j|,  i != j, i, j < n_e, |x_i|, |x_j| > 0,
// which is s_ij = (1 + G_ij / (|x_i||x_j|)) / 2 >= h without a division, packs 32 decisions per word
// and writes the word of (i, j) directly and the word of (j, i) through a warp-ballot bit transpose, so
// the adjacency is symmetric by construction.
#include <cuda.h>

#include "common.cuh"
#include "tc_common.cuh"

namespace luffy {
namespace {

constexpr int TS = 128, BK = 64, STAGES = 6;  // TS: rows per CTA; the pair tile is 2 TS x 2 TS
constexpr int T_BYTES = TS * BK * 2;  // 16 KiB per operand half-tile
constexpr int SMEM_BYTES = STAGES * 2 * T_BYTES + 1024 + 256;
constexpr int THREADS = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue

struct GramArgs {
  const int32_t* goff;
  const int32_t* gcnt;
  const int64_t* adjoff;
  const double* gnorm;
  uint32_t* adj;
  int E, d;
  double c2h;
  float* gdump;                   // debug (nullable): fp32 G of every computed block, group e at float
  int64_t gdump_cap;              //   offset adjoff[e] * 32, dense [npad_e][npad_e] row-major (j-block >= i-block)
  unsigned long long* band;       // stats (nullable): pairs i < j with |s_ij - h| <= 1e-5 (reading R18)
  // fast similarity measurement (HIST instantiation, readings R20/R21); adj layout bitmaps
  const uint32_t* dec1;           // previous block's s > S1 for this block's pairs (nullable: no history)
  const uint32_t* dec0;           // previous block's s < S2
  const uint8_t* tskip;           // [tiles] 1: every pair of the tile is decided -> no TMA, no MMA
  uint32_t* gdone;                // out (nullable): per group, pair tiles finished (+1 per CTA of the pair)
  uint32_t* hone;                 // out: this block's finalized weight > S1
  uint32_t* hzero;                // out: this block's finalized weight < S2
  double c2s1, c2s2;              // 2 S1 - 1, 2 S2 - 1
};

// Words of a 32x32 block: `word` for row li, columns j0.. (bit b = column j0 + b), stored directly and as
// its transpose (32x32 bit transpose across the warp, 5 shuffles), so the matrix is symmetric.
__device__ __forceinline__ void store_sym(uint32_t* base, int W, int li, int i0, int j0, int lane, uint32_t word,
                                          bool diag) {
  uint32_t tr = word;
#pragma unroll
  for (int sft = 16; sft >= 1; sft >>= 1) {
    const uint32_t lo = sft == 16 ? 0x0000FFFFu : sft == 8 ? 0x00FF00FFu : sft == 4 ? 0x0F0F0F0Fu
                                                    : sft == 2 ? 0x33333333u : 0x55555555u;
    const uint32_t oth = __shfl_xor_sync(0xffffffffu, tr, sft);
    tr = (lane & sft) ? ((tr & ~lo) | ((oth & ~lo) >> sft)) : ((tr & lo) | ((oth & lo) << sft));
  }
  __syncwarp();
  if (diag) {
    base[(size_t)li * W + (j0 >> 5)] = word | tr;
  } else {
    base[(size_t)li * W + (j0 >> 5)] = word;
    base[(size_t)(j0 + lane) * W + (i0 >> 5)] = tr;
  }
}

// Bits b where the fp64 relation  G_b (>, >=, <) thr * nj_b  holds, for the 32 fp32 accumulators of one row
// and the column norms njs / nj (fp64 per lane, shuffled): the fp32 products are within 1.8e-7 of the fp64
// ones, so outside a 1e-6 relative band the fp32 test IS the fp64 decision; elements inside the band are
// re-decided in fp64.  OP: 0 '>=', 1 '>', 2 '<'.
template <int OP>
__device__ __forceinline__ uint32_t decide_row(const uint32_t (&r)[32], const float* njs, double thr, double my_nj) {
  const float thr_f = (float)thr;
  const float big = thr_f >= 0.f ? thr_f * (1.f + 1e-6f) : thr_f * (1.f - 1e-6f);
  const float small = thr_f >= 0.f ? thr_f * (1.f - 1e-6f) : thr_f * (1.f + 1e-6f);
  uint32_t hi = 0, lo = 0;
#pragma unroll
  for (int b4 = 0; b4 < 8; ++b4) {
    const float4 nq = reinterpret_cast<const float4*>(njs)[b4];
    const float nv[4] = {nq.x, nq.y, nq.z, nq.w};
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
      const int b = 4 * b4 + k2;
      const float g = __uint_as_float(r[b]);
      if (OP == 0) { hi |= (uint32_t)(g >= big * nv[k2]) << b; lo |= (uint32_t)(g >= small * nv[k2]) << b; }
      if (OP == 1) { hi |= (uint32_t)(g > big * nv[k2]) << b; lo |= (uint32_t)(g > small * nv[k2]) << b; }
      if (OP == 2) { hi |= (uint32_t)(g < small * nv[k2]) << b; lo |= (uint32_t)(g < big * nv[k2]) << b; }
    }
  }
  uint32_t word = hi;
  const uint32_t amb = hi ^ lo;
  if (__any_sync(0xffffffffu, amb != 0u)) {
#pragma unroll
    for (int b = 0; b < 32; ++b) {
      const double nj = __shfl_sync(0xffffffffu, my_nj, b);
      if ((amb >> b) & 1u) {
        const double g = (double)__uint_as_float(r[b]), p = thr * nj;
        const bool on = OP == 0 ? g >= p : (OP == 1 ? g > p : g < p);
        word = on ? (word | (1u << b)) : (word & ~(1u << b));
      }
    }
  }
  return word;
}

// pair tiles (I, J), J >= I, over blocks of 2 TS rows of each group; groups in descending cost (n^2, ties
// to the lower group) -- the order the representative selection schedules them in, so the costliest
// group's selection can start first (greedy_cluster_kernel waits per group on GramArgs::gdone)
__device__ __forceinline__ int pair_blocks(int npad) { return (npad / TS + 1) / 2; }
__device__ __forceinline__ void group_order(const int32_t* gcnt_s, int E, int* order_s) {
  for (int i = threadIdx.x; i < E; i += blockDim.x) {
    const long long ci = (long long)gcnt_s[i] * gcnt_s[i];
    int rk = 0;
    for (int j = 0; j < E; ++j) {
      const long long cj = (long long)gcnt_s[j] * gcnt_s[j];
      rk += (cj > ci) || (cj == ci && j < i);
    }
    order_s[rk] = i;
  }
}
__device__ __forceinline__ bool decode_tile(int t, const int32_t* goff_s, const int* order_s, int E, int& e, int& I,
                                            int& J) {
  for (int r = 0; r < E; ++r) {
    e = order_s[r];
    const int nt = pair_blocks(goff_s[e + 1] - goff_s[e]);
    const int pairs = nt * (nt + 1) / 2;
    if (t < pairs) {
      int i = 0, rem = t;
      while (rem >= nt - i) { rem -= nt - i; ++i; }
      I = i;
      J = i + rem;
      return true;
    }
    t -= pairs;
  }
  return false;
}

template <bool HIST>
__global__ void __launch_bounds__(THREADS, 1) gram_tc_kernel(const __grid_constant__ CUtensorMap tX, const GramArgs a) {
  pdl_defer();
  extern __shared__ uint8_t smem_raw[];
  __shared__ int32_t goff_s[LUFFY_MAX_EXPERTS + 1];
  __shared__ int32_t gcnt_s[LUFFY_MAX_EXPERTS];
  __shared__ int ntiles_s;
  __shared__ int order_s[LUFFY_MAX_EXPERTS];
  __shared__ __align__(16) float njs_all[8 * 32];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * T_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * T_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = tc::cluster_rank();  // 0: leader (issues the MMA)
  const int E = a.E;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&tfull[s], 1);
      tc::mbar_init(&tempty[s], 16);  // the epilogue warps of both CTAs release the leader's buffer
    }
    tc::fence_barrier_init();
    tc::tma_prefetch(&tX);
  }
  if (warp == 1) tc::tmem_alloc_pair(tmem_holder, 512);
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  pdl_enter();  // from here on: the previous kernels' outputs (group offsets and rows, norms)
  for (int i = threadIdx.x; i <= E; i += blockDim.x) {
    goff_s[i] = a.goff[i];
    if (i < E) gcnt_s[i] = a.gcnt[i];
  }
  __syncthreads();
  group_order(gcnt_s, E, order_s);
  if (threadIdx.x == 0) {
    int n = 0;
    for (int e = 0; e < E; ++e) {
      const int nt = pair_blocks(goff_s[e + 1] - goff_s[e]);
      n += nt * (nt + 1) / 2;
    }
    ntiles_s = n;
  }
  __syncthreads();
  const uint32_t tmem_base = *tmem_holder;
  const int ntiles = ntiles_s;
  const int nkb = a.d / BK;
  const int tile0 = blockIdx.x >> 1, tstride = gridDim.x >> 1;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = tile0; t < ntiles; t += tstride) {
        if (HIST && a.tskip != nullptr && a.tskip[t]) continue;  // decided by history: nothing to measure
        int e, I, J;
        decode_tile(t, goff_s, order_s, E, e, I, J);
        const int h = (int)crank * TS;
        const int rI = goff_s[e] + I * 2 * TS + h, rJ = goff_s[e] + J * 2 * TS + h;
        for (int kb = 0; kb < nkb; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          if (crank == 0) tc::mbar_expect_tx(&full[stage], 4 * T_BYTES);
          const uint32_t barc = tc::map_rank(&full[stage], 0);
          tc::tma_load_2d_pair(sA + stage * T_BYTES, &tX, barc, kb * BK, rI);
          tc::tma_load_2d_pair(sB + stage * T_BYTES, &tX, barc, kb * BK, rJ);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && crank == 0) {
      constexpr uint32_t IDESC = tc::idesc_bf16(2 * TS, 2 * TS, 0, 0);
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      for (int t = tile0; t < ntiles; t += tstride) {
        if (HIST && a.tskip != nullptr && a.tskip[t]) continue;
        tc::mbar_wait(&tempty[acc], aphase ^ 1);
        tc::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 2 * TS;
        for (int kb = 0; kb < nkb; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::tc_fence_after();
          const uint32_t a0 = tc::smem_u32(sA + stage * T_BYTES);
          const uint32_t b0 = tc::smem_u32(sB + stage * T_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            tc::mma_bf16_pair(d_tmem, tc::smem_desc(a0 + kk * 32, 16, 1024), tc::smem_desc(b0 + kk * 32, 16, 1024),
                              IDESC, (kb | kk) != 0 ? 1u : 0u);
          tc::mma_commit_pair(&empty[stage], 3);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc::mma_commit_pair(&tfull[acc], 3);
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
      }
    }
  } else {
    const int q = warp & 3;
    const int hc = (warp - 2) >> 2;  // column half (128 of the 256 columns) handled by this warp
    float* njs = njs_all + (warp - 2) * 32;  // this warp's column norms (fp32)
    int acc = 0;
    uint32_t aphase = 0;
    // every epilogue thread's words of the tile are globally visible before its group's counter moves:
    // the epilogue warps meet at a CTA barrier, then one thread's gpu-scope fence (cumulative over what the
    // barrier ordered before it) and the increment
    auto tile_done = [&](int e) {
      if (a.gdone == nullptr) return;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (warp == 2 && lane == 0) {
        __threadfence();
        atomicAdd(a.gdone + e, 1u);
      }
    };
    for (int t = tile0; t < ntiles; t += tstride) {
      int e, I, J;
      decode_tile(t, goff_s, order_s, E, e, I, J);
      const int n = gcnt_s[e];
      const int npad = goff_s[e + 1] - goff_s[e];
      const int W = npad >> 5;
      uint32_t* base = a.adj + a.adjoff[e];
      const int i0 = I * 2 * TS + (int)crank * TS + 32 * q;  // first row (group-local) of this warp
      const int li = i0 + lane;
      // norms first (row, and the columns of this warp's four 32-column blocks), then the accumulator
      const double ni = i0 < npad ? a.gnorm[goff_s[e] + li] : 0.0;
      double njv[4];
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        const int jc = J * 2 * TS + 32 * (4 * hc + k4) + lane;
        njv[k4] = jc < npad ? a.gnorm[goff_s[e] + jc] : 0.0;
      }
      const double thr = a.c2h * ni;
      const float thr_f = (float)thr;
      const float thr_hi = thr_f >= 0.f ? thr_f * (1.f + 1e-6f) : thr_f * (1.f - 1e-6f);  // the larger bound
      const float thr_lo = thr_f >= 0.f ? thr_f * (1.f - 1e-6f) : thr_f * (1.f + 1e-6f);
      const bool rowok = li < n && ni > 0.0;
      const size_t hrow = (size_t)a.adjoff[e] + (size_t)li * W;  // this row's words in the history bitmaps
      if (HIST && a.tskip != nullptr && a.tskip[t]) {
        // every pair of the tile was decided by the previous block: weights 1 / 0, no MMA
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
          const int c = 4 * hc + k4;
          const int j0 = J * 2 * TS + 32 * c;
          if (i0 >= npad || j0 >= npad || j0 < i0) continue;
          const unsigned colok = __ballot_sync(0xffffffffu, j0 + lane < n && njv[k4] > 0.0);
          uint32_t m = rowok ? colok : 0u;
          const bool diag = (j0 == i0);
          if (diag) m &= (lane == 31) ? 0u : (0xffffffffu << (lane + 1));
          const uint32_t d1 = a.dec1[hrow + (j0 >> 5)] & m, d0 = a.dec0[hrow + (j0 >> 5)] & m;
          store_sym(base, W, li, i0, j0, lane, d1, diag);
          store_sym(a.hone + a.adjoff[e], W, li, i0, j0, lane, d1, diag);
          store_sym(a.hzero + a.adjoff[e], W, li, i0, j0, lane, d0, diag);
        }
        tile_done(e);
        continue;
      }
      tc::mbar_wait(&tfull[acc], aphase);
      tc::tc_fence_after();
      const uint32_t tb = tmem_base + ((uint32_t)(32 * q) << 16) + acc * 2 * TS;
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        const int c = 4 * hc + k4;
        const int j0 = J * 2 * TS + 32 * c;
        // rows / columns past the group's padded end, and blocks strictly below the diagonal (written as
        // the transpose of their mirror) are skipped (warp-uniform)
        if (i0 >= npad || j0 >= npad || j0 < i0) continue;
        uint32_t r[32];
        tc::tmem_ld32(tb + 32 * c, r);
        // column norms of this 32-column block: validity mask and fp32 copies broadcast from shared memory
        const double my_nj = njv[k4];
        const unsigned colok = __ballot_sync(0xffffffffu, j0 + lane < n && my_nj > 0.0);
        njs[lane] = (float)my_nj;
        __syncwarp();
        tc::tmem_ld_wait();
        if (a.gdump != nullptr) {  // debug export of the accumulator (tests: max |s_gpu - s_ref|, A18)
          const int64_t o = a.adjoff[e] * 32 + (int64_t)li * npad + j0;
          if (o + 32 <= a.gdump_cap) {
            float4* dst = reinterpret_cast<float4*>(a.gdump + o);
#pragma unroll
            for (int b4 = 0; b4 < 8; ++b4)
              dst[b4] = make_float4(__uint_as_float(r[4 * b4]), __uint_as_float(r[4 * b4 + 1]),
                                    __uint_as_float(r[4 * b4 + 2]), __uint_as_float(r[4 * b4 + 3]));
          }
        }
        uint32_t m = rowok ? colok : 0u;
        const bool diag = (j0 == i0);
        if (diag) m &= (lane == 31) ? 0u : (0xffffffffu << (lane + 1));  // keep j > i only
        uint32_t d1 = 0u, d0 = 0u;  // pairs decided by the previous block (HIST)
        if (HIST && a.dec1 != nullptr) {
          d1 = a.dec1[hrow + (j0 >> 5)] & m;
          d0 = a.dec0[hrow + (j0 >> 5)] & m;
        }
        if (a.band != nullptr) {  // near-threshold pairs: |G - (2h-1) n_i n_j| <= 2e-5 n_i n_j  <=>  |s - h| <= 1e-5
          const float blo = (float)((a.c2h - 2e-5) * ni), bhi = (float)((a.c2h + 2e-5) * ni);
          uint32_t bw = 0;
#pragma unroll
          for (int b = 0; b < 32; ++b) {
            const float g = __uint_as_float(r[b]), nv = njs[b];
            bw |= (uint32_t)(g >= blo * nv && g <= bhi * nv) << b;
          }
          bw &= m & ~(d1 | d0);
          const int cnt = __reduce_add_sync(0xffffffffu, __popc(bw));
          if (lane == 0 && cnt) atomicAdd(a.band, (unsigned long long)cnt);
        }
        // edge iff G >= thr * nj (thr = (2h-1)|x_i|, decided as in fp64): the fp32 product is within
        // 1.8e-7 (relative) of the fp64 one, so outside the band [p_lo, p_hi) = thr*nj*(1 -/+ 1e-6) the
        // fp32 comparison with either bound IS the fp64 decision; the rare elements inside the band are
        // re-decided in fp64 (two compares per element instead of a compare and an |G - p| test)
        uint32_t word = 0, lo = 0;
#pragma unroll
        for (int b4 = 0; b4 < 8; ++b4) {
          const float4 nq = reinterpret_cast<const float4*>(njs)[b4];
          const float nv[4] = {nq.x, nq.y, nq.z, nq.w};
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2) {
            const int b = 4 * b4 + k2;
            const float g = __uint_as_float(r[b]);
            word |= (uint32_t)(g >= thr_hi * nv[k2]) << b;
            lo |= (uint32_t)(g >= thr_lo * nv[k2]) << b;
          }
        }
        const uint32_t amb = word ^ lo;  // p_lo <= G < p_hi (column norms are >= 0, so the bounds stay ordered)
        if (__any_sync(0xffffffffu, amb != 0u)) {
#pragma unroll
          for (int b = 0; b < 32; ++b) {
            const double nj = __shfl_sync(0xffffffffu, my_nj, b);
            if ((amb >> b) & 1u) {
              const bool on = (double)__uint_as_float(r[b]) >= thr * nj;
              word = on ? (word | (1u << b)) : (word & ~(1u << b));
            }
          }
        }
        word &= m;
        if (HIST) {
          // decided pairs take weight 1 (edge for any h <= 1) or 0 (no edge); the finalized weights
          // are classified for the next block (reading R21): > S1, < S2 -- computed pairs in fp64 as above
          const uint32_t dec = d1 | d0;
          word = (word & ~dec) | d1;
          const uint32_t c1 = decide_row<1>(r, njs, a.c2s1 * ni, my_nj) & m & ~dec;
          const uint32_t c0 = decide_row<2>(r, njs, a.c2s2 * ni, my_nj) & m & ~dec;
          store_sym(a.hone + a.adjoff[e], W, li, i0, j0, lane, d1 | c1, diag);
          store_sym(a.hzero + a.adjoff[e], W, li, i0, j0, lane, d0 | c0, diag);
        }
        store_sym(base, W, li, i0, j0, lane, word, diag);
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster_relaxed(tc::map_rank(&tempty[acc], 0));
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
      tile_done(e);
    }
  }
  tc::tc_fence_before();
  tc::cluster_sync();  // neither CTA of the pair leaves while the other can still arrive on its barriers
  if (warp == 1) tc::tmem_dealloc_pair(tmem_base, 512);
}

// ---------------------------------------------------------------------------------------------------
// Fast similarity measurement, step 2: history of the previous block, readings R20/R21.

struct HistPrev {
  const int32_t* idx;     // [T, k] previous block's experts
  const int32_t* gloc;    // [T, k] its global (padded) group row of copy (t, j)
  const int32_t* goff;    // [E + 1]
  const int64_t* adjoff;  // [E + 1] word offsets of its group bitmaps
  const uint32_t* hone;   // its finalized weight > S1 (adj layout)
  const uint32_t* hzero;  // its finalized weight < S2
  int k;
};

// dec1 / dec0 (this block's adj layout): for each pair of this block's groups, the previous block's
// classification of the same token pair, read from the group of the first expert (in the row token's
// top-k order) the two tokens shared in the previous block; no shared expert -> no history (R20).  One warp
// per group row; lanes walk the columns, so a row's previous bitmap rows stay in L1.
__global__ void __launch_bounds__(256) hist_gather_kernel(const int32_t* __restrict__ goff, const int32_t* __restrict__ gcnt,
                                                          const int32_t* __restrict__ gtok, const int64_t* __restrict__ adjoff,
                                                          int E, HistPrev pv, uint32_t* __restrict__ dec1,
                                                          uint32_t* __restrict__ dec0) {
  pdl_enter();
  __shared__ int32_t goff_s[LUFFY_MAX_EXPERTS + 1];
  for (int i = threadIdx.x; i <= E; i += blockDim.x) goff_s[i] = goff[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int rows = goff_s[E];
  const int k = pv.k;
  for (int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < rows; g += (gridDim.x * blockDim.x) >> 5) {
    const int e = find_group(goff_s, E, g);
    const int g0 = goff_s[e], n = gcnt[e];
    const int W = (goff_s[e + 1] - g0) >> 5;
    const int li = g - g0;
    uint32_t* o1 = dec1 + adjoff[e] + (size_t)li * W;
    uint32_t* o0 = dec0 + adjoff[e] + (size_t)li * W;
    if (li >= n) {
      for (int w = lane; w < W; w += 32) o1[w] = o0[w] = 0u;
      continue;
    }
    const int ti = gtok[g];
    int pe[8];
    size_t pb[8];
    for (int j = 0; j < 8; ++j) {
      pe[j] = -1;
      pb[j] = 0;
      if (j < k) {
        pe[j] = pv.idx[(size_t)ti * k + j];
        const int p0 = pv.goff[pe[j]];
        const int pw = (pv.goff[pe[j] + 1] - p0) >> 5;
        pb[j] = (size_t)pv.adjoff[pe[j]] + (size_t)(pv.gloc[(size_t)ti * k + j] - p0) * pw;
      }
    }
    for (int w = 0; w < W; ++w) {
      const int lj = 32 * w + lane;
      bool b1 = false, b0 = false;
      if (lj < n && lj != li) {
        const int tj = gtok[g0 + lj];
        bool found = false;
        for (int j = 0; j < k && !found; ++j)
          for (int j2 = 0; j2 < k; ++j2)
            if (pv.idx[(size_t)tj * k + j2] == pe[j]) {
              const int col = pv.gloc[(size_t)tj * k + j2] - pv.goff[pe[j]];
              b1 = (pv.hone[pb[j] + (col >> 5)] >> (col & 31)) & 1u;
              b0 = (pv.hzero[pb[j] + (col >> 5)] >> (col & 31)) & 1u;
              found = true;
              break;
            }
      }
      const uint32_t w1 = __ballot_sync(0xffffffffu, b1), w0 = __ballot_sync(0xffffffffu, b0);
      if (lane == 0) {
        o1[w] = w1;
        o0[w] = w0;
      }
    }
  }
}

// tskip[t] = 1 iff every pair (i < j, both valid and of nonzero norm) of pair tile t is decided; also
// counts the decided pairs (stats).  One CTA of 2 TS threads (one per tile row) per tile, grid-stride.
__global__ void __launch_bounds__(2 * TS) hist_flags_kernel(const int32_t* __restrict__ goff, const int32_t* __restrict__ gcnt,
                                                            const int64_t* __restrict__ adjoff, const double* __restrict__ gnorm,
                                                            int E, const uint32_t* __restrict__ dec1,
                                                            const uint32_t* __restrict__ dec0, uint8_t* __restrict__ tskip,
                                                            unsigned long long* __restrict__ counts) {
  pdl_enter();
  __shared__ int32_t goff_s[LUFFY_MAX_EXPERTS + 1];
  __shared__ int32_t gcnt_s[LUFFY_MAX_EXPERTS];
  __shared__ int order_s[LUFFY_MAX_EXPERTS];
  __shared__ uint32_t colw[2 * TS / 32];
  __shared__ int ntiles_s;
  for (int i = threadIdx.x; i <= E; i += blockDim.x) {
    goff_s[i] = goff[i];
    if (i < E) gcnt_s[i] = gcnt[i];
  }
  __syncthreads();
  group_order(gcnt_s, E, order_s);  // the Gram's tile order (tskip is indexed by it)
  __syncthreads();
  if (threadIdx.x == 0) {
    int nt = 0;
    for (int e = 0; e < E; ++e) {
      const int pb = pair_blocks(goff_s[e + 1] - goff_s[e]);
      nt += pb * (pb + 1) / 2;
    }
    ntiles_s = nt;
  }
  __syncthreads();
  const int ntiles = ntiles_s;
  unsigned long long dec_pairs = 0, skipped = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int e, I, J;
    decode_tile(t, goff_s, order_s, E, e, I, J);
    const int g0 = goff_s[e], npad = goff_s[e + 1] - g0, n = gcnt[e], W = npad >> 5;
    const int lj = J * 2 * TS + threadIdx.x;
    const bool cv = lj < n && gnorm[g0 + lj] > 0.0;
    const uint32_t cb = __ballot_sync(0xffffffffu, cv);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) colw[threadIdx.x >> 5] = cb;
    __syncthreads();
    const int li = I * 2 * TS + threadIdx.x;
    const bool rv = li < n && gnorm[g0 + li] > 0.0;
    bool ok = true;
    if (rv) {
      for (int w = 0; w < 2 * TS / 32; ++w) {
        const int jw = J * (2 * TS / 32) + w;
        if (jw >= W) break;
        uint32_t need = colw[w];
        const int rel = li - 32 * jw;  // keep columns j > li
        if (rel >= 31) need = 0u;
        else if (rel >= 0) need &= 0xffffffffu << (rel + 1);
        const size_t o = (size_t)adjoff[e] + (size_t)li * W + jw;
        const uint32_t dec = (dec1[o] | dec0[o]) & need;
        ok = ok && dec == need;
        dec_pairs += __popc(dec);
      }
    }
    const int all = __syncthreads_and(ok);
    if (threadIdx.x == 0) {
      tskip[t] = (uint8_t)all;
      skipped += all;
    }
  }
  if (counts) {
    for (int o = 16; o > 0; o >>= 1) dec_pairs += __shfl_xor_sync(0xffffffffu, dec_pairs, o);
    if ((threadIdx.x & 31) == 0 && dec_pairs) atomicAdd(counts, dec_pairs);
    if (threadIdx.x == 0 && skipped) atomicAdd(counts + 1, skipped);
  }
}

}  // namespace

int make_tmap_bf16(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_stride_elems,
                   uint32_t box_outer);

int launch_gram_tc(luffy_layer* L, float h, unsigned long long* band, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  // (adjoff and the greedy control block are prepared by gather_norm_kernel)
  CUtensorMap tx;
  LUFFY_CUDA_TRY(make_tmap_bf16(&tx, L->xg, L->d, L->Cpad_max, L->d, TS));
  GramArgs a{};
  a.goff = L->goff;
  a.gcnt = L->gcnt;
  a.adjoff = L->adjoff;
  a.gnorm = L->gnorm;
  a.adj = L->adj;
  a.E = L->E;
  a.d = L->d;
  a.c2h = 2.0 * (double)h - 1.0;
  a.gdump = L->dbg_gram;
  a.gdump_cap = (int64_t)L->dbg_gram_cap;
  a.band = band;
  a.gdone = L->gdone;
  const bool hist = L->fast_measure;
  if (hist) {
    a.hone = L->hone;
    a.hzero = L->hzero;
    a.c2s1 = 2.0 * (double)L->hist_S1 - 1.0;
    a.c2s2 = 2.0 * (double)L->hist_S2 - 1.0;
    const luffy_layer* P = L->hist_prev;
    if (P != nullptr && P->hist_valid) {
      HistPrev pv{P->idx, P->gloc, P->goff, P->adjoff, P->hone, P->hzero, P->k};
      const int gblocks = (int)std::min<int64_t>((L->Cpad_max + 7) / 8, 148 * 8);
      launch_pdl(hist_gather_kernel, gblocks, 256, 0, st, (const int32_t*)L->goff, (const int32_t*)L->gcnt,
                 (const int32_t*)L->gtok, (const int64_t*)L->adjoff, L->E, pv, L->dec1, L->dec0);
      LUFFY_LAUNCHED();
      launch_pdl(hist_flags_kernel, 148 * 4, 2 * TS, 0, st, (const int32_t*)L->goff, (const int32_t*)L->gcnt,
                 (const int64_t*)L->adjoff, (const double*)L->gnorm, L->E, (const uint32_t*)L->dec1,
                 (const uint32_t*)L->dec0, L->tskip, band ? reinterpret_cast<unsigned long long*>(L->stat64) + 2 : nullptr);
      LUFFY_LAUNCHED();
      a.dec1 = L->dec1;
      a.dec0 = L->dec0;
      a.tskip = L->tskip;
    }
  }
  auto kern = hist ? gram_tc_kernel<true> : gram_tc_kernel<false>;
  LUFFY_CUDA_TRY(smem_optin((const void*)kern, SMEM_BYTES));
  const int sms = device_sms();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(sms & ~1);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  LUFFY_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, tx, a));
  LUFFY_LAUNCHED();
  return 0;
}

}  // namespace luffy
