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
};

// pair tiles (I, J), J >= I, over blocks of 2 TS rows of each group
__device__ __forceinline__ int pair_blocks(int npad) { return (npad / TS + 1) / 2; }
__device__ __forceinline__ bool decode_tile(int t, const int32_t* goff_s, int E, int& e, int& I, int& J) {
  for (e = 0; e < E; ++e) {
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

__global__ void __launch_bounds__(THREADS, 1) gram_tc_kernel(const __grid_constant__ CUtensorMap tX, const GramArgs a) {
  pdl_enter();
  extern __shared__ uint8_t smem_raw[];
  __shared__ int32_t goff_s[LUFFY_MAX_EXPERTS + 1];
  __shared__ int32_t gcnt_s[LUFFY_MAX_EXPERTS];
  __shared__ int ntiles_s;
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
  for (int i = threadIdx.x; i <= E; i += blockDim.x) {
    goff_s[i] = a.goff[i];
    if (i < E) gcnt_s[i] = a.gcnt[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int n = 0;
    for (int e = 0; e < E; ++e) {
      const int nt = pair_blocks(goff_s[e + 1] - goff_s[e]);
      n += nt * (nt + 1) / 2;
    }
    ntiles_s = n;
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
  const uint32_t tmem_base = *tmem_holder;
  const int ntiles = ntiles_s;
  const int nkb = a.d / BK;
  const int tile0 = blockIdx.x >> 1, tstride = gridDim.x >> 1;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = tile0; t < ntiles; t += tstride) {
        int e, I, J;
        decode_tile(t, goff_s, E, e, I, J);
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
    for (int t = tile0; t < ntiles; t += tstride) {
      int e, I, J;
      decode_tile(t, goff_s, E, e, I, J);
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
        // edge iff G >= thr * nj (thr = (2h-1)|x_i|, decided as in fp64): the fp32 product is within
        // 1.8e-7 (relative) of the fp64 one, so outside the band [p_lo, p_hi) = thr*nj*(1 -/+ 1e-6) the
        // fp32 comparison with either bound IS the fp64 decision; the rare elements inside the band are
        // re-decided in fp64 (two compares per element instead of a compare and an |G - p| test)
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
        if (a.band != nullptr) {  // near-threshold pairs: |G - (2h-1) n_i n_j| <= 2e-5 n_i n_j  <=>  |s - h| <= 1e-5
          const float blo = (float)((a.c2h - 2e-5) * ni), bhi = (float)((a.c2h + 2e-5) * ni);
          uint32_t bw = 0;
#pragma unroll
          for (int b = 0; b < 32; ++b) {
            const float g = __uint_as_float(r[b]), nv = njs[b];
            bw |= (uint32_t)(g >= blo * nv && g <= bhi * nv) << b;
          }
          bw &= rowok ? colok : 0u;
          if (j0 == i0) bw &= (lane == 31) ? 0u : (0xffffffffu << (lane + 1));
          const int c = __reduce_add_sync(0xffffffffu, __popc(bw));
          if (lane == 0 && c) atomicAdd(a.band, (unsigned long long)c);
        }
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
        word &= rowok ? colok : 0u;
        const bool diag = (j0 == i0);
        if (diag) word &= (lane == 31) ? 0u : (0xffffffffu << (lane + 1));  // keep j > i only
        // 32x32 bit transpose across the warp (recursive block swap, 5 shuffles): column b of the block
        // -> word of row j0 + b, so the adjacency is symmetric by construction
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
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster_relaxed(tc::map_rank(&tempty[acc], 0));
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  }
  tc::tc_fence_before();
  tc::cluster_sync();  // neither CTA of the pair leaves while the other can still arrive on its barriers
  if (warp == 1) tc::tmem_dealloc_pair(tmem_base, 512);
}

}  // namespace

int make_tmap_bf16(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_stride_elems,
                   uint32_t box_outer);

int launch_gram_tc(luffy_layer* L, float h, unsigned long long* band, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  // (adjoff and the greedy control block are prepared by gather_norm_kernel)
  CUtensorMap tx;
  LUFFY_CUDA_TRY(make_tmap_bf16(&tx, L->xg, L->d, L->Cpad_max, L->d, TS));
  GramArgs a;
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
  LUFFY_CUDA_TRY(smem_optin((const void*)gram_tc_kernel, SMEM_BYTES));
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
  LUFFY_CUDA_TRY(cudaLaunchKernelEx(&cfg, gram_tc_kernel, tx, a));
  LUFFY_LAUNCHED();
  return 0;
}

}  // namespace luffy
