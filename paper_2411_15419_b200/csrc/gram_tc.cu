// Similarity Gram + threshold on tcgen05 (bf16 groups), "calculating similarity of rest token pairs
// ... easily parallelized" and P:378 (threshold graph).
//
// Per expert group e (rows xg[goff[e] .. goff[e+1]), zero padded to 128), only upper-triangle tiles
// (I <= J) of G = Xg Xg^T are computed: 128x128 fp32 accumulators in TMEM from a 6-stage TMA ring of
// 128x64 bf16 tiles (both operands K-major, SWIZZLE_128B).  The epilogue decides each edge in fp64,
//     edge(i, j)  <=>  G_ij >= (2h - 1) |x_i| |x_j|,  i != j, i, j < n_e, |x_i|, |x_j| > 0,
// which is s_ij = (1 + G_ij / (|x_i||x_j|)) / 2 >= h without a division, packs 32 decisions per word
// and writes the word of (i, j) directly and the word of (j, i) through a warp-ballot bit transpose, so
// the adjacency is symmetric by construction.
#include <cuda.h>

#include "common.cuh"
#include "tc_common.cuh"

namespace luffy {
namespace {

constexpr int TS = 128, BK = 64, STAGES = 6;
constexpr int T_BYTES = TS * BK * 2;  // 16 KiB per operand tile
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
};

__device__ __forceinline__ bool decode_tile(int t, const int32_t* goff_s, int E, int& e, int& I, int& J) {
  for (e = 0; e < E; ++e) {
    const int nt = (goff_s[e + 1] - goff_s[e]) / TS;
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
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * T_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * T_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int E = a.E;
  for (int i = threadIdx.x; i <= E; i += blockDim.x) {
    goff_s[i] = a.goff[i];
    if (i < E) gcnt_s[i] = a.gcnt[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int n = 0;
    for (int e = 0; e < E; ++e) {
      const int nt = (goff_s[e + 1] - goff_s[e]) / TS;
      n += nt * (nt + 1) / 2;
    }
    ntiles_s = n;
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&tfull[s], 1);
      tc::mbar_init(&tempty[s], 8);
    }
    tc::fence_barrier_init();
    tc::tma_prefetch(&tX);
  }
  if (warp == 1) tc::tmem_alloc(tmem_holder, 256);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int ntiles = ntiles_s;
  const int nkb = a.d / BK;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int e, I, J;
        decode_tile(t, goff_s, E, e, I, J);
        const int rI = goff_s[e] + I * TS, rJ = goff_s[e] + J * TS;
        for (int kb = 0; kb < nkb; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          tc::mbar_expect_tx(&full[stage], 2 * T_BYTES);
          tc::tma_load_2d(sA + stage * T_BYTES, &tX, &full[stage], kb * BK, rI);
          tc::tma_load_2d(sB + stage * T_BYTES, &tX, &full[stage], kb * BK, rJ);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t IDESC = tc::idesc_bf16(TS, TS, 0, 0);
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        tc::mbar_wait(&tempty[acc], aphase ^ 1);
        tc::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * TS;
        for (int kb = 0; kb < nkb; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::tc_fence_after();
          const uint32_t a0 = tc::smem_u32(sA + stage * T_BYTES);
          const uint32_t b0 = tc::smem_u32(sB + stage * T_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            tc::mma_bf16(d_tmem, tc::smem_desc(a0 + kk * 32, 16, 1024), tc::smem_desc(b0 + kk * 32, 16, 1024), IDESC,
                         (kb | kk) != 0 ? 1u : 0u);
          tc::mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc::mma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
      }
    }
  } else {
    const int q = warp & 3;
    const int hc = (warp - 2) >> 2;  // column half of the tile handled by this warp
    int acc = 0;
    uint32_t aphase = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int e, I, J;
      decode_tile(t, goff_s, E, e, I, J);
      const int n = gcnt_s[e];
      const int W = (goff_s[e + 1] - goff_s[e]) >> 5;
      uint32_t* base = a.adj + a.adjoff[e];
      const int i0 = I * TS + 32 * q;          // first row (group-local) of this warp
      const int li = i0 + lane;
      const double ni = a.gnorm[goff_s[e] + li];
      const double thr = a.c2h * ni;
      tc::mbar_wait(&tfull[acc], aphase);
      tc::tc_fence_after();
      const uint32_t tb = tmem_base + ((uint32_t)(32 * q) << 16) + acc * TS;
#pragma unroll 1
      for (int c = 2 * hc; c < 2 * hc + 2; ++c) {
        uint32_t r[32];
        tc::tmem_ld32(tb + 32 * c, r);
        tc::tmem_ld_wait();
        const int j0 = J * TS + 32 * c;
        if (J == I && c < q) continue;  // strictly below the diagonal: written as the transpose of (c, q)
        const double my_nj = a.gnorm[goff_s[e] + j0 + lane];
        uint32_t word = 0;
#pragma unroll
        for (int b = 0; b < 32; ++b) {
          const double nj = __shfl_sync(0xffffffffu, my_nj, b);
          const int lj = j0 + b;
          const bool on = li < n && lj < n && ni > 0.0 && nj > 0.0 && (double)__uint_as_float(r[b]) >= thr * nj;
          word |= (uint32_t)on << b;
        }
        const bool diag = (j0 == i0);
        if (diag) word &= (lane == 31) ? 0u : (0xffffffffu << (lane + 1));  // keep j > i only
        // bit transpose through ballots: column b of the 32x32 block -> word of row j0 + b
        uint32_t tr = 0;
#pragma unroll
        for (int b = 0; b < 32; ++b) {
          const uint32_t col = __ballot_sync(0xffffffffu, (word >> b) & 1u);
          if (b == lane) tr = col;
        }
        if (diag) {
          base[(size_t)li * W + (j0 >> 5)] = word | tr;
        } else {
          base[(size_t)li * W + (j0 >> 5)] = word;
          base[(size_t)(j0 + lane) * W + (i0 >> 5)] = tr;
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  }
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem_base, 256);
}

__global__ void adj_offsets_tc_kernel(const int32_t* __restrict__ goff, int E, int64_t* __restrict__ adjoff) {
  pdl_enter();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int64_t o = 0;
    for (int e = 0; e < E; ++e) {
      adjoff[e] = o;
      const int64_t np = goff[e + 1] - goff[e];
      o += np * np / 32;
    }
    adjoff[E] = o;
  }
}

}  // namespace

int make_tmap_bf16(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_stride_elems,
                   uint32_t box_outer);

int launch_gram_tc(luffy_layer* L, float h, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  launch_pdl(adj_offsets_tc_kernel, 1, 32, 0, st, L->goff, L->E, L->adjoff);
  LUFFY_LAUNCHED();
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
  static bool attr = false;
  if (!attr) {
    LUFFY_CUDA_TRY(cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    attr = true;
  }
  int dev = 0, sms = 0;
  LUFFY_CUDA_TRY(cudaGetDevice(&dev));
  LUFFY_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  launch_pdl(gram_tc_kernel, sms, THREADS, SMEM_BYTES, st, tx, a);
  LUFFY_LAUNCHED();
  return 0;
}

}  // namespace luffy
