// tcgen05 grouped GEMMs for the expert FFN (bf16 in, fp32 accumulation in TMEM), sm_100a.
//
// One persistent CTA per SM, warp-specialized, as a CTA PAIR (cta_group::2, cluster of 2 on one TPC) or
// a single CTA (fallback, LUFFY_GEMM_CG=1):
//   warp 0      TMA producer: ring of (A 128x64, B (256/CG)x64) bf16 tiles, SWIZZLE_128B (6 stages of 32 KiB
//               per CTA for the pair, 4 of 48 KiB single); in the pair both CTAs load their own halves and
//               complete the bytes on the leader's barrier;
//   warp 1      MMA issuer: one thread of the leader issues tcgen05.mma.cta_group::{2,1}.kind::f16 (M=256 or
//               128, N=256, K=16) into a double-buffered TMEM accumulator (2 x 256 columns per CTA); the
//               pair halves the B bytes each SM stages and reads per MMA;
//   warps 2-9   epilogue (two per TMEM lane quarter, one column half each): tcgen05.ld 32x32b.x32 -> fused
//               GeLU / SwiGLU / GeLU' / SwiGLU' -> bf16 (or the fp32 weight gradient); each 32 x 32 block is
//               staged swizzled in shared memory and leaves through one TMA store (bf16 outputs kept on this
//               GPU) or coalesced per-lane stores (peer rows of the fused exchanges, SwiGLU, weight gradients).
// Tiles walk expert segments whose row offsets (multiples of 128) live on the device, so no host sync
// is needed to size the work.  Operands may be K-major or MN-major (the backward reads W1/W2 and the
// token-major activations transposed through the descriptor's major bit instead of transposing data).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "exchange.cuh"
#include "tc_common.cuh"

namespace luffy {
namespace {

constexpr int BM = 128, BN = 256, BK = 64;  // BM: accumulator rows per CTA (the pair's tile is 256 x 256)
constexpr int A_BYTES = BM * BK * 2;   // 16 KiB per CTA
constexpr int EPI_WARPS = 8;
constexpr int STG_BYTES = 4096;  // per epilogue warp: output staging (coalesced stores)
constexpr int THREADS = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue (2 per TMEM lane quarter)
template <int CG>
struct Pipe {
  static constexpr int STAGES = CG == 1 ? 4 : 6;
  static constexpr int B_ROWS = BN / CG;           // N rows of B staged by one CTA
  static constexpr int B_BYTES = B_ROWS * BK * 2;  // 32 KiB single, 16 KiB in the pair
  static constexpr int SMEM = STAGES * (A_BYTES + B_BYTES) + EPI_WARPS * STG_BYTES + 1024 + 256;
};

struct TcArgs {
  const int32_t* off;  // [G+1] segment offsets (rows), multiples of 128
  int G;
  int N, K, M;         // rows mode: D[rows, N] = A[rows, K] B^T.  wgrad: D[M, N] per group, K = segment rows
  int nbc;             // n-blocks per m-block
  int Nb, Kb;          // rows of one group's B in the B tensor map (K-major: Nb; MN-major: Kb)
  int ksplit;          // MN-major B split along K over (tB, tB3) at Kb
  void* D;
  void* aux;
  float* D3;
  int Msplit;
  int f;               // SwiGLU: d_ffn
  int has_rd;          // EPI_STORE rows: rows go to peer buffers (fused combine / dispatch-backward)
  XRedirect rd;
  int has_sig;         // publish completion to the peers when the kernel ends
  XSignal sig;
  int has_wr;          // fused dispatch: wait per tile for the source ranks of its A rows
  XWaitRows wr;
  int tma_out;         // rows mode: D (and the GeLU' aux) are stored through the tD / tD3 tensor maps
};

struct Tile {
  int g, m0, n0, nkb, krow0, mlim;  // mlim: end of the expert segment (rows mode)
};

// Pair tiles cover two consecutive 128-row blocks of ONE expert segment (the MMA shares B between the
// halves); a segment with an odd block count ends in a half-empty pair whose second half is not stored.
template <bool WG, int CG>
__device__ __forceinline__ int num_tiles(const TcArgs& a, const int32_t* off_s) {
  if (WG) return a.G * (a.M / (BM * CG)) * a.nbc;
  if (CG == 1) return (off_s[a.G] / BM) * a.nbc;
  int n = 0;
  for (int g = 0; g < a.G; ++g) n += ((off_s[g + 1] - off_s[g]) / BM + 1) / 2;
  return n * a.nbc;
}

template <int EPI, bool WG, int CG>
__device__ __forceinline__ Tile decode(int t, const TcArgs& a, const int32_t* off_s) {
  Tile x;
  if (WG) {
    const int tpg = (a.M / (BM * CG)) * a.nbc;
    x.g = t / tpg;
    const int r = t % tpg;
    x.m0 = (r / a.nbc) * BM * CG;
    x.n0 = (r % a.nbc) * BN;
    x.krow0 = off_s[x.g];
    x.nkb = (off_s[x.g + 1] - off_s[x.g]) / BK;
    x.mlim = a.M;
  } else {
    const int mb = t / a.nbc, nb = t % a.nbc;
    if (CG == 1) {
      x.m0 = mb * BM;
      x.g = find_group(off_s, a.G, x.m0);
    } else {
      int r = mb;
      x.g = 0;
      x.m0 = 0;
      for (int g = 0; g < a.G; ++g) {
        const int pb = ((off_s[g + 1] - off_s[g]) / BM + 1) / 2;
        if (r < pb) {
          x.g = g;
          x.m0 = off_s[g] + r * 2 * BM;
          break;
        }
        r -= pb;
      }
    }
    x.mlim = off_s[x.g + 1];
    x.n0 = nb * (EPI == EPI_SWIGLU ? BN / 2 : BN);
    x.nkb = a.K / BK;
    x.krow0 = 0;
  }
  return x;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void store32_bf16(bf16* dst, const float (&v)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u = make_uint4(pack_bf16(v[8 * q], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                         pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
    reinterpret_cast<uint4*>(dst)[q] = u;
  }
}
// ---- warp-cooperative staging of a 32-row x 32-column block (thread i owns row i): the block goes
// through a swizzled 2 KiB (bf16) / 4 KiB (fp32) shared-memory buffer so that every global access
// instruction covers 4 (8) whole 64-byte (128-byte) row segments instead of 32 scattered 16-byte pieces.
__device__ __forceinline__ uint4 pack8_bf16(const float* v) {
  return make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
}
__device__ __forceinline__ void stage_rows_bf16(uint8_t* buf, const float (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    *reinterpret_cast<uint4*>(buf + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)) = pack8_bf16(v + 8 * j);
  __syncwarp();
}
// dst: this thread's row pointer at the block's first column (nullptr: row not stored)
__device__ __forceinline__ void store_block_bf16(uint8_t* buf, const float (&v)[32], bf16* dst) {
  stage_rows_bf16(buf, v);
  const int lane = threadIdx.x & 31;
  const unsigned long long mine = reinterpret_cast<unsigned long long>(dst);
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int r = it * 8 + (lane >> 2), c = lane & 3;
    const uint4 u = *reinterpret_cast<const uint4*>(buf + r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
    const unsigned long long p = __shfl_sync(0xffffffffu, mine, r);
    if (p) reinterpret_cast<uint4*>(reinterpret_cast<bf16*>(p) + c * 8)[0] = u;
  }
  __syncwarp();
}
// multi-destination rows (fused combine with sequence migration): row r goes to every rank in mask[r],
// at row index r2[r] of that rank's buffer peer_base[g] (row length ld elements), column col.
__device__ __forceinline__ void store_block_bf16_multi(uint8_t* buf, const float (&v)[32], unsigned long long mask,
                                                       unsigned long long r2, void* const* peer_base, int ld, int col) {
  stage_rows_bf16(buf, v);
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int r = it * 8 + (lane >> 2), c = lane & 3;
    const uint4 u = *reinterpret_cast<const uint4*>(buf + r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
    unsigned long long m = __shfl_sync(0xffffffffu, mask, r);
    const unsigned long long rr = __shfl_sync(0xffffffffu, r2, r);
    while (m) {
      const int g = __ffsll((long long)m) - 1;
      m &= m - 1;
      reinterpret_cast<uint4*>(static_cast<bf16*>(peer_base[g]) + rr * ld + col + c * 8)[0] = u;
    }
  }
  __syncwarp();
}
// src: this thread's row pointer at the block's first column
__device__ __forceinline__ void load_block_bf16(uint8_t* buf, const bf16* src, float (&v)[32]) {
  const int lane = threadIdx.x & 31;
  const unsigned long long mine = reinterpret_cast<unsigned long long>(src);
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int r = it * 8 + (lane >> 2), c = lane & 3;
    const unsigned long long p = __shfl_sync(0xffffffffu, mine, r);
    *reinterpret_cast<uint4*>(buf + r * 64 + ((c ^ ((r >> 1) & 3)) << 4)) =
        reinterpret_cast<const uint4*>(reinterpret_cast<const bf16*>(p) + c * 8)[0];
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint4 u = *reinterpret_cast<const uint4*>(buf + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      v[8 * j + 2 * i] = f.x;
      v[8 * j + 2 * i + 1] = f.y;
    }
  }
  __syncwarp();
}
__device__ __forceinline__ void store_block_f32(uint8_t* buf, const float (&v)[32], float* dst) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    *reinterpret_cast<float4*>(buf + lane * 128 + ((j ^ (lane & 7)) << 4)) =
        make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  __syncwarp();
  const unsigned long long mine = reinterpret_cast<unsigned long long>(dst);
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int r = it * 4 + (lane >> 3), c = lane & 7;
    const float4 u = *reinterpret_cast<const float4*>(buf + r * 128 + ((c ^ (r & 7)) << 4));
    const unsigned long long p = __shfl_sync(0xffffffffu, mine, r);
    reinterpret_cast<float4*>(reinterpret_cast<float*>(p) + c * 4)[0] = u;
  }
  __syncwarp();
}

__device__ __forceinline__ void load32_bf16(const bf16* src, float (&v)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u = reinterpret_cast<const uint4*>(src)[q];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(h[i]);
      v[8 * q + 2 * i] = f.x;
      v[8 * q + 2 * i + 1] = f.y;
    }
  }
}

template <int EPI, bool A_MN, bool B_MN, bool WG, int CG>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                   const __grid_constant__ CUtensorMap tB3, const __grid_constant__ CUtensorMap tD,
                   const __grid_constant__ CUtensorMap tD3, const TcArgs a) {
  pdl_defer();
  constexpr int STAGES = Pipe<CG>::STAGES;
  constexpr int B_BYTES = Pipe<CG>::B_BYTES;
  constexpr int B_ROWS = Pipe<CG>::B_ROWS;
  extern __shared__ uint8_t smem_raw[];
  __shared__ int32_t off_s[LUFFY_MAX_EXPERTS + 1];
  const uint32_t crank = CG == 2 ? tc::cluster_rank() : 0u;  // 0: leader (issues the MMA)
  const int hm = (int)crank * BM;       // this CTA's accumulator rows within the pair tile
  const int hb = (int)crank * B_ROWS;   // this CTA's N rows of B within the tile
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint8_t* sStg = sB + STAGES * B_BYTES;  // epilogue staging, STG_BYTES per epilogue warp
  uint64_t* full = reinterpret_cast<uint64_t*>(sStg + EPI_WARPS * STG_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&tfull[s], 1);
      tc::mbar_init(&tempty[s], EPI_WARPS * CG);  // the pair's epilogue warps all release the leader's buffer
    }
    tc::fence_barrier_init();
    tc::tma_prefetch(&tA);
    tc::tma_prefetch(&tB);
    if (EPI == EPI_SWIGLU || B_MN) tc::tma_prefetch(&tB3);
  }
  if (warp == 1) {
    if (CG == 2) tc::tmem_alloc_pair(tmem_holder, 512);
    else tc::tmem_alloc(tmem_holder, 512);
  }
  tc::tc_fence_before();
  if (CG == 2) tc::cluster_sync();  // barrier inits visible to the peer before any remote arrive
  else __syncthreads();
  tc::tc_fence_after();
  pdl_enter();  // from here on: the previous kernel's outputs (expert offsets, operands)
  for (int i = threadIdx.x; i <= a.G; i += blockDim.x) off_s[i] = a.off[i];
  __syncthreads();
  const uint32_t tmem_base = *tmem_holder;
  const int ntiles = num_tiles<WG, CG>(a, off_s);
  const int tile0 = CG == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int tstride = CG == 2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = tile0; t < ntiles; t += tstride) {
        const Tile x = decode<EPI, WG, CG>(t, a, off_s);
        if (!WG && a.has_wr) xwait_rows(a.wr, x.g, x.m0 + hm, min(x.m0 + hm + BM, x.mlim));
        for (int kb = 0; kb < x.nkb; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* dA = sA + stage * A_BYTES;
          uint8_t* dB = sB + stage * B_BYTES;
          uint32_t barc = 0;  // pair: the leader's full barrier (both CTAs' bytes complete on it)
          if (CG == 2) {
            if (crank == 0) tc::mbar_expect_tx(&full[stage], 2 * (A_BYTES + B_BYTES));
            barc = tc::map_rank(&full[stage], 0);
          } else {
            tc::mbar_expect_tx(&full[stage], A_BYTES + B_BYTES);
          }
          auto LD = [&](void* dst, const CUtensorMap* m, int c0, int c1) {
            if (CG == 2) tc::tma_load_2d_pair(dst, m, barc, c0, c1);
            else tc::tma_load_2d(dst, m, &full[stage], c0, c1);
          };
          if (!A_MN) {
            LD(dA, &tA, kb * BK, x.m0 + hm);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) LD(dA + j * 8192, &tA, x.m0 + hm + 64 * j, x.krow0 + kb * BK);
          }
          if (WG) {
#pragma unroll
            for (int j = 0; j < B_ROWS / 64; ++j) LD(dB + j * 8192, &tB, x.n0 + hb + 64 * j, x.krow0 + kb * BK);
          } else if (!B_MN) {
            if (EPI == EPI_SWIGLU) {  // N = [W1 rows n0.. (128) | W3 rows n0.. (128)]; the pair splits them
              if (CG == 2) {
                LD(dB, crank == 0 ? &tB : &tB3, kb * BK, x.g * a.Nb + x.n0);
              } else {
                LD(dB, &tB, kb * BK, x.g * a.Nb + x.n0);
                LD(dB + B_BYTES / 2, &tB3, kb * BK, x.g * a.Nb + x.n0);
              }
            } else {
              LD(dB, &tB, kb * BK, x.g * a.Nb + x.n0 + hb);
            }
          } else {
            const int kk = kb * BK;
            const bool hi = a.ksplit && kk >= a.Kb;
            const CUtensorMap* mp = hi ? &tB3 : &tB;
            const int kl = hi ? kk - a.Kb : kk;
#pragma unroll
            for (int j = 0; j < B_ROWS / 64; ++j) LD(dB + j * 8192, mp, x.n0 + hb + 64 * j, x.g * a.Kb + kl);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && crank == 0) {
      // ------------------------------------------------------------------ MMA issuer (single thread)
      constexpr uint32_t IDESC = tc::idesc_bf16(BM * CG, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0;
      for (int t = tile0; t < ntiles; t += tstride) {
        const Tile x = decode<EPI, WG, CG>(t, a, off_s);
        tc::mbar_wait(&tempty[acc], aphase ^ 1);
        tc::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < x.nkb; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::tc_fence_after();
          const uint32_t a0 = tc::smem_u32(sA + stage * A_BYTES);
          const uint32_t b0 = tc::smem_u32(sB + stage * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = A_MN ? tc::smem_desc(a0 + kk * 2048, 8192, 1024) : tc::smem_desc(a0 + kk * 32, 16, 1024);
            const uint64_t bd = (B_MN || WG) ? tc::smem_desc(b0 + kk * 2048, 8192, 1024) : tc::smem_desc(b0 + kk * 32, 16, 1024);
            if (CG == 2) tc::mma_bf16_pair(d_tmem, ad, bd, IDESC, (kb | kk) != 0 ? 1u : 0u);
            else tc::mma_bf16(d_tmem, ad, bd, IDESC, (kb | kk) != 0 ? 1u : 0u);
          }
          if (CG == 2) tc::mma_commit_pair(&empty[stage], 3);
          else tc::mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (CG == 2) tc::mma_commit_pair(&tfull[acc], 3);
        else tc::mma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
      }
    }
  } else {
    // -------------------------------------------------------------------- epilogue warps 2..5
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int hc = (warp - 2) >> 2;  // column half handled by this warp
    const int rt = 32 * q + lane;
    uint8_t* stg = sStg + (warp - 2) * STG_BYTES;  // [0, 2K) and [2K, 4K): two bf16 blocks or one fp32 block
    int acc = 0;
    uint32_t aphase = 0;
    // aux (pre-activation) blocks of the backward epilogues are prefetched one 32-column chunk ahead with
    // coalesced loads (the first one before waiting for the accumulator), then re-laid through shared memory
    constexpr int NB = (EPI == EPI_DSWIGLU) ? 2 : ((EPI == EPI_DGELU) ? 1 : 0);
    uint4 pf[2][4];
    auto prefetch = [&](const Tile& x, int c0) {
      const size_t ldx = (EPI == EPI_DSWIGLU) ? 2 * (size_t)a.N : (size_t)a.N;
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int r = it * 8 + (lane >> 2), c = lane & 3;
          const bf16* src = static_cast<const bf16*>(a.aux) + (size_t)(x.m0 + hm + 32 * q + r) * ldx + (b ? a.N : 0) +
                            x.n0 + c0 + c * 8;
          pf[b][it] = *reinterpret_cast<const uint4*>(src);
        }
    };
    for (int t = tile0; t < ntiles; t += tstride) {
      const Tile x = decode<EPI, WG, CG>(t, a, off_s);
      const bool live = WG || x.m0 + hm < x.mlim;  // the second half of an expert's last pair may be empty
      if (NB && live) prefetch(x, hc * (BN / 2));
      tc::mbar_wait(&tfull[acc], aphase);
      tc::tc_fence_after();
      const uint32_t tb = tmem_base + ((uint32_t)(32 * q) << 16) + acc * BN;
      if (!live) {
      } else if (WG && !a.tma_out) {  // per-lane stores through the staging buffer (default)
        const int m = x.m0 + hm + rt;
        float* dst = m < a.Msplit ? static_cast<float*>(a.D) + ((size_t)x.g * a.Msplit + m) * a.N
                                  : a.D3 + ((size_t)x.g * (a.M - a.Msplit) + (m - a.Msplit)) * a.N;
        dst += x.n0;
#pragma unroll 1
        for (int c0 = hc * (BN / 2); c0 < (hc + 1) * (BN / 2); c0 += 32) {
          uint32_t r[32];
          tc::tmem_ld32(tb + c0, r);
          tc::tmem_ld_wait();
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = x.nkb > 0 ? __uint_as_float(r[i]) : 0.f;
          store_block_f32(stg, v, dst + c0);
        }
      } else if (WG) {
        // fp32 32x32 blocks leave through TMA stores (tensor maps tD / tD3, box 32 x 32, SWIZZLE_128B): the
        // staging layout below is the 128-byte swizzle, so one lane issues the whole 4 KiB block
        const int row0 = x.m0 + hm + 32 * q;  // Msplit is a multiple of 32: a block lies on one side
        const bool lo = row0 < a.Msplit;
        const CUtensorMap* md = lo ? &tD : &tD3;
        const int orow = lo ? x.g * a.Msplit + row0 : x.g * (a.M - a.Msplit) + (row0 - a.Msplit);
#pragma unroll 1
        for (int c0 = hc * (BN / 2); c0 < (hc + 1) * (BN / 2); c0 += 32) {
          uint32_t r[32];
          tc::tmem_ld32(tb + c0, r);
          tc::tmem_ld_wait();
          if (lane == 0) tc::bulk_wait_read();  // the previous block's store has read the buffer
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4 u = x.nkb > 0 ? make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                               __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
            *reinterpret_cast<float4*>(stg + lane * 128 + ((j ^ (lane & 7)) << 4)) = u;
          }
          tc::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) tc::tma_store_2d(md, stg, x.n0 + c0, orow);
        }
      } else {
        const size_t row = (size_t)(x.m0 + hm + rt);
        bf16* D = static_cast<bf16*>(a.D);
        bf16* X = static_cast<bf16*>(a.aux);
        // GEMM outputs that stay on this GPU leave through TMA stores (tD = D, tD3 = the GeLU' aux)
        const bool tma_out = (EPI == EPI_STORE || EPI == EPI_GELU || EPI == EPI_DGELU) && a.tma_out;
        if (EPI == EPI_SWIGLU) {
          const int f = a.f;
#pragma unroll 1
          for (int c0 = hc * (BN / 4); c0 < (hc + 1) * (BN / 4); c0 += 32) {
            uint32_t r1[32], r3[32];
            tc::tmem_ld32(tb + c0, r1);
            tc::tmem_ld32(tb + BN / 2 + c0, r3);
            tc::tmem_ld_wait();
            float p1[32], p3[32], o[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              p1[i] = __uint_as_float(r1[i]);
              p3[i] = __uint_as_float(r3[i]);
              o[i] = silu_f(p1[i]) * p3[i];
            }
            const int n = x.n0 + c0;
            store_block_bf16(stg, p1, X + row * (2 * f) + n);
            store_block_bf16(stg, p3, X + row * (2 * f) + f + n);
            store_block_bf16(stg, o, D + row * f + n);
          }
        } else {
#pragma unroll 1
          for (int c0 = hc * (BN / 2); c0 < (hc + 1) * (BN / 2); c0 += 32) {
            float pa[NB > 0 ? NB : 1][32];
#pragma unroll
            for (int b = 0; b < NB; ++b) {  // prefetched aux block -> own row through shared memory
              uint8_t* ab = stg + 2048;
#pragma unroll
              for (int it = 0; it < 4; ++it) {
                const int r = it * 8 + (lane >> 2), c = lane & 3;
                *reinterpret_cast<uint4*>(ab + r * 64 + ((c ^ ((r >> 1) & 3)) << 4)) = pf[b][it];
              }
              __syncwarp();
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const uint4 u = *reinterpret_cast<const uint4*>(ab + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4));
                const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const float2 f2 = __bfloat1622float2(h2[i]);
                  pa[b][8 * j + 2 * i] = f2.x;
                  pa[b][8 * j + 2 * i + 1] = f2.y;
                }
              }
              __syncwarp();
            }
            if (NB && c0 + 32 < (hc + 1) * (BN / 2)) prefetch(x, c0 + 32);  // next chunk in flight
            uint32_t r[32];
            tc::tmem_ld32(tb + c0, r);
            tc::tmem_ld_wait();
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
            const int n = x.n0 + c0;
            if (tma_out) {  // local output: 32 x 32 blocks leave through TMA stores (box 32 x 32, SWIZZLE_64B)
              float o[32];
              if (EPI == EPI_GELU) {
#pragma unroll
                for (int i = 0; i < 32; i += 2) {  // v <- GeLU'(pre), o <- GeLU(pre)
                  float2 gg, dd;
                  gelu_and_grad_as2(make_float2(v[i], v[i + 1]), gg, dd);
                  o[i] = gg.x;
                  o[i + 1] = gg.y;
                  v[i] = dd.x;
                  v[i + 1] = dd.y;
                }
              } else if (EPI == EPI_DGELU) {
#pragma unroll
                for (int i = 0; i < 32; i += 2) {
                  const float2 p = __fmul2_rn(make_float2(v[i], v[i + 1]), make_float2(pa[0][i], pa[0][i + 1]));
                  v[i] = p.x;
                  v[i + 1] = p.y;
                }
              }
              if (lane == 0) tc::bulk_wait_read();  // the previous chunk's stores have read the buffers
              __syncwarp();
              stage_rows_bf16(stg, EPI == EPI_GELU ? o : v);
              if (EPI == EPI_GELU) stage_rows_bf16(stg + 2048, v);
              tc::fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                const int row0 = x.m0 + hm + 32 * q;
                tc::tma_store_2d(&tD, stg, n, row0);
                if (EPI == EPI_GELU) tc::tma_store_2d(&tD3, stg + 2048, n, row0);
              }
            } else if (EPI == EPI_STORE) {
              if (a.has_rd) {  // fused exchange: the row goes straight to its rank's buffer over NVLink
                if (a.rd.mask) {  // combine: every destination rank of the row (sequence migration)
                  const unsigned long long m = a.rd.mask[row];
                  const int rk = a.rd.rank_of[row];
                  const unsigned long long r2 =
                      rk >= 0 ? (unsigned long long)rk * a.rd.stride + a.rd.slot_of[row] : 0ull;
                  store_block_bf16_multi(stg, v, rk >= 0 ? m : 0ull, r2, a.rd.peer_base, a.N, n);
                } else {
                  const int rk = a.rd.rank_of[row];
                  store_block_bf16(stg, v,
                                   rk >= 0 ? static_cast<bf16*>(a.rd.peer_base[rk]) + (size_t)a.rd.slot_of[row] * a.N + n
                                           : nullptr);
                }
              } else {
                store_block_bf16(stg, v, D + row * a.N + n);
              }
            } else if (EPI == EPI_GELU) {
              float o[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) gelu_and_grad_as(v[i], o[i], v[i]);  // v <- GeLU'(pre)
              store_block_bf16(stg, v, X + row * a.N + n);
              store_block_bf16(stg, o, D + row * a.N + n);
            } else if (EPI == EPI_DGELU) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] *= pa[0][i];  // aux holds GeLU'(pre) from the forward
              store_block_bf16(stg, v, D + row * a.N + n);
            } else {  // EPI_DSWIGLU: v = d_act, aux = pre [rows, 2N]
              float g1[32], g3[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const float p1 = pa[0][i], p3 = pa[NB - 1][i];
                g1[i] = v[i] * p3 * silu_grad_f(p1);
                g3[i] = v[i] * silu_f(p1);
              }
              store_block_bf16(stg, g1, D + row * (2 * a.N) + n);
              store_block_bf16(stg, g3, D + row * (2 * a.N) + a.N + n);
            }
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) tc::mbar_arrive_cluster_relaxed(tc::map_rank(&tempty[acc], 0));
        else tc::mbar_arrive(&tempty[acc]);
      }
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
    if (lane == 0) tc::bulk_wait_all();  // TMA stores complete before the CTA (and its buffers) retires
  }
  if (CG == 2) {
    tc::tc_fence_before();
    tc::cluster_sync();  // no CTA of the pair leaves while the other can still arrive on its barriers
    if (warp == 1) tc::tmem_dealloc_pair(tmem_base, 512);
  } else {
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem_base, 512);
  }
  if (a.has_sig) xsignal_done(a.sig);
}

int num_sms() { return device_sms(); }

// TMA stores for the bf16 outputs of the rows GEMMs that stay on this GPU.  LUFFY_TMA_STORE (A/B
// measurements): 0 = none, 1 = also the fp32 weight gradients, 2 = rows GEMMs only (default: with one
// 4 KiB staging buffer per warp the wgrad epilogue waits for each block's store to drain the buffer and
// measured ~0.5% slower per step than its per-lane stores; 0 is ~2% slower than 2)
int tma_store_mode() {
  static const int mode = [] {
    const char* v = std::getenv("LUFFY_TMA_STORE");
    return v && v[0] >= '0' && v[0] <= '2' ? v[0] - '0' : 2;
  }();
  return mode;
}

// CTA pairs unless LUFFY_GEMM_CG=1 (single-CTA fallback, A/B measurements)
bool use_pairs() {
  static const bool on = [] {
    const char* v = std::getenv("LUFFY_GEMM_CG");
    return !(v && v[0] == '1');
  }();
  return on;
}

template <int EPI, bool A_MN, bool B_MN, bool WG, int CG>
int launch_cg(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tb3, const CUtensorMap& td,
              const CUtensorMap& td3, const TcArgs& a, cudaStream_t s) {
  auto kern = gemm_tc_kernel<EPI, A_MN, B_MN, WG, CG>;
  constexpr int SMEM_BYTES = Pipe<CG>::SMEM;
  LUFFY_CUDA_TRY(smem_optin((const void*)kern, SMEM_BYTES));
  if (CG == 1) {
    launch_pdl(kern, num_sms(), THREADS, SMEM_BYTES, s, ta, tb, tb3, td, td3, a);
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    // persistent: as many pairs as can be co-resident (a TPC with one usable SM cannot host a pair)
    int pairs = 0;
    if (!dev_cache_get((const void*)kern, -1, &pairs)) {
      cfg.gridDim = dim3(num_sms() & ~1);
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1) n = num_sms() / 2;
      cudaGetLastError();
      pairs = std::min(n, num_sms() / 2);
      dev_cache_put((const void*)kern, -1, pairs);
      if (std::getenv("LUFFY_VERBOSE")) std::fprintf(stderr, "[luffy] gemm pair grid: %d co-resident pairs\n", pairs);
    }
    static const int cap = [] {  // LUFFY_GEMM_PAIRS: fewer pairs (bandwidth-sharing experiments only)
      const char* v = std::getenv("LUFFY_GEMM_PAIRS");
      return v ? std::atoi(v) : 0;
    }();
    if (cap > 0) pairs = std::min(pairs, cap);
    cfg.gridDim = dim3(2 * pairs);
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    cudaLaunchKernelEx(&cfg, kern, ta, tb, tb3, td, td3, a);
  }
  LUFFY_LAUNCHED();
  return 0;
}

template <int EPI, bool A_MN, bool B_MN, bool WG>
int launch(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tb3, const TcArgs& a, cudaStream_t s,
           const CUtensorMap* td = nullptr, const CUtensorMap* td3 = nullptr) {
  const CUtensorMap& d = td ? *td : ta;  // output maps: weight gradient only
  const CUtensorMap& d3 = td3 ? *td3 : d;
  return use_pairs() ? launch_cg<EPI, A_MN, B_MN, WG, 2>(ta, tb, tb3, d, d3, a, s)
                     : launch_cg<EPI, A_MN, B_MN, WG, 1>(ta, tb, tb3, d, d3, a, s);
}

}  // namespace

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return nullptr;
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  return encode;
}
// fp32 output [outer, inner] (row stride = inner), stored in 32 x 32 boxes with the 128-byte swizzle
int make_tmap_f32_store(CUtensorMap* m, void* ptr, uint64_t inner, uint64_t outer) {
  EncodeFn encode = encode_fn();
  if (!encode) return (int)cudaErrorNotSupported;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}
// bf16 output [outer, inner] (row stride = inner), stored in 32 x 32 boxes with the 64-byte swizzle
int make_tmap_bf16_store(CUtensorMap* m, void* ptr, uint64_t inner, uint64_t outer) {
  EncodeFn encode = encode_fn();
  if (!encode) return (int)cudaErrorNotSupported;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}
}  // namespace

int make_tmap_bf16(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_stride_elems,
                   uint32_t box_outer) {
  EncodeFn encode = encode_fn();
  if (!encode) return (int)cudaErrorNotSupported;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_elems * 2};
  cuuint32_t box[2] = {64, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}

// Rows GEMM: D[r, :] over expert segments; see luffy_internal.h (Epi) for the epilogues.
int gemm_rows_tc(int epi, const void* A, const void* B, const void* B3, void* D, void* aux0, const int32_t* off, int G,
                 int64_t max_rows, int N, int K, int b_kmajor, const XRedirect* rd, const XSignal* sig, void* s,
                 const XWaitRows* wr) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  TcArgs a{};
  if (wr) {
    a.has_wr = 1;
    a.wr = *wr;
  }
  if (rd) {
    a.has_rd = 1;
    a.rd = *rd;
  }
  if (sig) {
    a.has_sig = 1;
    a.sig = *sig;
  }
  a.off = off;
  a.G = G;
  a.N = N;
  a.K = K;
  a.D = D;
  a.aux = aux0;
  a.f = N / 2;
  CUtensorMap ta, tb, tb3, td, td3;
  LUFFY_CUDA_TRY(make_tmap_bf16(&ta, A, K, max_rows, K, BM));
  // outputs kept on this GPU (no peer redirect, no completion signal) use TMA stores; D (and aux) hold
  // max_rows rows like A
  a.tma_out = tma_store_mode() != 0 && !rd && !sig && (epi == EPI_STORE || epi == EPI_GELU || epi == EPI_DGELU);
  if (a.tma_out) {
    LUFFY_CUDA_TRY(make_tmap_bf16_store(&td, D, N, max_rows));
    if (epi == EPI_GELU) LUFFY_CUDA_TRY(make_tmap_bf16_store(&td3, aux0, N, max_rows));
    else td3 = td;
  } else {
    td = ta;
    td3 = ta;
  }
  if (b_kmajor) {
    const bool sw = epi == EPI_SWIGLU;
    a.Nb = sw ? N / 2 : N;
    a.nbc = sw ? (N / 2) / (BN / 2) : N / BN;
    LUFFY_CUDA_TRY(make_tmap_bf16(&tb, B, K, (uint64_t)G * a.Nb, K, sw ? BN / 2 : (use_pairs() ? BN / 2 : BN)));
    if (sw) LUFFY_CUDA_TRY(make_tmap_bf16(&tb3, B3, K, (uint64_t)G * a.Nb, K, BN / 2));
    else tb3 = tb;
    switch (epi) {
      case EPI_STORE: return launch<EPI_STORE, false, false, false>(ta, tb, tb3, a, st, &td, &td3);
      case EPI_GELU: return launch<EPI_GELU, false, false, false>(ta, tb, tb3, a, st, &td, &td3);
      case EPI_SWIGLU: return launch<EPI_SWIGLU, false, false, false>(ta, tb, tb3, a, st);
      default: return (int)cudaErrorNotSupported;
    }
  }
  a.ksplit = B3 != nullptr && epi == EPI_STORE;
  a.Kb = a.ksplit ? K / 2 : K;
  a.nbc = N / BN;
  LUFFY_CUDA_TRY(make_tmap_bf16(&tb, B, N, (uint64_t)G * a.Kb, N, 64));
  if (a.ksplit) LUFFY_CUDA_TRY(make_tmap_bf16(&tb3, B3, N, (uint64_t)G * a.Kb, N, 64));
  else tb3 = tb;
  switch (epi) {
    case EPI_STORE: return launch<EPI_STORE, false, true, false>(ta, tb, tb3, a, st, &td, &td3);
    case EPI_DGELU: return launch<EPI_DGELU, false, true, false>(ta, tb, tb3, a, st, &td, &td3);
    case EPI_DSWIGLU: return launch<EPI_DSWIGLU, false, true, false>(ta, tb, tb3, a, st);
    default: return (int)cudaErrorNotSupported;
  }
}

// Weight gradient: D_g[m, n] = sum over segment g rows of A[r, m] * B[r, n] (fp32 out, rows m >= Msplit -> D3).
int gemm_wgrad_tc(const void* A, const void* B, float* D, float* D3, int Msplit, const int32_t* off, int G, int M, int N,
                  int lda, int ldb, int64_t max_rows, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  TcArgs a{};
  a.off = off;
  a.G = G;
  a.M = M;
  a.N = N;
  a.nbc = N / BN;
  a.D = D;
  a.D3 = D3;
  a.Msplit = Msplit;
  if (Msplit % 32 != 0 || (Msplit < M && !D3)) return (int)cudaErrorInvalidValue;
  a.tma_out = tma_store_mode() == 1;
  CUtensorMap ta, tb, td, td3;
  LUFFY_CUDA_TRY(make_tmap_bf16(&ta, A, M, max_rows, lda, 64));
  LUFFY_CUDA_TRY(make_tmap_bf16(&tb, B, N, max_rows, ldb, 64));
  LUFFY_CUDA_TRY(make_tmap_f32_store(&td, D, N, (uint64_t)G * Msplit));
  if (Msplit < M) LUFFY_CUDA_TRY(make_tmap_f32_store(&td3, D3, N, (uint64_t)G * (M - Msplit)));
  else td3 = td;
  return launch<EPI_STORE, true, true, true>(ta, tb, tb, a, st, &td, &td3);
}

}  // namespace luffy
