// Top-k gate ("top-2 gating"; readings R1, R2) and its backward.
//
// Forward: one warp per token.  Lanes stream the token row with 16-byte loads, accumulate the E
// partial dot products with the fp32 gate weights in a fixed order (chunk order, then a butterfly
// reduction), so the result is bitwise reproducible.  Top-k by (logit desc, expert id asc) via a warp
// argmax; softmax over all experts is saved for the backward.
#include <algorithm>

#include "common.cuh"

namespace luffy {
namespace {

template <typename T, int EB>
__global__ void __launch_bounds__(256) route_kernel(const T* __restrict__ x, const float* __restrict__ wg,
                                                    int T_, int E, int d, int k, int renorm,
                                                    float* __restrict__ probs, int32_t* __restrict__ idx,
                                                    float* __restrict__ w, int32_t* __restrict__ idx_out,
                                                    float* __restrict__ w_out) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < T_; t += nwarps) {
    float mine[EB / 32 > 0 ? EB / 32 : 1];  // lane l keeps the logit of experts l, l+32, ...
#pragma unroll
    for (int i = 0; i < (EB / 32 > 0 ? EB / 32 : 1); ++i) mine[i] = -INFINITY;
    const T* xr = x + (size_t)t * d;
    for (int e0 = 0; e0 < E; e0 += EB) {
      float acc[EB];
#pragma unroll
      for (int e = 0; e < EB; ++e) acc[e] = 0.f;
      for (int c = lane * 8; c < d; c += 256) {
        float xv[8];
        load8(xr + c, xv);
#pragma unroll
        for (int e = 0; e < EB; ++e) {
          if (e0 + e < E) {
            float wv[8];
            load8(wg + (size_t)(e0 + e) * d + c, wv);
            float s = acc[e];
#pragma unroll
            for (int i = 0; i < 8; ++i) s = fmaf(xv[i], wv[i], s);
            acc[e] = s;
          }
        }
      }
#pragma unroll
      for (int e = 0; e < EB; ++e) {
        float s = warp_sum(acc[e]);
        int ge = e0 + e;
        if (ge < E && (ge & 31) == lane) mine[(ge >> 5) % (EB / 32 > 0 ? EB / 32 : 1)] = s;
      }
    }
    // mine[] holds expert (lane + 32*i) when E <= EB (host guarantees EB >= E rounded to 32)
    const int per = (E + 31) / 32;
    // softmax over all experts (fixed butterfly order)
    float mx = -INFINITY;
    for (int i = 0; i < per; ++i) mx = fmaxf(mx, mine[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float ex[EB / 32 > 0 ? EB / 32 : 1];
    float se = 0.f;
    for (int i = 0; i < per; ++i) {
      int e = lane + 32 * i;
      ex[i] = e < E ? expf(mine[i] - mx) : 0.f;
      se += ex[i];
    }
    se = warp_sum(se);
    for (int i = 0; i < per; ++i) {
      int e = lane + 32 * i;
      if (e < E) probs[(size_t)t * E + e] = ex[i] / se;
    }
    // top-k: repeated warp argmax of (logit, -id)
    float selv[8];
    int seli[8];
    unsigned taken[EB / 32 > 0 ? EB / 32 : 1];
    for (int i = 0; i < per; ++i) taken[i] = 0;
    for (int j = 0; j < k; ++j) {
      float bv = -INFINITY;
      int bi = 0x7fffffff;
      for (int i = 0; i < per; ++i) {
        int e = lane + 32 * i;
        if (e < E && !taken[i] && (mine[i] > bv || (mine[i] == bv && e < bi))) { bv = mine[i]; bi = e; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if ((bi & 31) == lane) taken[bi >> 5] = 1;
      selv[j] = bv;
      seli[j] = bi;
    }
    if (lane == 0) {
      if (renorm) {
        float s = 0.f, ev[8];
        for (int j = 0; j < k; ++j) { ev[j] = expf(selv[j] - selv[0]); s += ev[j]; }
        for (int j = 0; j < k; ++j) {
          float wv = ev[j] / s;
          w[(size_t)t * k + j] = wv;
          w_out[(size_t)t * k + j] = wv;
        }
      } else {
        for (int j = 0; j < k; ++j) {
          float wv = expf(selv[j] - mx) / se;
          w[(size_t)t * k + j] = wv;
          w_out[(size_t)t * k + j] = wv;
        }
      }
      for (int j = 0; j < k; ++j) {
        idx[(size_t)t * k + j] = seli[j];
        idx_out[(size_t)t * k + j] = seli[j];
      }
    }
  }
}

// Row fragments of 4 consecutive elements: raw load (8 bytes for bf16, 16 for fp32), conversion, store.
__device__ __forceinline__ uint2 ld4raw(const bf16* p) { return *reinterpret_cast<const uint2*>(p); }
__device__ __forceinline__ float4 ld4raw(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void cvt4(uint2 u, float (&f)[4]) {
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
  f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y;
}
__device__ __forceinline__ void cvt4(float4 u, float (&f)[4]) { f[0] = u.x; f[1] = u.y; f[2] = u.z; f[3] = u.w; }
__device__ __forceinline__ void st4(bf16* p, const float (&f)[4]) {
  const __nv_bfloat162 a = __floats2bfloat162_rn(f[0], f[1]);
  const __nv_bfloat162 b = __floats2bfloat162_rn(f[2], f[3]);
  uint2 u;
  u.x = *reinterpret_cast<const uint32_t*>(&a);
  u.y = *reinterpret_cast<const uint32_t*>(&b);
  *reinterpret_cast<uint2*>(p) = u;
}
__device__ __forceinline__ void st4(float* p, const float (&f)[4]) { *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]); }

// Gate for E <= 8, d % 256 == 0 (the GPT-MoE shapes): a CTA of 8 warps, 4 tokens per warp.  The row loads
// of up to 1024 columns of the warp's 4 tokens are issued first, W_g (<= 2048 columns per chunk, 64 KiB) is
// staged in shared memory meanwhile, and each float4 weight read feeds the 4 tokens.  The 32 partial sums
// (4 tokens x 8 experts) of every lane are then TRANSPOSE-reduced in 31 shuffles so that lane l holds the
// logit of (token l / 8, expert l % 8), and softmax / top-k / gate weights run lane-parallel in 8-lane
// groups.  Summation order is fixed (column order within a lane, then the halving tree): reproducible.
template <typename T>
__global__ void __launch_bounds__(256, 2) route_e8_kernel(const T* __restrict__ x, const float* __restrict__ wg, int T_,
                                                          int E, int d, int k, int renorm, float* __restrict__ probs,
                                                          int32_t* __restrict__ idx, float* __restrict__ w,
                                                          int32_t* __restrict__ idx_out, float* __restrict__ w_out) {
  pdl_enter();
  constexpr int TB = 4, EB = 8, RC = 2048;
  constexpr int SUB = sizeof(T) == 2 ? 4 : 2;  // 256-column sub-chunks per load batch
  using R = decltype(ld4raw(static_cast<const T*>(nullptr)));
  extern __shared__ __align__(16) float wsm[];  // [EB][RC]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int t0 = (blockIdx.x * 8 + wid) * TB;
  float v[TB * EB];
#pragma unroll
  for (int i = 0; i < TB * EB; ++i) v[i] = 0.f;
  for (int c0 = 0; c0 < d; c0 += RC) {
    const int rc = min(RC, d - c0);
    for (int s0 = 0; s0 < rc; s0 += 256 * SUB) {
      R raw[TB][SUB][2];
#pragma unroll
      for (int i = 0; i < TB; ++i)
#pragma unroll
        for (int u = 0; u < SUB; ++u)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = s0 + u * 256 + h * 128 + lane * 4;
            raw[i][u][h] = (t0 + i < T_ && c < rc) ? ld4raw(x + (size_t)(t0 + i) * d + c0 + c) : R{};
          }
      if (s0 == 0) {  // stage this chunk of W_g while the first row loads are in flight
        __syncthreads();
        // expert-pair layout: float4 ((2p + hf) * RC/4 + c/4) holds (w_2p, w_2p+1) at columns c + 2 hf and
        // c + 2 hf + 1, so one conflict-free float4 read feeds two packed FMAs; the partner of an odd last
        // expert is zero
        const int Ep = (E + 1) & ~1;
        for (int i = threadIdx.x; i < Ep * (rc / 4); i += blockDim.x) {
          const int e = i / (rc / 4), c = (i % (rc / 4)) * 4;
          const float4 q = e < E ? *reinterpret_cast<const float4*>(wg + (size_t)e * d + c0 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
          float* b0 = &wsm[((e >> 1) * 2 * (RC / 4) + (c >> 2)) * 4 + (e & 1)];
          float* b1 = b0 + RC;  // hf = 1: (RC / 4) float4 further
          b0[0] = q.x;
          b0[2] = q.y;
          b1[0] = q.z;
          b1[2] = q.w;
        }
        __syncthreads();
      }
#pragma unroll
      for (int u = 0; u < SUB; ++u) {
        if (s0 + u * 256 >= rc) break;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = s0 + u * 256 + h * 128 + lane * 4;
          float xv[TB][4];
#pragma unroll
          for (int i = 0; i < TB; ++i) cvt4(raw[i][u][h], xv[i]);
          // packed fp32x2 FMAs over expert pairs: each logit keeps its own column-ordered fmaf chain, so the
          // results are bit-identical to the scalar form at half the issue slots
#pragma unroll
          for (int p = 0; p < EB / 2; ++p) {
            if (2 * p < E) {
              const float4 w0 = *reinterpret_cast<const float4*>(&wsm[(p * 2 * (RC / 4) + (c >> 2)) * 4]);
              const float4 w1 = *reinterpret_cast<const float4*>(&wsm[((p * 2 + 1) * (RC / 4) + (c >> 2)) * 4]);
#pragma unroll
              for (int i = 0; i < TB; ++i) {
                float2 s2 = make_float2(v[i * EB + 2 * p], v[i * EB + 2 * p + 1]);
                s2 = __ffma2_rn(make_float2(xv[i][0], xv[i][0]), make_float2(w0.x, w0.y), s2);
                s2 = __ffma2_rn(make_float2(xv[i][1], xv[i][1]), make_float2(w0.z, w0.w), s2);
                s2 = __ffma2_rn(make_float2(xv[i][2], xv[i][2]), make_float2(w1.x, w1.y), s2);
                s2 = __ffma2_rn(make_float2(xv[i][3], xv[i][3]), make_float2(w1.z, w1.w), s2);
                v[i * EB + 2 * p] = s2.x;
                v[i * EB + 2 * p + 1] = s2.y;
              }
            }
          }
        }
      }
    }
  }
  // transpose-reduce: after the step with offset o, a lane keeps the half of its values selected by (lane & o)
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const bool hi = lane & 16;
    const float send = hi ? v[j] : v[j + 16];
    const float keep = hi ? v[j + 16] : v[j];
    v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const bool hi = lane & 8;
    const float send = hi ? v[j] : v[j + 8];
    const float keep = hi ? v[j + 8] : v[j];
    v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const bool hi = lane & 4;
    const float send = hi ? v[j] : v[j + 4];
    const float keep = hi ? v[j + 4] : v[j];
    v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const bool hi = lane & 2;
    const float send = hi ? v[j] : v[j + 2];
    const float keep = hi ? v[j + 2] : v[j];
    v[j] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  {
    const bool hi = lane & 1;
    const float send = hi ? v[0] : v[1];
    const float keep = hi ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
  }
  // lane l: token t0 + l / 8, expert e = l % 8 (8-lane groups, xor offsets < 8 stay inside a group)
  const int e = lane & 7;
  const int t = t0 + (lane >> 3);
  const float logit = e < E ? v[0] : -INFINITY;
  float mx = logit;
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const float ex = e < E ? expf(logit - mx) : 0.f;
  float se = ex;
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
  if (t < T_ && e < E) probs[(size_t)t * E + e] = expf(logit - mx) / se;
  // top-k by (logit desc, expert id asc)
  bool taken = e >= E;
  float selv[8];
  int seli[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (j >= k) break;
    float bv = taken ? -INFINITY : logit;
    int bi = taken ? 0x7fffffff : e;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    taken = taken || bi == e;
    selv[j] = bv;
    seli[j] = bi;
  }
  float ev[8], sum = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (j < k) {
      ev[j] = renorm ? expf(selv[j] - selv[0]) : expf(selv[j] - mx) / se;
      sum += ev[j];
    }
  float myw = 0.f;
  int myi = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (j < k && j == e) {
      myw = renorm ? ev[j] / sum : ev[j];
      myi = seli[j];
    }
  if (t < T_ && e < k) {
    w[(size_t)t * k + e] = myw;
    w_out[(size_t)t * k + e] = myw;
    idx[(size_t)t * k + e] = myi;
    idx_out[(size_t)t * k + e] = myi;
  }
}

// Gate for 8 < E <= 32 with W_g held in REGISTERS: warp w of a CTA owns 128 columns (4 per lane) of a
// 1024-column split of d and keeps those columns of all EB experts of W_g in registers (4 x EB floats), so
// a token costs one 8-byte load per lane, 4 x EB FMAs (packed over expert pairs) and a transpose-reduce
// (lane e ends with expert e's sum over the warp's 128 columns) -- no shared-memory traffic per FMA.  Warp
// partials of a batch of 8 tokens meet in shared memory and are summed in warp order; with one split the
// CTA finishes softmax / top-k itself (one warp per token, lane = expert), otherwise the split partials go
// to `part` and route_finish_kernel sums them in split order.  Summation order is fixed (4-column chain in
// a lane, the butterfly, warps, splits): reproducible.
constexpr int RW_SPLIT = 1024;  // columns per split (8 warps x 128)
constexpr int RW_NB = 8;        // tokens per shared-memory batch

__device__ __forceinline__ void gate_finish(float logit, bool valid_e, int e, int t, int T_, int E, int k, int renorm,
                                            float* __restrict__ probs, int32_t* __restrict__ idx, float* __restrict__ w,
                                            int32_t* __restrict__ idx_out, float* __restrict__ w_out) {
  // one warp per token, lane e = expert (e < E valid): softmax over E, top-k by (logit desc, id asc), gate weights
  const float lg = valid_e ? logit : -INFINITY;
  float mx = lg;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const float ex = valid_e ? expf(lg - mx) : 0.f;
  float se = ex;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
  if (t < T_ && valid_e) probs[(size_t)t * E + e] = ex / se;
  bool taken = !valid_e;
  float selv[8];
  int seli[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (j >= k) break;
    float bv = taken ? -INFINITY : lg;
    int bi = taken ? 0x7fffffff : e;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    taken = taken || bi == e;
    selv[j] = bv;
    seli[j] = bi;
  }
  float ev[8], sum = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (j < k) {
      ev[j] = renorm ? expf(selv[j] - selv[0]) : expf(selv[j] - mx) / se;
      sum += ev[j];
    }
  float myw = 0.f;
  int myi = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (j < k && j == e) {
      myw = renorm ? ev[j] / sum : ev[j];
      myi = seli[j];
    }
  if (t < T_ && e < k) {
    w[(size_t)t * k + e] = myw;
    w_out[(size_t)t * k + e] = myw;
    idx[(size_t)t * k + e] = myi;
    idx_out[(size_t)t * k + e] = myi;
  }
}

template <typename T, int EB>
__global__ void __launch_bounds__(256, 1) route_wreg_kernel(const T* __restrict__ x, const float* __restrict__ wg, int T_,
                                                            int E, int d, int k, int renorm, int tpc,
                                                            float* __restrict__ part, float* __restrict__ probs,
                                                            int32_t* __restrict__ idx, float* __restrict__ w,
                                                            int32_t* __restrict__ idx_out, float* __restrict__ w_out) {
  pdl_enter();
  using R = decltype(ld4raw(static_cast<const T*>(nullptr)));
  __shared__ float red[RW_NB][8][EB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int split = blockIdx.y, nsplit = gridDim.y;
  const int c = split * RW_SPLIT + wid * 128 + lane * 4;
  const bool active = c < d;
  float wr[EB][4];
#pragma unroll
  for (int e = 0; e < EB; ++e) {
    const float4 q = (e < E && active) ? *reinterpret_cast<const float4*>(wg + (size_t)e * d + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    wr[e][0] = q.x; wr[e][1] = q.y; wr[e][2] = q.z; wr[e][3] = q.w;
  }
  const int tg0 = blockIdx.x * tpc, tg1 = min(T_, tg0 + tpc);
  for (int tb = tg0; tb < tg1; tb += RW_NB) {
    R raw[RW_NB];
#pragma unroll
    for (int b = 0; b < RW_NB; ++b) raw[b] = (active && tb + b < tg1) ? ld4raw(x + (size_t)(tb + b) * d + c) : R{};
#pragma unroll
    for (int b = 0; b < RW_NB; ++b) {
      float xv[4];
      cvt4(raw[b], xv);
      float v[EB];
#pragma unroll
      for (int p = 0; p < EB / 2; ++p) {  // packed over expert pairs; each logit keeps its own column chain
        float2 s2 = __fmul2_rn(make_float2(xv[0], xv[0]), make_float2(wr[2 * p][0], wr[2 * p + 1][0]));
        s2 = __ffma2_rn(make_float2(xv[1], xv[1]), make_float2(wr[2 * p][1], wr[2 * p + 1][1]), s2);
        s2 = __ffma2_rn(make_float2(xv[2], xv[2]), make_float2(wr[2 * p][2], wr[2 * p + 1][2]), s2);
        s2 = __ffma2_rn(make_float2(xv[3], xv[3]), make_float2(wr[2 * p][3], wr[2 * p + 1][3]), s2);
        v[2 * p] = s2.x;
        v[2 * p + 1] = s2.y;
      }
      // lanes l and l + 32 - ... : butterfly over the offsets >= EB, then the transpose-reduce over offsets < EB
#pragma unroll
      for (int o = 16; o >= EB; o >>= 1)
#pragma unroll
        for (int j = 0; j < EB; ++j) v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
#pragma unroll
      for (int o = EB / 2; o >= 1; o >>= 1) {
        const bool hi = lane & o;
#pragma unroll
        for (int j = 0; j < o; ++j) {
          const float send = hi ? v[j] : v[j + o];
          const float keep = hi ? v[j + o] : v[j];
          v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      if (lane < EB) red[b][wid][lane] = v[0];  // lane e: expert e's sum over this warp's columns
    }
    __syncthreads();
    // warp b finishes token tb + b: lane e sums the 8 warps' partials in warp order
    {
      const int b = wid, e = lane;
      float s = 0.f;
      if (e < EB)
#pragma unroll
        for (int q = 0; q < 8; ++q) s += red[b][q][e];
      const int t = tb + b;
      if (nsplit == 1) {
        gate_finish(s, e < E, e, t, tg1, E, k, renorm, probs, idx, w, idx_out, w_out);
      } else if (t < tg1 && e < E) {
        part[((size_t)split * T_ + t) * E + e] = s;
      }
    }
    __syncthreads();
  }
}

// Sum of the split partials in split order, then softmax / top-k (one warp per token, lane = expert).
__global__ void __launch_bounds__(256) route_finish_kernel(const float* __restrict__ part, int nsplit, int T_, int E, int k,
                                                           int renorm, float* __restrict__ probs, int32_t* __restrict__ idx,
                                                           float* __restrict__ w, int32_t* __restrict__ idx_out,
                                                           float* __restrict__ w_out) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < T_; t += (gridDim.x * blockDim.x) >> 5) {
    float s = 0.f;
    if (lane < E)
      for (int q = 0; q < nsplit; ++q) s += part[((size_t)q * T_ + t) * E + lane];
    gate_finish(s, lane < E, lane, t, T_, E, k, renorm, probs, idx, w, idx_out, w_out);
  }
}


// Gate backward, per token: dl from dw (renormalized or raw softmax), then dx[t] += dl W_g.
template <typename T>
__global__ void __launch_bounds__(256) route_bwd_kernel(const float* __restrict__ wg, const float* __restrict__ probs,
                                                        const int32_t* __restrict__ idx, const float* __restrict__ w,
                                                        const float* __restrict__ dw, int T_, int E, int d, int k,
                                                        int renorm, float* __restrict__ dl, T* __restrict__ dx) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int t = warp; t < T_; t += nwarps) {
    // dl for experts lane + 32 i
    float s = 0.f;
    if (renorm) {
      for (int j = 0; j < k; ++j) s += w[(size_t)t * k + j] * dw[(size_t)t * k + j];
    } else {
      for (int j = 0; j < k; ++j) s += probs[(size_t)t * E + idx[(size_t)t * k + j]] * dw[(size_t)t * k + j];
    }
    for (int e = lane; e < E; e += 32) {
      float g = 0.f, wsel = 0.f;
      bool sel = false;
      for (int j = 0; j < k; ++j)
        if (idx[(size_t)t * k + j] == e) { g = dw[(size_t)t * k + j]; wsel = w[(size_t)t * k + j]; sel = true; }
      float v;
      if (renorm) v = sel ? wsel * (g - s) : 0.f;
      else v = probs[(size_t)t * E + e] * (g - s);
      dl[(size_t)t * E + e] = v;
    }
    __syncwarp();
    const float* dlt = dl + (size_t)t * E;
    T* dxr = dx + (size_t)t * d;
    for (int c = lane * 8; c < d; c += 256) {
      float acc[8];
      load8(dxr + c, acc);
      for (int e = 0; e < E; ++e) {
        float de = dlt[e];
        float wv[8];
        load8(wg + (size_t)e * d + c, wv);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fmaf(de, wv[i], acc[i]);
      }
      store8(dxr + c, acc);
    }
  }
}

// Fast gate backward for E <= 32, d % 256 == 0: CTA = 32 tokens (4 per warp).  dl (renormalized:
// w_j (dw_j - sum_i w_i dw_i); raw softmax: p (g - <p, g>)) is formed per token in shared memory, then
// dx[t] += dl[t] W_g with W_g chunks staged in shared memory (each float4 read feeds 4 tokens).
template <typename T, int EB>
__global__ void __launch_bounds__(256) route_bwd_fast_kernel(const float* __restrict__ wg, const float* __restrict__ probs,
                                                             const int32_t* __restrict__ idx, const float* __restrict__ w,
                                                             const float* __restrict__ dw, int T_, int E, int d, int k,
                                                             int renorm, float* __restrict__ dl, T* __restrict__ dx) {
  pdl_enter();
  constexpr int TB = 4, RC = 8192 / EB;
  __shared__ __align__(16) float ws[EB][RC];
  __shared__ float dls[32][EB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int tb0 = blockIdx.x * 32;
  // dl for the CTA's 32 tokens: thread (token lt, expert e)
  for (int i = threadIdx.x; i < 32 * EB; i += blockDim.x) {
    const int lt = i / EB, e = i % EB;
    const int t = tb0 + lt;
    float v = 0.f;
    if (t < T_ && e < E) {
      float s = 0.f, g = 0.f, wsel = 0.f;
      bool sel = false;
      for (int j = 0; j < k; ++j) {
        const int ej = idx[(size_t)t * k + j];
        const float dwj = dw[(size_t)t * k + j];
        s += (renorm ? w[(size_t)t * k + j] : probs[(size_t)t * E + ej]) * dwj;
        if (ej == e) { g = dwj; wsel = w[(size_t)t * k + j]; sel = true; }
      }
      v = renorm ? (sel ? wsel * (g - s) : 0.f) : probs[(size_t)t * E + e] * (g - s);
      dl[(size_t)t * E + e] = v;
    }
    dls[lt][e] = v;
  }
  const int t0 = tb0 + wid * TB;
  for (int c0 = 0; c0 < d; c0 += RC) {
    const int rc = min(RC, d - c0);
    __syncthreads();
    for (int i = threadIdx.x; i < E * (rc / 4); i += blockDim.x) {
      const int e = i / (rc / 4), c = (i % (rc / 4)) * 4;
      *reinterpret_cast<float4*>(&ws[e][c]) = *reinterpret_cast<const float4*>(wg + (size_t)e * d + c0 + c);
    }
    __syncthreads();
    for (int s0 = 0; s0 < rc; s0 += 256) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int cl = s0 + half * 128 + lane * 4;
        float acc[TB][4];
#pragma unroll
        for (int i = 0; i < TB; ++i) {
          const int t = t0 + i;
          if (t < T_) {
            T* p = dx + (size_t)t * d + c0 + cl;
            if constexpr (sizeof(T) == 2) {
              const uint2 u = *reinterpret_cast<const uint2*>(p);
              const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
              const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
              acc[i][0] = a.x; acc[i][1] = a.y; acc[i][2] = b.x; acc[i][3] = b.y;
            } else {
              const float4 u = *reinterpret_cast<const float4*>(p);
              acc[i][0] = u.x; acc[i][1] = u.y; acc[i][2] = u.z; acc[i][3] = u.w;
            }
          }
        }
#pragma unroll
        for (int e = 0; e < EB; ++e) {
          if (e < E) {
            const float4 wv = *reinterpret_cast<const float4*>(&ws[e][cl]);
#pragma unroll
            for (int i = 0; i < TB; ++i) {
              const float de = dls[wid * TB + i][e];
              acc[i][0] = fmaf(de, wv.x, acc[i][0]);
              acc[i][1] = fmaf(de, wv.y, acc[i][1]);
              acc[i][2] = fmaf(de, wv.z, acc[i][2]);
              acc[i][3] = fmaf(de, wv.w, acc[i][3]);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < TB; ++i) {
          const int t = t0 + i;
          if (t < T_) {
            T* p = dx + (size_t)t * d + c0 + cl;
            if constexpr (sizeof(T) == 2) {
              const __nv_bfloat162 a = __floats2bfloat162_rn(acc[i][0], acc[i][1]);
              const __nv_bfloat162 b = __floats2bfloat162_rn(acc[i][2], acc[i][3]);
              uint2 u;
              u.x = *reinterpret_cast<const uint32_t*>(&a);
              u.y = *reinterpret_cast<const uint32_t*>(&b);
              *reinterpret_cast<uint2*>(p) = u;
            } else {
              *reinterpret_cast<float4*>(p) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
            }
          }
        }
      }
    }
  }
}

// Fused gate backward for E <= 8, d % 1024 == 0: CTA = 32 tokens, thread = 4 columns of every 1024-column
// pass.  dl of the 32 tokens is formed in shared memory (as in route_bwd_fast_kernel); then each thread
// streams its columns of x and dx once: dx[t] += dl[t] W_g and part[p][e][c] = sum over the CTA's tokens (in
// token order) of dl[t][e] x[t][c], so x is read once for both products.  The partials are summed in a
// fixed order by wg_reduce_kernel (deterministic dW_g).
template <typename T>
__global__ void __launch_bounds__(256, 2) route_bwd_fused8_kernel(const float* __restrict__ wg, const float* __restrict__ probs,
                                                               const int32_t* __restrict__ idx, const float* __restrict__ w,
                                                               const float* __restrict__ dw, const T* __restrict__ x,
                                                               int T_, int E, int d, int k, int renorm, float* __restrict__ dl,
                                                               T* __restrict__ dx, float* __restrict__ part) {
  pdl_enter();
  constexpr int EB = 8, TT = 32, U = 4;
  __shared__ __align__(16) float dls[TT][EB];
  const int tb0 = blockIdx.x * TT;
  {
    const int i = threadIdx.x;  // 256 threads = 32 tokens x 8 experts
    const int lt = i / EB, e = i % EB;
    const int t = tb0 + lt;
    float v = 0.f;
    if (t < T_ && e < E) {
      float sacc = 0.f, g = 0.f, wsel = 0.f;
      bool sel = false;
      for (int j = 0; j < k; ++j) {
        const int ej = idx[(size_t)t * k + j];
        const float dwj = dw[(size_t)t * k + j];
        sacc += (renorm ? w[(size_t)t * k + j] : probs[(size_t)t * E + ej]) * dwj;
        if (ej == e) { g = dwj; wsel = w[(size_t)t * k + j]; sel = true; }
      }
      v = renorm ? (sel ? wsel * (g - sacc) : 0.f) : probs[(size_t)t * E + e] * (g - sacc);
      dl[(size_t)t * E + e] = v;
    }
    dls[lt][e] = v;
  }
  __syncthreads();
  const int nt = min(TT, T_ - tb0);
  for (int c = threadIdx.x * 4; c < d; c += 1024) {
    float wr[EB][4], acc[EB][4];
#pragma unroll
    for (int e = 0; e < EB; ++e) {
      const float4 q = e < E ? *reinterpret_cast<const float4*>(wg + (size_t)e * d + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      wr[e][0] = q.x; wr[e][1] = q.y; wr[e][2] = q.z; wr[e][3] = q.w;
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[e][j] = 0.f;
    }
    for (int t0 = 0; t0 < nt; t0 += U) {
      float xv[U][4], gv[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u) {  // all loads of the U tokens first
        const size_t o = (size_t)(tb0 + t0 + u) * d + c;
        if (t0 + u < nt) {
          if constexpr (sizeof(T) == 2) {
            const uint2 a = *reinterpret_cast<const uint2*>(x + o);
            const uint2 b = *reinterpret_cast<const uint2*>(dx + o);
            const float2 a0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&a.x));
            const float2 a1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&a.y));
            const float2 b0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&b.x));
            const float2 b1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&b.y));
            xv[u][0] = a0.x; xv[u][1] = a0.y; xv[u][2] = a1.x; xv[u][3] = a1.y;
            gv[u][0] = b0.x; gv[u][1] = b0.y; gv[u][2] = b1.x; gv[u][3] = b1.y;
          } else {
            const float4 a = *reinterpret_cast<const float4*>(x + o);
            const float4 b = *reinterpret_cast<const float4*>(dx + o);
            xv[u][0] = a.x; xv[u][1] = a.y; xv[u][2] = a.z; xv[u][3] = a.w;
            gv[u][0] = b.x; gv[u][1] = b.y; gv[u][2] = b.z; gv[u][3] = b.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) xv[u][j] = gv[u][j] = 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float4 l0 = *reinterpret_cast<const float4*>(&dls[t0 + u][0]);
        const float4 l1 = *reinterpret_cast<const float4*>(&dls[t0 + u][4]);
        const float lv[EB] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
        // packed fp32x2 FMAs over column pairs: every element keeps its own expert-ordered fmaf chain, so
        // the results are bit-identical to the scalar form at half the issue slots
#pragma unroll
        for (int e = 0; e < EB; ++e)
#pragma unroll
          for (int j = 0; j < 4; j += 2) {
            const float2 l2 = make_float2(lv[e], lv[e]);
            const float2 g2 = __ffma2_rn(l2, make_float2(wr[e][j], wr[e][j + 1]), make_float2(gv[u][j], gv[u][j + 1]));
            const float2 a2 = __ffma2_rn(l2, make_float2(xv[u][j], xv[u][j + 1]), make_float2(acc[e][j], acc[e][j + 1]));
            gv[u][j] = g2.x; gv[u][j + 1] = g2.y;
            acc[e][j] = a2.x; acc[e][j + 1] = a2.y;
          }
        if (t0 + u < nt) {
          const size_t o = (size_t)(tb0 + t0 + u) * d + c;
          if constexpr (sizeof(T) == 2) {
            const __nv_bfloat162 a = __floats2bfloat162_rn(gv[u][0], gv[u][1]);
            const __nv_bfloat162 b = __floats2bfloat162_rn(gv[u][2], gv[u][3]);
            uint2 q;
            q.x = *reinterpret_cast<const uint32_t*>(&a);
            q.y = *reinterpret_cast<const uint32_t*>(&b);
            *reinterpret_cast<uint2*>(dx + o) = q;
          } else {
            *reinterpret_cast<float4*>(dx + o) = make_float4(gv[u][0], gv[u][1], gv[u][2], gv[u][3]);
          }
        }
      }
    }
#pragma unroll
    for (int e = 0; e < EB; ++e)
      if (e < E)
        *reinterpret_cast<float4*>(part + ((size_t)blockIdx.x * E + e) * d + c) =
            make_float4(acc[e][0], acc[e][1], acc[e][2], acc[e][3]);
  }
}

// dW_g partials, fast path: CTA = (64 tokens, 256 columns); dl of the tile staged in shared memory,
// x streamed with unrolled loads; part[p][e][col] for token tile p.
template <typename T, int EB>
__global__ void __launch_bounds__(256) wg_partial_fast_kernel(const float* __restrict__ dl, const T* __restrict__ x,
                                                              int T_, int E, int d, float* __restrict__ part) {
  pdl_enter();
  constexpr int TT = 64;
  __shared__ float dls[TT][EB];
  const int col = blockIdx.x * 256 + threadIdx.x;
  const int p = blockIdx.y;
  const int t0 = p * TT;
  for (int i = threadIdx.x; i < TT * EB; i += 256) {
    const int lt = i / EB, e = i % EB;
    dls[lt][e] = (t0 + lt < T_ && e < E) ? dl[(size_t)(t0 + lt) * E + e] : 0.f;
  }
  __syncthreads();
  float acc[EB];
#pragma unroll
  for (int e = 0; e < EB; ++e) acc[e] = 0.f;
  const int nt = min(TT, T_ - t0);
#pragma unroll 8
  for (int lt = 0; lt < nt; ++lt) {
    const float xv = to_f(x[(size_t)(t0 + lt) * d + col]);
#pragma unroll
    for (int e = 0; e < EB; ++e) acc[e] = fmaf(dls[lt][e], xv, acc[e]);
  }
#pragma unroll
  for (int e = 0; e < EB; ++e)
    if (e < E) part[((size_t)p * E + e) * d + col] = acc[e];
}

// dW_g partials: part p covers tokens [p*chunk, (p+1)*chunk); one thread per column, E accumulators.
template <typename T, int EB>
__global__ void __launch_bounds__(256) wg_partial_kernel(const float* __restrict__ dl, const T* __restrict__ x,
                                                         int T_, int E, int d, int chunk, float* __restrict__ part) {
  pdl_enter();
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  const int p = blockIdx.y;
  const int e0 = blockIdx.z * EB;
  if (col >= d) return;
  float acc[EB];
#pragma unroll
  for (int e = 0; e < EB; ++e) acc[e] = 0.f;
  const int t0 = p * chunk, t1 = min(T_, t0 + chunk);
  for (int t = t0; t < t1; ++t) {
    float xv = to_f(x[(size_t)t * d + col]);
    const float* dlt = dl + (size_t)t * E + e0;
#pragma unroll
    for (int e = 0; e < EB; ++e)
      if (e0 + e < E) acc[e] = fmaf(dlt[e], xv, acc[e]);
  }
#pragma unroll
  for (int e = 0; e < EB; ++e)
    if (e0 + e < E) part[((size_t)p * E + e0 + e) * d + col] = acc[e];
}

// dW_g = sum of the partials in a fixed order: CTA = 32 outputs x 8 warps; warp w sums parts w, w+8, ...
// (coalesced 128-byte rows), then the 8 warp sums are added in warp order.
__global__ void __launch_bounds__(256) wg_reduce_kernel(const float* __restrict__ part, int parts, int n,
                                                        float* __restrict__ out) {
  pdl_enter();
  __shared__ float red[8][33];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (i < n) {
#pragma unroll 4
    for (int p = wid; p < parts; p += 8) s += part[(size_t)p * n + i];
  }
  red[wid][lane] = s;
  __syncthreads();
  if (wid == 0 && i < n) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][lane];
    out[i] = t;
  }
}

template <typename T>
int route_dispatch(const luffy_layer* L, const void* x, const float* wg, int32_t* idx_out, float* w_out, cudaStream_t s) {
  const int warps_per_block = 8;
  int blocks = (L->T + warps_per_block - 1) / warps_per_block;
  blocks = blocks > 148 * 16 ? 148 * 16 : blocks;
  const T* xp = static_cast<const T*>(x);
  if (L->E <= 32 && L->d % 256 == 0) {
    const int fb = (L->T + 31) / 32;
    if (L->E <= 8) {
      LUFFY_CUDA_TRY(smem_optin((const void*)route_e8_kernel<T>, 65536));
      launch_pdl(route_e8_kernel<T>, fb, 256, 65536, s, xp, wg, L->T, L->E, L->d, L->k, L->renorm, L->probs, L->idx, L->w,
                 idx_out, w_out);
      LUFFY_LAUNCHED();
    } else {
      // W_g in registers (route_wreg_kernel): ~148 CTAs over the token ranges of every column split
      const int nsplit = (L->d + RW_SPLIT - 1) / RW_SPLIT;
      int tpc = (int)(((int64_t)L->T * nsplit + device_sms() - 1) / device_sms());
      tpc = std::max(RW_NB, (tpc + RW_NB - 1) / RW_NB * RW_NB);
      const dim3 grid((L->T + tpc - 1) / tpc, nsplit);
      if (L->E <= 16)
        launch_pdl(route_wreg_kernel<T, 16>, grid, 256, 0, s, xp, wg, L->T, L->E, L->d, L->k, L->renorm, tpc, L->rpart,
                   L->probs, L->idx, L->w, idx_out, w_out);
      else
        launch_pdl(route_wreg_kernel<T, 32>, grid, 256, 0, s, xp, wg, L->T, L->E, L->d, L->k, L->renorm, tpc, L->rpart,
                   L->probs, L->idx, L->w, idx_out, w_out);
      LUFFY_LAUNCHED();
      if (nsplit > 1) {
        launch_pdl(route_finish_kernel, std::max(1, std::min((L->T + 7) / 8, 148 * 8)), 256, 0, s, (const float*)L->rpart,
                   nsplit, L->T, L->E, L->k, L->renorm, L->probs, L->idx, L->w, idx_out, w_out);
        LUFFY_LAUNCHED();
      }
    }
    return 0;
  }
#define LUFFY_ROUTE(EBV)                                                                                 \
  launch_pdl(route_kernel<T, EBV>, blocks, 256, 0, s, xp, wg, L->T, L->E, L->d, L->k, L->renorm, L->probs, L->idx, \
                                              L->w, idx_out, w_out)
  if (L->E <= 32) LUFFY_ROUTE(32);
  else if (L->E <= 64) LUFFY_ROUTE(64);
  else if (L->E <= 128) LUFFY_ROUTE(128);
  else LUFFY_ROUTE(256);
#undef LUFFY_ROUTE
  LUFFY_LAUNCHED();
  return 0;
}

}  // namespace

// Near-tie report (reading R2, stats only): a token whose k+1 largest logits, in the gate's order (logit
// desc, expert asc), have an adjacent gap <= 1e-5 * max(1, |l_1|).  One warp per token: the order and a
// loose screen come from the saved softmax probabilities (log p_a - log p_b = l_a - l_b); only screened
// tokens recompute their k+1 logits from x and W_g (fp32) for the exact tolerance test.
template <typename T>
__global__ void __launch_bounds__(256) near_tie_kernel(const float* __restrict__ probs, const T* __restrict__ x,
                                                       const float* __restrict__ wg, int T_, int E, int d, int k,
                                                       unsigned long long* __restrict__ out) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int nk = min(k + 1, E);
  int cnt = 0;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < T_; t += (gridDim.x * blockDim.x) >> 5) {
    int sel[9];
    float ps[9];
    float pv[8];  // experts 0..E-1 in chunks of 32 lanes: E <= 256 -> up to 8 values per lane
    for (int c = 0; c < 8; ++c) pv[c] = (c * 32 + lane < E) ? probs[(size_t)t * E + c * 32 + lane] : -1.f;
    for (int i = 0; i < nk; ++i) {  // arg-max by (p desc, expert asc), k+1 times
      float best = -2.f;
      int be = 0x7fffffff;
      for (int c = 0; c < 8; ++c) {
        const int e = c * 32 + lane;
        if (e < E && pv[c] > best) { best = pv[c]; be = e; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const float ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oe = __shfl_xor_sync(0xffffffffu, be, o);
        if (ob > best || (ob == best && oe < be)) { best = ob; be = oe; }
      }
      sel[i] = be;
      ps[i] = best;
      if ((be & 31) == lane) pv[be >> 5] = -1.f;  // remove
    }
    bool screen = false;
    for (int i = 0; i + 1 < nk; ++i) {
      const float a = ps[i], b = ps[i + 1];
      if (b <= 0.f) continue;                       // underflowed runner-up: far from a tie
      screen |= (logf(a) - logf(b)) <= 1e-3f;
    }
    if (!screen) continue;
    float l[9];
    for (int i = 0; i < nk; ++i) {
      float acc = 0.f;
      for (int c = lane; c < d; c += 32) acc = fmaf(to_f(x[(size_t)t * d + c]), wg[(size_t)sel[i] * d + c], acc);
      l[i] = warp_sum(acc);
    }
    const float tol = 1e-5f * fmaxf(1.f, fabsf(l[0]));
    bool tie = false;
    for (int i = 0; i + 1 < nk; ++i) tie |= fabsf(l[i] - l[i + 1]) <= tol;
    cnt += tie ? 1 : 0;
  }
  if (lane == 0 && cnt) atomicAdd(out, (unsigned long long)cnt);
}

int launch_near_tie(const luffy_layer* L, const void* x, const float* wg, unsigned long long* out, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  const int blocks = std::max(1, std::min((L->T + 7) / 8, 148 * 8));
  if (L->dtype == LUFFY_BF16)
    launch_pdl(near_tie_kernel<bf16>, blocks, 256, 0, st, L->probs, static_cast<const bf16*>(x), wg, L->T, L->E, L->d,
               L->k, out);
  else
    launch_pdl(near_tie_kernel<float>, blocks, 256, 0, st, L->probs, static_cast<const float*>(x), wg, L->T, L->E, L->d,
               L->k, out);
  LUFFY_LAUNCHED();
  return 0;
}

int launch_route(const luffy_layer* L, const void* x, const float* wg, int32_t* idx_out, float* w_out, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  return L->dtype == LUFFY_BF16 ? route_dispatch<bf16>(L, x, wg, idx_out, w_out, st)
                                : route_dispatch<float>(L, x, wg, idx_out, w_out, st);
}

int launch_route_bwd(const luffy_layer* L, const void* x, const float* wg, const float* dw, void* dx, float* dwg, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  const bool fast = L->E <= 32 && L->d % 256 == 0;
  if (L->E <= 8 && L->d % 1024 == 0) {  // fused: one pass over x for dx and the dW_g partials
    const int parts = (L->T + 31) / 32;
    if (L->dtype == LUFFY_BF16)
      launch_pdl(route_bwd_fused8_kernel<bf16>, parts, 256, 0, st, wg, L->probs, L->idx, L->w, dw,
                 static_cast<const bf16*>(x), L->T, L->E, L->d, L->k, L->renorm, L->dl, static_cast<bf16*>(dx), L->wg_part);
    else
      launch_pdl(route_bwd_fused8_kernel<float>, parts, 256, 0, st, wg, L->probs, L->idx, L->w, dw,
                 static_cast<const float*>(x), L->T, L->E, L->d, L->k, L->renorm, L->dl, static_cast<float*>(dx), L->wg_part);
    LUFFY_LAUNCHED();
    const int n = L->E * L->d;
    launch_pdl(wg_reduce_kernel, (n + 31) / 32, 256, 0, st, L->wg_part, parts, n, dwg);
    LUFFY_LAUNCHED();
    return 0;
  }
  // (a one-pass backward for 8 < E <= 32 holding W_g and the dW_g partials in registers was measured slower
  // than the two kernels below -- C3 74 vs 38 us, C4 179 vs 142 us: 8 warps per SM cannot hide its loads)
  if (fast) {
    const int fb = (L->T + 31) / 32;
    const int parts = (L->T + 63) / 64;
    dim3 pg(L->d / 256, parts);
#define LUFFY_RB(EBV)                                                                                               \
  do {                                                                                                              \
    if (L->dtype == LUFFY_BF16) {                                                                                   \
      launch_pdl(route_bwd_fast_kernel<bf16, EBV>, fb, 256, 0, st, wg, L->probs, L->idx, L->w, dw, L->T, L->E, L->d, L->k,  \
                                                          L->renorm, L->dl, static_cast<bf16*>(dx));                \
      LUFFY_LAUNCHED();                                                                                             \
      launch_pdl(wg_partial_fast_kernel<bf16, EBV>, pg, 256, 0, st, L->dl, static_cast<const bf16*>(x), L->T, L->E, L->d,    \
                                                           L->wg_part);                                             \
    } else {                                                                                                        \
      launch_pdl(route_bwd_fast_kernel<float, EBV>, fb, 256, 0, st, wg, L->probs, L->idx, L->w, dw, L->T, L->E, L->d, L->k, \
                                                           L->renorm, L->dl, static_cast<float*>(dx));              \
      LUFFY_LAUNCHED();                                                                                             \
      launch_pdl(wg_partial_fast_kernel<float, EBV>, pg, 256, 0, st, L->dl, static_cast<const float*>(x), L->T, L->E, L->d,  \
                                                            L->wg_part);                                            \
    }                                                                                                               \
    LUFFY_LAUNCHED();                                                                                               \
  } while (0)
    if (L->E <= 8) LUFFY_RB(8);
    else if (L->E <= 16) LUFFY_RB(16);
    else LUFFY_RB(32);
#undef LUFFY_RB
    const int n = L->E * L->d;
    launch_pdl(wg_reduce_kernel, (n + 31) / 32, 256, 0, st, L->wg_part, parts, n, dwg);
    LUFFY_LAUNCHED();
    return 0;
  }
  int blocks = (L->T + 7) / 8;
  blocks = blocks > 148 * 16 ? 148 * 16 : blocks;
  if (L->dtype == LUFFY_BF16)
    launch_pdl(route_bwd_kernel<bf16>, blocks, 256, 0, st, wg, L->probs, L->idx, L->w, dw, L->T, L->E, L->d, L->k, L->renorm,
                                                   L->dl, static_cast<bf16*>(dx));
  else
    launch_pdl(route_bwd_kernel<float>, blocks, 256, 0, st, wg, L->probs, L->idx, L->w, dw, L->T, L->E, L->d, L->k, L->renorm,
                                                    L->dl, static_cast<float*>(dx));
  LUFFY_LAUNCHED();
  const int parts = wg_parts(L->E, L->d);
  const int chunk = (L->T + parts - 1) / parts;
  constexpr int EB = 16;
  dim3 grid((L->d + 255) / 256, parts, (L->E + EB - 1) / EB);
  if (L->dtype == LUFFY_BF16)
    launch_pdl(wg_partial_kernel<bf16, EB>, grid, 256, 0, st, L->dl, static_cast<const bf16*>(x), L->T, L->E, L->d, chunk, L->wg_part);
  else
    launch_pdl(wg_partial_kernel<float, EB>, grid, 256, 0, st, L->dl, static_cast<const float*>(x), L->T, L->E, L->d, chunk, L->wg_part);
  LUFFY_LAUNCHED();
  const int n = L->E * L->d;
  launch_pdl(wg_reduce_kernel, (n + 31) / 32, 256, 0, st, L->wg_part, parts, n, dwg);
  LUFFY_LAUNCHED();
  return 0;
}

}  // namespace luffy
