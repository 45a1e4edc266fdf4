// Top-k gate ("top-2 gating"; readings R1, R2) and its backward.
//
// Forward: one warp per token.  Lanes stream the token row with 16-byte loads, accumulate the E
// partial dot products with the fp32 gate weights in a fixed order (chunk order, then a butterfly
// reduction), so the result is bitwise reproducible.  Top-k by (logit desc, expert id asc) via a warp
// argmax; softmax over all experts is saved for the backward.
#include "common.cuh"

namespace luffy {
namespace {

template <typename T, int EB>
__global__ void __launch_bounds__(256) route_kernel(const T* __restrict__ x, const float* __restrict__ wg,
                                                    int T_, int E, int d, int k, int renorm,
                                                    float* __restrict__ probs, int32_t* __restrict__ idx,
                                                    float* __restrict__ w, int32_t* __restrict__ idx_out,
                                                    float* __restrict__ w_out) {
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

// Gate backward, per token: dl from dw (renormalized or raw softmax), then dx[t] += dl W_g.
template <typename T>
__global__ void __launch_bounds__(256) route_bwd_kernel(const float* __restrict__ wg, const float* __restrict__ probs,
                                                        const int32_t* __restrict__ idx, const float* __restrict__ w,
                                                        const float* __restrict__ dw, int T_, int E, int d, int k,
                                                        int renorm, float* __restrict__ dl, T* __restrict__ dx) {
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

// dW_g partials: part p covers tokens [p*chunk, (p+1)*chunk); one thread per column, E accumulators.
template <typename T, int EB>
__global__ void __launch_bounds__(256) wg_partial_kernel(const float* __restrict__ dl, const T* __restrict__ x,
                                                         int T_, int E, int d, int chunk, float* __restrict__ part) {
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

__global__ void wg_reduce_kernel(const float* __restrict__ part, int parts, int n, float* __restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float s = 0.f;
  for (int p = 0; p < parts; ++p) s += part[(size_t)p * n + i];
  out[i] = s;
}

template <typename T>
int route_dispatch(const luffy_layer* L, const void* x, const float* wg, int32_t* idx_out, float* w_out, cudaStream_t s) {
  const int warps_per_block = 8;
  int blocks = (L->T + warps_per_block - 1) / warps_per_block;
  blocks = blocks > 148 * 16 ? 148 * 16 : blocks;
  const T* xp = static_cast<const T*>(x);
#define LUFFY_ROUTE(EBV)                                                                                   \
  route_kernel<T, EBV><<<blocks, 256, 0, s>>>(xp, wg, L->T, L->E, L->d, L->k, L->renorm, L->probs, L->idx, \
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

int launch_route(const luffy_layer* L, const void* x, const float* wg, int32_t* idx_out, float* w_out, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  return L->dtype == LUFFY_BF16 ? route_dispatch<bf16>(L, x, wg, idx_out, w_out, st)
                                : route_dispatch<float>(L, x, wg, idx_out, w_out, st);
}

int launch_route_bwd(const luffy_layer* L, const void* x, const float* wg, const float* dw, void* dx, float* dwg, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  int blocks = (L->T + 7) / 8;
  blocks = blocks > 148 * 16 ? 148 * 16 : blocks;
  if (L->dtype == LUFFY_BF16)
    route_bwd_kernel<bf16><<<blocks, 256, 0, st>>>(wg, L->probs, L->idx, L->w, dw, L->T, L->E, L->d, L->k, L->renorm,
                                                   L->dl, static_cast<bf16*>(dx));
  else
    route_bwd_kernel<float><<<blocks, 256, 0, st>>>(wg, L->probs, L->idx, L->w, dw, L->T, L->E, L->d, L->k, L->renorm,
                                                    L->dl, static_cast<float*>(dx));
  LUFFY_LAUNCHED();
  const int parts = wg_parts(L->E, L->d);
  const int chunk = (L->T + parts - 1) / parts;
  constexpr int EB = 16;
  dim3 grid((L->d + 255) / 256, parts, (L->E + EB - 1) / EB);
  if (L->dtype == LUFFY_BF16)
    wg_partial_kernel<bf16, EB><<<grid, 256, 0, st>>>(L->dl, static_cast<const bf16*>(x), L->T, L->E, L->d, chunk, L->wg_part);
  else
    wg_partial_kernel<float, EB><<<grid, 256, 0, st>>>(L->dl, static_cast<const float*>(x), L->T, L->E, L->d, chunk, L->wg_part);
  LUFFY_LAUNCHED();
  const int n = L->E * L->d;
  wg_reduce_kernel<<<(n + 255) / 256, 256, 0, st>>>(L->wg_part, parts, n, dwg);
  LUFFY_LAUNCHED();
  return 0;
}

}  // namespace luffy
