// Device helpers shared by the libluffy kernels (sm_100a).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "luffy_internal.h"

namespace luffy {

#define LUFFY_CUDA_TRY(expr)                          \
  do {                                                \
    cudaError_t _e = (cudaError_t)(expr);             \
    if (_e != cudaSuccess) return (int)_e;            \
  } while (0)

#define LUFFY_LAUNCHED() \
  do {                   \
    note_launch();       \
    LUFFY_CUDA_TRY(cudaGetLastError()); \
  } while (0)

typedef __nv_bfloat16 bf16;

// Programmatic dependent launch.  Every kernel is launched with programmatic stream serialization and
// begins with pdl_enter(): wait until the preceding kernel of the stream has completed and flushed
// (griddepcontrol.wait), then allow the next kernel's CTAs to be scheduled (launch_dependents), so its
// launch latency overlaps this kernel instead of following it.  Because every kernel waits before its
// first global access, completion stays transitive along the stream exactly as without PDL.
// tests/test_abi_cpu.py checks that every __global__ kernel calls it.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Kernels whose prologue touches nothing the preceding kernel writes (mbarrier init, TMEM allocation,
// tensor-map prefetch, cluster barrier) start with pdl_defer() and call pdl_enter() right after that
// prologue and before their first global-memory access, so a CTA that becomes resident while the previous
// kernel is still draining spends the wait with its prologue already done.
__device__ __forceinline__ void pdl_defer() {}
// griddepcontrol.launch_dependents alone: for a kernel that synchronises with its predecessor through
// explicit counters instead of waiting for the whole grid (greedy_cluster_kernel after the Gram)
__device__ __forceinline__ void pdl_launch_only() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Per-device launch caches (api.cu).  Function attributes and occupancy answers belong to a (kernel,
// device) pair, so they are cached per current device and per `extra` key (e.g. the shared-memory size or
// the group count they were computed for) -- a process driving several devices or layers of different
// shapes never reuses another's answer.
bool dev_cache_get(const void* key, int64_t extra, int* value);
void dev_cache_put(const void* key, int64_t extra, int value);
int device_sms();                                      // SM count of the current device
int smem_optin(const void* kernel, int bytes);         // cudaFuncAttributeMaxDynamicSharedMemorySize, once per device

bool pdl_enabled();  // api.cu: LUFFY_PDL=0 in the environment disables the attribute (A/B measurements)

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, static_cast<Args&&>(args)...);  // errors surface via LUFFY_LAUNCHED
}

// 8 consecutive elements <-> 8 floats (one 16-byte load for bf16, two for fp32)
__device__ __forceinline__ void load8(const bf16* p, float (&v)[8]) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void load8(const float* p, float (&v)[8]) {
  float4 a = *reinterpret_cast<const float4*>(p);
  float4 b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void store8(bf16* p, const float (&v)[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}
__device__ __forceinline__ void store8(float* p, const float (&v)[8]) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ void zero8(bf16* p) { *reinterpret_cast<uint4*>(p) = make_uint4(0, 0, 0, 0); }
__device__ __forceinline__ void zero8(float* p) {
  *reinterpret_cast<float4*>(p) = make_float4(0.f, 0.f, 0.f, 0.f);
  *reinterpret_cast<float4*>(p + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
}

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(bf16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float x) { return __float2bfloat16_rn(x); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u > v ? u : v;
  }
  return v;
}

// GeLU with the exact erf form (R12) and its derivative.
__device__ __forceinline__ float gelu_f(float x) { return 0.5f * x * (1.f + erff(x * 0.70710678118654752f)); }
__device__ __forceinline__ float gelu_grad_f(float x) {
  float cdf = 0.5f * (1.f + erff(x * 0.70710678118654752f));
  float pdf = 0.3989422804014327f * expf(-0.5f * x * x);
  return cdf + x * pdf;
}
// GeLU(x) and GeLU'(x) sharing one erf: the forward saves GeLU'(pre), so the backward needs no erf.
__device__ __forceinline__ void gelu_and_grad_f(float x, float& g, float& dg) {
  const float cdf = 0.5f * (1.f + erff(x * 0.70710678118654752f));
  g = x * cdf;
  dg = cdf + x * 0.3989422804014327f * __expf(-0.5f * x * x);
}
// The same pair for the bf16 tensor-core epilogue (reading R12b): Phi from one exponential via Abramowitz &
// Stegun 26.2.17, Q(|x|) = phi(|x|) (b1 t + ... + b5 t^5), t = 1 / (1 + p |x|), |error| < 7.5e-8 -- far below
// the bf16 resolution of the stored activation -- so GeLU and GeLU' cost ~17 instructions instead of erff's
// two-range polynomial plus a second exponential.
__device__ __forceinline__ void gelu_and_grad_as(float x, float& g, float& dg) {
  // e = exp(-x^2/2) = 2^(x * (x * -log2(e)/2)); MUFU ex2 / rcp without range fix-ups (ftz: only values
  // below 1e-38 are affected); 1/sqrt(2 pi) is folded into the polynomial coefficients
  float e, t;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * (x * -0.72134752044448170368f)));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.2316419f, fabsf(x), 1.f)));
  float poly = fmaf(t, 0.3989422804014327f * 1.330274429f, 0.3989422804014327f * -1.821255978f);
  poly = fmaf(t, poly, 0.3989422804014327f * 1.781477937f);
  poly = fmaf(t, poly, 0.3989422804014327f * -0.356563782f);
  poly = fmaf(t, poly, 0.3989422804014327f * 0.319381530f);
  const float q = e * (poly * t);  // upper tail Q(|x|) = 1 - Phi(|x|) = phi(|x|) (b1 t + ... + b5 t^5)
  const float cdf = x >= 0.f ? 1.f - q : q;
  g = x * cdf;
  dg = fmaf(x * 0.3989422804014327f, e, cdf);  // Phi(x) + x phi(x)
}
// The same arithmetic on two values with the packed fp32x2 instructions of sm_100 (FFMA2 / FMUL2: one
// issue slot for two lanes of work); every step rounds exactly as in gelu_and_grad_as, so the results are
// bit-identical to it.
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ void gelu_and_grad_as2(float2 x, float2& g, float2& dg) {
  float2 e, t;
  const float2 a = __fmul2_rn(x, __fmul2_rn(x, f2(-0.72134752044448170368f)));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.x) : "f"(a.x));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.y) : "f"(a.y));
  const float2 den = __ffma2_rn(f2(0.2316419f), make_float2(fabsf(x.x), fabsf(x.y)), f2(1.f));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t.x) : "f"(den.x));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t.y) : "f"(den.y));
  float2 poly = __ffma2_rn(t, f2(0.3989422804014327f * 1.330274429f), f2(0.3989422804014327f * -1.821255978f));
  poly = __ffma2_rn(t, poly, f2(0.3989422804014327f * 1.781477937f));
  poly = __ffma2_rn(t, poly, f2(0.3989422804014327f * -0.356563782f));
  poly = __ffma2_rn(t, poly, f2(0.3989422804014327f * 0.319381530f));
  const float2 q = __fmul2_rn(e, __fmul2_rn(poly, t));
  const float2 omq = __ffma2_rn(q, f2(-1.f), f2(1.f));  // 1 - q, rounded once as in the scalar form
  const float2 cdf = make_float2(x.x >= 0.f ? omq.x : q.x, x.y >= 0.f ? omq.y : q.y);
  g = __fmul2_rn(x, cdf);
  dg = __ffma2_rn(__fmul2_rn(x, f2(0.3989422804014327f)), e, cdf);
}
__device__ __forceinline__ float silu_f(float x) { return x / (1.f + expf(-x)); }
__device__ __forceinline__ float silu_grad_f(float x) {
  float s = 1.f / (1.f + expf(-x));
  return s * (1.f + x * (1.f - s));
}

// Group of a padded row: off[0..G] ascending; returns g with off[g] <= r < off[g+1] (or G if beyond).
__device__ __forceinline__ int find_group(const int32_t* off, int G, int64_t r) {
  int lo = 0, hi = G;  // invariant: off[lo] <= r
  if (r >= off[G]) return G;
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (off[mid] <= r) lo = mid; else hi = mid;
  }
  return lo;
}

}  // namespace luffy
