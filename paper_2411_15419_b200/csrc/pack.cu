// Representative layout, pack, output reuse and their backward.
//
//  layout:      only representatives are dispatched ("keep the token ... for transmission"); send
//               order = expert asc (= destination rank asc under contiguous placement, R14), token asc
//               (R15); each expert segment padded to LUFFY_ROW_ALIGN rows.  pos[t, j] = slot of the
//               representative of copy (t, j); rep[t, j] = its token (token_to_token).
//  pack_rows:   dst[slot] = x[perm[slot]] with 16-byte vector copies (zero rows for padding).
//  uncondense:  y_t = sum_j w_tj * gathered[pos_tj] -- a condensed token reuses its representative's
//               expert output with its own gate weight (R10); fp32 accumulation.
//  backward:    d_gathered[slot] = sum over the copies it represents (token order) of w * dy; the
//               members are read from the slot's adjacency row (they are exactly its neighbours whose
//               rep is the slot, plus itself), so no atomics and a fixed summation order.
#include "common.cuh"

namespace luffy {
namespace {

__device__ __forceinline__ int block_scan_flag2(bool flag, int* warp_sums, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned b = __ballot_sync(0xffffffffu, flag);
  int pre = __popc(b & ((1u << lane) - 1u));
  if (lane == 0) warp_sums[wid] = __popc(b);
  __syncthreads();
  if (wid == 0) {
    int v = lane < nw ? warp_sums[lane] : 0;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    if (lane < nw) warp_sums[lane] = inc - v;
    if (lane == 31) warp_sums[32] = inc;
  }
  __syncthreads();
  pre += warp_sums[wid];
  total = warp_sums[32];
  __syncthreads();
  return pre;
}

// One CTA per expert.  Every CTA recounts the representatives of all experts (cheap) so that the
// padded send offsets need no second launch.
__global__ void __launch_bounds__(1024) layout_kernel(const int32_t* __restrict__ goff, const int32_t* __restrict__ gcnt,
                                                      const int32_t* __restrict__ gtok, const int32_t* __restrict__ rep_local,
                                                      const int32_t* __restrict__ idx, int E, int k,
                                                      int32_t* __restrict__ nrep, int32_t* __restrict__ soff,
                                                      int32_t* __restrict__ lslot, int32_t* __restrict__ perm,
                                                      int32_t* __restrict__ slot_gl, int32_t* __restrict__ pos,
                                                      int32_t* __restrict__ rep) {
  __shared__ int cnt[LUFFY_MAX_EXPERTS];
  __shared__ int offs[LUFFY_MAX_EXPERTS + 1];
  __shared__ int32_t goff_s[LUFFY_MAX_EXPERTS + 1];
  __shared__ int warp_sums[33];
  const int e = blockIdx.x;
  for (int i = threadIdx.x; i <= E; i += blockDim.x) {
    goff_s[i] = goff[i];
    if (i < E) cnt[i] = 0;
  }
  __syncthreads();
  const int rows = goff_s[E];
  for (int g = threadIdx.x; g < rows; g += blockDim.x)
    if (rep_local[g] == g) atomicAdd(&cnt[find_group(goff_s, E, g)], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    offs[0] = 0;
    for (int x = 0; x < E; ++x) offs[x + 1] = offs[x] + (cnt[x] + kRowAlign - 1) / kRowAlign * kRowAlign;
  }
  __syncthreads();
  if (e == 0)
    for (int i = threadIdx.x; i <= E; i += blockDim.x) {
      soff[i] = offs[i];
      if (i < E) nrep[i] = cnt[i];
    }
  const int g0 = goff_s[e], n = gcnt[e];
  int base = offs[e];
  for (int c0 = 0; c0 < n; c0 += blockDim.x) {
    const int g = g0 + c0 + threadIdx.x;
    const bool inr = c0 + threadIdx.x < n;
    const bool isrep = inr && rep_local[g] == g;
    int total;
    const int pre = block_scan_flag2(isrep, warp_sums, total);
    if (isrep) {
      const int slot = base + pre;
      lslot[g] = slot;
      perm[slot] = gtok[g];
      slot_gl[slot] = g;
    } else if (inr) {
      lslot[g] = -1;
    }
    base += total;
  }
  for (int s = offs[e] + cnt[e] + threadIdx.x; s < offs[e + 1]; s += blockDim.x) {
    perm[s] = -1;
    slot_gl[s] = -1;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    const int g = g0 + c;
    const int t = gtok[g];
    const int r = rep_local[g];
    int jj = 0;
    for (int j = 0; j < k; ++j)
      if (idx[(size_t)t * k + j] == e) jj = j;
    pos[(size_t)t * k + jj] = lslot[r];
    rep[(size_t)t * k + jj] = gtok[r];
  }
}

template <typename T>
__global__ void __launch_bounds__(256) pack_rows_kernel(const T* __restrict__ x, const int32_t* __restrict__ perm,
                                                        const int32_t* __restrict__ soff, int E, int d,
                                                        T* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t rows = soff[E];
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < rows; s += nw) {
    const int t = perm[s];
    T* o = dst + s * d;
    if (t < 0) {
      for (int c = lane * 8; c < d; c += 256) zero8(o + c);
    } else {
      const T* src = x + (size_t)t * d;
      for (int c = lane * 8; c < d; c += 256) {
        if constexpr (sizeof(T) == 2) {
          *reinterpret_cast<uint4*>(o + c) = *reinterpret_cast<const uint4*>(src + c);
        } else {
          *reinterpret_cast<float4*>(o + c) = *reinterpret_cast<const float4*>(src + c);
          *reinterpret_cast<float4*>(o + c + 4) = *reinterpret_cast<const float4*>(src + c + 4);
        }
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) uncondense_kernel(const T* __restrict__ gathered, const int32_t* __restrict__ pos,
                                                         const float* __restrict__ w, int T_, int k, int d,
                                                         T* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < T_; t += nw) {
    for (int c = lane * 8; c < d; c += 256) {
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int j = 0; j < k; ++j) {
        const float wj = w[(size_t)t * k + j];
        float v[8];
        load8(gathered + (size_t)pos[(size_t)t * k + j] * d + c, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fmaf(wj, v[i], acc[i]);
      }
      store8(y + (size_t)t * d + c, acc);
    }
  }
}

// d_topk_w[t, j] = <dy_t, gathered[pos_tj]>
template <typename T>
__global__ void __launch_bounds__(256) dw_kernel(const T* __restrict__ dy, const T* __restrict__ gathered,
                                                 const int32_t* __restrict__ pos, int T_, int k, int d,
                                                 float* __restrict__ dw) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < T_; t += nw) {
    for (int j = 0; j < k; ++j) {
      const T* o = gathered + (size_t)pos[(size_t)t * k + j] * d;
      float s = 0.f;
      for (int c = lane * 8; c < d; c += 256) {
        float a[8], b[8];
        load8(dy + (size_t)t * d + c, a);
        load8(o + c, b);
#pragma unroll
        for (int i = 0; i < 8; ++i) s = fmaf(a[i], b[i], s);
      }
      s = warp_sum(s);
      if (lane == 0) dw[(size_t)t * k + j] = s;
    }
  }
}

// d_gathered[slot] = sum_{members m of the slot, token order} gw[m] * dy[gtok[m]]; padding -> 0.
// One warp per slot; columns in passes of 256 * CH elements (CH 16-byte chunks per lane).
template <typename T, int CH>
__global__ void __launch_bounds__(256) uncondense_bwd_kernel(const T* __restrict__ dy, const int32_t* __restrict__ slot_gl,
                                                             const int32_t* __restrict__ soff, const int32_t* __restrict__ goff,
                                                             const int32_t* __restrict__ gtok, const float* __restrict__ gw,
                                                             const int32_t* __restrict__ rep_local,
                                                             const int64_t* __restrict__ adjoff, const uint32_t* __restrict__ adj,
                                                             int has_adj, int E, int d, T* __restrict__ dg) {
  __shared__ int32_t goff_s[LUFFY_MAX_EXPERTS + 1];
  for (int i = threadIdx.x; i <= E; i += blockDim.x) goff_s[i] = goff[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t rows = soff[E];
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < rows; s += nw) {
    const int u = slot_gl[s];
    T* out = dg + s * d;
    if (u < 0) {
      for (int c = lane * 8; c < d; c += 256) zero8(out + c);
      continue;
    }
    const int g = find_group(goff_s, E, u);
    const int W = (goff_s[g + 1] - goff_s[g]) >> 5;
    const uint32_t* row = has_adj ? adj + adjoff[g] + (int64_t)(u - goff_s[g]) * W : nullptr;
    for (int c0 = 0; c0 < d; c0 += 256 * CH) {
      float acc[CH][8];
#pragma unroll
      for (int q = 0; q < CH; ++q)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[q][i] = 0.f;
      auto add_member = [&](int m) {
        const float wm = gw[m];
        const T* src = dy + (size_t)gtok[m] * d;
#pragma unroll
        for (int q = 0; q < CH; ++q) {
          const int c = c0 + q * 256 + lane * 8;
          if (c < d) {
            float v[8];
            load8(src + c, v);
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[q][i] = fmaf(wm, v[i], acc[q][i]);
          }
        }
      };
      bool self_done = false;
      if (has_adj) {
        for (int wd = 0; wd < W; ++wd) {
          uint32_t bits = row[wd];  // warp-uniform broadcast load
          while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const int m = goff_s[g] + wd * 32 + b;
            if (!self_done && m > u) { add_member(u); self_done = true; }
            if (rep_local[m] == u) add_member(m);
          }
        }
      }
      if (!self_done) add_member(u);
#pragma unroll
      for (int q = 0; q < CH; ++q) {
        const int c = c0 + q * 256 + lane * 8;
        if (c < d) store8(out + c, acc[q]);
      }
    }
  }
}

// dx[t] = sum_{j : rep(t, j) == t} d_send[pos_tj]   (condensed copies get no expert-path gradient, R11)
template <typename T>
__global__ void __launch_bounds__(256) unpack_bwd_kernel(const T* __restrict__ dsend, const int32_t* __restrict__ pos,
                                                         const int32_t* __restrict__ rep, int T_, int k, int d,
                                                         T* __restrict__ dx) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < T_; t += nw) {
    for (int c = lane * 8; c < d; c += 256) {
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int j = 0; j < k; ++j) {
        if (rep[(size_t)t * k + j] != t) continue;
        float v[8];
        load8(dsend + (size_t)pos[(size_t)t * k + j] * d + c, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += v[i];
      }
      store8(dx + (size_t)t * d + c, acc);
    }
  }
}

inline int grid_for_warps(int64_t warps) {
  int64_t b = (warps + 7) / 8;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}

}  // namespace

int launch_pack(luffy_layer* L, const void* x, void* dst_rows, int32_t* rep_out, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  layout_kernel<<<L->E, 1024, 0, st>>>(L->goff, L->gcnt, L->gtok, L->rep_local, L->idx, L->E, L->k, L->nrep, L->soff,
                                       L->lslot, L->perm, L->slot_gl, L->pos, L->rep);
  LUFFY_LAUNCHED();
  if (rep_out) {
    LUFFY_CUDA_TRY(cudaMemcpyAsync(rep_out, L->rep, sizeof(int32_t) * L->T * L->k, cudaMemcpyDeviceToDevice, st));
  }
  if (dst_rows) {
    const int blocks = grid_for_warps(L->Rpad_max);
    if (L->dtype == LUFFY_BF16)
      pack_rows_kernel<bf16><<<blocks, 256, 0, st>>>(static_cast<const bf16*>(x), L->perm, L->soff, L->E, L->d,
                                                     static_cast<bf16*>(dst_rows));
    else
      pack_rows_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(x), L->perm, L->soff, L->E, L->d,
                                                      static_cast<float*>(dst_rows));
    LUFFY_LAUNCHED();
  }
  return 0;
}

int launch_pack_rows(luffy_layer* L, const void* x, void* dst_rows, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  const int blocks = grid_for_warps(L->Rpad_max);
  if (L->dtype == LUFFY_BF16)
    pack_rows_kernel<bf16><<<blocks, 256, 0, st>>>(static_cast<const bf16*>(x), L->perm, L->soff, L->E, L->d,
                                                   static_cast<bf16*>(dst_rows));
  else
    pack_rows_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(x), L->perm, L->soff, L->E, L->d,
                                                    static_cast<float*>(dst_rows));
  LUFFY_LAUNCHED();
  return 0;
}

int launch_uncondense(const luffy_layer* L, const void* gathered, void* y, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  const int blocks = grid_for_warps(L->T);
  if (L->dtype == LUFFY_BF16)
    uncondense_kernel<bf16><<<blocks, 256, 0, st>>>(static_cast<const bf16*>(gathered), L->pos, L->w, L->T, L->k, L->d,
                                                    static_cast<bf16*>(y));
  else
    uncondense_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(gathered), L->pos, L->w, L->T, L->k, L->d,
                                                     static_cast<float*>(y));
  LUFFY_LAUNCHED();
  return 0;
}

int launch_uncondense_bwd(const luffy_layer* L, const void* dy, const void* gathered, void* dg, float* dw, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  const int bt = grid_for_warps(L->T);
  const int bs = grid_for_warps(L->Rpad_max);
  if (L->dtype == LUFFY_BF16) {
    dw_kernel<bf16><<<bt, 256, 0, st>>>(static_cast<const bf16*>(dy), static_cast<const bf16*>(gathered), L->pos, L->T,
                                        L->k, L->d, dw);
    LUFFY_LAUNCHED();
    uncondense_bwd_kernel<bf16, 4><<<bs, 256, 0, st>>>(static_cast<const bf16*>(dy), L->slot_gl, L->soff, L->goff, L->gtok,
                                                       L->gw, L->rep_local, L->adjoff, L->adj, L->has_adj ? 1 : 0, L->E,
                                                       L->d, static_cast<bf16*>(dg));
  } else {
    dw_kernel<float><<<bt, 256, 0, st>>>(static_cast<const float*>(dy), static_cast<const float*>(gathered), L->pos, L->T,
                                         L->k, L->d, dw);
    LUFFY_LAUNCHED();
    uncondense_bwd_kernel<float, 4><<<bs, 256, 0, st>>>(static_cast<const float*>(dy), L->slot_gl, L->soff, L->goff,
                                                        L->gtok, L->gw, L->rep_local, L->adjoff, L->adj,
                                                        L->has_adj ? 1 : 0, L->E, L->d, static_cast<float*>(dg));
  }
  LUFFY_LAUNCHED();
  return 0;
}

int launch_unpack_bwd(const luffy_layer* L, const void* dsend, void* dx, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  const int blocks = grid_for_warps(L->T);
  if (L->dtype == LUFFY_BF16)
    unpack_bwd_kernel<bf16><<<blocks, 256, 0, st>>>(static_cast<const bf16*>(dsend), L->pos, L->rep, L->T, L->k, L->d,
                                                    static_cast<bf16*>(dx));
  else
    unpack_bwd_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(dsend), L->pos, L->rep, L->T, L->k, L->d,
                                                     static_cast<float*>(dx));
  LUFFY_LAUNCHED();
  return 0;
}

}  // namespace luffy
