// Representative layout, pack, output reuse and their backward.
//
//  layout:      only representatives are dispatched ("keep the token ... for transmission"); send
//               order = expert asc (= destination rank asc under contiguous placement, R14), token asc
//               (R15); each expert segment padded to LUFFY_ROW_ALIGN rows.  pos[t, j] = slot of the
//               representative of copy (t, j); rep[t, j] = its token (token_to_token).
//  pack_rows:   dst[slot] = x[perm[slot]] with 16-byte vector copies (zero rows for padding).
//  uncondense:  y_t = sum_j w_tj * gathered[pos_tj] -- a condensed token reuses its representative's
//               expert output with its own gate weight (R10); fp32 accumulation.
//  backward:    d_gathered[slot] = sum over the copies it represents (token order) of w * dy, from the
//               slot-sorted member CSR built by layout (no atomics, fixed summation order); the same
//               pass computes the gate-weight gradient dw[t, j] = <dy_t, gathered[slot of (t, j)]>.
#include <cstdlib>

#include "common.cuh"
#include "exchange.cuh"

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

// Block-wide exclusive scan of one int per thread.
__device__ __forceinline__ int block_scan_value(int v, int* warp_sums, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) warp_sums[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const int w = lane < nw ? warp_sums[lane] : 0;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += u;
    }
    if (lane < nw) warp_sums[lane] = wi - w;
    if (lane == 31) warp_sums[32] = wi;
  }
  __syncthreads();
  const int pre = inc - v + warp_sums[wid];
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
                                                      int32_t* __restrict__ rep, int32_t* __restrict__ mstart,
                                                      int32_t* __restrict__ mcnt, int32_t* __restrict__ mcur,
                                                      int32_t* __restrict__ marr,
                                                      int32_t* __restrict__ members, int32_t* __restrict__ mslot,
                                                      int32_t* __restrict__ rep_out,
                                                      const int32_t* __restrict__ gnrep, int cur_cap,
                                                      const int32_t* __restrict__ mrank,
                                                      const int32_t* __restrict__ mcnt_row) {
  pdl_enter();
  extern __shared__ int cur_smem[];
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
  if (gnrep) {  // published by the representative selection of this step
    for (int i = threadIdx.x; i < E; i += blockDim.x) cnt[i] = gnrep[i];
  } else {
    const int rows = goff_s[E];
    for (int g = threadIdx.x; g < rows; g += blockDim.x)
      if (rep_local[g] == g) atomicAdd(&cnt[find_group(goff_s, E, g)], 1);
  }
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
  if (5 * n <= cur_cap) {
    // The group's rows, their representatives and slots live in shared memory, so the dependent lookups
    // (slot of a row's representative, its token) cost no global round trips.
    const int s0 = offs[e], ns = cnt[e];
    int* s_rep = cur_smem;   // [n] representative of each row (group-local index)
    int* s_tok = s_rep + n;  // [n] token of each row
    int* s_ls = s_tok + n;   // [n] slot (relative to s0) of each representative row, -1 otherwise
    int* s_cnt = s_ls + n;   // [ns] members per slot
    int* s_cur = s_cnt + ns; // [ns] placement cursors
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
      s_rep[c] = rep_local[g0 + c] - g0;
      s_tok[c] = gtok[g0 + c];
    }
    for (int i = threadIdx.x; i < ns; i += blockDim.x) s_cnt[i] = 0;
    for (int sl = s0 + ns + threadIdx.x; sl < offs[e + 1]; sl += blockDim.x) {
      perm[sl] = -1;
      slot_gl[sl] = -1;
      mcnt[sl] = 0;
      marr[sl] = 0;
    }
    for (int g = g0 + n + threadIdx.x; g < goff_s[e + 1]; g += blockDim.x) {
      members[g] = -1;
      mslot[g] = -1;
    }
    __syncthreads();
    if (mrank) {
      // member ranks and list lengths came from representative selection (greedy_cluster_kernel, phase D0):
      // slots and list starts are two prefix sums over the group's rows, every member a direct store
      int* s_mst = s_cnt;  // [n] start of the member list of each representative row (reuses s_cnt/s_cur)
      int baseR = 0, baseM = g0;
      for (int c0 = 0; c0 < n; c0 += blockDim.x) {
        const int c = c0 + threadIdx.x;
        const bool inr = c < n;
        const bool isrep = inr && s_rep[c] == c;
        const int mc = isrep ? mcnt_row[g0 + c] : 0;
        int totR, totM;
        const int preR = block_scan_flag2(isrep, warp_sums, totR);
        const int preM = block_scan_value(mc, warp_sums, totM);
        if (isrep) {
          const int ls = baseR + preR;
          s_ls[c] = ls;
          s_mst[c] = baseM + preM;
          lslot[g0 + c] = s0 + ls;
          perm[s0 + ls] = s_tok[c];
          slot_gl[s0 + ls] = g0 + c;
          mstart[s0 + ls] = baseM + preM;
          mcnt[s0 + ls] = mc;
          marr[s0 + ls] = 0;
        } else if (inr) {
          s_ls[c] = -1;
          lslot[g0 + c] = -1;
        }
        baseR += totR;
        baseM += totM;
      }
      __syncthreads();
      for (int c = threadIdx.x; c < n; c += blockDim.x) {
        const int t = s_tok[c];
        const int r = s_rep[c];
        int jj = 0;
        for (int j = 0; j < k; ++j)
          if (idx[(size_t)t * k + j] == e) jj = j;
        const int ls = s_ls[r];
        pos[(size_t)t * k + jj] = s0 + ls;
        rep[(size_t)t * k + jj] = s_tok[r];
        if (rep_out) rep_out[(size_t)t * k + jj] = s_tok[r];
        const int p = s_mst[r] + mrank[g0 + c];
        members[p] = g0 + c;
        mslot[p] = s0 + ls;
      }
      return;
    }
    int base = 0;
    for (int c0 = 0; c0 < n; c0 += blockDim.x) {
      const int c = c0 + threadIdx.x;
      const bool inr = c < n;
      const bool isrep = inr && s_rep[c] == c;
      int total;
      const int pre = block_scan_flag2(isrep, warp_sums, total);
      if (isrep) {
        const int ls = base + pre;
        s_ls[c] = ls;
        lslot[g0 + c] = s0 + ls;
        perm[s0 + ls] = s_tok[c];
        slot_gl[s0 + ls] = g0 + c;
      } else if (inr) {
        s_ls[c] = -1;
        lslot[g0 + c] = -1;
      }
      base += total;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
      const int t = s_tok[c];
      const int r = s_rep[c];
      int jj = 0;
      for (int j = 0; j < k; ++j)
        if (idx[(size_t)t * k + j] == e) jj = j;
      const int ls = s_ls[r];
      pos[(size_t)t * k + jj] = s0 + ls;
      rep[(size_t)t * k + jj] = s_tok[r];
      if (rep_out) rep_out[(size_t)t * k + jj] = s_tok[r];
      atomicAdd(&s_cnt[ls], 1);
    }
    __syncthreads();
    // member CSR (see below): counts -> exclusive scan -> stable placement in group-row order
    int run = g0;
    for (int c0 = 0; c0 < ns; c0 += blockDim.x) {
      const int i = c0 + threadIdx.x;
      const int v = i < ns ? s_cnt[i] : 0;
      int total;
      const int pre = block_scan_value(v, warp_sums, total);
      if (i < ns) {
        mstart[s0 + i] = run + pre;
        mcnt[s0 + i] = v;
        marr[s0 + i] = 0;
        s_cur[i] = run + pre;
      }
      run += total;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    for (int c0 = 0; c0 < n; c0 += blockDim.x) {
      const int c = c0 + threadIdx.x;
      const bool valid = c < n;
      const int key = valid ? s_ls[s_rep[c]] : -1 - lane;  // invalid lanes never group
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      const int leader = __ffs(peers) - 1;
      int b = 0;
      const int nwv = min(nwb, (n - c0 + 31) >> 5);
      for (int w = 0; w < nwv; ++w) {  // warps claim their runs in order: stable across the block
        if (wid == w && valid && lane == leader) {
          b = s_cur[key];
          s_cur[key] = b + __popc(peers);
        }
        __syncthreads();
      }
      b = __shfl_sync(0xffffffffu, b, leader);
      if (valid) {
        const int p = b + __popc(peers & ((1u << lane) - 1u));
        members[p] = g0 + c;
        mslot[p] = key + s0;
      }
    }
    return;
  }
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
    if (rep_out) rep_out[(size_t)t * k + jj] = gtok[r];
  }
  // ---- member CSR of every slot of this expert, members in token (= group row) order, stored in the
  // group-row space [g0, g0 + n) (padding rows of the space hold -1): mstart[slot], mcnt[slot],
  // members[], mslot[] (the slot of each member).  Deterministic: integer-atomic counts, then a stable
  // block-wide placement (in-warp ranks by __match_any_sync, cross-warp order by warp index).
  const int s0 = offs[e], ns = cnt[e];
  for (int s = s0 + threadIdx.x; s < offs[e + 1]; s += blockDim.x) {
    mcnt[s] = 0;
    marr[s] = 0;
  }
  for (int g = g0 + n + threadIdx.x; g < goff_s[e + 1]; g += blockDim.x) {
    members[g] = -1;
    mslot[g] = -1;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < n; c += blockDim.x) atomicAdd(&mcnt[lslot[rep_local[g0 + c]]], 1);
  __syncthreads();
  int* cur = ns <= cur_cap ? cur_smem : mcur + s0;  // placement cursors (shared memory when they fit)
  int run = g0;
  for (int c0 = 0; c0 < ns; c0 += blockDim.x) {
    const int s = s0 + c0 + threadIdx.x;
    const int v = c0 + threadIdx.x < ns ? mcnt[s] : 0;
    int total;
    const int pre = block_scan_value(v, warp_sums, total);
    if (c0 + threadIdx.x < ns) {
      mstart[s] = run + pre;
      cur[c0 + threadIdx.x] = run + pre;
    }
    run += total;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  for (int c0 = 0; c0 < n; c0 += blockDim.x) {
    const bool valid = c0 + threadIdx.x < n;
    const int g = g0 + c0 + threadIdx.x;
    const int key = valid ? lslot[rep_local[g]] - s0 : -1 - lane;  // invalid lanes never group
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int leader = __ffs(peers) - 1;
    int b = 0;
    const int nwv = min(nwb, (n - c0 + 31) >> 5);  // warps holding rows of this chunk (uniform)
    for (int w = 0; w < nwv; ++w) {  // warps claim their runs in order: stable across the block
      if (wid == w && valid && lane == leader) {
        b = cur[key];
        cur[key] = b + __popc(peers);
      }
      __syncthreads();
    }
    b = __shfl_sync(0xffffffffu, b, leader);
    if (valid) {
      const int p = b + __popc(peers & ((1u << lane) - 1u));
      members[p] = g;
      mslot[p] = key + s0;
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) pack_rows_kernel(const T* __restrict__ x, const int32_t* __restrict__ perm,
                                                        const int32_t* __restrict__ soff, int E, int d,
                                                        T* __restrict__ dst) {
  pdl_enter();
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

// y[t] = sum_j w[t, j] * gathered[pos(t, j)] (j in order, fp32): one warp per token, the token's k slots
// and weights read once (lanes < k), every row load of a 512-column block issued before the arithmetic.
template <typename T, int KM>
__global__ void __launch_bounds__(256) uncondense_kernel(const T* __restrict__ gathered, const int32_t* __restrict__ pos,
                                                         const float* __restrict__ w, int T_, int k, int d,
                                                         const T* __restrict__ res, T* __restrict__ y);
template <typename T, int KM>
__global__ void __launch_bounds__(256) unpack_bwd_kernel(const T* __restrict__ dsend, const int32_t* __restrict__ pos,
                                                         const int32_t* __restrict__ rep, int T_, int k, int d,
                                                         const T* __restrict__ res, T* __restrict__ dx);

// d_gathered[slot] = sum_{members m of the slot, token order} gw[m] * dy[gtok[m]]; padding -> 0.
//
// Load-balanced and deterministic: the slot-sorted member array (group-row space) is cut into fixed
// windows of WIN members; one warp per window walks its members in order, accumulating the current
// slot in fp32.  A slot that lies inside one window is written directly; a slot crossing window
// boundaries leaves fp32 partials (the head run of a window at part[w][0], the tail run at part[w][1]);
// the window delivering a slot's last partial sums them in window order (arrival counter per slot).
constexpr int WIN = 16;

// 8 consecutive elements: raw 16-byte (bf16) / 32-byte (fp32) load, then conversion
struct F8 {
  float4 a, b;
};
__device__ __forceinline__ uint4 ldraw8(const bf16* p) { return *reinterpret_cast<const uint4*>(p); }
__device__ __forceinline__ F8 ldraw8(const float* p) {
  return F8{*reinterpret_cast<const float4*>(p), *reinterpret_cast<const float4*>(p + 4)};
}
__device__ __forceinline__ void cvt8(const uint4& u, float (&v)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void cvt8(const F8& u, float (&v)[8]) {
  v[0] = u.a.x; v[1] = u.a.y; v[2] = u.a.z; v[3] = u.a.w;
  v[4] = u.b.x; v[5] = u.b.y; v[6] = u.b.z; v[7] = u.b.w;
}

// Destination of the backward rows of send slots: local d_gathered, or (fused combine-backward) the
// owning rank's dexp buffer at row dst_base[e] + (slot - soff[e]).
struct XDest {
  int remote;
  const int32_t* soff;
  const int32_t* dst_base;
  void* const* peer;
  int E, El;
  template <typename T>
  __device__ __forceinline__ T* row(int slot, int d) const {
    int lo = 0, hi = E;  // expert of the slot: soff[lo] <= slot < soff[lo+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (soff[mid] <= slot) lo = mid; else hi = mid;
    }
    return static_cast<T*>(peer[lo / El]) + ((int64_t)dst_base[lo] + (slot - soff[lo])) * d;
  }
};

template <typename T>
__global__ void __launch_bounds__(256) uncondense_bwd_window_kernel(
    const T* __restrict__ dy, const int32_t* __restrict__ goff, int E, const int32_t* __restrict__ members,
    const int32_t* __restrict__ mslot, const int32_t* __restrict__ mstart, const int32_t* __restrict__ mcnt,
    const int32_t* __restrict__ gtok, const float* __restrict__ gw, const int32_t* __restrict__ gcopy, int d,
    const T* __restrict__ gathered, float* __restrict__ dw, T* __restrict__ dg, float* __restrict__ part,
    int32_t* __restrict__ marr, const int32_t* __restrict__ perm, const int32_t* __restrict__ soff, XDest xd,
    XSignal sig) {
  pdl_enter();
  using R = decltype(ldraw8(static_cast<const T*>(nullptr)));
  const int lane = threadIdx.x & 31;
  const int64_t nwin = goff[E] / WIN;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (!xd.remote) {  // padding slots of d_gathered are zero (remote: the expert rank zeroes its own)
    const int64_t rows = soff[E];
    for (int64_t b = gwarp * 32; b < rows; b += nw * 32) {  // 32 slots per warp step, one perm load each
      unsigned pad = __ballot_sync(0xffffffffu, b + lane < rows && perm[b + lane] < 0);
      while (pad) {
        const int u = __ffs(pad) - 1;
        pad &= pad - 1u;
        for (int c = lane * 8; c < d; c += 256) zero8(dg + (b + u) * d + c);
      }
    }
  }
  for (int64_t wi = gwarp; wi < nwin; wi += nw) {
    const int m0 = (int)(wi * WIN);
    // per-member metadata, resolved once per window (lane u = member u): slot, token, gate weight, copy,
    // whether the member ends its slot's run inside the window, and where that run's sum goes
    int my_slot = -1, my_tok = 0, my_copy = -1;
    float my_w = 0.f;
    if (lane < WIN) {
      const int g = members[m0 + lane];
      if (g >= 0) {
        my_slot = mslot[m0 + lane];
        my_tok = gtok[g];
        my_w = gw[g];
        my_copy = gcopy[g];
      }
    }
    const unsigned live = __ballot_sync(0xffffffffu, my_slot >= 0);
    if (!live) continue;
    const int nxt = __shfl_down_sync(0xffffffffu, my_slot, 1);
    bool my_end = false, my_inside = false;
    unsigned long long my_dst = 0ull;
    int my_ms = 0, my_me = 0;
    if (my_slot >= 0) {
      my_end = lane == WIN - 1 || nxt != my_slot;
      if (my_end) {
        const int ms = mstart[my_slot], me = ms + mcnt[my_slot];
        my_ms = ms;
        my_me = me;
        my_inside = ms >= m0 && me <= m0 + WIN;
        my_dst = my_inside ? reinterpret_cast<unsigned long long>(xd.remote ? xd.row<T>(my_slot, d) : dg + (size_t)my_slot * d)
                           : reinterpret_cast<unsigned long long>(part + ((size_t)wi * 2 + (ms < m0 ? 0 : 1)) * d);
      }
    }
    const unsigned ends = __ballot_sync(0xffffffffu, my_end);
    const unsigned inside = __ballot_sync(0xffffffffu, my_inside);
    float dot[WIN];  // this lane's partial of <dy_t, gathered[slot]> for every member (gate-weight gradient)
#pragma unroll
    for (int u = 0; u < WIN; ++u) dot[u] = 0.f;
    for (int c0 = 0; c0 < d; c0 += 256) {
      const int c = c0 + lane * 8;
      // issue the row loads of the whole window first: dy of every member and, for the gate-weight
      // gradient, the expert output row of its slot (8 elements per lane each)
      R rdy[WIN], rg[WIN];
#pragma unroll
      for (int u = 0; u < WIN; ++u) {
        const int tok = __shfl_sync(0xffffffffu, my_tok, u);
        const int slot = __shfl_sync(0xffffffffu, my_slot, u);
        const bool ok = ((live >> u) & 1u) && c < d;
        rdy[u] = ok ? ldraw8(dy + (size_t)tok * d + c) : R{};
        rg[u] = (ok && dw) ? ldraw8(gathered + (size_t)slot * d + c) : R{};
      }
      float acc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = 0.f;
#pragma unroll
      for (int u = 0; u < WIN; ++u) {
        const float wm = __shfl_sync(0xffffffffu, my_w, u);
        const unsigned long long dst = __shfl_sync(0xffffffffu, my_dst, u);
        if (!((live >> u) & 1u)) continue;  // padding rows (warp-uniform)
        float v[8], o[8];
        cvt8(rdy[u], v);
        cvt8(rg[u], o);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          acc[i] = fmaf(wm, v[i], acc[i]);
          dot[u] = fmaf(v[i], o[i], dot[u]);
        }
        if ((ends >> u) & 1u) {  // the slot's run ends here: write it (whole slot or a partial), restart
          if (c < d) {
            if ((inside >> u) & 1u) store8(reinterpret_cast<T*>(dst) + c, acc);
            else store8(reinterpret_cast<float*>(dst) + c, acc);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] = 0.f;
        }
      }
    }
    if (dw) {
#pragma unroll
      for (int u = 0; u < WIN; ++u) {
        const float sdot = warp_sum(dot[u]);
        const int cp = __shfl_sync(0xffffffffu, my_copy, u);
        if (lane == 0 && cp >= 0) dw[cp] = sdot;
      }
    }
    // runs left as partials (a slot crossing window boundaries): the window that delivers a slot's LAST
    // partial sums all of them in window order (the tail partial of the first window, then the head
    // partials) -- a fixed order, so the result does not depend on which window arrives last
    unsigned pm = ends & ~inside & live;
    if (pm) {
      __threadfence();
      while (pm) {
        const int u = __ffs(pm) - 1;
        pm &= pm - 1u;
        const int slot = __shfl_sync(0xffffffffu, my_slot, u);
        const int ms = __shfl_sync(0xffffffffu, my_ms, u), me = __shfl_sync(0xffffffffu, my_me, u);
        const int ws = ms / WIN, we = (me - 1) / WIN, n = we - ws + 1;
        int last = 0;
        if (lane == 0) last = atomicAdd(marr + slot, 1) == n - 1;
        last = __shfl_sync(0xffffffffu, last, 0);
        if (!last) continue;
        __threadfence();
        T* out = xd.remote ? xd.row<T>(slot, d) : dg + (size_t)slot * d;
        // partials summed in window order j = 0 .. n-1 for up to 4 column chunks at once (two windows
        // of loads in flight), chunk groups of 1024 columns
        for (int cg = 0; cg < d; cg += 1024) {
          float a[4][8];
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[q][i] = 0.f;
#pragma unroll 2
          for (int j = 0; j < n; ++j) {
            const float* src = part + ((size_t)(ws + j) * 2 + (j == 0 ? 1 : 0)) * d;
            float4 x[4][2] = {};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int c = cg + q * 256 + lane * 8;
              if (c < d) {
                x[q][0] = __ldcg(reinterpret_cast<const float4*>(src + c));
                x[q][1] = __ldcg(reinterpret_cast<const float4*>(src + c) + 1);
              }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              a[q][0] += x[q][0].x; a[q][1] += x[q][0].y; a[q][2] += x[q][0].z; a[q][3] += x[q][0].w;
              a[q][4] += x[q][1].x; a[q][5] += x[q][1].y; a[q][6] += x[q][1].z; a[q][7] += x[q][1].w;
            }
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int c = cg + q * 256 + lane * 8;
            if (c < d) store8(out + c, a[q]);
          }
        }
        if (lane == 0) marr[slot] = 0;  // ready for the next backward over the same layout
      }
    }
  }
  if (xd.remote) {
    __threadfence_system();
    xsignal_done(sig);
  }
}

// dx[t] = [res[t] +] sum_{j : rep(t, j) == t} d_send[pos_tj]   (condensed copies get no expert-path
// gradient, R11; res: the residual branch's gradient dY of a block y = x + MoE(x))
template <typename T, int KM>
__global__ void __launch_bounds__(256) unpack_bwd_kernel(const T* __restrict__ dsend, const int32_t* __restrict__ pos,
                                                         const int32_t* __restrict__ rep, int T_, int k, int d,
                                                         const T* __restrict__ res, T* __restrict__ dx) {
  pdl_enter();
  using R = decltype(ldraw8(static_cast<const T*>(nullptr)));
  constexpr int HC = KM <= 2 ? 2 : 1;  // 256-column chunks per load batch
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < T_; t += nw) {
    int my_pos = -1;
    if (lane < k && rep[(size_t)t * k + lane] == t) my_pos = pos[(size_t)t * k + lane];
    int row[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) row[j] = __shfl_sync(0xffffffffu, my_pos, j);
    for (int c0 = 0; c0 < d; c0 += 256 * HC) {
      R raw[HC][KM];
#pragma unroll
      for (int h = 0; h < HC; ++h)
#pragma unroll
        for (int j = 0; j < KM; ++j) {
          const int c = c0 + h * 256 + lane * 8;
          raw[h][j] = (j < k && row[j] >= 0 && c < d) ? ldraw8(dsend + (size_t)row[j] * d + c) : R{};
        }
#pragma unroll
      for (int h = 0; h < HC; ++h) {
        const int c = c0 + h * 256 + lane * 8;
        if (c >= d) break;
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (res != nullptr) load8(res + (size_t)t * d + c, acc);
#pragma unroll
        for (int j = 0; j < KM; ++j) {
          if (j < k && row[j] >= 0) {
            float v[8];
            cvt8(raw[h][j], v);
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] += v[i];
          }
        }
        store8(dx + (size_t)t * d + c, acc);
      }
    }
  }
}

template <typename T, int KM>
__global__ void __launch_bounds__(256) uncondense_kernel(const T* __restrict__ gathered, const int32_t* __restrict__ pos,
                                                         const float* __restrict__ w, int T_, int k, int d,
                                                         const T* __restrict__ res, T* __restrict__ y) {
  pdl_enter();
  using R = decltype(ldraw8(static_cast<const T*>(nullptr)));
  constexpr int HC = KM <= 2 ? 2 : 1;
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < T_; t += nw) {
    int my_pos = 0;
    float my_w = 0.f;
    if (lane < k) {
      my_pos = pos[(size_t)t * k + lane];
      my_w = w[(size_t)t * k + lane];
    }
    int row[KM];
    float wt[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      row[j] = __shfl_sync(0xffffffffu, my_pos, j);
      wt[j] = __shfl_sync(0xffffffffu, my_w, j);
    }
    for (int c0 = 0; c0 < d; c0 += 256 * HC) {
      R raw[HC][KM];
#pragma unroll
      for (int h = 0; h < HC; ++h)
#pragma unroll
        for (int j = 0; j < KM; ++j) {
          const int c = c0 + h * 256 + lane * 8;
          raw[h][j] = (j < k && c < d) ? ldraw8(gathered + (size_t)row[j] * d + c) : R{};
        }
#pragma unroll
      for (int h = 0; h < HC; ++h) {
        const int c = c0 + h * 256 + lane * 8;
        if (c >= d) break;
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (res != nullptr) load8(res + (size_t)t * d + c, acc);  // residual block: y = x + sum_j w o
#pragma unroll
        for (int j = 0; j < KM; ++j) {
          if (j < k) {
            float v[8];
            cvt8(raw[h][j], v);
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = fmaf(wt[j], v[i], acc[i]);
          }
        }
        store8(y + (size_t)t * d + c, acc);
      }
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
  // dynamic shared memory (ints): the staged group state, or the placement cursors of the global-memory
  // path (LUFFY_LAYOUT_SMEM=0 forces that path, for tests)
  static const int cur_cap = [] {
    const char* v = std::getenv("LUFFY_LAYOUT_SMEM");
    return v && v[0] == '0' ? 0 : 40000;
  }();
  LUFFY_CUDA_TRY(smem_optin((const void*)layout_kernel, 40000 * 4));
  launch_pdl(layout_kernel, L->E, 1024, (size_t)std::max(cur_cap, 1) * 4, st, L->goff, L->gcnt, L->gtok, L->rep_local, L->idx, L->E, L->k, L->nrep,
                                                 L->soff, L->lslot, L->perm, L->slot_gl, L->pos, L->rep, L->mstart,
                                                 L->mcnt, L->mcur, L->marr, L->members, L->mslot, rep_out,
                                                 L->gnrep_valid ? L->gnrep : nullptr, cur_cap,
                                                 L->mrank_valid ? L->mrank : nullptr, L->mcnt_row);
  LUFFY_LAUNCHED();

  if (dst_rows) {
    const int blocks = grid_for_warps(L->Rpad_max);
    if (L->dtype == LUFFY_BF16)
      launch_pdl(pack_rows_kernel<bf16>, blocks, 256, 0, st, static_cast<const bf16*>(x), L->perm, L->soff, L->E, L->d,
                                                     static_cast<bf16*>(dst_rows));
    else
      launch_pdl(pack_rows_kernel<float>, blocks, 256, 0, st, static_cast<const float*>(x), L->perm, L->soff, L->E, L->d,
                                                      static_cast<float*>(dst_rows));
    LUFFY_LAUNCHED();
  }
  return 0;
}

int launch_pack_rows(luffy_layer* L, const void* x, void* dst_rows, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  const int blocks = grid_for_warps(L->Rpad_max);
  if (L->dtype == LUFFY_BF16)
    launch_pdl(pack_rows_kernel<bf16>, blocks, 256, 0, st, static_cast<const bf16*>(x), L->perm, L->soff, L->E, L->d,
                                                   static_cast<bf16*>(dst_rows));
  else
    launch_pdl(pack_rows_kernel<float>, blocks, 256, 0, st, static_cast<const float*>(x), L->perm, L->soff, L->E, L->d,
                                                    static_cast<float*>(dst_rows));
  LUFFY_LAUNCHED();
  return 0;
}

int launch_uncondense(const luffy_layer* L, const void* gathered, const void* res, void* y, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  const int blocks = grid_for_warps(L->T);
  if (L->dtype == LUFFY_BF16)
    launch_pdl(L->k <= 2 ? uncondense_kernel<bf16, 2> : uncondense_kernel<bf16, 8>, blocks, 256, 0, st, static_cast<const bf16*>(gathered), L->pos, L->w, L->T, L->k, L->d,
                                                    static_cast<const bf16*>(res), static_cast<bf16*>(y));
  else
    launch_pdl(L->k <= 2 ? uncondense_kernel<float, 2> : uncondense_kernel<float, 8>, blocks, 256, 0, st, static_cast<const float*>(gathered), L->pos, L->w, L->T, L->k, L->d,
                                                     static_cast<const float*>(res), static_cast<float*>(y));
  LUFFY_LAUNCHED();
  return 0;
}

int launch_uncondense_bwd(const luffy_layer* L, const void* dy, const void* gathered, void* dg, float* dw, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  XDest xd{};
  XSignal sig{};
  if (L->P > 1) {
    xd.remote = 1;
    xd.soff = L->soff;
    xd.dst_base = L->x_dst_base;
    xd.peer = L->x_peer_dexp;
    xd.E = L->E;
    xd.El = L->El;
    sig = make_signal(L, XP_CBWD);
  }
  const int bw = grid_for_warps(L->Cpad_max / WIN);
  if (L->dtype == LUFFY_BF16) {
    launch_pdl(uncondense_bwd_window_kernel<bf16>, bw, 256, 0, st, static_cast<const bf16*>(dy), L->goff, L->E, L->members,
               L->mslot, L->mstart, L->mcnt, L->gtok, L->gw, L->gcopy, L->d, static_cast<const bf16*>(gathered), dw,
               static_cast<bf16*>(dg), L->mpart, L->marr, L->perm, L->soff, xd, sig);
  } else {
    launch_pdl(uncondense_bwd_window_kernel<float>, bw, 256, 0, st, static_cast<const float*>(dy), L->goff, L->E, L->members,
               L->mslot, L->mstart, L->mcnt, L->gtok, L->gw, L->gcopy, L->d, static_cast<const float*>(gathered), dw,
               static_cast<float*>(dg), L->mpart, L->marr, L->perm, L->soff, xd, sig);
  }
  LUFFY_LAUNCHED();
  return 0;
}

int launch_unpack_bwd(const luffy_layer* L, const void* dsend, const void* res, void* dx, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  const int blocks = grid_for_warps(L->T);
  if (L->dtype == LUFFY_BF16)
    launch_pdl(L->k <= 2 ? unpack_bwd_kernel<bf16, 2> : unpack_bwd_kernel<bf16, 8>, blocks, 256, 0, st, static_cast<const bf16*>(dsend), L->pos, L->rep, L->T, L->k, L->d,
                                                    static_cast<const bf16*>(res), static_cast<bf16*>(dx));
  else
    launch_pdl(L->k <= 2 ? unpack_bwd_kernel<float, 2> : unpack_bwd_kernel<float, 8>, blocks, 256, 0, st, static_cast<const float*>(dsend), L->pos, L->rep, L->T, L->k, L->d,
                                                     static_cast<const float*>(res), static_cast<float*>(dx));
  LUFFY_LAUNCHED();
  return 0;
}

}  // namespace luffy
