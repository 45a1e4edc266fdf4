// Dispatch-push pattern probe (2 GPUs, one process, peer access): scattered 2 KB rows (a random
// permutation of a 16 MB bf16 [8192, 1024] x) pushed into a peer's contiguous receive buffer, as the fused
// pack + dispatch does, in several warp schedules; and the contiguous copy as the upper bound.  Sizes: the
// C2 N = 2 push (4250 rows, 8.7 MB).  Used to pick xpack_push_kernel's schedule.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/nvpush tools/nvlink_push_probe.cu && /tmp/nvpush
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

constexpr int D = 1024;  // bf16 elements per row -> 2 KB, 128 uint4

// (a) warp per row, per 16-byte piece: load then store (the shipped schedule)
__global__ void push_a(const uint4* __restrict__ x, const int* __restrict__ perm, uint4* dst, int rows) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < rows; s += nw) {
    const uint4* src = x + (size_t)perm[s] * (D / 8);
    uint4* d = dst + (size_t)s * (D / 8);
    for (int c = lane; c < D / 8; c += 32) d[c] = src[c];
  }
}
// (b) warp per row, all four loads first, then the four stores
__global__ void push_b(const uint4* __restrict__ x, const int* __restrict__ perm, uint4* dst, int rows) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < rows; s += nw) {
    const uint4* src = x + (size_t)perm[s] * (D / 8);
    uint4* d = dst + (size_t)s * (D / 8);
    uint4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = src[lane + 32 * j];
#pragma unroll
    for (int j = 0; j < 4; ++j) d[lane + 32 * j] = v[j];
  }
}
// (c) warp per R rows at once: 4R loads in flight, then 4R stores
template <int R>
__global__ void push_c(const uint4* __restrict__ x, const int* __restrict__ perm, uint4* dst, int rows) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * R; s0 < rows; s0 += nw * R) {
    uint4 v[R][4];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int s = s0 + r;
      const uint4* src = x + (size_t)perm[s < rows ? s : rows - 1] * (D / 8);
#pragma unroll
      for (int j = 0; j < 4; ++j) v[r][j] = src[lane + 32 * j];
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (s0 + r >= rows) break;
      uint4* d = dst + (size_t)(s0 + r) * (D / 8);
#pragma unroll
      for (int j = 0; j < 4; ++j) d[lane + 32 * j] = v[r][j];
    }
  }
}
// (d) stores only (no source reads): the NVLink write path alone
__global__ void push_d(uint4* dst, int rows) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const uint4 v = make_uint4(lane, 1, 2, 3);
  for (int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < rows; s += nw) {
    uint4* d = dst + (size_t)s * (D / 8);
#pragma unroll
    for (int j = 0; j < 4; ++j) d[lane + 32 * j] = v;
  }
}
// (e) st.global with .L2::... none; use 16-byte stores with the no-allocate hint (st.global.cs)
__global__ void push_e(const uint4* __restrict__ x, const int* __restrict__ perm, uint4* dst, int rows) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < rows; s += nw) {
    const uint4* src = x + (size_t)perm[s] * (D / 8);
    uint4* d = dst + (size_t)s * (D / 8);
    uint4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = __ldcs(src + lane + 32 * j);
#pragma unroll
    for (int j = 0; j < 4; ++j) __stcs(d + lane + 32 * j, v[j]);
  }
}

int main() {
  int n = 0;
  cudaGetDeviceCount(&n);
  if (n < 2) { printf("need 2 GPUs\n"); return 0; }
  const int T = 8192;
  const size_t xbytes = (size_t)T * D * 2;
  uint4 *x, *dst;
  int* perm;
  cudaSetDevice(1); cudaMalloc(&dst, xbytes); cudaDeviceEnablePeerAccess(0, 0);
  cudaSetDevice(0); cudaMalloc(&x, xbytes); cudaMalloc(&perm, T * 4); cudaDeviceEnablePeerAccess(1, 0);
  uint4* flush; cudaMalloc(&flush, 256ull << 20);
  cudaMemset(x, 1, xbytes);
  std::vector<int> h(T);
  for (int i = 0; i < T; ++i) h[i] = i;
  std::mt19937 g(7); std::shuffle(h.begin(), h.end(), g);
  cudaMemcpy(perm, h.data(), T * 4, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch, int rows) {
    float best = 1e9;
    for (int rep = 0; rep < 8; ++rep) {
      cudaMemset(flush, rep, 256ull << 20);  // evict x from L2
      cudaEventRecord(e0); launch(rows); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    }
    const double b = (double)rows * D * 2;
    printf("%-34s rows %5d  %7.1f us  %6.0f GB/s  (%s)\n", name, rows, best * 1e3, b / best / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int rows : {4250, 6350, 8192}) {
    const int w1 = (rows + 7) / 8;  // CTAs of 8 warps, one warp per row
    run("a  warp/row ld-st (shipped)", [&](int r) { push_a<<<w1, 256>>>(x, perm, dst, r); }, rows);
    run("b  warp/row 4 ld then 4 st", [&](int r) { push_b<<<w1, 256>>>(x, perm, dst, r); }, rows);
    run("c2 warp/2 rows", [&](int r) { push_c<2><<<(w1 + 1) / 2, 256>>>(x, perm, dst, r); }, rows);
    run("c4 warp/4 rows", [&](int r) { push_c<4><<<(w1 + 3) / 4, 256>>>(x, perm, dst, r); }, rows);
    run("b  grid 148x8 warps (persistent)", [&](int r) { push_b<<<148, 256>>>(x, perm, dst, r); }, rows);
    run("b  grid 296x8 warps", [&](int r) { push_b<<<296, 256>>>(x, perm, dst, r); }, rows);
    run("e  ldcs/stcs", [&](int r) { push_e<<<w1, 256>>>(x, perm, dst, r); }, rows);
    run("d  stores only", [&](int r) { push_d<<<w1, 256>>>(dst, r); }, rows);
    run("memcpy peer (contiguous)", [&](int r) { cudaMemcpyPeerAsync(dst, 1, x, 0, (size_t)r * D * 2); }, rows);
  }
  return 0;
}
