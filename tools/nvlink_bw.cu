// NVLink peer bandwidth probe (2 GPUs, one process, peer access): warp 16-byte stores to the peer
// (push), 16-byte loads from the peer (pull), and bulk async copies (cp.async.bulk) smem -> peer.
// Used to choose the data-movement primitive of the fused exchange.  Build/run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/nvbw tools/nvlink_bw.cu && /tmp/nvbw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void push_st(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) dst[i] = src[i];
}
__global__ void pull_ld(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) dst[i] = src[i];
}
// each CTA: load 16 KB chunks into smem, then one thread bulk-copies them to the peer
__global__ void push_bulk(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  __shared__ __align__(128) uint4 buf[1024];
  const size_t chunk = 1024;
  for (size_t c = blockIdx.x; c * chunk < n; c += gridDim.x) {
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = src[c * chunk + i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * chunk),
                   "r"((unsigned)__cvta_generic_to_shared(buf)), "r"(16384) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int n = 0;
  cudaGetDeviceCount(&n);
  if (n < 2) { printf("need 2 GPUs\n"); return 0; }
  const size_t bytes = 256ull << 20, N = bytes / 16;
  uint4 *a0, *b0, *a1;
  cudaSetDevice(1); cudaMalloc(&a1, bytes); cudaDeviceEnablePeerAccess(0, 0);
  cudaSetDevice(0); cudaMalloc(&a0, bytes); cudaMalloc(&b0, bytes); cudaDeviceEnablePeerAccess(1, 0);
  cudaMemset(a0, 1, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int grid : {148, 296, 592, 1184}) {
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0); push_st<<<grid, 512>>>(a0, a1, N); cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1); printf("push  st.128  grid %5d: %7.1f GB/s\n", grid, bytes / ms / 1e6);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0); pull_ld<<<grid, 512>>>(a1, b0, N); cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1); printf("pull  ld.128  grid %5d: %7.1f GB/s\n", grid, bytes / ms / 1e6);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0); push_bulk<<<grid, 256>>>(a0, a1, N); cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1); printf("push  bulk    grid %5d: %7.1f GB/s  (%s)\n", grid, bytes / ms / 1e6,
                                              cudaGetErrorString(cudaGetLastError()));
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); cudaMemcpyPeerAsync(a1, 1, a0, 0, bytes); cudaEventRecord(e1); cudaEventSynchronize(e1);
  }
  float ms; cudaEventElapsedTime(&ms, e0, e1); printf("cudaMemcpyPeer        : %7.1f GB/s\n", bytes / ms / 1e6);
  // small transfers: 8 MB like one dispatch of C2 at P=2
  const size_t sb = 8ull << 20;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); push_st<<<1184, 512>>>(a0, a1, sb / 16); cudaEventRecord(e1); cudaEventSynchronize(e1);
  }
  cudaEventElapsedTime(&ms, e0, e1); printf("push st.128 8 MB       : %7.1f GB/s (%.1f us)\n", sb / ms / 1e6, ms * 1e3);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); pull_ld<<<1184, 512>>>(a1, b0, sb / 16); cudaEventRecord(e1); cudaEventSynchronize(e1);
  }
  cudaEventElapsedTime(&ms, e0, e1); printf("pull ld.128 8 MB       : %7.1f GB/s (%.1f us)\n", sb / ms / 1e6, ms * 1e3);
  return 0;
}
