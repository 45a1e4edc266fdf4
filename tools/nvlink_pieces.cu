// NVLink remote-store bandwidth vs. contiguous piece size per destination row (the fused-exchange epilogues
// write each output row as pieces of 64 B (4 lanes x 16 B, 8 rows per warp instruction)).  2 GPUs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/nvp tools/nvlink_pieces.cu && /tmp/nvp
#include <cstdio>
#include <cuda_runtime.h>

// rows of 2 KB; each warp instruction stores PIECE bytes to each of 512 / PIECE rows (scattered row order)
template <int PIECE>
__global__ void pieces(const uint4* __restrict__ src, uint4* __restrict__ dst, int rows, const int* __restrict__ perm) {
  constexpr int LPR = PIECE / 16;  // lanes per row
  constexpr int RPI = 32 / LPR;    // rows per instruction
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w * RPI < rows; w += warps) {
    const int r = w * RPI + lane / LPR;
    const int dr = perm[r];
    for (int c = (lane % LPR); c < 128; c += LPR)  // 128 x 16 B = 2 KB row
      dst[(size_t)dr * 128 + c] = src[(size_t)r * 128 + c];
  }
}

int main() {
  int n = 0;
  cudaGetDeviceCount(&n);
  if (n < 2) { printf("need 2 GPUs\n"); return 0; }
  const int rows = 8192;  // 16 MB
  const size_t bytes = (size_t)rows * 2048;
  uint4 *a0, *a1;
  int* perm;
  cudaSetDevice(1); cudaMalloc(&a1, bytes); cudaDeviceEnablePeerAccess(0, 0);
  cudaSetDevice(0); cudaMalloc(&a0, bytes); cudaDeviceEnablePeerAccess(1, 0);
  cudaMalloc(&perm, rows * sizeof(int));
  int* h = new int[rows];
  for (int i = 0; i < rows; ++i) h[i] = (int)(((long long)i * 2654435761LL) % rows);  // scattered, bijective-ish
  for (int i = 0; i < rows; ++i) h[i] = (i * 4099) % rows;                           // bijective (4099 odd prime)
  cudaMemcpy(perm, h, rows * sizeof(int), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
#define RUN(P, DST)                                                                              \
  for (int rep = 0; rep < 3; ++rep) {                                                            \
    cudaEventRecord(e0); pieces<P><<<1184, 256>>>(a0, DST, rows, perm); cudaEventRecord(e1);     \
    cudaEventSynchronize(e1);                                                                    \
  }                                                                                              \
  cudaEventElapsedTime(&ms, e0, e1);                                                             \
  printf("%-6s piece %4d B: %7.1f GB/s (%.1f us for 16 MB)\n", #DST, P, bytes / ms / 1e6, ms * 1e3);
  RUN(64, a1) RUN(128, a1) RUN(256, a1) RUN(512, a1)
  uint4* l0; cudaMalloc(&l0, bytes);
  RUN(64, l0) RUN(512, l0)
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
