// SIMT grouped GEMMs over expert segments: exact fp32 FFMA.  This is the fp32 path of the expert FFN
// (fp32 configs must not use tf32 tensor cores: the 1e-4 bound) and the reference
// shape of the tcgen05 kernels in gemm_tc.cu (same layouts, same fused epilogues).
#include "common.cuh"
#include "exchange.cuh"

namespace luffy {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;

template <typename T>
__device__ __forceinline__ void store1(T* p, float v) { *p = from_f<T>(v); }

// Thread (ty, tx) owns rows ty*4 + i and tile columns {2tx, 2tx+1, 32+2tx, 33+2tx} (so that SwiGLU's
// pre1/pre3 pairs land in one thread).
__device__ __forceinline__ int tcol(int tx, int j) { return (j < 2 ? 2 * tx + j : 32 + 2 * tx + (j - 2)); }

template <typename T, int EPI>
__global__ void __launch_bounds__(256) gemm_rows_kernel(const T* __restrict__ A, const T* __restrict__ B,
                                                        const T* __restrict__ B3, T* __restrict__ D, T* __restrict__ aux0,
                                                        const int32_t* __restrict__ off, int G, int N, int K, int bkm,
                                                        XRedirect rd, int has_rd, XSignal sig, int has_sig) {
  pdl_enter();
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int64_t row0 = (int64_t)blockIdx.y * BM;
  const int32_t rows = off[G];
  if (row0 >= rows) {
    if (has_sig) xsignal_done(sig);
    return;
  }
  const int g = find_group(off, G, row0);
  // Column mapping.  SWIGLU: f = N / 2 logical columns, tile covers f-cols [n0, n0+32) of W1 and W3.
  const int f = N / 2;
  const int n0 = EPI == EPI_SWIGLU ? blockIdx.x * 32 : blockIdx.x * BN;
  // B_g base and leading dims.  b_kmajor: B_g is [Nb, K]; else B_g is [K, Nb].
  const int Nb = EPI == EPI_SWIGLU ? f : N;
  // K split over [B; B3] (the SwiGLU input-gradient GEMM d_pre [rows, 2f] x [W1; W3]).
  const bool ksplit = EPI != EPI_SWIGLU && B3 != nullptr;
  const int Kb = ksplit ? K / 2 : K;
  const T* Bg = B + (size_t)g * Nb * Kb;
  const T* B3g = B3 ? B3 + (size_t)g * Nb * Kb : nullptr;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += BK) {
    for (int i = threadIdx.x; i < BM * BK; i += 256) {
      const int r = i / BK, kk = i % BK;
      As[kk][r] = to_f(A[(row0 + r) * K + k0 + kk]);
    }
    for (int i = threadIdx.x; i < BN * BK; i += 256) {
      int c, kk;
      if (bkm) { c = i / BK; kk = i % BK; } else { kk = i / BN; c = i % BN; }
      const int kg = k0 + kk;
      float v;
      if (EPI == EPI_SWIGLU) {
        const int nf = n0 + (c & 31);
        const T* src = c < 32 ? Bg : B3g;
        v = to_f(src[(size_t)nf * Kb + kg]);  // W1/W3 are [f, d] = [Nb, K] (K-major)
      } else if (ksplit) {
        const T* src = kg < Kb ? Bg : B3g;
        const int kl = kg < Kb ? kg : kg - Kb;
        const int n = n0 + c;
        v = bkm ? to_f(src[(size_t)n * Kb + kl]) : to_f(src[(size_t)kl * Nb + n]);
      } else {
        const int n = n0 + c;
        v = bkm ? to_f(Bg[(size_t)n * Kb + kg]) : to_f(Bg[(size_t)kg * Nb + n]);
      }
      Bs[kk][c] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tcol(tx, j)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = row0 + ty * 4 + i;
    if (EPI == EPI_SWIGLU) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int nf = n0 + 2 * tx + j;
        const float p1 = acc[i][j], p3 = acc[i][j + 2];
        store1(aux0 + r * (2 * f) + nf, p1);
        store1(aux0 + r * (2 * f) + f + nf, p3);
        store1(D + r * f + nf, silu_f(p1) * p3);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = n0 + tcol(tx, j);
        const float v = acc[i][j];
        if (EPI == EPI_STORE) {
          if (has_rd) {
            if (rd.mask) {
              unsigned long long m = rd.mask[r];
              const size_t r2 = (size_t)rd.rank_of[r] * rd.stride + rd.slot_of[r];
              while (m) {
                const int g = __ffsll((long long)m) - 1;
                m &= m - 1;
                store1(static_cast<T*>(rd.peer_base[g]) + r2 * N + n, v);
              }
            } else {
              const int rk = rd.rank_of[r];
              if (rk >= 0) store1(static_cast<T*>(rd.peer_base[rk]) + (size_t)rd.slot_of[r] * N + n, v);
            }
          } else {
            store1(D + r * N + n, v);
          }
        } else if (EPI == EPI_GELU) {
          float g, dg;
          gelu_and_grad_f(v, g, dg);
          store1(aux0 + r * N + n, dg);  // saved for the backward: GeLU'(pre)
          store1(D + r * N + n, g);
        } else if (EPI == EPI_DGELU) {
          store1(D + r * N + n, v * to_f(aux0[r * N + n]));
        } else {  // EPI_DSWIGLU: v = d_act[r, n], N = f
          const float p1 = to_f(aux0[r * (2 * N) + n]), p3 = to_f(aux0[r * (2 * N) + N + n]);
          store1(D + r * (2 * N) + n, v * p3 * silu_grad_f(p1));
          store1(D + r * (2 * N) + N + n, v * silu_f(p1));
        }
      }
    }
  }
  if (has_sig) xsignal_done(sig);
}

// D_g[m, n] = sum_{r in segment g} A[r, m] * B[r, n], fp32 output; rows m >= Msplit go to D3.
template <typename T>
__global__ void __launch_bounds__(256) gemm_wgrad_kernel(const T* __restrict__ A, const T* __restrict__ B,
                                                         float* __restrict__ D, float* __restrict__ D3, int Msplit,
                                                         const int32_t* __restrict__ off, int M, int N, int lda, int ldb) {
  pdl_enter();
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int g = blockIdx.z;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int r0 = off[g], r1 = off[g + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int k0 = r0; k0 < r1; k0 += BK) {
    for (int i = threadIdx.x; i < BM * BK; i += 256) {
      const int kk = i / BM, c = i % BM;
      As[kk][c] = to_f(A[(size_t)(k0 + kk) * lda + m0 + c]);
      Bs[kk][c] = to_f(B[(size_t)(k0 + kk) * ldb + n0 + c]);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tcol(tx, j)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    float* dst = m < Msplit ? D + ((size_t)g * Msplit + m) * N : D3 + ((size_t)g * (M - Msplit) + (m - Msplit)) * N;
#pragma unroll
    for (int j = 0; j < 4; ++j) dst[n0 + tcol(tx, j)] = acc[i][j];
  }
}

template <typename T>
int gemm_rows_t(int epi, const void* A, const void* B, const void* B3, void* D, void* aux0, const int32_t* off, int G,
                int64_t max_rows, int N, int K, int bkm, const XRedirect* rdp, const XSignal* sgp, cudaStream_t s) {
  XRedirect rd{};
  XSignal sg{};
  const int has_rd = rdp != nullptr, has_sig = sgp != nullptr;
  if (rdp) rd = *rdp;
  if (sgp) sg = *sgp;
  dim3 grid(epi == EPI_SWIGLU ? (N / 2) / 32 : N / BN, (unsigned)((max_rows + BM - 1) / BM));
  const T* a = static_cast<const T*>(A);
  const T* b = static_cast<const T*>(B);
  const T* b3 = static_cast<const T*>(B3);
  T* d = static_cast<T*>(D);
  T* x = static_cast<T*>(aux0);
  switch (epi) {
    case EPI_STORE: launch_pdl(gemm_rows_kernel<T, EPI_STORE>, grid, 256, 0, s, a, b, b3, d, x, off, G, N, K, bkm, rd, has_rd, sg, has_sig); break;
    case EPI_GELU: launch_pdl(gemm_rows_kernel<T, EPI_GELU>, grid, 256, 0, s, a, b, b3, d, x, off, G, N, K, bkm, rd, has_rd, sg, has_sig); break;
    case EPI_SWIGLU: launch_pdl(gemm_rows_kernel<T, EPI_SWIGLU>, grid, 256, 0, s, a, b, b3, d, x, off, G, N, K, bkm, rd, has_rd, sg, has_sig); break;
    case EPI_DGELU: launch_pdl(gemm_rows_kernel<T, EPI_DGELU>, grid, 256, 0, s, a, b, b3, d, x, off, G, N, K, bkm, rd, has_rd, sg, has_sig); break;
    default: launch_pdl(gemm_rows_kernel<T, EPI_DSWIGLU>, grid, 256, 0, s, a, b, b3, d, x, off, G, N, K, bkm, rd, has_rd, sg, has_sig); break;
  }
  LUFFY_LAUNCHED();
  return 0;
}

}  // namespace

int gemm_rows_simt(int dtype, int epi, const void* A, const void* B, const void* B3, void* D, void* aux0,
                   const int32_t* off, int G, int64_t max_rows, int N, int K, int b_kmajor, const XRedirect* rd,
                   const XSignal* sig, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  return dtype == LUFFY_BF16 ? gemm_rows_t<bf16>(epi, A, B, B3, D, aux0, off, G, max_rows, N, K, b_kmajor, rd, sig, st)
                             : gemm_rows_t<float>(epi, A, B, B3, D, aux0, off, G, max_rows, N, K, b_kmajor, rd, sig, st);
}

int gemm_wgrad_simt(int dtype, const void* A, const void* B, float* D, float* D3, int Msplit, const int32_t* off, int G,
                    int M, int N, int lda, int ldb, void* s) {
  cudaStream_t st = static_cast<cudaStream_t>(s);
  dim3 grid(N / BN, M / BM, G);
  if (dtype == LUFFY_BF16)
    launch_pdl(gemm_wgrad_kernel<bf16>, grid, 256, 0, st, static_cast<const bf16*>(A), static_cast<const bf16*>(B), D, D3, Msplit,
                                                  off, M, N, lda, ldb);
  else
    launch_pdl(gemm_wgrad_kernel<float>, grid, 256, 0, st, static_cast<const float*>(A), static_cast<const float*>(B), D, D3,
                                                   Msplit, off, M, N, lda, ldb);
  LUFFY_LAUNCHED();
  return 0;
}

}  // namespace luffy
