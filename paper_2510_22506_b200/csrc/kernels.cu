// K1: generic labeled contraction (merge of factors / partials into M_k,
// network.py:249-258 over tensor.py:156-200) by offset tables, the generic
// permutation, and the dtype conversion.  See DESIGN.md.
#include <cuda_runtime.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "kernels.cuh"

namespace fctn {

static void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// ============================================================ K1 contract

template <typename T>
__global__ void __launch_bounds__(256) k_contract(const T* __restrict__ A, const T* __restrict__ B,
                                                  T* __restrict__ C, const int64_t* __restrict__ rowA,
                                                  const int64_t* __restrict__ rowC,
                                                  const int64_t* __restrict__ colB,
                                                  const int64_t* __restrict__ colC,
                                                  const int64_t* __restrict__ kA,
                                                  const int64_t* __restrict__ kB, int64_t rows,
                                                  int64_t cols, int64_t K, int64_t tiles_r) {
  constexpr int BR = 64, BC = 64, KC = 16;
  __shared__ T As[KC][BR + 1];
  __shared__ T Bs[KC][BC + 1];
  __shared__ int64_t sRA[BR], sCB[BC];
  const int64_t tile = blockIdx.x;
  const int64_t r0 = (tile % tiles_r) * BR;
  const int64_t c0 = (tile / tiles_r) * BC;
  const int tid = threadIdx.x;
  if (tid < BR) {
    sRA[tid] = (r0 + tid < rows) ? rowA[r0 + tid] : -1;
  } else if (tid < BR + BC) {
    int c = tid - BR;
    sCB[c] = (c0 + c < cols) ? colB[c0 + c] : -1;
  }
  __syncthreads();
  const int tx = tid & 15, ty = tid >> 4;
  T acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = T(0);
  for (int64_t k0 = 0; k0 < K; k0 += KC) {
    for (int e = tid; e < KC * BR; e += 256) {
      int kk = e / BR, r = e % BR;
      int64_t ra = sRA[r];
      T v = T(0);
      if (ra >= 0 && k0 + kk < K) v = A[ra + kA[k0 + kk]];
      As[kk][r] = v;
    }
    for (int e = tid; e < KC * BC; e += 256) {
      int kk = e / BC, c = e % BC;
      int64_t cb = sCB[c];
      T v = T(0);
      if (cb >= 0 && k0 + kk < K) v = B[cb + kB[k0 + kk]];
      Bs[kk][c] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      T av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[kk][tx + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Bs[kk][ty + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] += av[a] * bv[b];
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    int64_t r = r0 + tx + 16 * a;
    if (r >= rows) continue;
    int64_t rc = rowC[r];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      int64_t c = c0 + ty + 16 * b;
      if (c < cols) C[rc + colC[c]] = acc[a][b];
    }
  }
}

template <typename T>
void launch_contract(const T* A, const T* B, T* C, const int64_t* rowA, const int64_t* rowC,
                     const int64_t* colB, const int64_t* colC, const int64_t* kA, const int64_t* kB,
                     int64_t rows, int64_t cols, int64_t K, cudaStream_t st) {
  int64_t tr = (rows + 63) / 64, tc = (cols + 63) / 64;
  int64_t tiles = tr * tc;
  if (tiles <= 0) return;
  k_contract<T><<<(unsigned)tiles, 256, 0, st>>>(A, B, C, rowA, rowC, colB, colC, kA, kB, rows, cols, K, tr);
  check_launch("contract");
}
template void launch_contract<double>(const double*, const double*, double*, const int64_t*, const int64_t*,
                                      const int64_t*, const int64_t*, const int64_t*, const int64_t*, int64_t,
                                      int64_t, int64_t, cudaStream_t);
template void launch_contract<float>(const float*, const float*, float*, const int64_t*, const int64_t*,
                                     const int64_t*, const int64_t*, const int64_t*, const int64_t*, int64_t,
                                     int64_t, int64_t, cudaStream_t);

template <typename T>
__global__ void k_permute(const T* __restrict__ in, T* __restrict__ out, PermDesc d, int64_t numel) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < numel;
       o += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = o, off = 0;
    for (int q = 0; q < d.nd; ++q) {
      int64_t dg = rem % d.ext[q];
      rem /= d.ext[q];
      off += dg * d.in_stride[q];
    }
    out[o] = in[off];
  }
}

template <typename T>
void launch_permute(const T* in, T* out, const PermDesc& d, int64_t numel, cudaStream_t st) {
  if (numel <= 0) return;
  int64_t blocks = (numel + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_permute<T><<<(unsigned)blocks, 256, 0, st>>>(in, out, d, numel);
  check_launch("permute");
}
template void launch_permute<double>(const double*, double*, const PermDesc&, int64_t, cudaStream_t);
template void launch_permute<float>(const float*, float*, const PermDesc&, int64_t, cudaStream_t);

__global__ void k_convert(const double* __restrict__ in, float* __restrict__ out, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = (float)in[e];
}

void launch_convert_f64_f32(const double* in, float* out, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_convert<<<(unsigned)blocks, 256, 0, st>>>(in, out, n);
  check_launch("convert");
}

}  // namespace fctn
