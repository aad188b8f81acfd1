// K4 (SIMT path): C = A_(k) M_k (network.py:313-332) fused with the P_Omega
// blend (solver.py:227-237) and the sweep reductions (solver.py:220,346-354,
// 382).  C never touches HBM: each CTA computes a TI x PC tile of C in
// registers, blends it with X_old, writes X_new and emits four fixed-order
// partial sums.  M_k is p-fastest (M[p + pk s]).
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <string>

#include "kernels.cuh"

namespace fctn {

// separately rounded multiply / add / divide (no FMA contraction)
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }

static void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T, bool XFAST>
__global__ void __launch_bounds__(256) k_compose(const T* __restrict__ A, const T* __restrict__ M,
                                                 const T* __restrict__ Xo, const uint8_t* __restrict__ mask,
                                                 T* __restrict__ Xn, int64_t I, int64_t P, int64_t S, int64_t p,
                                                 double rho, int objective_only, int64_t tiles_i,
                                                 double* __restrict__ partials) {
  constexpr int TI = 64, PC = 64, KC = 16;
  __shared__ T As[KC][TI + 1];
  __shared__ T Ms[KC][PC + 1];
  __shared__ double red[4][256];
  const int tid = threadIdx.x;
  const int64_t i0 = (blockIdx.x % tiles_i) * TI;
  const int64_t p0 = (blockIdx.x / tiles_i) * PC;
  const int tx = tid & 15, ty = tid >> 4;
  // the fastest-varying thread index walks the contiguous axis of X_(k)
  const int ti = XFAST ? tx : ty, tp = XFAST ? ty : tx;
  T acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = T(0);
  for (int64_t s0 = 0; s0 < S; s0 += KC) {
    for (int e = tid; e < KC * TI; e += 256) {
      const int i = e % TI, kk = e / TI;
      const int64_t gi = i0 + i, gs = s0 + kk;
      As[kk][i] = (gi < I && gs < S) ? A[gi + I * gs] : T(0);
    }
    for (int e = tid; e < KC * PC; e += 256) {
      const int pp = e % PC, kk = e / PC;
      const int64_t gp = p0 + pp, gs = s0 + kk;
      Ms[kk][pp] = (gp < p && gs < S) ? M[gp + p * gs] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      T av[4], mv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[kk][ti + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) mv[b] = Ms[kk][tp + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] += av[a] * mv[b];
    }
    __syncthreads();
  }
  double s_d = 0.0, s_b = 0.0, s_c = 0.0, s_n = 0.0;
  const T r = (T)rho;
  const T onep = (T)(1.0 + rho);
  const int64_t PI = P * I;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t gi = i0 + ti + 16 * a;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t gp = p0 + tp + 16 * b;
      if (gi >= I || gp >= p) continue;
      const int64_t off = XFAST ? gi + I * gp : (gp % P) + P * gi + PI * (gp / P);
      const T x = Xo[off];
      const T c = acc[a][b];
      if (objective_only) {
        const double d = (double)x - (double)c;
        s_c += d * d;
      } else {
        T xn;
        if (mask[off]) {
          xn = x;  // observed entries restored bit for bit (solver.py:235-236)
        } else {
          // (x*rho + c)/(1+rho) in the reference's operation order and
          // rounding (solver.py:232-234: multiply, add, divide, each rounded;
          // the _rn intrinsics keep nvcc from contracting them into an FMA)
          xn = div_rn(add_rn(mul_rn(x, r), c), onep);
        }
        Xn[off] = xn;
        const double dx = (double)xn - (double)x;
        const double dc = (double)xn - (double)c;
        s_d += dx * dx;
        s_b += (double)x * (double)x;
        s_c += dc * dc;
        s_n += (double)xn * (double)xn;
      }
    }
  }
  red[0][tid] = s_d;
  red[1][tid] = s_b;
  red[2][tid] = s_c;
  red[3][tid] = s_n;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if (tid < off)
      for (int q = 0; q < 4; ++q) red[q][tid] += red[q][tid + off];
    __syncthreads();
  }
  if (tid < 4) partials[blockIdx.x * 4 + tid] = red[tid][0];
}

template <typename T>
int launch_compose(const T* A, const T* M, const T* Xo, const uint8_t* mask, T* Xn, int64_t I, int64_t P,
                   int64_t S, int64_t p, double rho, bool objective_only, double* partials, int64_t partial_cap,
                   cudaStream_t st) {
  const int64_t ti = (I + 63) / 64, tp = (p + 63) / 64;
  const int64_t blocks = ti * tp;
  if (blocks > partial_cap) throw std::runtime_error("compose partial buffer too small");
  if (P == 1)
    k_compose<T, true><<<(unsigned)blocks, 256, 0, st>>>(A, M, Xo, mask, Xn, I, P, S, p, rho, objective_only, ti,
                                                           partials);
  else
    k_compose<T, false><<<(unsigned)blocks, 256, 0, st>>>(A, M, Xo, mask, Xn, I, P, S, p, rho, objective_only, ti,
                                                            partials);
  check_launch("compose");
  return (int)blocks;
}
template int launch_compose<double>(const double*, const double*, const double*, const uint8_t*, double*, int64_t,
                                    int64_t, int64_t, int64_t, double, bool, double*, int64_t, cudaStream_t);
template int launch_compose<float>(const float*, const float*, const float*, const uint8_t*, float*, int64_t,
                                   int64_t, int64_t, int64_t, double, bool, double*, int64_t, cudaStream_t);

// Fixed-order final reduction of n x 4 partials: 1024 threads stride the
// partials, then a tree in smem.
__global__ void __launch_bounds__(1024) k_reduce4(const double* __restrict__ part, int64_t n,
                                                  double* __restrict__ out) {
  __shared__ double red[4][1024];
  const int tid = threadIdx.x;
  double v[4] = {0, 0, 0, 0};
  for (int64_t e = tid; e < n; e += 1024)
    for (int q = 0; q < 4; ++q) v[q] += part[e * 4 + q];
  for (int q = 0; q < 4; ++q) red[q][tid] = v[q];
  __syncthreads();
  for (int off = 512; off > 0; off >>= 1) {
    if (tid < off)
      for (int q = 0; q < 4; ++q) red[q][tid] += red[q][tid + off];
    __syncthreads();
  }
  if (tid < 4) out[tid] = red[tid][0];
}

// The P_Omega blend of an already formed C (compose through the partials,
// fctn_ctx.cu compose_via_partials): X_new = Omega ? X_old : (rho X_old + C) /
// (1 + rho) in the reference's rounding, and the same four per-block sums as
// k_compose (solver.py:220,227-237,346-354,382).
__global__ void __launch_bounds__(256) k_blend(const double* __restrict__ C, const double* __restrict__ Xo,
                                               const uint8_t* __restrict__ mask, double* __restrict__ Xn,
                                               int64_t T, double r, double* __restrict__ partials) {
  __shared__ double red[4][256];
  const int tid = threadIdx.x;
  const double onep = 1.0 + r;
  double s_d = 0.0, s_b = 0.0, s_c = 0.0, s_n = 0.0;
  for (int64_t e = blockIdx.x * 256LL + tid; e < T; e += (int64_t)gridDim.x * 256) {
    const double x = Xo[e], c = C[e];
    const double xn = mask[e] ? x : div_rn(add_rn(mul_rn(x, r), c), onep);
    Xn[e] = xn;
    const double dx = xn - x, dc = xn - c;
    s_d += dx * dx;
    s_b += x * x;
    s_c += dc * dc;
    s_n += xn * xn;
  }
  red[0][tid] = s_d;
  red[1][tid] = s_b;
  red[2][tid] = s_c;
  red[3][tid] = s_n;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if (tid < off)
      for (int q = 0; q < 4; ++q) red[q][tid] += red[q][tid + off];
    __syncthreads();
  }
  if (tid < 4) partials[blockIdx.x * 4 + tid] = red[tid][0];
}

int launch_blend(const double* C, const double* Xo, const uint8_t* mask, double* Xn, int64_t T, double rho,
                 double* partials, int64_t partial_cap, cudaStream_t st) {
  const int64_t blocks = std::min<int64_t>(std::min<int64_t>((T + 255) / 256, 148 * 8), partial_cap);
  k_blend<<<(unsigned)blocks, 256, 0, st>>>(C, Xo, mask, Xn, T, rho, partials);
  check_launch("blend");
  return (int)blocks;
}

void launch_reduce4(const double* partials, int64_t n, double* out, cudaStream_t st) {
  k_reduce4<<<1, 1024, 0, st>>>(partials, n, out);
  check_launch("reduce4");
}

}  // namespace fctn
