// sm_100a kernels of the PAM sweep (first generation: tiled SIMT, fixed-order
// split-K reductions).  See DESIGN.md for each kernel's roofline.
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

// ============================================================ K2 stream

StreamPlan plan_stream(int64_t I, int64_t S, int64_t p, int target_ctas) {
  StreamPlan sp;
  sp.ts = S <= 16 ? 16 : S <= 32 ? 32 : S <= 64 ? 64 : 128;
  sp.ti = 4096 / sp.ts;
  sp.n_itiles = (int)((I + sp.ti - 1) / sp.ti);
  int64_t want = target_ctas / sp.n_itiles;
  if (want < 1) want = 1;
  int64_t max_split = (p + 63) / 64;  // at least 64 columns per split
  if (want > max_split) want = max_split;
  if (want < 1) want = 1;
  int64_t chunk = (p + want - 1) / want;
  chunk = (chunk + 15) / 16 * 16;
  sp.chunk = chunk;
  sp.nsplit = (int)((p + chunk - 1) / chunk);
  if (sp.nsplit < 1) sp.nsplit = 1;
  return sp;
}

template <typename T, int TS, bool XFAST>
__global__ void __launch_bounds__(256) k_stream(const T* __restrict__ X, const T* __restrict__ M,
                                                double* __restrict__ part, int64_t I, int64_t P, int64_t S,
                                                int64_t p, int64_t chunk) {
  constexpr int TI = 4096 / TS;
  constexpr int PC = 16;
  constexpr int NTS = TS / 4;  // threads along s
  __shared__ T Xs[PC][TI + 1];
  __shared__ T Ms[PC][TS + 1];
  const int tid = threadIdx.x;
  const int ts = tid % NTS, ti = tid / NTS;
  const int64_t i0 = (int64_t)blockIdx.x * TI;
  const int64_t split = blockIdx.y;
  const int64_t pb = split * chunk;
  int64_t pe = pb + chunk;
  if (pe > p) pe = p;
  const int64_t PI = P * I;
  T acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = T(0);
  for (int64_t p0 = pb; p0 < pe; p0 += PC) {
    for (int e = tid; e < PC * TI; e += 256) {
      int i, pp;
      if (XFAST) {
        i = e % TI;
        pp = e / TI;
      } else {
        pp = e % PC;
        i = e / PC;
      }
      int64_t gp = p0 + pp, gi = i0 + i;
      T v = T(0);
      if (gp < pe && gi < I) {
        int64_t off = XFAST ? gi + I * gp : (gp % P) + P * gi + PI * (gp / P);
        v = X[off];
      }
      Xs[pp][i] = v;
    }
    for (int e = tid; e < PC * TS; e += 256) {
      int s = e % TS, pp = e / TS;
      int64_t gp = p0 + pp;
      T v = T(0);
      if (gp < pe && s < S) v = M[s + S * gp];
      Ms[pp][s] = v;
    }
    __syncthreads();
#pragma unroll
    for (int pp = 0; pp < PC; ++pp) {
      T xv[4], mv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) xv[a] = Xs[pp][ti + (TI / 4) * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) mv[b] = Ms[pp][ts + NTS * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] += xv[a] * mv[b];
    }
    __syncthreads();
  }
  double* out = part + split * I * S;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    int64_t gi = i0 + ti + (TI / 4) * a;
    if (gi >= I) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      int64_t s = ts + NTS * b;
      if (s < S) out[gi + I * s] = (double)acc[a][b];
    }
  }
}

template <typename T, int TS>
static void stream_dispatch_fast(const T* X, const T* M, double* part, int64_t I, int64_t P, int64_t S,
                                 int64_t p, const StreamPlan& sp, cudaStream_t st) {
  dim3 grid(sp.n_itiles, sp.nsplit);
  if (P == 1)
    k_stream<T, TS, true><<<grid, 256, 0, st>>>(X, M, part, I, P, S, p, sp.chunk);
  else
    k_stream<T, TS, false><<<grid, 256, 0, st>>>(X, M, part, I, P, S, p, sp.chunk);
}

template <typename T>
void launch_stream(const T* X, const T* M, double* part, int64_t I, int64_t P, int64_t S, int64_t p,
                   const StreamPlan& sp, cudaStream_t st) {
  switch (sp.ts) {
    case 16: stream_dispatch_fast<T, 16>(X, M, part, I, P, S, p, sp, st); break;
    case 32: stream_dispatch_fast<T, 32>(X, M, part, I, P, S, p, sp, st); break;
    case 64: stream_dispatch_fast<T, 64>(X, M, part, I, P, S, p, sp, st); break;
    default: stream_dispatch_fast<T, 128>(X, M, part, I, P, S, p, sp, st); break;
  }
  check_launch("stream");
}
template void launch_stream<double>(const double*, const double*, double*, int64_t, int64_t, int64_t, int64_t,
                                    const StreamPlan&, cudaStream_t);
template void launch_stream<float>(const float*, const float*, double*, int64_t, int64_t, int64_t, int64_t,
                                   const StreamPlan&, cudaStream_t);

__global__ void k_reduce_y(const double* __restrict__ part, int nsplit, int64_t IS,
                           const double* __restrict__ aprev, double rho, double* __restrict__ Y) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < IS; e += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int s = 0; s < nsplit; ++s) acc += part[s * IS + e];
    Y[e] = acc + rho * aprev[e];
  }
}

void launch_reduce_y(const double* part, int nsplit, int64_t I, int64_t S, const double* aprev, double rho,
                     double* Y, cudaStream_t st) {
  int64_t n = I * S;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_reduce_y<<<(unsigned)blocks, 256, 0, st>>>(part, nsplit, n, aprev, rho, Y);
  check_launch("reduce_y");
}

__global__ void k_reduce_g(const double* __restrict__ part, int nsplit, int64_t S, double* __restrict__ G) {
  int64_t SS = S * S;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < SS; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = e % S, b = e / S;
    double x = 0.0, y = 0.0;
    for (int s = 0; s < nsplit; ++s) {
      x += part[s * SS + a + S * b];
      y += part[s * SS + b + S * a];
    }
    G[e] = 0.5 * (x + y);
  }
}

void launch_reduce_g(const double* part, int nsplit, int64_t S, double* G, cudaStream_t st) {
  int64_t n = S * S;
  int64_t blocks = (n + 255) / 256;
  k_reduce_g<<<(unsigned)blocks, 256, 0, st>>>(part, nsplit, S, G);
  check_launch("reduce_g");
}

// ============================================================ K3 solve

__global__ void k_dft_fwd(const double* __restrict__ Y, int64_t I, int64_t S, int64_t H1,
                          const double* __restrict__ cosT, const double* __restrict__ sinT,
                          double* __restrict__ Fr, double* __restrict__ Fi) {
  int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t s = blockIdx.y;
  if (w >= H1) return;
  const double* y = Y + I * s;
  double cr = 0.0, ci = 0.0;
  int64_t idx = 0;
  for (int64_t j = 0; j < I; ++j) {
    double v = y[j];
    cr += v * cosT[idx];
    ci += v * sinT[idx];
    idx += w;
    if (idx >= I) idx -= I;
  }
  Fr[w + H1 * s] = cr;
  Fi[w + H1 * s] = ci;
}

void launch_dft_fwd(const double* Y, int64_t I, int64_t S, const double* cosT, const double* sinT, double* Fr,
                    double* Fi, cudaStream_t st) {
  int64_t H1 = I / 2 + 1;
  dim3 grid((unsigned)((H1 + 127) / 128), (unsigned)S);
  k_dft_fwd<<<grid, 128, 0, st>>>(Y, I, S, H1, cosT, sinT, Fr, Fi);
  check_launch("dft_fwd");
}

// One CTA per frequency: Cholesky of H = G + mu I (row-major in smem), then
// two triangular solves for the cosine and sine right-hand sides.  The CTA
// with blockIdx.x == H1 (if present) only factorises G + check_mu I.
__global__ void __launch_bounds__(256) k_chol_solve(const double* __restrict__ G, int64_t S, int64_t H1,
                                                    const double* __restrict__ mu, double* __restrict__ Fr,
                                                    double* __restrict__ Fi, double check_mu,
                                                    int* __restrict__ status) {
  extern __shared__ double sm[];
  double* L = sm;
  double* b0 = sm + S * S;
  double* b1 = b0 + S;
  __shared__ int bad;
  const int tid = threadIdx.x;
  const int64_t w = blockIdx.x;
  const bool is_check = (w == H1);
  const double shift = is_check ? check_mu : mu[w];
  if (tid == 0) bad = 0;
  for (int64_t e = tid; e < S * S; e += blockDim.x) {
    int64_t i = e / S, j = e % S;
    double v = G[i + S * j];
    if (i == j) v += shift;
    L[e] = v;
  }
  if (!is_check)
    for (int64_t i = tid; i < S; i += blockDim.x) {
      b0[i] = Fr[w + H1 * i];
      b1[i] = Fi[w + H1 * i];
    }
  __syncthreads();
  for (int64_t k = 0; k < S; ++k) {
    if (tid == 0) {
      double d = L[k * S + k];
      if (!(d > 0.0) || !isfinite(d)) {
        bad = 1;
        d = 1.0;
      }
      L[k * S + k] = sqrt(d);
    }
    __syncthreads();
    const double dk = L[k * S + k];
    for (int64_t i = k + 1 + tid; i < S; i += blockDim.x) L[i * S + k] /= dk;
    __syncthreads();
    const int64_t m = S - k - 1;
    for (int64_t e = tid; e < m * m; e += blockDim.x) {
      int64_t i = k + 1 + e / m, j = k + 1 + e % m;
      if (j <= i) L[i * S + j] -= L[i * S + k] * L[j * S + k];
    }
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) atomicOr(status, is_check ? 1 : 2);
    return;
  }
  if (is_check) return;
  for (int64_t k = 0; k < S; ++k) {  // L z = b
    if (tid == 0) {
      b0[k] /= L[k * S + k];
      b1[k] /= L[k * S + k];
    }
    __syncthreads();
    for (int64_t i = k + 1 + tid; i < S; i += blockDim.x) {
      b0[i] -= L[i * S + k] * b0[k];
      b1[i] -= L[i * S + k] * b1[k];
    }
    __syncthreads();
  }
  for (int64_t k = S - 1; k >= 0; --k) {  // L^T x = z
    if (tid == 0) {
      b0[k] /= L[k * S + k];
      b1[k] /= L[k * S + k];
    }
    __syncthreads();
    for (int64_t i = tid; i < k; i += blockDim.x) {
      b0[i] -= L[k * S + i] * b0[k];
      b1[i] -= L[k * S + i] * b1[k];
    }
    __syncthreads();
  }
  for (int64_t i = tid; i < S; i += blockDim.x) {
    Fr[w + H1 * i] = b0[i];
    Fi[w + H1 * i] = b1[i];
  }
}

void launch_chol_solve(const double* G, int64_t S, int64_t H1, const double* mu, double* Fr, double* Fi,
                       double check_mu, int* status, cudaStream_t st) {
  size_t smem = (size_t)(S * S + 2 * S) * sizeof(double);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_chol_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  unsigned blocks = (unsigned)H1 + (isfinite(check_mu) ? 1u : 0u);
  k_chol_solve<<<blocks, 256, smem, st>>>(G, S, H1, mu, Fr, Fi, check_mu, status);
  check_launch("chol_solve");
}

template <typename T>
__global__ void k_dft_inv(const double* __restrict__ Fr, const double* __restrict__ Fi, int64_t I, int64_t S,
                          int64_t H1, const double* __restrict__ cosT, const double* __restrict__ sinT,
                          const double* __restrict__ Aold, double* __restrict__ Anew, T* __restrict__ Ac,
                          int extrap, double alpha, double beta) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t s = blockIdx.y;
  if (j >= I) return;
  const double* fr = Fr + H1 * s;
  const double* fi = Fi + H1 * s;
  const bool even = (I % 2) == 0;
  const int64_t wmax = even ? I / 2 - 1 : (I - 1) / 2;
  double acc2 = 0.0;
  int64_t idx = 0;
  for (int64_t w = 1; w <= wmax; ++w) {
    idx += j;
    if (idx >= I) idx -= I;
    acc2 += fr[w] * cosT[idx] + fi[w] * sinT[idx];
  }
  double acc = fr[0] + 2.0 * acc2;
  if (even) acc += (j & 1) ? -fr[I / 2] : fr[I / 2];
  double a = acc / (double)I;
  const int64_t e = j + I * s;
  if (extrap) {
    double ao = Aold[e];
    a = a + alpha * (a - beta * ao);
  }
  Anew[e] = a;
  if (Ac) Ac[e] = (T)a;
}

template <typename T>
void launch_dft_inv(const double* Fr, const double* Fi, int64_t I, int64_t S, const double* cosT,
                    const double* sinT, const double* Aold, double* Anew, T* Ac, int extrap, double alpha,
                    double beta, cudaStream_t st) {
  int64_t H1 = I / 2 + 1;
  dim3 grid((unsigned)((I + 127) / 128), (unsigned)S);
  k_dft_inv<T><<<grid, 128, 0, st>>>(Fr, Fi, I, S, H1, cosT, sinT, Aold, Anew, Ac, extrap, alpha, beta);
  check_launch("dft_inv");
}
template void launch_dft_inv<double>(const double*, const double*, int64_t, int64_t, const double*, const double*,
                                     const double*, double*, double*, int, double, double, cudaStream_t);
template void launch_dft_inv<float>(const double*, const double*, int64_t, int64_t, const double*, const double*,
                                    const double*, double*, float*, int, double, double, cudaStream_t);

template <int NT>
__device__ void block_sum3(double* v, double (*sh)[NT]) {
  const int tid = threadIdx.x;
  for (int q = 0; q < 3; ++q) sh[q][tid] = v[q];
  __syncthreads();
  for (int off = NT / 2; off > 0; off >>= 1) {
    if (tid < off)
      for (int q = 0; q < 3; ++q) sh[q][tid] += sh[q][tid + off];
    __syncthreads();
  }
  for (int q = 0; q < 3; ++q) v[q] = sh[q][0];
}

__global__ void __launch_bounds__(256) k_factor_stats(const double* __restrict__ A, const double* __restrict__ Ao,
                                                      int64_t I, int64_t S, double delta, double sgn,
                                                      double* __restrict__ out) {
  __shared__ double sh[3][256];
  double v[3] = {0.0, 0.0, 0.0};
  const int64_t n = I * S;
  for (int64_t e = threadIdx.x; e < n; e += 256) {
    int64_t j = e % I, s = e / I;
    double a = A[e];
    double d = a - Ao[e];
    int64_t jm = (j == 0) ? I - 1 : j - 1;
    int64_t jp = (j == I - 1) ? 0 : j + 1;
    double la = sgn * ((-2.0 - delta) * a + A[jm + I * s] + A[jp + I * s]);
    v[0] += d * d;
    v[1] += a * a;
    v[2] += a * la;
  }
  block_sum3<256>(v, sh);
  if (threadIdx.x == 0) {
    out[0] = v[0];
    out[1] = v[1];
    out[2] = v[2];
  }
}

void launch_factor_stats(const double* Anew, const double* Aold, int64_t I, int64_t S, double delta, double sgn,
                         double* out, cudaStream_t st) {
  k_factor_stats<<<1, 256, 0, st>>>(Anew, Aold, I, S, delta, sgn, out);
  check_launch("factor_stats");
}

// ============================================================ K4 compose

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
  T acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = T(0);
  for (int64_t s0 = 0; s0 < S; s0 += KC) {
    for (int e = tid; e < KC * TI; e += 256) {
      int i = e % TI, kk = e / TI;
      int64_t gi = i0 + i, gs = s0 + kk;
      As[kk][i] = (gi < I && gs < S) ? A[gi + I * gs] : T(0);
    }
    for (int e = tid; e < KC * PC; e += 256) {
      int kk = e % KC, pp = e / KC;
      int64_t gp = p0 + pp, gs = s0 + kk;
      Ms[kk][pp] = (gp < p && gs < S) ? M[gs + S * gp] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      T av[4], mv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[kk][(XFAST ? tx : ty) + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) mv[b] = Ms[kk][(XFAST ? ty : tx) + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] += av[a] * mv[b];
    }
    __syncthreads();
  }
  double s_d = 0.0, s_b = 0.0, s_c = 0.0, s_n = 0.0;
  const T r = (T)rho;
  const T inv = (T)(1.0 + rho);
  const int64_t PI = P * I;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    int64_t gi = i0 + (XFAST ? tx : ty) + 16 * a;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      int64_t gp = p0 + (XFAST ? ty : tx) + 16 * b;
      if (gi >= I || gp >= p) continue;
      int64_t off = XFAST ? gi + I * gp : (gp % P) + P * gi + PI * (gp / P);
      T x = Xo[off];
      T c = acc[a][b];
      if (objective_only) {
        double d = (double)x - (double)c;
        s_c += d * d;
      } else {
        T xn;
        if (mask[off]) {
          xn = x;  // observed entries restored bit for bit (solver.py:235-236)
        } else {
          // (x*rho + c)/(1+rho) in the reference's operation order (solver.py:232-234)
          T t = x * r;
          t = t + c;
          xn = t / inv;
        }
        Xn[off] = xn;
        double dx = (double)xn - (double)x;
        double dc = (double)xn - (double)c;
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
                   int64_t S, int64_t p, double rho, bool objective_only, double* partials,
                   int64_t partial_cap, cudaStream_t st) {
  int64_t ti = (I + 63) / 64, tp = (p + 63) / 64;
  int64_t blocks = ti * tp;
  if (blocks > partial_cap) throw std::runtime_error("compose partial buffer too small");
  if (P == 1)
    k_compose<T, true><<<(unsigned)blocks, 256, 0, st>>>(A, M, Xo, mask, Xn, I, P, S, p, rho, objective_only,
                                                           ti, partials);
  else
    k_compose<T, false><<<(unsigned)blocks, 256, 0, st>>>(A, M, Xo, mask, Xn, I, P, S, p, rho, objective_only,
                                                            ti, partials);
  check_launch("compose");
  return (int)blocks;
}
template int launch_compose<double>(const double*, const double*, const double*, const uint8_t*, double*, int64_t,
                                    int64_t, int64_t, int64_t, double, bool, double*, int64_t, cudaStream_t);
template int launch_compose<float>(const float*, const float*, const float*, const uint8_t*, float*, int64_t,
                                   int64_t, int64_t, int64_t, double, bool, double*, int64_t, cudaStream_t);

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

void launch_reduce4(const double* partials, int64_t n, double* out, cudaStream_t st) {
  k_reduce4<<<1, 1024, 0, st>>>(partials, n, out);
  check_launch("reduce4");
}

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
