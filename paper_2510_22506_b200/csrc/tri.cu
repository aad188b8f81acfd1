// K3 with one decomposition of G_k per update (the reference's structure,
// sylvester.py:51-61, 98-116, with its eigendecomposition replaced by a
// tridiagonal one):
//
//   G = Q T Q^T                 Householder tridiagonalisation, one CTA
//   (A Q) (T + mu_w I) = DFT... per frequency w the subproblem
//       a_w (G + mu_w I) = y_w   becomes   a~_w (T + mu_w I) = (y Q)_w,
//   a tridiagonal SPD system solved in O(s) (Thomas), then A = A~ Q^T.
//
// Exact like the eigenbasis form (T and the eigen-diagonal are similar
// matrices), O(s^3) once per update instead of per frequency (the Cholesky
// form factorises H1 = I/2 + 1 shifted copies of G), and the decomposition
// needs only the other factors' Grams, so the context runs it on the side
// stream concurrently with the Y_k pass.  After Y_k the critical path is
// Y Q -> DFT -> per-frequency tridiagonal solves -> inverse DFT -> (.) Q^T.
#include <cuda_runtime.h>

#include <cmath>
#include <stdexcept>
#include <string>

#include "kernels.cuh"

namespace fctn {

static void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {

constexpr int TRI_THREADS = 256;
constexpr int TRI_WARPS = TRI_THREADS / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide fixed-order sum (deterministic); red: TRI_WARPS doubles of smem
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int q = 0; q < TRI_WARPS; ++q) t += red[q];
  return t;
}

// G (S x S, global, symmetric) -> Q (S x S, global), d (S), e (S - 1).
// Shared memory: A (S x LD, LD = S + 1; below the sub-diagonal, column j
// keeps v_j[1..] of reflector j like LAPACK dsytd2), Q (S x S), v / p
// scratch (2 S).
__global__ void __launch_bounds__(TRI_THREADS, 1)
    k_tridiag(const double* __restrict__ G, int S, double* __restrict__ Qg, double* __restrict__ dg,
              double* __restrict__ eg) {
  extern __shared__ double tsm[];
  const int LD = S + 1;
  double* A = tsm;
  double* Q = A + (size_t)S * LD;
  double* v = Q + (size_t)S * S;
  double* pv = v + S;
  double* taus = Q;  // Q is built after the reduction: borrow its first column for tau_j
  __shared__ double red[TRI_WARPS];
  __shared__ double sh_k;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < S * S; e += TRI_THREADS) {
    const int i = e % S, j = e / S;
    A[i + LD * j] = G[e];
  }
  __syncthreads();
  for (int j = 0; j + 2 < S; ++j) {
    const int n = S - j - 1;  // rows / columns j+1 .. S-1; v[0 .. n) <-> rows j+1 ..
    // Householder vector of x = A[j+1:, j] (LAPACK dlarfg)
    double ss = 0.0;
    for (int r = 1 + tid; r < n; r += TRI_THREADS) {
      const double x = A[(j + 1 + r) + LD * j];
      ss = fma(x, x, ss);
    }
    ss = block_sum(ss, red);
    const double alpha = A[(j + 1) + LD * j];
    double tau = 0.0, beta = alpha, scale = 0.0;
    if (ss > 0.0) {
      beta = -copysign(sqrt(fma(alpha, alpha, ss)), alpha);
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    __syncthreads();  // every thread has read alpha before column j is overwritten
    for (int r = tid; r < n; r += TRI_THREADS) {
      const double vr = r == 0 ? 1.0 : A[(j + 1 + r) + LD * j] * scale;
      v[r] = vr;
      if (r > 0) A[(j + 1 + r) + LD * j] = vr;  // kept for the Q accumulation
    }
    if (tid == 0) {
      taus[j] = tau;
      eg[j] = beta;
    }
    __syncthreads();
    if (tau == 0.0) continue;  // uniform: every thread computed the same tau
    // p = tau A22 v
    for (int r = tid; r < n; r += TRI_THREADS) {
      const double* ar = A + (j + 1 + r);
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int c = 0;
      for (; c + 3 < n; c += 4) {
        a0 = fma(ar[LD * (j + 1 + c)], v[c], a0);
        a1 = fma(ar[LD * (j + 2 + c)], v[c + 1], a1);
        a2 = fma(ar[LD * (j + 3 + c)], v[c + 2], a2);
        a3 = fma(ar[LD * (j + 4 + c)], v[c + 3], a3);
      }
      for (; c < n; ++c) a0 = fma(ar[LD * (j + 1 + c)], v[c], a0);
      pv[r] = tau * ((a0 + a1) + (a2 + a3));
    }
    __syncthreads();
    // K = (tau / 2) p . v ; w = p - K v
    double pd = 0.0;
    for (int r = tid; r < n; r += TRI_THREADS) pd = fma(pv[r], v[r], pd);
    pd = block_sum(pd, red);
    if (tid == 0) sh_k = 0.5 * tau * pd;
    __syncthreads();
    const double K = sh_k;
    // A22 -= v w^T + w v^T (both triangles; warps over columns, lanes over rows)
    for (int c = warp; c < n; c += TRI_WARPS) {
      const double vc = v[c], wc = pv[c] - K * vc;
      double* ac = A + (size_t)LD * (j + 1 + c) + (j + 1);
      for (int r = lane; r < n; r += 32) {
        const double vr = v[r], wr = pv[r] - K * vr;
        ac[r] -= fma(vr, wc, wr * vc);
      }
    }
    __syncthreads();
  }
  // T: diagonal and the sub-diagonal of the last 2 x 2 block
  for (int j = tid; j < S; j += TRI_THREADS) dg[j] = A[j + LD * j];
  if (tid == 0 && S >= 2) eg[S - 2] = A[(S - 1) + LD * (S - 2)];
  // Q = H_0 H_1 ... H_{S-3} by backward accumulation (LAPACK dorgtr order)
  __syncthreads();
  for (int j = tid; j + 2 < S; j += TRI_THREADS) pv[j] = taus[j];  // free Q's first column
  __syncthreads();
  for (int j = tid; j + 2 < S; j += TRI_THREADS) v[j] = pv[j];  // taus now live in v
  __syncthreads();
  for (int e = tid; e < S * S; e += TRI_THREADS) Q[e] = (e % S == e / S) ? 1.0 : 0.0;
  double* tv = v;   // tau_j
  double* vb = pv;  // reflector j, contiguous
  __syncthreads();
  for (int j = S - 3; j >= 0; --j) {
    const double tau = tv[j];
    if (tau == 0.0) continue;
    const int n = S - j - 1;
    // reflector j into vb[0 .. n), then u_c into the tail of A's column j
    // (rows <= j of column j are no longer needed: d and e are written)
    for (int r = tid; r < n; r += TRI_THREADS) vb[r] = r == 0 ? 1.0 : A[(j + 1 + r) + LD * j];
    __syncthreads();
    const double* vv = vb;
    double* uu = A + (size_t)LD * (S - 1);  // last column of A: free after the reduction (n <= S - 1)
    // u_c = tau v . Q[j+1:, j+1+c]
    for (int c = warp; c < n; c += TRI_WARPS) {
      const double* qc = Q + (size_t)S * (j + 1 + c) + (j + 1);
      double acc = 0.0;
      for (int r = lane; r < n; r += 32) acc = fma(vv[r], qc[r], acc);
      acc = warp_sum(acc);
      if (lane == 0) uu[c] = tau * acc;
    }
    __syncthreads();
    for (int c = warp; c < n; c += TRI_WARPS) {
      const double uc = uu[c];
      double* qc = Q + (size_t)S * (j + 1 + c) + (j + 1);
      for (int r = lane; r < n; r += 32) qc[r] = fma(-vv[r], uc, qc[r]);
    }
    __syncthreads();
  }
  for (int e = tid; e < S * S; e += TRI_THREADS) Qg[e] = Q[e];
}

// Per frequency w (one thread): (T + mu_w I) x = b for b = the real and the
// imaginary row w of F (F[w + H1 s]), in place.  T SPD + mu_w > 0: Thomas
// elimination without pivoting is stable; a non-positive pivot (non-finite
// input) sets status bit 2 like the Cholesky form.
template <int SMAX>
__global__ void __launch_bounds__(128) k_thomas(const double* __restrict__ d, const double* __restrict__ e, int S,
                                               int64_t H1, const double* __restrict__ mu, double* __restrict__ Fr,
                                               double* __restrict__ Fi, int* __restrict__ status) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= H1) return;
  const double m = mu[w];
  double cp[SMAX];  // c'_s of the elimination (local memory for large s)
  double prev_c = 0.0, prev_r = 0.0, prev_i = 0.0;
  bool bad = false;
  for (int s = 0; s < S; ++s) {
    const double es = s > 0 ? e[s - 1] : 0.0;
    const double piv = d[s] + m - es * prev_c;
    if (!(piv > 0.0) || !isfinite(piv)) bad = true;
    const double inv = 1.0 / piv;
    const double cs = s + 1 < S ? e[s] * inv : 0.0;
    const double br = (Fr[w + H1 * s] - es * prev_r) * inv;
    const double bi = (Fi[w + H1 * s] - es * prev_i) * inv;
    Fr[w + H1 * s] = br;
    Fi[w + H1 * s] = bi;
    cp[s] = cs;
    prev_c = cs;
    prev_r = br;
    prev_i = bi;
  }
  double xr = 0.0, xi = 0.0;
  for (int s = S - 1; s >= 0; --s) {
    xr = Fr[w + H1 * s] - cp[s] * xr;
    xi = Fi[w + H1 * s] - cp[s] * xi;
    Fr[w + H1 * s] = xr;
    Fi[w + H1 * s] = xi;
  }
  if (bad) atomicOr(status, 2);
}

}  // namespace

size_t tridiag_smem_bytes(int64_t S) { return (size_t)(S * (S + 1) + S * S + 2 * S) * sizeof(double); }
bool tridiag_fits_smem(int64_t S) { return S <= 256 && tridiag_smem_bytes(S) <= 220 * 1024; }

void launch_tridiag(const double* G, int64_t S, double* Q, double* d, double* e, cudaStream_t st) {
  if (!tridiag_fits_smem(S)) throw std::runtime_error("tridiag: s too large for the shared-memory form");
  const size_t smem = tridiag_smem_bytes(S);
  if (smem > 48 * 1024) {
    cudaError_t err =
        cudaFuncSetAttribute((const void*)k_tridiag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) throw std::runtime_error(std::string("tridiag smem: ") + cudaGetErrorString(err));
  }
  k_tridiag<<<1, TRI_THREADS, smem, st>>>(G, (int)S, Q, d, e);
  check_launch("tridiag");
}

void launch_thomas(const double* d, const double* e, int64_t S, int64_t H1, const double* mu, double* Fr, double* Fi,
                   int* status, cudaStream_t st) {
  const unsigned blocks = (unsigned)((H1 + 127) / 128);
  if (S <= 64)
    k_thomas<64><<<blocks, 128, 0, st>>>(d, e, (int)S, H1, mu, Fr, Fi, status);
  else if (S <= 128)
    k_thomas<128><<<blocks, 128, 0, st>>>(d, e, (int)S, H1, mu, Fr, Fi, status);
  else
    throw std::runtime_error("thomas: s > 128");
  check_launch("thomas");
}

}  // namespace fctn
