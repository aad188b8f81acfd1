// K3, the reference's own formulation of the factor subproblem
// (sylvester.py:51-61, 98-116):
//
//   G = V diag(phi) V^T            one symmetric eigendecomposition per update
//   T[w, v] = lam Lambda_w + phi_v + rho
//   A = Re(F^H [(F (Y V)) / T]) V^T
//
// Eigendecomposition: two-sided cyclic Jacobi in one CTA on G' = V0^T G V0
// (V0: the previous update's basis for the same mode, identity on the first
// sweep).  Rounds follow the round-robin (circle) order: s/2 disjoint pairs
// (p, q) per round; phase 0 computes every pair's rotation from (g_pp, g_qq,
// g_pq) with one sqrt and one rsqrt (no divisions), phase 1 rotates rows p, q,
// phase 2 columns p, q of G and of V.  A pair is skipped once |g_pq| <=
// s eps sqrt(g_pp g_qq) (the relative criterion under which Jacobi is
// accurate for positive definite matrices); the sweep loop ends when a whole
// sweep rotates nothing.  phi = diag(G) at the end, clamped at 0 like
// sylvester.py:61.  Once the iteration settles, G moves little between
// sweeps, so the warm start needs 1-3 Jacobi sweeps instead of ~8.  Any
// orthonormal eigenbasis gives the same A up to rounding (sign and
// degenerate-rotation invariance of the closed form), so the warm start
// changes no result beyond ~1e-15.
//
// The eigendecomposition depends only on the other factors' Grams, not on
// Y_k, so the context runs it on a side stream concurrently with the Y_k
// pass; the critical path after Y_k is two small GEMMs and two DFTs.
#include <cuda_runtime.h>

#include <algorithm>
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

constexpr int EIGH_THREADS = 1024;
constexpr int EIGH_WARPS = EIGH_THREADS / 32;
constexpr int EIGH_PPW_MAX = 16;  // pairs per warp of the global-memory form: s <= 1024


// pair i of round r in the circle schedule over m (even) indices
__device__ __forceinline__ void rr_pair(int m, int r, int i, int& p, int& q) {
  if (i == 0) {
    p = m - 1;
    q = r;
  } else {
    p = r + i;  // r, i < m - 1: one conditional subtraction instead of a modulo
    if (p >= m - 1) p -= m - 1;
    q = r - i;
    if (q < 0) q += m - 1;
  }
}

// Gs: S x LD (LD = S + 1: row sweeps are bank-conflict free), V: S x S,
// both column-major in shared memory (GLOBAL: in a global scratch, for
// large S).  G: global, symmetric.  Vg in/out (global): warm start / result.
// One warp per pair: every lane computes the pair's rotation from the three
// broadcast entries (no shuffles, no shared rotation table), rotates rows p,
// q with lanes across columns, then -- after one barrier -- columns p, q of G
// and V; a second barrier ends the round.
template <bool GLOBAL, int EIGH_PAIRS_PER_WARP>
__global__ void __launch_bounds__(EIGH_THREADS, 1)
    k_eigh_jacobi(const double* __restrict__ G, int S, double* __restrict__ Vg, double* __restrict__ phi,
                  double* __restrict__ work, int max_sweeps, double tol, double floor_shift,
                  int* __restrict__ status, int* __restrict__ nsweeps) {
  extern __shared__ double esm[];
  const int LD = S + 1;
  double* Gs = GLOBAL ? work : esm;
  double* V = Gs + (size_t)S * LD;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int SS = S * S;
  // G' = V0^T (G V0): W = G V0 into V's buffer, then G' = V0^T W into Gs
  for (int j = warp; j < S; j += EIGH_WARPS)
    for (int r = lane; r < S; r += 32) {
      double acc = 0.0;
      for (int l = 0; l < S; ++l) acc = fma(G[r + (size_t)S * l], Vg[l + (size_t)S * j], acc);
      V[r + S * j] = acc;
    }
  __syncthreads();
  for (int j = warp; j < S; j += EIGH_WARPS)
    for (int i = lane; i < S; i += 32) {
      double acc = 0.0;
      for (int r = 0; r < S; ++r) acc = fma(Vg[r + (size_t)S * i], V[r + S * j], acc);
      Gs[i + LD * j] = acc;
    }
  __syncthreads();
  for (int e = tid; e < SS; e += EIGH_THREADS) V[e] = Vg[e];
  // symmetrise (the two products round differently above and below the diagonal)
  for (int j = warp; j < S; j += EIGH_WARPS)
    for (int i = lane; i < j; i += 32) {
      const double v = 0.5 * (Gs[i + LD * j] + Gs[j + LD * i]);
      Gs[i + LD * j] = v;
      Gs[j + LD * i] = v;
    }
  __syncthreads();
  const int m = S + (S & 1);
  const int npairs = m / 2;
  const double tol2 = tol * tol;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    int rotated = 0;
    for (int r = 0; r < m - 1; ++r) {
      double cs[EIGH_PAIRS_PER_WARP], sn[EIGH_PAIRS_PER_WARP];
      int pp[EIGH_PAIRS_PER_WARP], qq[EIGH_PAIRS_PER_WARP];
#pragma unroll
      for (int u = 0; u < EIGH_PAIRS_PER_WARP; ++u) {
        const int i = warp + EIGH_WARPS * u;
        sn[u] = 0.0;
        cs[u] = 1.0;
        pp[u] = qq[u] = 0;
        if (i >= npairs) continue;
        int p, q;
        rr_pair(m, r, i, p, q);
        if (p >= S || q >= S) continue;
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        pp[u] = p;
        qq[u] = q;
        const double app = Gs[p + LD * p], aqq = Gs[q + LD * q], apq = Gs[p + LD * q];
        if (apq != 0.0 && apq * apq > tol2 * fabs(app * aqq)) {
          // zero g_pq (Golub-Van Loan symSchur2) without divisions:
          // tau = g_qq - g_pp, g2 = 2 g_pq, r = |(tau, g2)|, h = |tau| + r:
          // c = h / |(h, g2)|, s = sign(tau) g2 / |(h, g2)|
          const double tau = aqq - app, g2 = 2.0 * apq;
          const double x = fma(tau, tau, g2 * g2);
          const double rr = x * rsqrt(x);  // x > 0 (g_pq != 0)
          const double h = fabs(tau) + rr;
          const double qn = rsqrt(fma(h, h, g2 * g2));
          cs[u] = h * qn;
          sn[u] = (tau >= 0.0 ? g2 : -g2) * qn;
          rotated = 1;
        }
      }
      // rows p, q of G <- J^T G
#pragma unroll
      for (int u = 0; u < EIGH_PAIRS_PER_WARP; ++u) {
        if (sn[u] == 0.0) continue;
        const int p = pp[u], q = qq[u];
        for (int j = lane; j < S; j += 32) {
          const double gp = Gs[p + LD * j], gq = Gs[q + LD * j];
          Gs[p + LD * j] = cs[u] * gp - sn[u] * gq;
          Gs[q + LD * j] = sn[u] * gp + cs[u] * gq;
        }
      }
      __syncthreads();
      // columns p, q of G and V <- (.) J
#pragma unroll
      for (int u = 0; u < EIGH_PAIRS_PER_WARP; ++u) {
        if (sn[u] == 0.0) continue;
        double* gpc = Gs + LD * pp[u];
        double* gqc = Gs + LD * qq[u];
        double* vp = V + (size_t)S * pp[u];
        double* vq = V + (size_t)S * qq[u];
        for (int j = lane; j < S; j += 32) {
          const double gp = gpc[j], gq = gqc[j];
          gpc[j] = cs[u] * gp - sn[u] * gq;
          gqc[j] = sn[u] * gp + cs[u] * gq;
          const double a = vp[j], b = vq[j];
          vp[j] = cs[u] * a - sn[u] * b;
          vq[j] = sn[u] * a + cs[u] * b;
        }
      }
      __syncthreads();
    }
    if (!__syncthreads_or(rotated)) break;
  }
  if (nsweeps && tid == 0) *nsweeps = sweep + (sweep < max_sweeps ? 1 : 0);
  for (int j = tid; j < S; j += EIGH_THREADS) {
    const double d = Gs[j + LD * j];
    phi[j] = d > 0.0 ? d : 0.0;
  }
  for (int e = tid; e < SS; e += EIGH_THREADS) Vg[e] = V[e];
  __syncthreads();
  // T-floor guard (sylvester.py:108-113): min T = lam min(Lambda) + rho + min(phi)
  if (tid == 0) {
    double pmin = INFINITY;
    bool bad = false;
    for (int j = 0; j < S; ++j) {
      pmin = fmin(pmin, phi[j]);
      bad |= !isfinite(phi[j]);
    }
    if (bad) atomicOr(status, 2);
    else if (floor_shift + pmin <= 1e-10) atomicOr(status, 1);
  }
}

// out[i, s] = sum_v A[i, v] W(v, s) with W = V (trans = false) or V^T
// (trans = true); A, out: I x S column-major; V: S x S.  With `aold` the
// epilogue applies the extrapolation of solver.py:240-243 and writes the
// compute-dtype copy.  A CTA owns 32 rows x all S columns; V in shared memory.
template <typename T, bool VG>
__global__ void __launch_bounds__(256) k_rotate(const double* __restrict__ A, int64_t I, int S,
                                               const double* __restrict__ Vm, bool trans, double* __restrict__ out,
                                               const double* __restrict__ aold, int extrap, double alpha,
                                               double beta, T* __restrict__ acomp) {
  // VG (large s): the basis is read from global memory (L1 / L2) instead of
  // being staged in shared memory
  extern __shared__ double rsm[];
  double* Vs = rsm;                                 // S x S, Vs[v + S s] = W(v, s)
  double* As = VG ? rsm : rsm + (size_t)S * S;      // 32 x (S + 1)
  const int tid = threadIdx.x;
  const int64_t i0 = (int64_t)blockIdx.x * 32;
  if (!VG)
    for (int e = tid; e < S * S; e += 256) {
      const int v = e % S, s = e / S;
      Vs[e] = trans ? Vm[s + (size_t)S * v] : Vm[e];
    }
  const int LD = S + 1;
  for (int e = tid; e < 32 * S; e += 256) {
    const int r = e % 32, v = e / 32;
    const int64_t gi = i0 + r;
    As[r * LD + v] = gi < I ? A[gi + I * v] : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < 32 * S; e += 256) {
    const int r = e % 32, s = e / 32;
    const int64_t gi = i0 + r;
    if (gi >= I) continue;
    const double* ar = As + r * LD;
    double acc = 0.0;
    if (VG) {
      for (int v = 0; v < S; ++v) acc = fma(ar[v], trans ? Vm[s + (size_t)S * v] : Vm[v + (size_t)S * s], acc);
    } else {
      const double* vs = Vs + (size_t)S * s;
      for (int v = 0; v < S; ++v) acc = fma(ar[v], vs[v], acc);
    }
    const int64_t g = gi + I * s;
    if (aold && extrap) acc = acc + alpha * (acc - beta * aold[g]);
    out[g] = acc;
    if (acomp) acomp[g] = (T)acc;
  }
}

}  // namespace

size_t eigh_smem_bytes(int64_t S) { return (size_t)(S * (S + 1) + S * S) * sizeof(double); }
bool eigh_fits_smem(int64_t S) { return eigh_smem_bytes(S) <= 220 * 1024; }

void launch_eigh(const double* G, int64_t S, double* V, double* phi, double* work, double floor_shift, int* status,
                 int max_sweeps, cudaStream_t st, int* nsweeps) {
  const bool sm = eigh_fits_smem(S);
  if (!sm && !work) throw std::runtime_error("eigh: global work buffer required for s > 117");
  if (S > 2 * EIGH_WARPS * EIGH_PPW_MAX) throw std::runtime_error("eigh: s > 1024 is not supported");
  // tol: a pair is rotated while |g_pq| > s eps sqrt(g_pp g_qq) (the
  // rounding floor of the rotated entries; a tighter threshold never stops
  // rotating); V^T G V is then diagonal to ~s eps relative.
  const double tol = (double)S * 2.220446049250313e-16;
  if (sm) {
    const size_t smem = eigh_smem_bytes(S);
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute((const void*)k_eigh_jacobi<false, 2>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) throw std::runtime_error(std::string("eigh smem attribute: ") + cudaGetErrorString(e));
    }
    k_eigh_jacobi<false, 2><<<1, EIGH_THREADS, smem, st>>>(G, (int)S, V, phi, nullptr, max_sweeps, tol, floor_shift,
                                                        status, nsweeps);
  } else {
    k_eigh_jacobi<true, EIGH_PPW_MAX><<<1, EIGH_THREADS, 0, st>>>(G, (int)S, V, phi, work, max_sweeps, tol, floor_shift, status,
                                                    nsweeps);
  }
  check_launch("eigh");
}

template <typename T>
void launch_rotate(const double* A, int64_t I, int64_t S, const double* V, bool trans, double* out,
                   const double* aold, int extrap, double alpha, double beta, T* acomp, cudaStream_t st) {
  const size_t tile = (size_t)32 * (S + 1) * sizeof(double);
  const size_t full = (size_t)S * S * sizeof(double) + tile;
  const bool vg = full > 200 * 1024;
  const size_t smem = vg ? tile : full;
  if (smem > 200 * 1024) throw std::runtime_error("rotate: s too large");
  const void* fn = vg ? (const void*)k_rotate<T, true> : (const void*)k_rotate<T, false>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) throw std::runtime_error(std::string("rotate smem attribute: ") + cudaGetErrorString(e));
  }
  const unsigned blocks = (unsigned)((I + 31) / 32);
  if (vg)
    k_rotate<T, true><<<blocks, 256, smem, st>>>(A, I, (int)S, V, trans, out, aold, extrap, alpha, beta, acomp);
  else
    k_rotate<T, false><<<blocks, 256, smem, st>>>(A, I, (int)S, V, trans, out, aold, extrap, alpha, beta, acomp);
  check_launch("rotate");
}
template void launch_rotate<double>(const double*, int64_t, int64_t, const double*, bool, double*, const double*, int,
                                    double, double, double*, cudaStream_t);
template void launch_rotate<float>(const double*, int64_t, int64_t, const double*, bool, double*, const double*, int,
                                   double, double, float*, cudaStream_t);

// V <- I (S x S)
__global__ void k_identity(double* V, int64_t S) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < S * S; e += (int64_t)gridDim.x * blockDim.x)
    V[e] = (e % S == e / S) ? 1.0 : 0.0;
}
void launch_identity(double* V, int64_t S, cudaStream_t st) {
  k_identity<<<(unsigned)std::min<int64_t>((S * S + 255) / 256, 1024), 256, 0, st>>>(V, S);
  check_launch("identity");
}

}  // namespace fctn
