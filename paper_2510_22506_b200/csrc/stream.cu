// K2 (SIMT path): Y_k partials = X_(k) M_k^T over the long reduction axis
// p = (modes before k, modes after k), sylvester.py:104.  X is read in place
// as the 3-D view [P, I_k, Q] of the first-index-fastest tensor (no unfold
// copy, solver.py:320 / tensor.py:107); M_k is stored p-fastest (M[p + pk s]),
// the column order chosen so that it matches X's (network.py:360-371).
//
// Split-K with per-split partials in fp64 and a fixed-order second stage:
// deterministic, no floating-point atomics (test_acceptance.py:407-443).
// The fp32 path on B200 tensor cores is stream_tc.cu; this kernel is the
// fp64 workhorse and the fallback for shapes TMA cannot describe.
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "kernels.cuh"

namespace fctn {

static void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

StreamPlan plan_stream(int64_t I, int64_t S, int64_t p, int target_ctas) {
  StreamPlan sp;
  sp.ts = S <= 16 ? 16 : S <= 32 ? 32 : S <= 64 ? 64 : 128;
  const int nts = sp.ts / 4;
  const int nti = 256 / nts;
  sp.ri = I <= nti ? 1 : 4;
  sp.ti = nti * sp.ri;
  sp.n_itiles = (int)((I + sp.ti - 1) / sp.ti);
  int64_t want = target_ctas / sp.n_itiles;
  if (want < 1) want = 1;
  int64_t max_split = (p + 127) / 128;  // at least 128 columns per split
  if (want > max_split) want = max_split;
  if (want < 1) want = 1;
  int64_t chunk = (p + want - 1) / want;
  chunk = (chunk + 15) / 16 * 16;
  sp.chunk = chunk;
  sp.nsplit = (int)((p + chunk - 1) / chunk);
  if (sp.nsplit < 1) sp.nsplit = 1;
  return sp;
}

// CTA: TI (= NTI*RI) rows of mode k x TS bond columns (column tile z), one p-chunk.
template <typename T, int TS, int RI, bool XFAST>
__global__ void __launch_bounds__(256) k_stream(const T* __restrict__ X, const T* __restrict__ M,
                                                double* __restrict__ part, int64_t I, int64_t P, int64_t S,
                                                int64_t p, int64_t chunk) {
  constexpr int NTS = TS / 4;
  constexpr int NTI = 256 / NTS;
  constexpr int TI = NTI * RI;
  constexpr int PC = (TI * sizeof(T) >= 2048) ? 16 : 32;  // static smem <= 48 KB
  __shared__ T Xs[PC][TI + 1];
  __shared__ T Ms[PC][TS + 1];
  const int tid = threadIdx.x;
  const int ts = tid % NTS, ti = tid / NTS;
  const int64_t i0 = (int64_t)blockIdx.x * TI;
  const int64_t split = blockIdx.y;
  const int64_t pb = split * chunk;
  const int64_t s0 = (int64_t)blockIdx.z * TS;  // column tile (s > TS)
  int64_t pe = pb + chunk;
  if (pe > p) pe = p;
  const int64_t PI = P * I;
  T acc[RI][4];
#pragma unroll
  for (int a = 0; a < RI; ++a)
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
      const int64_t gp = p0 + pp, gi = i0 + i;
      T v = T(0);
      if (gp < pe && gi < I) v = X[XFAST ? gi + I * gp : (gp % P) + P * gi + PI * (gp / P)];
      Xs[pp][i] = v;
    }
    for (int e = tid; e < PC * TS; e += 256) {
      const int pp = e % PC, s = e / PC;
      const int64_t gp = p0 + pp;
      Ms[pp][s] = (gp < pe && s0 + s < S) ? M[gp + p * (s0 + s)] : T(0);
    }
    __syncthreads();
#pragma unroll 4
    for (int pp = 0; pp < PC; ++pp) {
      T xv[RI], mv[4];
#pragma unroll
      for (int a = 0; a < RI; ++a) xv[a] = Xs[pp][ti + NTI * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) mv[b] = Ms[pp][ts + NTS * b];
#pragma unroll
      for (int a = 0; a < RI; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] += xv[a] * mv[b];
    }
    __syncthreads();
  }
  double* out = part + split * I * S;
#pragma unroll
  for (int a = 0; a < RI; ++a) {
    const int64_t gi = i0 + ti + NTI * a;
    if (gi >= I) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t s = s0 + ts + NTS * b;
      if (s < S) out[gi + I * s] = (double)acc[a][b];
    }
  }
}

template <typename T, int TS, int RI>
static void stream_go(const T* X, const T* M, double* part, int64_t I, int64_t P, int64_t S, int64_t p,
                      const StreamPlan& sp, cudaStream_t st) {
  dim3 grid(sp.n_itiles, sp.nsplit, (unsigned)((S + TS - 1) / TS));
  if (P == 1)
    k_stream<T, TS, RI, true><<<grid, 256, 0, st>>>(X, M, part, I, P, S, p, sp.chunk);
  else
    k_stream<T, TS, RI, false><<<grid, 256, 0, st>>>(X, M, part, I, P, S, p, sp.chunk);
}

template <typename T, int TS>
static void stream_ri(const T* X, const T* M, double* part, int64_t I, int64_t P, int64_t S, int64_t p,
                      const StreamPlan& sp, cudaStream_t st) {
  if (sp.ri == 1)
    stream_go<T, TS, 1>(X, M, part, I, P, S, p, sp, st);
  else
    stream_go<T, TS, 4>(X, M, part, I, P, S, p, sp, st);
}

template <typename T>
void launch_stream(const T* X, const T* M, double* part, int64_t I, int64_t P, int64_t S, int64_t p,
                   const StreamPlan& sp, cudaStream_t st) {
  switch (sp.ts) {
    case 16: stream_ri<T, 16>(X, M, part, I, P, S, p, sp, st); break;
    case 32: stream_ri<T, 32>(X, M, part, I, P, S, p, sp, st); break;
    case 64: stream_ri<T, 64>(X, M, part, I, P, S, p, sp, st); break;
    default: stream_ri<T, 128>(X, M, part, I, P, S, p, sp, st); break;
  }
  check_launch("stream");
}
template void launch_stream<double>(const double*, const double*, double*, int64_t, int64_t, int64_t, int64_t,
                                    const StreamPlan&, cudaStream_t);
template void launch_stream<float>(const float*, const float*, double*, int64_t, int64_t, int64_t, int64_t,
                                   const StreamPlan&, cudaStream_t);

// out[e] = sum_{split} part[split*n + e] (+ rho * aprev[e]).  A CTA owns 32
// consecutive outputs; its 8 warps take the splits round-robin (fixed
// assignment), then combine in warp order: a fixed summation tree.
template <typename PT>
__global__ void __launch_bounds__(256) k_reduce_splits(const PT* __restrict__ part, int nsplit, int64_t n,
                                                       const double* __restrict__ aprev, double rho,
                                                       double* __restrict__ out) {
  __shared__ double red[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e = blockIdx.x * 32LL + lane;
  double a0 = 0.0, a1 = 0.0;
  if (e < n) {
    int sp = w;
    for (; sp + 8 < nsplit; sp += 16) {
      a0 += (double)part[(int64_t)sp * n + e];
      a1 += (double)part[(int64_t)(sp + 8) * n + e];
    }
    if (sp < nsplit) a0 += (double)part[(int64_t)sp * n + e];
  }
  red[w][lane] = a0 + a1;
  __syncthreads();
  if (w == 0 && e < n) {
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) v += red[q][lane];
    if (aprev) v = __dadd_rn(v, __dmul_rn(rho, aprev[e]));  // y + rho a_prev rounded like numpy (no FMA)
    out[e] = v;
  }
}

void launch_reduce_splits(const double* part, int nsplit, int64_t n, const double* aprev, double rho, double* out,
                          cudaStream_t st) {
  int64_t blocks = (n + 31) / 32;
  k_reduce_splits<double><<<(unsigned)blocks, 256, 0, st>>>(part, nsplit, n, aprev, rho, out);
  check_launch("reduce_splits");
}
void launch_reduce_splits_f32(const float* part, int nsplit, int64_t n, const double* aprev, double rho,
                              double* out, cudaStream_t st) {
  int64_t blocks = (n + 31) / 32;
  k_reduce_splits<float><<<(unsigned)blocks, 256, 0, st>>>(part, nsplit, n, aprev, rho, out);
  check_launch("reduce_splits_f32");
}

}  // namespace fctn
