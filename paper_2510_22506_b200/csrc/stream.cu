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

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <type_traits>
#include <string>

#include "kernels.cuh"

namespace fctn {

#define CK_STREAM(x)                                                                          \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) throw std::runtime_error(std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

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

// FP64 on the tensor cores (DMMA: mma.sync.aligned.m8n8k4 f64, exact IEEE
// double FMAs): the same split-K product for the FP64 path.  CTA = 64 rows
// (mode k) x 64 bond columns x one p-chunk, 8 warps of 32 x 16; K stages of
// 32 p staged in shared memory (padded leading dimensions: the fragment
// reads are conflict-free at the 64-bit two-wavefront minimum).  Register
// reuse: 4 A + 2 B fragments feed 8 DMMAs per K = 4 step, against one shared
// load per 2 FMAs in the SIMT tile above (shared-memory bound at ~25 % of
// the FP64 peak on c3).
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <bool XFAST>
__global__ void __launch_bounds__(256) k_stream_dmma(const double* __restrict__ X, const double* __restrict__ M,
                                                     double* __restrict__ part, int64_t I, int64_t P, int64_t S,
                                                     int64_t p, int64_t chunk) {
  constexpr int BI = 64, BS = 64, KC = 32;
  __shared__ double Xs[BI][KC + 4];  // [i][p]
  __shared__ double Ms[KC][BS + 8];  // [p][s]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wi = w >> 2, ws = w & 3;  // warp tile: rows 32 wi .. +32, cols 16 ws .. +16
  const int64_t i0 = (int64_t)blockIdx.x * BI, s0 = (int64_t)blockIdx.z * BS;
  const int64_t split = blockIdx.y;
  const int64_t pb = split * chunk;
  int64_t pe = pb + chunk;
  if (pe > p) pe = p;
  const int64_t PI = P * I;
  double acc[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int64_t p0 = pb; p0 < pe; p0 += KC) {
    // p = (r, q) with r = p % P: one 64-bit division per stage, then at most
    // one wrap inside the 32-wide stage when P >= 32
    const int64_t q0 = XFAST ? 0 : p0 / P, r0 = XFAST ? 0 : p0 - q0 * P;
#pragma unroll
    for (int j = 0; j < (BI * KC) / 256; ++j) {
      const int e = tid + 256 * j;
      int il, pl;
      if (XFAST) {
        il = e % BI;
        pl = e / BI;
      } else {
        pl = e % KC;
        il = e / KC;
      }
      const int64_t gp = p0 + pl, gi = i0 + il;
      double v = 0.0;
      if (gp < pe && gi < I) {
        if (XFAST) {
          v = X[gi + I * gp];
        } else {
          int64_t rr = r0 + pl, qq = q0;
          if (P >= KC) {
            if (rr >= P) {
              rr -= P;
              ++qq;
            }
          } else {
            qq += rr / P;
            rr %= P;
          }
          v = X[rr + P * gi + PI * qq];
        }
      }
      Xs[il][pl] = v;
    }
#pragma unroll
    for (int j = 0; j < (KC * BS) / 256; ++j) {
      const int e = tid + 256 * j;
      const int pl = e % KC, sl = e / KC;
      const int64_t gp = p0 + pl, gs = s0 + sl;
      Ms[pl][sl] = (gp < pe && gs < S) ? M[gp + p * gs] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      double av[4], bv[2];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = Xs[32 * wi + 8 * a + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
      for (int b = 0; b < 2; ++b) bv[b] = Ms[kk + (lane & 3)][16 * ws + 8 * b + (lane >> 2)];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) dmma_8x8x4(acc[a][b], av[a], bv[b]);
    }
    __syncthreads();
  }
  double* out = part + split * I * S;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t gi = i0 + 32 * wi + 8 * a + (lane >> 2);
    if (gi >= I) continue;
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gs = s0 + 16 * ws + 8 * b + 2 * (lane & 3) + h;
        if (gs < S) out[gi + I * gs] = acc[a][b][h];
      }
  }
}

// the DMMA form for the FP64 path when the tile is not mostly padding; it
// uses at most the split count the SIMT plan reserved partials for
static bool dmma_ok(int64_t I, int64_t S) {
  static const bool off = getenv("FCTN_NO_DMMA") != nullptr;
  return !off && I >= 16 && S >= 16;
}

template <typename T>
void launch_stream(const T* X, const T* M, double* part, int64_t I, int64_t P, int64_t S, int64_t p,
                   const StreamPlan& sp, cudaStream_t st) {
  if constexpr (std::is_same<T, double>::value) {
    if (dmma_ok(I, S)) {
      const int64_t ti = (I + 63) / 64, ts = (S + 63) / 64;
      int64_t want = std::max<int64_t>(1, (2 * 148 + ti * ts - 1) / (ti * ts));
      want = std::min<int64_t>(want, std::max<int64_t>(1, (p + 255) / 256));
      want = std::min<int64_t>(want, sp.nsplit);  // the partial buffer is sized for sp.nsplit
      int64_t chunk = (p + want - 1) / want;
      chunk = (chunk + 31) / 32 * 32;
      const int64_t ns = (p + chunk - 1) / chunk;
      // k_reduce_splits reads sp.nsplit partials: zero the ones this grid leaves empty
      if (ns < sp.nsplit) CK_STREAM(cudaMemsetAsync(part + ns * I * S, 0, (sp.nsplit - ns) * I * S * sizeof(double), st));
      dim3 grid((unsigned)ti, (unsigned)ns, (unsigned)ts);
      if (P == 1)
        k_stream_dmma<true><<<grid, 256, 0, st>>>(X, M, part, I, P, S, p, chunk);
      else
        k_stream_dmma<false><<<grid, 256, 0, st>>>(X, M, part, I, P, S, p, chunk);
      check_launch("stream_dmma");
      return;
    }
  }
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
