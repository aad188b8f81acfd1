// K1: generic labeled contraction (merge of factors / partials into M_k,
// network.py:249-258 over tensor.py:156-200), the generic
// permutation, and the dtype conversion.  See DESIGN.md.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <type_traits>

#include "kernels.cuh"

namespace fctn {

static void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// ============================================================ K1 contract
//
// C[r, c] = sum_k A[r, k] B[c, k] where r, c, k are mixed-radix multi-indices
// over labels (ContractDesc): every offset is computed on device from the
// extents/strides, so a new visiting order or rank table needs no host
// tables.  Rows enumerate the operand holding C's fastest label, so the
// stores are coalesced.  Small-output / long-K contractions (the doubled
// network of the Gram) split K over CTAs and reduce in a fixed order.

__device__ __forceinline__ void md_offsets(int64_t idx, int nd, const int64_t* ext, const int64_t* s1,
                                           const int64_t* s2, int64_t& o1, int64_t& o2) {
  o1 = 0;
  o2 = 0;
  for (int q = 0; q < nd; ++q) {
    const int64_t d = idx % ext[q];
    idx /= ext[q];
    o1 += d * s1[q];
    o2 += d * s2[q];
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_contract(const T* __restrict__ A, const T* __restrict__ B,
                                                  T* __restrict__ C, T* __restrict__ part, const ContractDesc d,
                                                  int64_t tiles_r, int64_t kchunk) {
  constexpr int BR = 64, BC = 64, KC = 16;
  __shared__ T As[KC][BR + 1];
  __shared__ T Bs[KC][BC + 1];
  __shared__ int64_t sRA[BR], sRC[BR], sCB[BC], sCC[BC];
  extern __shared__ int64_t sK[];  // [kA | kB] for this CTA's K range
  const int64_t tile = blockIdx.x;
  const int64_t r0 = (tile % tiles_r) * BR;
  const int64_t c0 = (tile / tiles_r) * BC;
  const int64_t kb = blockIdx.y * kchunk;
  int64_t ke = kb + kchunk;
  if (ke > d.K) ke = d.K;
  const int64_t nk = ke - kb;
  const int tid = threadIdx.x;
  if (tid < BR) {
    const int64_t r = r0 + tid;
    int64_t oa = -1, oc = 0;
    if (r < d.rows) md_offsets(r, d.nr, d.r_ext, d.r_sa, d.r_sc, oa, oc);
    sRA[tid] = oa;
    sRC[tid] = oc;
  } else if (tid < BR + BC) {
    const int c = tid - BR;
    int64_t ob = -1, oc = 0;
    if (c0 + c < d.cols) md_offsets(c0 + c, d.nc, d.c_ext, d.c_sb, d.c_sc, ob, oc);
    sCB[c] = ob;
    sCC[c] = oc;
  }
  for (int64_t k = tid; k < nk; k += 256) {
    int64_t oa, ob;
    md_offsets(kb + k, d.nk, d.k_ext, d.k_sa, d.k_sb, oa, ob);
    sK[k] = oa;
    sK[nk + k] = ob;
  }
  __syncthreads();
  const int tx = tid & 15, ty = tid >> 4;
  T acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = T(0);
  for (int64_t k0 = 0; k0 < nk; k0 += KC) {
    for (int e = tid; e < KC * BR; e += 256) {
      const int kk = e / BR, r = e % BR;
      const int64_t ra = sRA[r];
      As[kk][r] = (ra >= 0 && k0 + kk < nk) ? A[ra + sK[k0 + kk]] : T(0);
    }
    for (int e = tid; e < KC * BC; e += 256) {
      const int kk = e / BC, c = e % BC;
      const int64_t cb = sCB[c];
      Bs[kk][c] = (cb >= 0 && k0 + kk < nk) ? B[cb + sK[nk + k0 + kk]] : T(0);
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
    const int rl = tx + 16 * a;
    if (r0 + rl >= d.rows) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int cl = ty + 16 * b;
      if (c0 + cl >= d.cols) continue;
      if (part)
        part[blockIdx.y * d.rows * d.cols + (r0 + rl) + d.rows * (c0 + cl)] = acc[a][b];
      else
        C[sRC[rl] + sCC[cl]] = acc[a][b];
    }
  }
}

// FP64 contraction on the tensor cores (DMMA, mma.sync m8n8k4 f64): the same
// descriptor-driven tile (64 x 64 output, offset tables in shared memory) as
// k_contract, with 8 warps of 32 x 16 and 4 A + 2 B fragments feeding 8
// DMMAs per K = 4 step (the SIMT tile is shared-memory bound at ~2 TFLOP/s on
// c3's joins).  Padded K-major stages keep fragment reads at the 64-bit
// two-wavefront minimum.
__device__ __forceinline__ void dmma_884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) k_contract_dmma(const double* __restrict__ A, const double* __restrict__ B,
                                                       double* __restrict__ C, double* __restrict__ part,
                                                       const ContractDesc d, int64_t tiles_r, int64_t kchunk) {
  constexpr int BR = 64, BC = 64, KC = 16, LD = 72;
  __shared__ double As[KC][LD];
  __shared__ double Bs[KC][LD];
  __shared__ int64_t sRA[BR], sRC[BR], sCB[BC], sCC[BC];
  extern __shared__ int64_t sK[];  // [kA | kB] for this CTA's K range
  const int64_t tile = blockIdx.x;
  const int64_t r0 = (tile % tiles_r) * BR;
  const int64_t c0 = (tile / tiles_r) * BC;
  const int64_t kb = blockIdx.y * kchunk;
  int64_t ke = kb + kchunk;
  if (ke > d.K) ke = d.K;
  const int64_t nk = ke - kb;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wr = w >> 2, wc = w & 3;  // warp tile: rows 32 wr .. +32, cols 16 wc .. +16
  if (tid < BR) {
    const int64_t r = r0 + tid;
    int64_t oa = -1, oc = 0;
    if (r < d.rows) md_offsets(r, d.nr, d.r_ext, d.r_sa, d.r_sc, oa, oc);
    sRA[tid] = oa;
    sRC[tid] = oc;
  } else if (tid < BR + BC) {
    const int c = tid - BR;
    int64_t ob = -1, oc = 0;
    if (c0 + c < d.cols) md_offsets(c0 + c, d.nc, d.c_ext, d.c_sb, d.c_sc, ob, oc);
    sCB[c] = ob;
    sCC[c] = oc;
  }
  for (int64_t k = tid; k < nk; k += 256) {
    int64_t oa, ob;
    md_offsets(kb + k, d.nk, d.k_ext, d.k_sa, d.k_sb, oa, ob);
    sK[k] = oa;
    sK[nk + k] = ob;
  }
  __syncthreads();
  double acc[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int64_t k0 = 0; k0 < nk; k0 += KC) {
    for (int e = tid; e < KC * BR; e += 256) {
      const int kk = e / BR, r = e % BR;
      const int64_t ra = sRA[r];
      As[kk][r] = (ra >= 0 && k0 + kk < nk) ? A[ra + sK[k0 + kk]] : 0.0;
    }
    for (int e = tid; e < KC * BC; e += 256) {
      const int kk = e / BC, c = e % BC;
      const int64_t cb = sCB[c];
      Bs[kk][c] = (cb >= 0 && k0 + kk < nk) ? B[cb + sK[nk + k0 + kk]] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      double av[4], bv[2];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[kk + (lane & 3)][32 * wr + 8 * a + (lane >> 2)];
#pragma unroll
      for (int b = 0; b < 2; ++b) bv[b] = Bs[kk + (lane & 3)][16 * wc + 8 * b + (lane >> 2)];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) dmma_884(acc[a][b], av[a], bv[b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int rl = 32 * wr + 8 * a + (lane >> 2);
    if (r0 + rl >= d.rows) continue;
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cl = 16 * wc + 8 * b + 2 * (lane & 3) + h;
        if (c0 + cl >= d.cols) continue;
        if (part)
          part[blockIdx.y * d.rows * d.cols + (r0 + rl) + d.rows * (c0 + cl)] = acc[a][b][h];
        else
          C[sRC[rl] + sCC[cl]] = acc[a][b][h];
      }
  }
}

// Split-K reduction: a CTA owns 32 consecutive outputs; its 8 warps take the
// splits round-robin with two independent accumulators each (many splits over
// a small output, e.g. 296 x 375 for c3's Y_2 = W (*) L, would otherwise be one
// dependent chain of loads per thread), combined in warp order: a fixed
// summation tree.
template <typename T>
__global__ void __launch_bounds__(256) k_contract_reduce(const T* __restrict__ part, int nsplit, const ContractDesc d,
                                                         T* __restrict__ C) {
  __shared__ T red[8][33];
  const int64_t n = d.rows * d.cols;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e = blockIdx.x * 32LL + lane;
  T a0 = T(0), a1 = T(0);
  if (e < n) {
    int sp = w;
    for (; sp + 8 < nsplit; sp += 16) {
      a0 += part[(int64_t)sp * n + e];
      a1 += part[(int64_t)(sp + 8) * n + e];
    }
    if (sp < nsplit) a0 += part[(int64_t)sp * n + e];
  }
  red[w][lane] = a0 + a1;
  __syncthreads();
  if (w == 0 && e < n) {
    T v = T(0);
#pragma unroll
    for (int q = 0; q < 8; ++q) v += red[q][lane];
    int64_t x, rc, cc;
    md_offsets(e % d.rows, d.nr, d.r_ext, d.r_sa, d.r_sc, x, rc);
    md_offsets(e / d.rows, d.nc, d.c_ext, d.c_sb, d.c_sc, x, cc);
    C[rc + cc] = v;
  }
}

// Resident-rows contraction for large outputs with a short side (the merges
// that write M_k or big partials): the whole row operand (rows x K, rows <=
// 512) stays in shared memory for the CTA's lifetime, CTAs walk column tiles
// persistently, lanes run along rows (the operand holding C's fastest label,
// so stores coalesce) and each thread keeps RPT rows x CPT columns in
// registers.  Only the streamed column operand is gathered per tile.
template <typename T, int RPT, int CPT>
__global__ void __launch_bounds__(256) k_contract_res(const T* __restrict__ A, const T* __restrict__ B,
                                                      T* __restrict__ C, const ContractDesc d, int64_t n_ctiles) {
  constexpr int CT = 8 * CPT;  // columns per tile: 8 warps x CPT
  extern __shared__ __align__(16) unsigned char smraw[];
  const int K = (int)d.K;
  const int rows = (int)d.rows;
  T* As = reinterpret_cast<T*>(smraw);                     // [K][32*RPT]
  T* Bs = As + (size_t)K * 32 * RPT;                       // [K][CT]
  int64_t* sRC = reinterpret_cast<int64_t*>(Bs + (size_t)K * CT);  // [32*RPT]
  int64_t* sKB = sRC + 32 * RPT;                           // [K]
  int64_t* sCB = sKB + K;                                  // [CT]
  int64_t* sCC = sCB + CT;                                 // [CT]
  const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;
  // resident rows: A[r, k] and the output row offsets
  for (int e = tid; e < K * 32 * RPT; e += 256) {
    const int k = e / (32 * RPT), r = e % (32 * RPT);
    T v = T(0);
    if (r < rows) {
      int64_t oa, oc, ka, kb;
      md_offsets(r, d.nr, d.r_ext, d.r_sa, d.r_sc, oa, oc);
      md_offsets(k, d.nk, d.k_ext, d.k_sa, d.k_sb, ka, kb);
      v = A[oa + ka];
    }
    As[e] = v;
  }
  for (int r = tid; r < 32 * RPT; r += 256) {
    int64_t oa = 0, oc = 0;
    if (r < rows) md_offsets(r, d.nr, d.r_ext, d.r_sa, d.r_sc, oa, oc);
    sRC[r] = oc;
  }
  for (int k = tid; k < K; k += 256) {
    int64_t ka, kb;
    md_offsets(k, d.nk, d.k_ext, d.k_sa, d.k_sb, ka, kb);
    sKB[k] = kb;
  }
  for (int64_t ct = blockIdx.x; ct < n_ctiles; ct += gridDim.x) {
    const int64_t c0 = ct * CT;
    __syncthreads();  // previous tile's Bs / sCC readers are done
    for (int c = tid; c < CT; c += 256) {
      int64_t ob = -1, oc = 0;
      if (c0 + c < d.cols) md_offsets(c0 + c, d.nc, d.c_ext, d.c_sb, d.c_sc, ob, oc);
      sCB[c] = ob;
      sCC[c] = oc;
    }
    __syncthreads();
    for (int e = tid; e < K * CT; e += 256) {
      const int k = e / CT, c = e % CT;
      const int64_t ob = sCB[c];
      Bs[e] = ob >= 0 ? B[ob + sKB[k]] : T(0);
    }
    __syncthreads();
    T acc[RPT][CPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i)
#pragma unroll
      for (int j = 0; j < CPT; ++j) acc[i][j] = T(0);
    for (int k = 0; k < K; ++k) {
      T a[RPT], b[CPT];
#pragma unroll
      for (int i = 0; i < RPT; ++i) a[i] = As[k * 32 * RPT + lane + 32 * i];
#pragma unroll
      for (int j = 0; j < CPT; ++j) b[j] = Bs[k * CT + wy * CPT + j];
#pragma unroll
      for (int i = 0; i < RPT; ++i)
#pragma unroll
        for (int j = 0; j < CPT; ++j) acc[i][j] += a[i] * b[j];
    }
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int c = wy * CPT + j;
      if (sCB[c] < 0) continue;
      const int64_t cc = sCC[c];
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int r = lane + 32 * i;
        if (r < rows) C[sRC[r] + cc] = acc[i][j];
      }
    }
  }
}

template <typename T, int RPT, int CPT>
static bool res_go(const T* A, const T* B, T* C, const ContractDesc& d, int n_sm, cudaStream_t st) {
  constexpr int CT = 8 * CPT;
  const size_t smem = (size_t)d.K * (32 * RPT + CT) * sizeof(T) + (32 * RPT + d.K + 2 * CT) * sizeof(int64_t);
  if (smem > 160 * 1024) return false;
  auto fn = k_contract_res<T, RPT, CPT>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) throw std::runtime_error(std::string("contract_res smem: ") + cudaGetErrorString(e));
  }
  const int64_t n_ct = (d.cols + CT - 1) / CT;
  const int64_t grid = std::min<int64_t>(n_ct, (int64_t)n_sm * 4);
  fn<<<(unsigned)grid, 256, smem, st>>>(A, B, C, d, n_ct);
  check_launch("contract_res");
  return true;
}

// Resident-columns variant: the short side is the column operand (<= 256
// columns) and the long row operand holds C's fastest label.  Each thread
// owns one streamed row (its K values in registers) and sweeps all resident
// columns, CB at a time; lanes run along rows, so both the row gathers and
// the stores coalesce.
template <typename T, int KMAX, int CB>
__global__ void __launch_bounds__(256) k_contract_rescol(const T* __restrict__ A, const T* __restrict__ B,
                                                         T* __restrict__ C, const ContractDesc d) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int K = (int)d.K, cols = (int)d.cols;
  T* Bs = reinterpret_cast<T*>(smraw);                            // [K][cols]
  // the int64 tables start 8-byte aligned whatever K * cols is
  int64_t* sCC = reinterpret_cast<int64_t*>(smraw + (((size_t)K * cols * sizeof(T) + 7) & ~(size_t)7));  // [cols]
  int64_t* sKA = sCC + cols;                                      // [K]
  for (int e = threadIdx.x; e < K * cols; e += blockDim.x) {
    const int k = e / cols, c = e % cols;
    int64_t ob, oc, ka, kb;
    md_offsets(c, d.nc, d.c_ext, d.c_sb, d.c_sc, ob, oc);
    md_offsets(k, d.nk, d.k_ext, d.k_sa, d.k_sb, ka, kb);
    Bs[e] = B[ob + kb];
  }
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    int64_t ob, oc;
    md_offsets(c, d.nc, d.c_ext, d.c_sb, d.c_sc, ob, oc);
    sCC[c] = oc;
  }
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    int64_t ka, kb;
    md_offsets(k, d.nk, d.k_ext, d.k_sa, d.k_sb, ka, kb);
    sKA[k] = ka;
  }
  __syncthreads();
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < d.rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t oa, orc;
    md_offsets(r, d.nr, d.r_ext, d.r_sa, d.r_sc, oa, orc);
    T a[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) a[k] = k < K ? A[oa + sKA[k]] : T(0);
    for (int c0 = 0; c0 < cols; c0 += CB) {
      T acc[CB];
#pragma unroll
      for (int j = 0; j < CB; ++j) acc[j] = T(0);
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
        if (k >= K) break;
#pragma unroll
        for (int j = 0; j < CB; ++j) acc[j] += a[k] * Bs[k * cols + (c0 + j < cols ? c0 + j : 0)];
      }
#pragma unroll
      for (int j = 0; j < CB; ++j)
        if (c0 + j < cols) C[orc + sCC[c0 + j]] = acc[j];
    }
  }
}

template <typename T, int KMAX>
static bool rescol_go(const T* A, const T* B, T* C, const ContractDesc& d, int n_sm, cudaStream_t st) {
  constexpr int CB = 8;
  const size_t smem = (((size_t)d.K * d.cols * sizeof(T) + 7) & ~(size_t)7) + (d.cols + d.K) * sizeof(int64_t);
  if (smem > 160 * 1024) return false;
  auto fn = k_contract_rescol<T, KMAX, CB>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) throw std::runtime_error(std::string("contract_rescol smem: ") + cudaGetErrorString(e));
  }
  const int64_t grid = std::min<int64_t>((d.rows + 255) / 256, (int64_t)n_sm * 8);
  fn<<<(unsigned)grid, 256, smem, st>>>(A, B, C, d);
  check_launch("contract_rescol");
  return true;
}

// dispatch for large outputs with a short row side; false = not applicable
template <typename T>
static bool contract_resident(const T* A, const T* B, T* C, const ContractDesc& d, int n_sm, cudaStream_t st) {
  if (d.cols <= 256 && d.rows >= 65536 && d.K <= 32) {  // long rows, short resident columns
    if (d.K <= 8) return rescol_go<T, 8>(A, B, C, d, n_sm, st);
    if (d.K <= 16) return rescol_go<T, 16>(A, B, C, d, n_sm, st);
    return rescol_go<T, 32>(A, B, C, d, n_sm, st);
  }
  if (d.rows > 512 || d.cols < 4096 || d.K > 1024) return false;
  const int rpt = (int)((d.rows + 31) / 32);
  if (rpt <= 1) return res_go<T, 1, 8>(A, B, C, d, n_sm, st);
  if (rpt <= 2) return res_go<T, 2, 8>(A, B, C, d, n_sm, st);
  if (rpt <= 4) return res_go<T, 4, 8>(A, B, C, d, n_sm, st);
  if (rpt <= 8) return res_go<T, 8, 4>(A, B, C, d, n_sm, st);
  return res_go<T, 16, 2>(A, B, C, d, n_sm, st);
}

int64_t contract_split_scratch(const ContractDesc& d, int n_sm) {
  const int64_t tiles = ((d.rows + 63) / 64) * ((d.cols + 63) / 64);
  if (tiles >= n_sm || d.K < 256) return 0;
  int64_t ns = std::min<int64_t>(d.K / 64, (2 * n_sm + tiles - 1) / tiles);
  if (ns < 2) return 0;
  return ns * d.rows * d.cols;
}

// Small outputs (a handful of 64 x 64 tiles, e.g. the fp64 Gram network's
// s_k x s_k result at c4: one tile, one CTA, ~25 us of serial K loop): one
// warp per output column block, lanes along rows, K split over the 8 warps
// of a CTA and reduced in shared memory in a fixed order.
template <typename T>
__global__ void __launch_bounds__(256) k_contract_small(const T* __restrict__ A, const T* __restrict__ B,
                                                        T* __restrict__ C, const ContractDesc d) {
  __shared__ T red[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r = (int64_t)blockIdx.x * 32 + lane;  // output row (lanes: C's fastest label)
  const int64_t c = blockIdx.y;                       // output column
  int64_t oa = 0, orc = 0, ob = 0, oc = 0;
  const bool ok = r < d.rows;
  if (ok) md_offsets(r, d.nr, d.r_ext, d.r_sa, d.r_sc, oa, orc);
  md_offsets(c, d.nc, d.c_ext, d.c_sb, d.c_sc, ob, oc);
  T acc = T(0);
  if (ok)
    for (int64_t k = warp; k < d.K; k += 8) {
      int64_t ka, kb;
      md_offsets(k, d.nk, d.k_ext, d.k_sa, d.k_sb, ka, kb);
      acc += A[oa + ka] * B[ob + kb];
    }
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && ok) {
    T v = red[0][lane];
#pragma unroll
    for (int w = 1; w < 8; ++w) v += red[w][lane];
    C[orc + oc] = v;
  }
}

template <typename T>
void launch_contract(const T* A, const T* B, T* C, const ContractDesc& d, T* scratch, int64_t scratch_cap, int n_sm,
                     cudaStream_t st) {
  const int64_t tr = (d.rows + 63) / 64, tcn = (d.cols + 63) / 64;
  const int64_t tiles = tr * tcn;
  if (tiles <= 0) return;
  if (tiles <= 4 && d.K <= 4096 && d.cols <= 65535 && d.rows * d.cols >= 256 && !getenv("FCTN_NO_SMALL_CONTRACT")) {
    dim3 grid((unsigned)((d.rows + 31) / 32), (unsigned)d.cols);
    k_contract_small<T><<<grid, 256, 0, st>>>(A, B, C, d);
    check_launch("contract_small");
    return;
  }
  if constexpr (std::is_same<T, float>::value) {
    if (tc_join_applicable(d)) {
      launch_join_tc(A, B, C, d, n_sm, st);
      return;
    }
  }
  if (join_applicable(d, sizeof(T))) {
    launch_join<T>(A, B, C, d, n_sm, st);
    return;
  }
  if (contract_resident<T>(A, B, C, d, n_sm, st)) return;
  // what the specialised forms above do not take: FP64 on the tensor cores
  // (measured faster than the SIMT tile, slower than k_join on the joins)
  static const bool no_dmma = getenv("FCTN_NO_DMMA") != nullptr;
  const bool dmma = std::is_same<T, double>::value && !no_dmma && d.K >= 4;
  int64_t ns = 1;
  if (scratch && tiles < n_sm && d.K >= 256) {
    ns = std::min<int64_t>(d.K / 64, (2 * n_sm + tiles - 1) / tiles);
    while (ns > 1 && ns * d.rows * d.cols > scratch_cap) --ns;
  }
  int64_t kchunk = (d.K + ns - 1) / ns;
  ns = (d.K + kchunk - 1) / kchunk;
  if (kchunk > 6144) throw std::runtime_error("contraction K chunk too long for the on-chip offset table");
  const size_t smem = (size_t)2 * kchunk * sizeof(int64_t);
  // the kernel also holds ~19 KB of static tiles: opt in above 48 KB in total
  if (smem > 24 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_contract<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024);
    if (e != cudaSuccess) throw std::runtime_error(std::string("contract smem: ") + cudaGetErrorString(e));
  }
  dim3 grid((unsigned)tiles, (unsigned)ns);
  if constexpr (std::is_same<T, double>::value) {
    if (dmma) {
      if (smem > 24 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_contract_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem + 1024);
        if (e != cudaSuccess) throw std::runtime_error(std::string("contract_dmma smem: ") + cudaGetErrorString(e));
      }
      k_contract_dmma<<<grid, 256, smem, st>>>(A, B, C, ns > 1 ? scratch : nullptr, d, tr, kchunk);
      check_launch("contract_dmma");
    }
  }
  if (!dmma) {
    k_contract<T><<<grid, 256, smem, st>>>(A, B, C, ns > 1 ? scratch : nullptr, d, tr, kchunk);
    check_launch("contract");
  }
  if (ns > 1) {
    const int64_t n = d.rows * d.cols;
    k_contract_reduce<T><<<(unsigned)((n + 31) / 32), 256, 0, st>>>(scratch, (int)ns, d, C);
    check_launch("contract_reduce");
  }
}
template void launch_contract<double>(const double*, const double*, double*, const ContractDesc&, double*, int64_t,
                                      int, cudaStream_t);
template void launch_contract<float>(const float*, const float*, float*, const ContractDesc&, float*, int64_t, int,
                                     cudaStream_t);

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

// rows [lo, lo+rows) of a column-major I x S fp64 matrix -> rows x S (T)
template <typename T>
__global__ void k_copy_rows(const double* __restrict__ A, int64_t I, int64_t S, int64_t lo, int64_t rows,
                            T* __restrict__ out) {
  const int64_t n = rows * S;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % rows, s = e / rows;
    out[e] = (T)A[lo + i + I * s];
  }
}

void launch_copy_rows(const double* A, int64_t I, int64_t S, int64_t lo, int64_t rows, void* out, bool f32,
                      cudaStream_t st) {
  const int64_t n = rows * S;
  if (n <= 0) return;
  const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8);
  if (f32)
    k_copy_rows<float><<<blocks, 256, 0, st>>>(A, I, S, lo, rows, (float*)out);
  else
    k_copy_rows<double><<<blocks, 256, 0, st>>>(A, I, S, lo, rows, (double*)out);
  check_launch("copy_rows");
}

// all-gathered blocks [rank][rows_r x S, ld rows_r] (padded to slab_max*S)
// -> Y (I x S column-major), rank r owning rows [r*I/n, (r+1)*I/n)
__global__ void k_scatter_rows(const double* __restrict__ g, int nranks, int64_t slab_max, int64_t I, int64_t S,
                               double* __restrict__ Y) {
  const int64_t n = I * S;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % I, s = e / I;
    int r = (int)((i * nranks) / I);  // owner: largest r with r*I/n <= i
    while (r + 1 < nranks && (r + 1) * I / nranks <= i) ++r;
    while (r > 0 && r * I / nranks > i) --r;
    const int64_t lo = r * I / nranks, rows = (r + 1) * I / nranks - lo;
    Y[e] = g[(int64_t)r * slab_max * S + (i - lo) + rows * s];
  }
}

void launch_scatter_rows(const double* g, int nranks, int64_t slab_max, int64_t I, int64_t S, double* Y,
                         cudaStream_t st) {
  const int64_t n = I * S;
  const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8);
  k_scatter_rows<<<blocks, 256, 0, st>>>(g, nranks, slab_max, I, S, Y);
  check_launch("scatter_rows");
}

__global__ void k_axpy(double* __restrict__ y, const double* __restrict__ x, double a, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    y[e] = __dadd_rn(y[e], __dmul_rn(a, x[e]));  // y += a x rounded like numpy (sylvester.py:106), no FMA
}

void launch_axpy(double* y, const double* x, double a, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8);
  k_axpy<<<blocks, 256, 0, st>>>(y, x, a, n);
  check_launch("axpy");
}

// N = 3 schedule, Y_k = Z_j (*) A_(l) (kernels.cuh: YzArgs).
//  long_l (contract the fast row mode r = i_l):
//     Y[o, bz, ba] = sum_{r, bc} Z[r, o, bc, bz] A[r, bc, ba]
//     CTA per (bz, group of G o); a thread keeps A[r, :, :] in registers for
//     its r and accumulates G x RA sums; fixed-order block tree.
//  otherwise (contract the slow row mode o = i_l, rows r = i_k):
//     Y[r, bz, ba] = sum_{o, bc} Z[r, o, bc, bz] A[o, bc, ba]
//     thread per (r, bz), CTAs also split bc (partials reduced in order);
//     A values are warp-uniform.
// fp64 accumulation, deterministic.
template <typename T, int RC, int RA, int G>
__global__ void __launch_bounds__(256, 2) k_yzl(const T* __restrict__ Z, const T* __restrict__ A, YzArgs p,
                                             double* __restrict__ Y, int64_t r_chunk,
                                             const double* __restrict__ aprev, double rho) {
  const int64_t bz = blockIdx.x % p.Rz, o0 = (blockIdx.x / p.Rz) * G;
  const int64_t rows = p.Ir * p.Io;
  const int64_t r_lo = blockIdx.y * r_chunk, r_hi = (p.Ir < r_lo + r_chunk) ? p.Ir : r_lo + r_chunk;
  Y += blockIdx.y * (p.Io * p.Rz * RA);  // this r-split's partial
  double acc[G][RA];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int c = 0; c < RA; ++c) acc[g][c] = 0.0;
  for (int64_t r = r_lo + threadIdx.x; r < r_hi; r += 256) {
    // the RC-term inner products in the data precision (fp32 for the FP32
    // variant: FFMA at 2x the fp64 rate), accumulated over rows in fp64; one
    // bond of A at a time keeps the register tile small
    T in[G][RA];
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int c = 0; c < RA; ++c) in[g][c] = T(0);
#pragma unroll
    for (int b = 0; b < RC; ++b) {
      T ab[RA];
#pragma unroll
      for (int c = 0; c < RA; ++c) ab[c] = A[r + p.Ir * (b * p.ac + c * p.aa)];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int64_t o = o0 + g < p.Io ? o0 + g : p.Io - 1;  // clamped; rows past Io are never stored
        const T z = Z[r + p.Ir * o + rows * (b * p.zc + bz * p.zk)];
#pragma unroll
        for (int c = 0; c < RA; ++c) in[g][c] = fma(z, ab[c], in[g][c]);
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int c = 0; c < RA; ++c) acc[g][c] += (double)in[g][c];
  }
  __shared__ double red[8][G * RA];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int c = 0; c < RA; ++c) {
      double v = acc[g][c];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[wid][g * RA + c] = v;
    }
  __syncthreads();
  for (int e = threadIdx.x; e < G * RA; e += 256) {
    const int g = e / RA, c = e % RA;
    const int64_t o = o0 + g;
    if (o >= p.Io) continue;
    double v = 0.0;
    for (int q = 0; q < 8; ++q) v += red[q][e];
    const int64_t yi = o + p.Io * (bz * p.yz + c * p.ya);
    if (aprev) v = __dadd_rn(v, __dmul_rn(rho, aprev[yi]));  // + rho A_prev (sylvester.py:106), unsplit; no FMA
    Y[yi] = v;
  }
}

template <typename T, int RB>
__global__ void __launch_bounds__(256) k_yzs(const T* __restrict__ Z, const T* __restrict__ A, YzArgs p,
                                             double* __restrict__ part) {
  constexpr int OC = 64;  // o values per shared-memory chunk of A
  __shared__ double as[OC][RB];
  const int64_t r = blockIdx.x * 256LL + threadIdx.x;
  const int bz = blockIdx.y, bc = blockIdx.z;
  const bool live = r < p.Ir;
  const int64_t rows = p.Ir * p.Io;
  const T* zp = Z + (live ? r : 0) + rows * (bc * p.zc + bz * p.zk);
  const T* ap = A + p.Io * (bc * p.ac);
  double acc[RB];
#pragma unroll
  for (int c = 0; c < RB; ++c) acc[c] = 0.0;
  for (int64_t o0 = 0; o0 < p.Io; o0 += OC) {
    const int on = (int)(p.Io - o0 < OC ? p.Io - o0 : OC);
    __syncthreads();
    for (int e = threadIdx.x; e < OC * RB; e += 256) {
      const int o = e % OC, c = e / OC;
      as[o][c] = (o < on && c < p.Ra) ? (double)ap[o0 + o + p.Io * (c * p.aa)] : 0.0;
    }
    __syncthreads();
    if (live) {
#pragma unroll 8
      for (int o = 0; o < on; ++o) {
        const double z = (double)zp[p.Ir * (o0 + o)];
#pragma unroll
        for (int c = 0; c < RB; ++c) acc[c] = fma(z, as[o][c], acc[c]);
      }
    }
  }
  if (!live) return;
  const int64_t n = p.Ir * p.Rz * p.Ra;
#pragma unroll
  for (int c = 0; c < RB; ++c)
    if (c < p.Ra) part[bc * n + r + p.Ir * (bz * p.yz + c * p.ya)] = acc[c];
}

template <typename T, int R>
static int yzl_go(const T* Z, const T* Al, const YzArgs& a, double* Y, double* part, const double* aprev,
                  double rho, cudaStream_t st) {
  constexpr int G = R * R > 32 ? 4 : 8;  // G x R fp64 accumulators + R x R operands stay in registers
  const int64_t nxy = a.Rz * ((a.Io + G - 1) / G);
  // split the contracted rows so that the grid covers the GPU, but keep >= 4
  // rows per thread so the CTA's G x R-value reduction stays amortised;
  // partials reduced in order
  int64_t rs = (148 + nxy - 1) / nxy;
  rs = std::max<int64_t>(1, std::min<int64_t>(rs, (a.Ir + 1023) / 1024));
  const int64_t chunk = (a.Ir + rs - 1) / rs;
  rs = (a.Ir + chunk - 1) / chunk;
  dim3 grid((unsigned)nxy, (unsigned)rs);
  k_yzl<T, R, R, G><<<grid, 256, 0, st>>>(Z, Al, a, rs > 1 ? part : Y, chunk, rs > 1 ? nullptr : aprev, rho);
  if (rs > 1) launch_reduce_splits(part, (int)rs, a.Io * a.Rz * R, aprev, rho, Y, st);
  return rs > 1 ? 2 : 1;
}

template <typename T>
int launch_y_from_z(const T* Z, const T* Al, const YzArgs& a, double* Y, double* part, const double* aprev,
                    double rho, cudaStream_t st) {
  if (a.long_l) {
    int nl = 0;
    if (a.Rc != a.Ra || a.Rc > 8) throw std::runtime_error("y_from_z: non-uniform bonds need the generic contraction");
    switch (a.Rc) {
      case 1: nl = yzl_go<T, 1>(Z, Al, a, Y, part, aprev, rho, st); break;
      case 2: nl = yzl_go<T, 2>(Z, Al, a, Y, part, aprev, rho, st); break;
      case 3: nl = yzl_go<T, 3>(Z, Al, a, Y, part, aprev, rho, st); break;
      case 4: nl = yzl_go<T, 4>(Z, Al, a, Y, part, aprev, rho, st); break;
      case 5: nl = yzl_go<T, 5>(Z, Al, a, Y, part, aprev, rho, st); break;
      case 6: nl = yzl_go<T, 6>(Z, Al, a, Y, part, aprev, rho, st); break;
      case 7: nl = yzl_go<T, 7>(Z, Al, a, Y, part, aprev, rho, st); break;
      default: nl = yzl_go<T, 8>(Z, Al, a, Y, part, aprev, rho, st); break;
    }
    check_launch("y_from_z_long");
    return nl;
  }
  if (a.Ra > 16) throw std::runtime_error("y_from_z: bond > 16");
  dim3 grid((unsigned)((a.Ir + 255) / 256), (unsigned)a.Rz, (unsigned)a.Rc);
  if (a.Ra <= 8) k_yzs<T, 8><<<grid, 256, 0, st>>>(Z, Al, a, part);
  else k_yzs<T, 16><<<grid, 256, 0, st>>>(Z, Al, a, part);
  check_launch("y_from_z_short");
  launch_reduce_splits(part, a.Rc, a.Ir * a.Rz * a.Ra, aprev, rho, Y, st);
  return 2;
}
template int launch_y_from_z<float>(const float*, const float*, const YzArgs&, double*, double*, const double*, double,
                                    cudaStream_t);
template int launch_y_from_z<double>(const double*, const double*, const YzArgs&, double*, double*, const double*,
                                     double, cudaStream_t);

__global__ void k_convert(const double* __restrict__ in, float* __restrict__ out, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = (float)in[e];
}

__global__ void k_convert_up(const float* __restrict__ in, double* __restrict__ out, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = (double)in[e];
}

void launch_convert_f32_f64(const float* in, double* out, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_convert_up<<<(unsigned)blocks, 256, 0, st>>>(in, out, n);
  check_launch("convert_up");
}

void launch_convert_f64_f32(const double* in, float* out, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_convert<<<(unsigned)blocks, 256, 0, st>>>(in, out, n);
  check_launch("convert");
}

}  // namespace fctn
