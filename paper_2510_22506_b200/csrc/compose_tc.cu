// K4 on the B200 tensor cores: C = A_(k) M_k (network.py:313-332) with tcgen05
// kind::tf32, fused with the P_Omega blend (solver.py:227-237) and the four
// sweep reductions (solver.py:220,346-354,382).  C exists only in TMEM.
//
// The accumulator rows are the contiguous axis of X_(k) so the epilogue's
// X_old loads and X_new stores are coalesced:
//   P > 1  (k > 0): rows = p (M_k columns), cols = i (mode-k rows)
//   P == 1 (k = 0): rows = i, cols = p
// Both operands are MN-major 32-bit tiles (SWIZZLE_128B_BASE32B, TMA 32-B
// atoms) with K = s.  Persistent CTAs (one per SM) walk the tiles with one
// operand stage and a double-buffered TMEM accumulator, so the MMA of tile
// t+1 overlaps the epilogue of tile t; the producer also bulk-prefetches each
// tile's X_old rows into L2 so the epilogue's loads hit L2.
// Warp roles (704 threads): warp 0 TMA (lane 0) + L2 prefetch (all lanes),
// warp 1 TMEM alloc + MMA issue, warps 2..5 TF32 rounding / 3xTF32 split of
// operand tiles that were not pre-split in HBM, warps 6..21 epilogue (four
// warps per TMEM lane quadrant, column quarters).  K = s runs through a ring
// of 32-row stages.
// The observation mask is read bit-packed (1 bit per entry, F order).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace fctn {

CUtensorMap tc_make_map_f32(const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                            const uint32_t* box, bool mn32);
CUtensorMap tc_make_map_f32_plain(const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                                  const uint32_t* box);
CUtensorMap tc_make_map_u32_plain(const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                                  const uint32_t* box);

namespace {

constexpr int KB = 32;  // K rows per pipeline stage
constexpr int CONV_WARPS = 4;
constexpr int EPI_WARPS = 16;
constexpr int CONV0 = 2;                       // first converter warp
constexpr int EPI0 = CONV0 + CONV_WARPS;       // first epilogue warp
constexpr int NWARPS = EPI0 + EPI_WARPS;
constexpr int THREADS = 32 * NWARPS;

struct ComposeArgs {
  const float* Xo;
  float* Xn;
  const uint32_t* maskbits;
  double* partials;
  long long rows, cols;       // accumulator extents (row axis = contiguous axis of X_(k))
  long long n_rb, n_tiles;
  long long P, PI, I;         // X view
  int nkb;                    // K blocks per tile (s padded to 32)
  int stages;
  int rows_are_p;
  int prefetch;               // L2 bulk prefetch of each tile's X_old: 1 rows contiguous per column,
                              // 2 the tile's X block contiguous (rows = p, P == 1), 3 rows = p in
                              // runs of P (P % 128 != 0)
  int a_pre, b_pre;           // operand arrives pre-split (hi and lo tensors) from HBM
  float rho, onep, inv_onep;
  int objective_only;
};

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(p)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Stage layout: [A hi | B hi | A lo | B lo]; A = 128 rows, B = N cols, each
// a set of 32 x 32 MN-major boxes (4 KB, SWIZZLE_128B_BASE32B).
template <int N, bool SPLIT>
__global__ void __launch_bounds__(THREADS, 1)
    k_compose_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmAl,
                 const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmBl,
                 const ComposeArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr uint32_t A_B = 128u * KB * 4u, B_B = (uint32_t)N * KB * 4u;
  constexpr uint32_t HI = A_B + B_B;
  constexpr uint32_t STAGE = HI * (SPLIT ? 2 : 1);
  const int S_ = args.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S_ * STAGE);
  uint64_t* conv = full + S_;
  uint64_t* empty = conv + S_;
  uint64_t* tfull = empty + S_;   // [2]
  uint64_t* tempty = tfull + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ double red[4][NWARPS];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NCOLS = 2 * N <= 32 ? 32 : 2 * N <= 64 ? 64 : 2 * N <= 128 ? 128 : 2 * N <= 256 ? 256 : 512;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
    for (int s = 0; s < S_; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&conv[s], CONV_WARPS);
      tc::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&tfull[s], 1);
      tc::mbar_init(&tempty[s], EPI_WARPS);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<NCOLS>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  double s_d = 0.0, s_b = 0.0, s_c = 0.0, s_n = 0.0;

  if (warp == 0) {
    // ---- TMA producer (lane 0) + L2 prefetch of each tile's X_old rows and
    // mask words (all lanes, paced by the stage ring, so ~one tile ahead of
    // the MMA and two ahead of the epilogue)
    uint32_t tx = HI;
    if (SPLIT) tx += (args.a_pre ? A_B : 0) + (args.b_pre ? B_B : 0);
    int g = 0;
    for (long long t = blockIdx.x; t < args.n_tiles; t += gridDim.x) {
      const int r0 = (int)((t % args.n_rb) * 128), c0 = (int)((t / args.n_rb) * N);
      if (lane == 0) {
        for (int kb = 0; kb < args.nkb; ++kb, ++g) {
          const int s = g % S_;
          tc::mbar_wait(&empty[s], ((g / S_) & 1) ^ 1);
          tc::mbar_expect_tx(&full[s], tx);
          uint8_t* st = smem + s * STAGE;
#pragma unroll
          for (int c = 0; c < 4; ++c) tc::tma_load_2d(st + c * 4096, &tmA, &full[s], r0 + 32 * c, kb * KB);
#pragma unroll
          for (int c = 0; c < N / 32; ++c)
            tc::tma_load_2d(st + A_B + c * 4096, &tmB, &full[s], c0 + 32 * c, kb * KB);
          if (SPLIT && args.a_pre)
#pragma unroll
            for (int c = 0; c < 4; ++c) tc::tma_load_2d(st + HI + c * 4096, &tmAl, &full[s], r0 + 32 * c, kb * KB);
          if (SPLIT && args.b_pre)
#pragma unroll
            for (int c = 0; c < N / 32; ++c)
              tc::tma_load_2d(st + HI + A_B + c * 4096, &tmBl, &full[s], c0 + 32 * c, kb * KB);
        }
      }
      __syncwarp();
      if (args.prefetch == 2) {
        // rows = p with P == 1: the tile's X_old is one contiguous block of
        // nrow * I entries (and nrow * I bits of mask)
        const long long nrow = args.rows - r0 < 128 ? args.rows - r0 : 128;
        const long long base = (long long)r0 * args.I, cnt = nrow * args.I;
        const long long b0 = (base * 4) & ~15LL, b1 = ((base + cnt) * 4 + 15) & ~15LL;
        for (long long o = b0 + (long long)lane * 1024; o < b1; o += 32 * 1024)
          prefetch_l2(reinterpret_cast<const char*>(args.Xo) + o, (uint32_t)(b1 - o < 1024 ? b1 - o : 1024));
        if (!args.objective_only && lane == 0) {
          const long long w0 = (base >> 5) & ~3LL, w1 = ((base + cnt + 31) >> 5) + 4;
          prefetch_l2(args.maskbits + w0, (uint32_t)(((w1 - w0) * 4 + 15) & ~15LL));
        }
      } else if (args.prefetch == 3) {
        // rows = p in runs of P (not 128-aligned): prefetch run segment by segment
        const long long nrow = args.rows - r0 < 128 ? args.rows - r0 : 128;
        for (long long r = r0; r < r0 + nrow;) {
          const long long in = r % args.P;
          const long long seg = (args.P - in) < (r0 + nrow - r) ? (args.P - in) : (r0 + nrow - r);
          const long long rb = in + args.PI * (r / args.P);
          for (int c = lane; c < N; c += 32) {
            const long long gc = c0 + c;
            if (gc >= args.cols) break;
            const long long off = rb + args.P * gc;
            const long long b0 = (off * 4) & ~15LL, b1 = ((off + seg) * 4 + 15) & ~15LL;
            prefetch_l2(reinterpret_cast<const char*>(args.Xo) + b0, (uint32_t)(b1 - b0));
          }
          r += seg;
        }
      } else if (args.prefetch) {
        const long long rbase = args.rows_are_p ? (r0 % args.P) + args.PI * (r0 / args.P) : r0;
        const long long cstride = args.rows_are_p ? args.P : args.I;
        const long long nrow = args.rows - r0 < 128 ? args.rows - r0 : 128;
        for (int c = lane; c < N; c += 32) {
          const long long gc = c0 + c;
          if (gc >= args.cols) break;
          const long long off = rbase + cstride * gc;
          prefetch_l2(args.Xo + off, (uint32_t)(((nrow * 4) + 15) & ~15LL));
          if (!args.objective_only)
            prefetch_l2(reinterpret_cast<const void*>(reinterpret_cast<uintptr_t>(args.maskbits + (off >> 5)) &
                                                      ~uintptr_t(15)),
                        32);
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer
    constexpr uint32_t idesc = tc::idesc_tf32(128, N, true, true);
    int g = 0, j = 0;
    for (long long t = blockIdx.x; t < args.n_tiles; t += gridDim.x, ++j) {
      const int acc = j & 1;
      tc::mbar_wait(&tempty[acc], ((j >> 1) & 1) ^ 1);
      for (int kb = 0; kb < args.nkb; ++kb, ++g) {
        const int s = g % S_;
        tc::mbar_wait(&conv[s], (g / S_) & 1);
        tc::fence_after_sync();
        const uint32_t a = tc::smem_u32(smem + s * STAGE), b = a + A_B;
#pragma unroll
        for (int kk = 0; kk < KB / 8; ++kk) {
          const uint64_t ad = tc::sdesc(a + kk * 1024, 4096, 512, 1);
          const uint64_t bd = tc::sdesc(b + kk * 1024, 4096, 512, 1);
          const uint32_t first = (kb | kk) != 0;
          if (SPLIT) {
            tc::mma_tf32(tmem + acc * N, tc::sdesc(a + HI + kk * 1024, 4096, 512, 1), bd, idesc, first);
            tc::mma_tf32(tmem + acc * N, ad, tc::sdesc(b + HI + kk * 1024, 4096, 512, 1), idesc, 1);
          }
          tc::mma_tf32(tmem + acc * N, ad, bd, idesc, SPLIT ? 1u : first);
        }
        tc::mma_commit(&empty[s]);
      }
      tc::mma_commit(&tfull[acc]);
    }
  } else if (warp >= CONV0 && warp < EPI0) {
    // ---- operand rounding (TF32 round-to-nearest) or 3xTF32 hi/lo split of
    // the operands that did not arrive pre-split
    const int ct = threadIdx.x - 32 * CONV0;
    int g = 0;
    for (long long t = blockIdx.x; t < args.n_tiles; t += gridDim.x) {
      for (int kb = 0; kb < args.nkb; ++kb, ++g) {
        const int s = g % S_;
        tc::mbar_wait(&full[s], (g / S_) & 1);
        uint8_t* st = smem + s * STAGE;
        if (!args.a_pre) tc::tf32_split_tile<SPLIT>(st, st + HI, (int)(A_B / 4), ct, 32 * CONV_WARPS);
        if (!args.b_pre) tc::tf32_split_tile<SPLIT>(st + A_B, st + HI + A_B, (int)(B_B / 4), ct, 32 * CONV_WARPS);
        tc::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&conv[s]);
      }
    }
  } else if (warp >= EPI0) {
    // ---- epilogue: TMEM -> registers, blend with X_old, write X_new, reduce
    const int ew = warp - EPI0;
    const int quad = warp & 3;
    const int part = ew >> 2;                  // column quarter of this warp
    constexpr int CW = N / 4;                  // columns per warp (multiple of 16)
    const int row = 32 * quad + lane;
    int j = 0;
    for (long long t = blockIdx.x; t < args.n_tiles; t += gridDim.x, ++j) {
      const int acc = j & 1;
      tc::mbar_wait(&tfull[acc], (j >> 1) & 1);
      tc::fence_after_sync();
      const long long gr = (t % args.n_rb) * 128 + row;
      const long long cb = (t / args.n_rb) * N + part * CW;
      const bool row_ok = gr < args.rows;
      const long long rowbase = args.rows_are_p ? (gr % args.P) + args.PI * (gr / args.P) : gr;
      const long long colstride = args.rows_are_p ? args.P : args.I;
      const uint32_t taddr = tmem + acc * N + ((uint32_t)(32 * quad) << 16) + part * CW;
      float f_d = 0.f, f_b = 0.f, f_c = 0.f, f_n = 0.f;  // per-tile partials (fp32), folded into fp64
#pragma unroll 1
      for (int c0 = 0; c0 < CW; c0 += 16) {
        uint32_t r[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr + c0));
        float x[16];
        uint32_t mw[16];
        const long long off0 = rowbase + colstride * (cb + c0);
        const long long rem = args.cols - (cb + c0);
        const int nc = rem < 16 ? (int)rem : 16;
        // a row's 16 columns contiguous and 16-B aligned (rows = p with P == 1,
        // c5's k = 0): four 16-B loads instead of sixteen 4-B ones
        const bool vec = colstride == 1 && nc == 16 && (off0 & 3) == 0;
        if (vec && row_ok) {
          const float4* src = reinterpret_cast<const float4*>(args.Xo + off0);
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const float4 t = __ldcs(src + v);
            x[4 * v] = t.x;
            x[4 * v + 1] = t.y;
            x[4 * v + 2] = t.z;
            x[4 * v + 3] = t.w;
          }
          const uint32_t w0 = args.objective_only ? 0u : __ldg(args.maskbits + (off0 >> 5));
          const uint32_t w1 = args.objective_only ? 0u : __ldg(args.maskbits + ((off0 + 15) >> 5));
#pragma unroll
          for (int q = 0; q < 16; ++q) mw[q] = ((off0 + q) >> 5) == (off0 >> 5) ? w0 : w1;
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q) {  // all loads in flight before the TMEM wait
            const long long off = off0 + colstride * q;
            x[q] = (row_ok && q < nc) ? __ldcs(args.Xo + off) : 0.0f;
            mw[q] = (row_ok && q < nc && !args.objective_only) ? __ldg(args.maskbits + (off >> 5)) : 0u;
          }
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (!row_ok) continue;
        float xo[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          if (q >= nc) break;
          const long long off = off0 + colstride * q;
          const float c = __uint_as_float(r[q]);
          if (args.objective_only) {
            const float d = x[q] - c;
            f_c += d * d;
          } else {
            float xn;
            if ((mw[q] >> (off & 31)) & 1u) {
              xn = x[q];  // observed entries restored bit for bit (solver.py:235-236)
            } else {
              // (x*rho + c)/(1+rho) (solver.py:232-234); the fp32 variant
              // multiplies by the rounded reciprocal (<= 1 ulp)
              xn = fmaf(x[q], args.rho, c) * args.inv_onep;
            }
            if (vec) xo[q] = xn;
            else __stcs(args.Xn + off, xn);
            const float dx = xn - x[q], dc = xn - c;
            f_d += dx * dx;
            f_b += x[q] * x[q];
            f_c += dc * dc;
            f_n += xn * xn;
          }
        }
        if (vec && !args.objective_only) {
          float4* dst = reinterpret_cast<float4*>(args.Xn + off0);
#pragma unroll
          for (int v = 0; v < 4; ++v) __stcs(dst + v, make_float4(xo[4 * v], xo[4 * v + 1], xo[4 * v + 2], xo[4 * v + 3]));
        }
      }
      s_d += (double)f_d;
      s_b += (double)f_b;
      s_c += (double)f_c;
      s_n += (double)f_n;
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
  }
  // fixed-order reduction: warp shuffle tree, then warps in index order
  s_d = warp_sum(s_d);
  s_b = warp_sum(s_b);
  s_c = warp_sum(s_c);
  s_n = warp_sum(s_n);
  if (lane == 0) {
    red[0][warp] = s_d;
    red[1][warp] = s_b;
    red[2][warp] = s_c;
    red[3][warp] = s_n;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 4) {
    double v = 0.0;
    for (int q = 0; q < NWARPS; ++q) v += red[threadIdx.x][q];
    args.partials[blockIdx.x * 4 + threadIdx.x] = v;
  }
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc<NCOLS>(tmem);
  }
}

// ---------------------------------------------------------------------------
// TMA-ring variant (X views TMA can describe): the epilogue never touches
// global memory for X.  A producer warp streams X_old sub-tiles (128 rows x
// 32 columns, 16 KB) into a ring of shared-memory slots; the epilogue blends
// each slot in place and one thread TMA-stores it back as X_new, keeping a
// few bulk groups in flight.  The bulk engines, not registers, hold the bytes
// in flight.  Operands stream through 16-row K stages.
// K rows per operand stage: 8 (one K=8 MMA step) for wide tiles; 16 or 32 for
// narrow ones (c5: N = 64), where with K = 8 each 3-MMA stage paid a full
// barrier / fence / commit round trip (ncu: tensor pipe 10 %, epilogue
// waiting on the MMA 45 %)
constexpr int KB2 = 8;
template <int KB>
__host__ __device__ constexpr int boxb() { return 32 * KB * 4; }  // bytes of one 32-row MN-major operand box
constexpr int XC = 32;       // columns per X sub-tile
constexpr int XS_DEFAULT = 9;  // X ring slots
constexpr int XKEEP = 3;     // TMA stores allowed in flight
constexpr int T_CONV0 = 3, T_EPI0 = T_CONV0 + CONV_WARPS, T_NWARPS = T_EPI0 + EPI_WARPS;
constexpr int T_THREADS = 32 * T_NWARPS;
constexpr int XBYTES = 128 * XC * 4;
constexpr int MBYTES = XC * 4 * 4;  // mask bits of a sub-tile: 4 words (128 rows) per column

struct ComposeTmaArgs {
  const uint32_t* maskbits;
  double* partials;
  long long rows, cols, n_rb, n_tiles;
  long long P, PI, I;
  int nkb;                     // K stages per tile
  int rows_are_p;
  int a_pre, b_pre;
  float rho, inv_onep;
  int objective_only;
  int op3d;  // operand maps are 3-D [32, S, extent/32] views: one TMA per operand per stage
};

template <int N>
__device__ __forceinline__ void x_coords(const ComposeTmaArgs& a, long long t, int j, int& c0, int& c1, int& c2) {
  const long long r0 = (t % a.n_rb) * 128, col = (t / a.n_rb) * N + (long long)j * XC;
  if (a.rows_are_p) {  // 3-D view (P, I, Q): rows = fastest-mode run, cols = i
    c0 = (int)(r0 % a.P);
    c1 = (int)col;
    c2 = (int)(r0 / a.P);
  } else {             // 2-D view (I, p): rows = i, cols = p
    c0 = (int)r0;
    c1 = (int)col;
    c2 = 0;
  }
}

// shared memory: OPS operand stages + XS X/mask slots + barriers; the
// operand ring takes whatever the X ring leaves of the 227 KB
constexpr int T_SMEM_MAX = 232448 - 1024 /*static red[]*/;
constexpr int T_TAIL = 1024 /*align*/ + 512 /*barriers*/;
template <int N, bool SPLIT, int KB = KB2>
__host__ __device__ constexpr int t_stage() { return (128 + N) * KB * 4 * (SPLIT ? 2 : 1); }
template <int N, bool SPLIT, int XS, int KB = KB2>
__host__ __device__ constexpr int t_ops() {
  constexpr int o = (T_SMEM_MAX - T_TAIL - XS * (XBYTES + MBYTES)) / t_stage<N, SPLIT, KB>();
  return o > 8 ? 8 : o;
}

template <int N, bool SPLIT, int XS, int KB>
__global__ void __launch_bounds__(T_THREADS, 1)
    k_compose_tma(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmAl,
                  const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmBl,
                  const __grid_constant__ CUtensorMap tmXo, const __grid_constant__ CUtensorMap tmXn,
                  const __grid_constant__ CUtensorMap tmMask, const ComposeTmaArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr uint32_t A_B = 128u * KB * 4u, B_B = (uint32_t)N * KB * 4u;
  constexpr int BOXB = boxb<KB>();
  constexpr uint32_t HI = A_B + B_B;
  constexpr uint32_t STAGE = HI * (SPLIT ? 2 : 1);
  constexpr int OPS = t_ops<N, SPLIT, XS, KB>();
  static_assert(OPS >= 2, "operand ring");
  uint8_t* xring = smem + OPS * STAGE;
  uint32_t* mring = reinterpret_cast<uint32_t*>(xring + XS * XBYTES);  // [XS][XC][4] mask words
  uint64_t* full = reinterpret_cast<uint64_t*>(xring + XS * (XBYTES + MBYTES));
  uint64_t* conv = full + OPS;
  uint64_t* empty = conv + OPS;
  uint64_t* tfull = empty + OPS;   // [2]
  uint64_t* tempty = tfull + 2;    // [2]
  uint64_t* xfull = tempty + 2;    // [XS]
  uint64_t* xempty = xfull + XS;   // [XS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xempty + XS);
  __shared__ double red[4][T_NWARPS];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NCOLS = 2 * N <= 32 ? 32 : 2 * N <= 64 ? 64 : 2 * N <= 128 ? 128 : 2 * N <= 256 ? 256 : 512;
  constexpr int NX = N / XC;  // X sub-tiles per tile

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
    tc::tma_prefetch(&tmXo);
    tc::tma_prefetch(&tmXn);
    for (int s = 0; s < OPS; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&conv[s], CONV_WARPS);
      tc::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&tfull[s], 1);
      tc::mbar_init(&tempty[s], EPI_WARPS);
    }
    for (int s = 0; s < XS; ++s) {
      tc::mbar_init(&xfull[s], 1);
      tc::mbar_init(&xempty[s], 1);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<NCOLS>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  double s_d = 0.0, s_b = 0.0, s_c = 0.0, s_n = 0.0;

  if (warp == 0 && lane == 0) {
    // ---- operand producer
    uint32_t tx = HI;
    if (SPLIT) tx += (args.a_pre ? A_B : 0) + (args.b_pre ? B_B : 0);
    int g = 0;
    for (long long t = blockIdx.x; t < args.n_tiles; t += gridDim.x) {
      const int r0 = (int)((t % args.n_rb) * 128), c0 = (int)((t / args.n_rb) * N);
      for (int kb = 0; kb < args.nkb; ++kb, ++g) {
        const int s = g % OPS;
        tc::mbar_wait(&empty[s], ((g / OPS) & 1) ^ 1);
        tc::mbar_expect_tx(&full[s], tx);
        uint8_t* st = smem + s * STAGE;
        if (args.op3d) {  // box [32 rows, KB2, chunks] lands as chunk-major 1 KB boxes
          tc::tma_load_3d(st, &tmA, &full[s], 0, kb * KB, r0 / 32);
          tc::tma_load_3d(st + A_B, &tmB, &full[s], 0, kb * KB, c0 / 32);
          if (SPLIT && args.a_pre) tc::tma_load_3d(st + HI, &tmAl, &full[s], 0, kb * KB, r0 / 32);
          if (SPLIT && args.b_pre) tc::tma_load_3d(st + HI + A_B, &tmBl, &full[s], 0, kb * KB, c0 / 32);
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) tc::tma_load_2d(st + c * BOXB, &tmA, &full[s], r0 + 32 * c, kb * KB);
#pragma unroll
          for (int c = 0; c < N / 32; ++c)
            tc::tma_load_2d(st + A_B + c * BOXB, &tmB, &full[s], c0 + 32 * c, kb * KB);
          if (SPLIT && args.a_pre)
#pragma unroll
            for (int c = 0; c < 4; ++c) tc::tma_load_2d(st + HI + c * BOXB, &tmAl, &full[s], r0 + 32 * c, kb * KB);
          if (SPLIT && args.b_pre)
#pragma unroll
            for (int c = 0; c < N / 32; ++c)
              tc::tma_load_2d(st + HI + A_B + c * BOXB, &tmBl, &full[s], c0 + 32 * c, kb * KB);
        }
      }
    }
  } else if (warp == 2 && lane == 0) {
    // ---- X_old producer: sub-tiles into the ring
    int g = 0;
    for (long long t = blockIdx.x; t < args.n_tiles; t += gridDim.x) {
      for (int j = 0; j < NX; ++j, ++g) {
        const int s = g % XS;
        tc::mbar_wait(&xempty[s], ((g / XS) & 1) ^ 1);
        tc::mbar_expect_tx(&xfull[s], XBYTES + (args.objective_only ? 0 : MBYTES));
        int c0, c1, c2;
        x_coords<N>(args, t, j, c0, c1, c2);
        if (args.rows_are_p) {
          tc::tma_load_3d(xring + s * XBYTES, &tmXo, &xfull[s], c0, c1, c2);
          if (!args.objective_only) tc::tma_load_3d(mring + s * (MBYTES / 4), &tmMask, &xfull[s], c0 / 32, c1, c2);
        } else {
          tc::tma_load_2d(xring + s * XBYTES, &tmXo, &xfull[s], c0, c1);
          if (!args.objective_only) tc::tma_load_2d(mring + s * (MBYTES / 4), &tmMask, &xfull[s], c0 / 32, c1);
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer
    constexpr uint32_t idesc = tc::idesc_tf32(128, N, true, true);
    int g = 0, j = 0;
    for (long long t = blockIdx.x; t < args.n_tiles; t += gridDim.x, ++j) {
      const int acc = j & 1;
      tc::mbar_wait(&tempty[acc], ((j >> 1) & 1) ^ 1);
      for (int kb = 0; kb < args.nkb; ++kb, ++g) {
        const int s = g % OPS;
        tc::mbar_wait(&conv[s], (g / OPS) & 1);
        tc::fence_after_sync();
        const uint32_t a = tc::smem_u32(smem + s * STAGE), b = a + A_B;
#pragma unroll
        for (int kk = 0; kk < KB / 8; ++kk) {
          const uint64_t ad = tc::sdesc(a + kk * 1024, BOXB, 512, 1);
          const uint64_t bd = tc::sdesc(b + kk * 1024, BOXB, 512, 1);
          const uint32_t first = (kb | kk) != 0;
          if (SPLIT) {
            tc::mma_tf32(tmem + acc * N, tc::sdesc(a + HI + kk * 1024, BOXB, 512, 1), bd, idesc, first);
            tc::mma_tf32(tmem + acc * N, ad, tc::sdesc(b + HI + kk * 1024, BOXB, 512, 1), idesc, 1);
          }
          tc::mma_tf32(tmem + acc * N, ad, bd, idesc, SPLIT ? 1u : first);
        }
        tc::mma_commit(&empty[s]);
      }
      tc::mma_commit(&tfull[acc]);
    }
  } else if (warp >= T_CONV0 && warp < T_EPI0) {
    // ---- operand rounding / 3xTF32 split of operands not pre-split in HBM
    const int ct = threadIdx.x - 32 * T_CONV0;
    int g = 0;
    for (long long t = blockIdx.x; t < args.n_tiles; t += gridDim.x) {
      for (int kb = 0; kb < args.nkb; ++kb, ++g) {
        const int s = g % OPS;
        tc::mbar_wait(&full[s], (g / OPS) & 1);
        uint8_t* st = smem + s * STAGE;
        if (!args.a_pre) tc::tf32_split_tile<SPLIT>(st, st + HI, (int)(A_B / 4), ct, 32 * CONV_WARPS);
        if (!args.b_pre) tc::tf32_split_tile<SPLIT>(st + A_B, st + HI + A_B, (int)(B_B / 4), ct, 32 * CONV_WARPS);
        tc::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&conv[s]);
      }
    }
  } else if (warp >= T_EPI0) {
    // ---- epilogue: per X sub-tile, warp (quad, part) blends 32 rows x 8 cols
    const int ew = warp - T_EPI0;
    const int quad = warp & 3;
    const int part = ew >> 2;
    const int row = 32 * quad + lane;
    const bool leader = (ew == 0 && lane == 0);
    int g = 0, j = 0;
    for (long long t = blockIdx.x; t < args.n_tiles; t += gridDim.x, ++j) {
      const int acc = j & 1;
      tc::mbar_wait(&tfull[acc], (j >> 1) & 1);
      tc::fence_after_sync();
      const long long gr = (t % args.n_rb) * 128 + row;
      const bool row_ok = gr < args.rows;
      const long long rowbase = args.rows_are_p ? (gr % args.P) + args.PI * (gr / args.P) : gr;
      const long long colstride = args.rows_are_p ? args.P : args.I;
      float f_d = 0.f, f_b = 0.f, f_c = 0.f, f_n = 0.f;
      for (int xj = 0; xj < NX; ++xj, ++g) {
        const int s = g % XS;
        const int col0 = xj * XC + part * 8;                  // column within the tile
        const long long gc0 = (t / args.n_rb) * N + col0;     // global column
        uint32_t r[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                       "=r"(r[7])
                     : "r"(tmem + acc * N + ((uint32_t)(32 * quad) << 16) + col0));
        tc::mbar_wait(&xfull[s], (g / XS) & 1);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float* xs = reinterpret_cast<float*>(xring + s * XBYTES);
        const uint32_t* ms = mring + s * (MBYTES / 4);  // [col][4 words]
        if (row_ok) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (gc0 + q >= args.cols) break;
            float* px = xs + (part * 8 + q) * 128 + row;
            const float x = *px;
            const float c = __uint_as_float(r[q]);
            if (args.objective_only) {
              const float d = x - c;
              f_c += d * d;
            } else {
              const uint32_t mw = ms[(part * 8 + q) * 4 + (row >> 5)];  // warp-uniform word
              float xn;
              if ((mw >> (row & 31)) & 1u) {
                xn = x;  // observed entries restored bit for bit (solver.py:235-236)
              } else {
                xn = fmaf(x, args.rho, c) * args.inv_onep;  // solver.py:232-234 (fp32: reciprocal, <= 1 ulp)
              }
              *px = xn;
              const float dx = xn - x, dc = xn - c;
              f_d += dx * dx;
              f_b += x * x;
              f_c += dc * dc;
              f_n += xn * xn;
            }
          }
        }
        // all epilogue warps done with this slot -> one thread stores it
        tc::fence_proxy_async_smem();
        tc::named_bar(1, 32 * EPI_WARPS);
        if (leader) {
          if (!args.objective_only) {
            int c0, c1, c2;
            x_coords<N>(args, t, xj, c0, c1, c2);
            if (args.rows_are_p)
              tc::tma_store_3d(&tmXn, xs, c0, c1, c2);
            else
              tc::tma_store_2d(&tmXn, xs, c0, c1);
          }
          tc::bulk_commit();
          constexpr int XK = XS >= 7 ? XKEEP : 2;
          tc::bulk_wait_read<XK>();
          if (g >= XK) tc::mbar_arrive(&xempty[(g - XK) % XS]);
        }
      }
      s_d += (double)f_d;
      s_b += (double)f_b;
      s_c += (double)f_c;
      s_n += (double)f_n;
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
    if (leader) tc::bulk_wait<0>();  // X_new fully written before exit
  }
  s_d = warp_sum(s_d);
  s_b = warp_sum(s_b);
  s_c = warp_sum(s_c);
  s_n = warp_sum(s_n);
  if (lane == 0) {
    red[0][warp] = s_d;
    red[1][warp] = s_b;
    red[2][warp] = s_c;
    red[3][warp] = s_n;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 4) {
    double v = 0.0;
    for (int q = 0; q < T_NWARPS; ++q) v += red[threadIdx.x][q];
    args.partials[blockIdx.x * 4 + threadIdx.x] = v;
  }
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc<NCOLS>(tmem);
  }
}

template <int N, bool SPLIT, int XS, int KB>
int go_tma_xs(const CUtensorMap* maps, const ComposeTmaArgs& a, int grid, cudaStream_t st) {
  const int smem = t_ops<N, SPLIT, XS, KB>() * t_stage<N, SPLIT, KB>() + XS * (XBYTES + MBYTES) + T_TAIL;
  auto fn = k_compose_tma<N, SPLIT, XS, KB>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) throw std::runtime_error(std::string("compose_tma smem: ") + cudaGetErrorString(e));
  fn<<<grid, T_THREADS, smem, st>>>(maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], maps[6], a);
  e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("compose_tma: ") + cudaGetErrorString(e));
  return grid;
}

int compose_xs() {
  static const int v = [] {
    const char* e = getenv("FCTN_COMPOSE_XS");
    const int x = e ? atoi(e) : XS_DEFAULT;
    return (x == 5 || x == 7) ? x : 9;
  }();
  return v;
}

// K rows per operand stage for an N-wide tile (FCTN_COMPOSE_KB overrides for N = 64)
int compose_kb(int N) {
  static const int env = [] {
    const char* e = getenv("FCTN_COMPOSE_KB");
    const int x = e ? atoi(e) : 0;
    return (x == 8 || x == 16 || x == 32) ? x : 0;
  }();
  if (N != 64) return KB2;
  return env ? env : 16;
}

template <int N, bool SPLIT>
int go_tma(const CUtensorMap* maps, const ComposeTmaArgs& a, int grid, cudaStream_t st) {
  if constexpr (N == 64) {
    const int kb = compose_kb(N);
    if (kb == 16) return go_tma_xs<N, SPLIT, 5, 16>(maps, a, grid, st);
    if (kb == 32) return go_tma_xs<N, SPLIT, 5, 32>(maps, a, grid, st);
  }
  switch (compose_xs()) {
    case 5: return go_tma_xs<N, SPLIT, 5, KB2>(maps, a, grid, st);
    case 7: return go_tma_xs<N, SPLIT, 7, KB2>(maps, a, grid, st);
    default: return go_tma_xs<N, SPLIT, 9, KB2>(maps, a, grid, st);
  }
}

template <int N, bool SPLIT>
int go2(const CUtensorMap* maps, ComposeArgs a, int grid, cudaStream_t st) {
  constexpr int STAGE = (128 + N) * KB * 4 * (SPLIT ? 2 : 1);
  a.stages = std::min(4, (200 * 1024) / STAGE);
  if (a.stages < 1) throw std::runtime_error("compose_tc: tile does not fit in shared memory");
  const int smem = a.stages * STAGE + 1024 + 256;
  auto fn = k_compose_tc<N, SPLIT>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) throw std::runtime_error(std::string("compose_tc smem: ") + cudaGetErrorString(e));
  fn<<<grid, THREADS, smem, st>>>(maps[0], maps[1], maps[2], maps[3], a);
  e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("compose_tc: ") + cudaGetErrorString(e));
  return grid;
}

template <int N>
int go(const CUtensorMap* maps, const ComposeArgs& a, int grid, bool split3, cudaStream_t st) {
  return split3 ? go2<N, true>(maps, a, grid, st) : go2<N, false>(maps, a, grid, st);
}

}  // namespace

bool tc_compose_supported(int64_t I, int64_t P, int64_t p, int64_t S) {
  if (S > 128) return false;
  if (I % 4 != 0 || p % 4 != 0) return false;  // TMA row strides of A_(k) [I, S] and M [p, S]
  if (I > (1LL << 31) || p > (1LL << 31)) return false;
  (void)P;
  return true;
}

int launch_compose_tc(const ComposeOperands& op, const float* Xo, const uint32_t* maskbits, float* Xn, int64_t I,
                      int64_t P, int64_t S, int64_t p, double rho, bool objective_only, double* partials,
                      int64_t partial_cap, int n_sm, bool split3, cudaStream_t st) {
  ComposeArgs a;
  a.Xo = Xo;
  a.Xn = Xn;
  a.maskbits = maskbits;
  a.partials = partials;
  a.P = P;
  a.PI = P * I;
  a.I = I;
  a.nkb = (int)((S + KB - 1) / KB);
  // accumulator rows = the contiguous axis of X_(k) when it spans a 128-row
  // tile (i for k = 0, p for k > 0); a short mode 0 (I < 128, c5: 48) takes
  // rows = p instead, so the MMA's 128 rows are all live (with rows = i only
  // I of 128 were)
  static const bool rows_i = getenv("FCTN_COMPOSE_ROWS_I") != nullptr;  // A/B: the former rows = i for k = 0
  a.rows_are_p = P > 1 || (I < 128 && !rows_i);
  a.rho = (float)rho;
  a.onep = (float)(1.0 + rho);
  a.inv_onep = (float)(1.0 / (1.0 + rho));
  a.objective_only = objective_only ? 1 : 0;
  a.rows = a.rows_are_p ? p : I;
  a.cols = a.rows_are_p ? I : p;
  int N = 256;
  if (a.rows_are_p) {
    N = (int)((I + 63) / 64 * 64);  // epilogue warps take N/4 columns in chunks of 16
    if (N > 256) N = 256;
  }
  a.n_rb = (a.rows + 127) / 128;
  // a tile's 128 rows are one contiguous run of X when rows = i, or rows = p
  // within one run of the fastest modes (P a multiple of 128)
  a.prefetch = (!a.rows_are_p || P % 128 == 0) ? 1 : (P == 1 ? 2 : 3);
  const long long n_cb = (a.cols + N - 1) / N;
  a.n_tiles = a.n_rb * n_cb;
  int grid = (int)std::min<long long>(a.n_tiles, n_sm);
  if (grid > partial_cap) throw std::runtime_error("compose partial buffer too small");
  // the rows operand and the cols operand, each [extent, S] 32-bit MN-major;
  // "pre" tensors: hi = rn_tf32(x), lo = x - hi already in HBM
  const float* Mh = op.m_hi ? op.m_hi : op.m;
  const float* Ah = op.a_hi ? op.a_hi : op.a;
  uint64_t dm[2] = {(uint64_t)p, (uint64_t)S}, sm_[1] = {(uint64_t)p * 4};
  uint64_t da[2] = {(uint64_t)I, (uint64_t)S}, sa[1] = {(uint64_t)I * 4};
  uint32_t box[2] = {32, KB};
  CUtensorMap mM = tc_make_map_f32(Mh, 2, dm, sm_, box, true);
  CUtensorMap mMl = op.m_lo ? tc_make_map_f32(op.m_lo, 2, dm, sm_, box, true) : mM;
  CUtensorMap mA = tc_make_map_f32(Ah, 2, da, sa, box, true);
  CUtensorMap mAl = op.a_lo ? tc_make_map_f32(op.a_lo, 2, da, sa, box, true) : mA;
  const bool m_pre = op.m_hi != nullptr && (op.m_lo != nullptr || !split3);
  const bool a_pre = op.a_hi != nullptr && (op.a_lo != nullptr || !split3);
  CUtensorMap maps[7];
  if (a.rows_are_p) {
    maps[0] = mM; maps[1] = mMl; maps[2] = mA; maps[3] = mAl;
    a.a_pre = m_pre; a.b_pre = a_pre;
  } else {
    maps[0] = mA; maps[1] = mAl; maps[2] = mM; maps[3] = mMl;
    a.a_pre = a_pre; a.b_pre = m_pre;
  }
  // TMA-ring variant when TMA can describe the X tiles (rows = a contiguous
  // run of 128): rows = i (P == 1), or rows = p inside runs of P (P % 128 == 0)
  // (the mask words ride along by TMA too: rows must start on 32-entry words)
  const bool tma_x = ((!a.rows_are_p && I % 128 == 0) || (a.rows_are_p && P % 128 == 0)) &&
                     !getenv("FCTN_COMPOSE_DIRECT");
  if (tma_x) {
    ComposeTmaArgs t;
    t.maskbits = maskbits;
    t.partials = partials;
    t.rows = a.rows;
    t.cols = a.cols;
    t.n_rb = a.n_rb;
    t.n_tiles = a.n_tiles;
    t.P = P;
    t.PI = P * I;
    t.I = I;
    if (N % XC != 0) N = (N + XC - 1) / XC * XC;
    const uint32_t kbr = (uint32_t)compose_kb(N);  // K rows per operand stage
    t.nkb = (int)((S + kbr - 1) / kbr);
    t.rows_are_p = a.rows_are_p;
    t.a_pre = a.a_pre;
    t.b_pre = a.b_pre;
    t.rho = a.rho;
    t.inv_onep = a.inv_onep;
    t.objective_only = a.objective_only;
    if (N % XC != 0) N = (N + XC - 1) / XC * XC;
    // operand maps with KB2-row K boxes; when both extents are multiples of 32
    // a 3-D view [32, S, extent / 32] fetches a whole stage operand in one TMA
    t.op3d = (p % 32 == 0 && I % 32 == 0 && !getenv("FCTN_COMPOSE_OP2D")) ? 1 : 0;
    const uint32_t nb_m = a.rows_are_p ? 4u : (uint32_t)(N / 32), nb_a = a.rows_are_p ? (uint32_t)(N / 32) : 4u;
    auto mk = [&](const float* base, int64_t ext, uint32_t nb) {
      if (t.op3d) {
        uint64_t d[3] = {32, (uint64_t)S, (uint64_t)(ext / 32)}, sd[2] = {(uint64_t)ext * 4, 128};
        uint32_t b[3] = {32, kbr, nb};
        return tc_make_map_f32(base, 3, d, sd, b, true);
      }
      uint64_t d[2] = {(uint64_t)ext, (uint64_t)S}, sd[1] = {(uint64_t)ext * 4};
      uint32_t b[2] = {32, kbr};
      return tc_make_map_f32(base, 2, d, sd, b, true);
    };
    CUtensorMap tM = mk(Mh, p, nb_m);
    CUtensorMap tMl = op.m_lo ? mk(op.m_lo, p, nb_m) : tM;
    CUtensorMap tA = mk(Ah, I, nb_a);
    CUtensorMap tAl = op.a_lo ? mk(op.a_lo, I, nb_a) : tA;
    if (a.rows_are_p) {
      maps[0] = tM; maps[1] = tMl; maps[2] = tA; maps[3] = tAl;
    } else {
      maps[0] = tA; maps[1] = tAl; maps[2] = tM; maps[3] = tMl;
    }
    if (a.rows_are_p) {
      const uint64_t Q = (uint64_t)(p / P);
      uint64_t dx[3] = {(uint64_t)P, (uint64_t)I, Q}, sx[2] = {(uint64_t)P * 4, (uint64_t)P * I * 4};
      uint32_t bx[3] = {128, XC, 1};
      maps[4] = tc_make_map_f32_plain(Xo, 3, dx, sx, bx);
      maps[5] = tc_make_map_f32_plain(Xn, 3, dx, sx, bx);
      uint64_t dmk[3] = {(uint64_t)(P / 32), (uint64_t)I, Q}, smk[2] = {(uint64_t)(P / 32) * 4, (uint64_t)(P / 32) * I * 4};
      uint32_t bmk[3] = {4, XC, 1};
      maps[6] = tc_make_map_u32_plain(maskbits, 3, dmk, smk, bmk);
    } else {
      uint64_t dx[2] = {(uint64_t)I, (uint64_t)p}, sx[1] = {(uint64_t)I * 4};
      uint32_t bx[2] = {128, XC};
      maps[4] = tc_make_map_f32_plain(Xo, 2, dx, sx, bx);
      maps[5] = tc_make_map_f32_plain(Xn, 2, dx, sx, bx);
      uint64_t dmk[2] = {(uint64_t)(I / 32), (uint64_t)p}, smk[1] = {(uint64_t)(I / 32) * 4};
      uint32_t bmk[2] = {4, XC};
      maps[6] = tc_make_map_u32_plain(maskbits, 2, dmk, smk, bmk);
    }
    if (N % XC != 0) N = (N + XC - 1) / XC * XC;
    switch (N) {
      case 64: return split3 ? go_tma<64, true>(maps, t, grid, st) : go_tma<64, false>(maps, t, grid, st);
      case 128: return split3 ? go_tma<128, true>(maps, t, grid, st) : go_tma<128, false>(maps, t, grid, st);
      case 192: return split3 ? go_tma<192, true>(maps, t, grid, st) : go_tma<192, false>(maps, t, grid, st);
      default: return split3 ? go_tma<256, true>(maps, t, grid, st) : go_tma<256, false>(maps, t, grid, st);
    }
  }
  switch (N) {
    case 64: return go<64>(maps, a, grid, split3, st);
    case 128: return go<128>(maps, a, grid, split3, st);
    case 192: return go<192>(maps, a, grid, split3, st);
    default: return go<256>(maps, a, grid, split3, st);
  }
}

// hi = rn_tf32(x), lo = x - hi (lo may be null: round only)
__global__ void k_tf32_split(const float* __restrict__ x, float* __restrict__ hi, float* __restrict__ lo, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[e];
    const float h = tc::tf32_rn(v);
    hi[e] = h;
    if (lo) lo[e] = v - h;
  }
}

void launch_tf32_split(const float* x, float* hi, float* lo, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_tf32_split<<<(unsigned)blocks, 256, 0, st>>>(x, hi, lo, n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("tf32_split: ") + cudaGetErrorString(e));
}

// 1 bit per entry, F order: bits[w] bit b <-> mask[32 w + b]
__global__ void k_pack_mask(const uint8_t* __restrict__ mask, int64_t T, uint32_t* __restrict__ bits) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w * 32 >= T) return;
  uint32_t v = 0;
  for (int b = 0; b < 32; ++b) {
    const int64_t e = w * 32 + b;
    if (e < T && mask[e]) v |= 1u << b;
  }
  bits[w] = v;
}

void launch_pack_mask(const uint8_t* mask, int64_t T, uint32_t* bits, cudaStream_t st) {
  const int64_t words = (T + 31) / 32;
  k_pack_mask<<<(unsigned)((words + 255) / 256), 256, 0, st>>>(mask, T, bits);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("pack_mask: ") + cudaGetErrorString(e));
}

}  // namespace fctn
