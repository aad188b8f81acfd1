// K4 on the B200 tensor cores: C = A_(k) M_k (network.py:313-332) with tcgen05
// kind::tf32, fused with the P_Omega blend (solver.py:227-237) and the four
// sweep reductions (solver.py:220,346-354,382).  C exists only in TMEM.
//
// The accumulator rows are the contiguous axis of X_(k) so the epilogue's
// X_old loads and X_new stores are coalesced:
//   P > 1  (k > 0): rows = p (M_k columns), cols = i (mode-k rows)
//   P == 1 (k = 0): rows = i, cols = p
// Both operands are MN-major 32-bit tiles (SWIZZLE_128B_BASE32B, TMA 32-B
// atoms) with K = s.  Persistent CTAs (one per SM) walk the tiles with a
// 2-stage smem ring and a double-buffered TMEM accumulator, so the MMA of
// tile t+1 overlaps the epilogue of tile t.
// Warp roles (448 threads): warp 0 TMA, warp 1 TMEM alloc + MMA issue,
// warps 2..5 TF32 rounding / 3xTF32 split of the landed operand tiles,
// warps 6..13 epilogue (two warps per TMEM lane quadrant, column halves).
// The observation mask is read bit-packed (1 bit per entry, F order).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <string>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace fctn {

CUtensorMap tc_make_map_f32(const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                            const uint32_t* box, bool mn32);

namespace {

constexpr int CONV_WARPS = 4;
constexpr int EPI_WARPS = 8;
constexpr int EPI0 = 2 + CONV_WARPS;  // first epilogue warp
constexpr int THREADS = 32 * (EPI0 + EPI_WARPS);

struct ComposeArgs {
  const float* Xo;
  float* Xn;
  const uint32_t* maskbits;
  double* partials;
  long long rows, cols;       // accumulator extents (row axis = contiguous axis of X_(k))
  long long n_rb, n_tiles;
  long long P, PI, I;         // X view
  int kp;                     // K (= s padded to 8)
  int rows_are_p;
  float rho, onep;
  int objective_only;
};

template <int N, bool SPLIT>
__global__ void __launch_bounds__(THREADS, 1)
    k_compose_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const ComposeArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int kp = args.kp;
  const uint32_t a_bytes = 128u * kp * 4u, b_bytes = (uint32_t)N * kp * 4u;
  const uint32_t tma_bytes = a_bytes + b_bytes;
  const uint32_t stage_bytes = tma_bytes * (SPLIT ? 2 : 1);  // [A hi | B hi | (A lo | B lo)]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * stage_bytes);
  uint64_t* conv = full + 2;
  uint64_t* empty = conv + 2;
  uint64_t* tfull = empty + 2;
  uint64_t* tempty = tfull + 2;  // (barrier block: 10 x 8 B)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ double red[4][THREADS];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NCOLS = 2 * N <= 32 ? 32 : 2 * N <= 64 ? 64 : 2 * N <= 128 ? 128 : 2 * N <= 256 ? 256 : 512;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&conv[s], CONV_WARPS);
      tc::mbar_init(&empty[s], 1);
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

  if (warp == 0 && lane == 0) {
    int j = 0;
    for (long long t = blockIdx.x; t < args.n_tiles; t += gridDim.x, ++j) {
      const int s = j & 1;
      tc::mbar_wait(&empty[s], ((j >> 1) & 1) ^ 1);
      tc::mbar_expect_tx(&full[s], tma_bytes);
      const int r0 = (int)((t % args.n_rb) * 128), c0 = (int)((t / args.n_rb) * N);
      uint8_t* a = smem + s * stage_bytes;
      uint8_t* b = a + a_bytes;
      const uint32_t chunk = 32u * kp * 4u;
#pragma unroll
      for (int c = 0; c < 4; ++c) tc::tma_load_2d(a + c * chunk, &tmA, &full[s], r0 + 32 * c, 0);
#pragma unroll
      for (int c = 0; c < N / 32; ++c) tc::tma_load_2d(b + c * chunk, &tmB, &full[s], c0 + 32 * c, 0);
    }
  } else if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = tc::idesc_tf32(128, N, true, true);
    const uint32_t chunk = 32u * kp * 4u;
    int j = 0;
    for (long long t = blockIdx.x; t < args.n_tiles; t += gridDim.x, ++j) {
      const int s = j & 1;
      const uint32_t ph = (j >> 1) & 1;
      tc::mbar_wait(&tempty[s], ph ^ 1);
      tc::mbar_wait(&conv[s], ph);
      tc::fence_after_sync();
      const uint32_t a = tc::smem_u32(smem + s * stage_bytes);
      const uint32_t b = a + a_bytes;
      for (int kk = 0; kk < kp / 8; ++kk) {
        const uint64_t ad = tc::sdesc(a + kk * 1024, chunk, 512, 1);
        const uint64_t bd = tc::sdesc(b + kk * 1024, chunk, 512, 1);
        if (SPLIT) {
          tc::mma_tf32(tmem + s * N, tc::sdesc(a + tma_bytes + kk * 1024, chunk, 512, 1), bd, idesc, kk != 0);
          tc::mma_tf32(tmem + s * N, ad, tc::sdesc(b + tma_bytes + kk * 1024, chunk, 512, 1), idesc, 1);
        }
        tc::mma_tf32(tmem + s * N, ad, bd, idesc, SPLIT || kk != 0);
      }
      tc::mma_commit(&empty[s]);
      tc::mma_commit(&tfull[s]);
    }
  } else if (warp >= 2 && warp < EPI0) {
    // operand rounding (TF32 round-to-nearest) or 3xTF32 hi/lo split
    const int ct = threadIdx.x - 64;
    int j = 0;
    for (long long t = blockIdx.x; t < args.n_tiles; t += gridDim.x, ++j) {
      const int s = j & 1;
      tc::mbar_wait(&full[s], (j >> 1) & 1);
      uint8_t* a = smem + s * stage_bytes;
      tc::tf32_split_tile<SPLIT>(a, a + tma_bytes, (int)(tma_bytes / 4), ct, 32 * CONV_WARPS);
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&conv[s]);
    }
  } else if (warp >= EPI0) {
    const int ew = warp - EPI0;
    const int quad = warp & 3;
    const int half = ew >> 2;  // column half handled by this warp
    const int row = 32 * quad + lane;
    int j = 0;
    for (long long t = blockIdx.x; t < args.n_tiles; t += gridDim.x, ++j) {
      const int s = j & 1;
      tc::mbar_wait(&tfull[s], (j >> 1) & 1);
      tc::fence_after_sync();
      const long long gr = (t % args.n_rb) * 128 + row;
      const long long cb = (t / args.n_rb) * N;
      const bool row_ok = gr < args.rows;
      long long rowbase, colstride;
      if (args.rows_are_p) {
        rowbase = (gr % args.P) + args.PI * (gr / args.P);
        colstride = args.P;
      } else {
        rowbase = gr;
        colstride = args.I;
      }
#pragma unroll 1
      for (int c0 = half * (N / 2); c0 < (half + 1) * (N / 2); c0 += 16) {
        float v[16];
        tc::tmem_ld16(tmem + s * N + ((uint32_t)(32 * quad) << 16) + c0, v);
        if (row_ok) {
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const long long gc = cb + c0 + q;
            if (gc < args.cols) {
              const long long off = rowbase + colstride * gc;
              const float x = __ldcs(args.Xo + off);
              const float c = v[q];
              if (args.objective_only) {
                const double d = (double)x - (double)c;
                s_c += d * d;
              } else {
                const bool obs = (__ldg(args.maskbits + (off >> 5)) >> (off & 31)) & 1u;
                float xn;
                if (obs) {
                  xn = x;  // observed entries restored bit for bit (solver.py:235-236)
                } else {
                  float tt = x * args.rho;  // (x*rho + c)/(1+rho), solver.py:232-234
                  tt = tt + c;
                  xn = tt / args.onep;
                }
                __stcs(args.Xn + off, xn);
                const double dx = (double)xn - (double)x;
                const double dc = (double)xn - (double)c;
                s_d += dx * dx;
                s_b += (double)x * (double)x;
                s_c += dc * dc;
                s_n += (double)xn * (double)xn;
              }
            }
          }
        }
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[s]);
    }
  }
  red[0][threadIdx.x] = s_d;
  red[1][threadIdx.x] = s_b;
  red[2][threadIdx.x] = s_c;
  red[3][threadIdx.x] = s_n;
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 4) {
    double v = 0.0;
    for (int q = 0; q < THREADS; ++q) v += red[threadIdx.x][q];  // fixed order
    args.partials[blockIdx.x * 4 + threadIdx.x] = v;
  }
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc<NCOLS>(tmem);
  }
}

template <int N, bool SPLIT>
int go2(const CUtensorMap& ma, const CUtensorMap& mb, const ComposeArgs& a, int grid, cudaStream_t st) {
  const int smem = 2 * (128 + N) * a.kp * 4 * (SPLIT ? 2 : 1) + 1024 + 256;
  auto fn = k_compose_tc<N, SPLIT>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) throw std::runtime_error(std::string("compose_tc smem: ") + cudaGetErrorString(e));
  fn<<<grid, THREADS, smem, st>>>(ma, mb, a);
  e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("compose_tc: ") + cudaGetErrorString(e));
  return grid;
}

template <int N>
int go(const CUtensorMap& ma, const CUtensorMap& mb, const ComposeArgs& a, int grid, bool split3, cudaStream_t st) {
  return split3 ? go2<N, true>(ma, mb, a, grid, st) : go2<N, false>(ma, mb, a, grid, st);
}

}  // namespace

bool tc_compose_supported(int64_t I, int64_t P, int64_t p, int64_t S) {
  if (S > 128) return false;
  if (I % 4 != 0 || p % 4 != 0) return false;  // TMA row strides of A_(k) [I, S] and M [p, S]
  if (I > (1LL << 31) || p > (1LL << 31)) return false;
  (void)P;
  return true;
}

int launch_compose_tc(const float* A, const float* M, const float* Xo, const uint32_t* maskbits, float* Xn,
                      int64_t I, int64_t P, int64_t S, int64_t p, double rho, bool objective_only, double* partials,
                      int64_t partial_cap, int n_sm, bool split3, cudaStream_t st) {
  ComposeArgs a;
  a.Xo = Xo;
  a.Xn = Xn;
  a.maskbits = maskbits;
  a.partials = partials;
  a.P = P;
  a.PI = P * I;
  a.I = I;
  a.kp = (int)((S + 7) / 8 * 8);
  a.rows_are_p = P > 1;
  a.rho = (float)rho;
  a.onep = (float)(1.0 + rho);
  a.objective_only = objective_only ? 1 : 0;
  a.rows = a.rows_are_p ? p : I;
  a.cols = a.rows_are_p ? I : p;
  int N = 256;
  if (a.rows_are_p) {
    N = (int)((I + 31) / 32 * 32);
    if (N > 256) N = 256;
  }
  while (N > 32 && 2 * (128 + N) * a.kp * 4 * (split3 ? 2 : 1) + 1280 > 200 * 1024) N /= 2;
  if (N != 32 && N != 64 && N != 96 && N != 128 && N != 160 && N != 192 && N != 224 && N != 256) N = 256;
  a.n_rb = (a.rows + 127) / 128;
  const long long n_cb = (a.cols + N - 1) / N;
  a.n_tiles = a.n_rb * n_cb;
  int grid = (int)std::min<long long>(a.n_tiles, n_sm);
  if (grid > partial_cap) throw std::runtime_error("compose partial buffer too small");
  // operand maps: rows operand (A) and cols operand (B), both [extent, S] 32-bit MN-major
  uint64_t dm[2] = {(uint64_t)p, (uint64_t)S}, sm_[1] = {(uint64_t)p * 4};
  uint64_t da[2] = {(uint64_t)I, (uint64_t)S}, sa[1] = {(uint64_t)I * 4};
  uint32_t box[2] = {32, (uint32_t)a.kp};
  CUtensorMap mM = tc_make_map_f32(M, 2, dm, sm_, box, true);
  CUtensorMap mA = tc_make_map_f32(A, 2, da, sa, box, true);
  const CUtensorMap& rowsmap = a.rows_are_p ? mM : mA;
  const CUtensorMap& colsmap = a.rows_are_p ? mA : mM;
  switch (N) {
    case 32: return go<32>(rowsmap, colsmap, a, grid, split3, st);
    case 64: return go<64>(rowsmap, colsmap, a, grid, split3, st);
    case 96: return go<96>(rowsmap, colsmap, a, grid, split3, st);
    case 128: return go<128>(rowsmap, colsmap, a, grid, split3, st);
    case 160: return go<160>(rowsmap, colsmap, a, grid, split3, st);
    case 192: return go<192>(rowsmap, colsmap, a, grid, split3, st);
    case 224: return go<224>(rowsmap, colsmap, a, grid, split3, st);
    default: return go<256>(rowsmap, colsmap, a, grid, split3, st);
  }
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
