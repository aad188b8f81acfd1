// K2 on the B200 tensor cores (fp32 data, tcgen05 kind::tf32, fp32
// accumulation in TMEM): Y_k partials = X_(k) M_k^T (sylvester.py:104).
//
// One CTA = one 128-row tile of mode k x one split of the reduction axis p.
// Warp roles (192 threads):
//   warp 0      TMA producer: X tile (128 x 32 fp32) + M tile (NT x 32) per stage
//   warp 1      TMEM allocator + single-thread MMA issuer (4 x K=8 per stage,
//               x3 for the 3xTF32 split)
//   warps 2..5  per stage: round the landed tiles to TF32 (round-to-nearest)
//               or split them hi/lo for 3xTF32 (tc_common.cuh); at the end:
//               tcgen05.ld the 128 x NT accumulator, write fp32 partials
// X is read in place through a TMA descriptor of the mode-k view:
//   P > 1  (modes before k exist): 3-D [P, I, Q], K-major A tile (rows = i,
//          128 B = 32 consecutive p along the fastest mode)
//   P == 1 (k = 0): 2-D [I, Q], MN-major A tile (i contiguous), four 32-row
//          boxes per 128-row tile, SWIZZLE_128B with 32-byte atoms (the only
//          MN-major smem layout UMMA accepts for 32-bit operands)
// M_k (p-fastest) is a 3-D [P, Q, S] (or 2-D [Q, S]) K-major B tile.  Both
// use SWIZZLE_128B; OOB boxes are zero-filled by TMA, so ragged P, I, S need
// no special casing.  Partials are combined by the fixed-order split reduce.
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

namespace {

constexpr int BK = 32;  // fp32 per 128-byte row
constexpr int A_BYTES = 128 * BK * 4;  // 16 KB

// stage = [A hi | B hi | (A lo | B lo)]; TMA bytes = A + B
template <int NT, bool SPLIT>
struct StreamSmem {
  static constexpr int B_BYTES = NT * BK * 4;
  static constexpr int TMA_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGE_BYTES = TMA_BYTES * (SPLIT ? 2 : 1);
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 6 ? 6 : (200 * 1024) / STAGE_BYTES;
  static constexpr int TOTAL = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

template <int NT, bool AMN, bool SPLIT>
__global__ void __launch_bounds__(192, 1)
    k_stream_tc(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmM,
                const __grid_constant__ CUtensorMap tmMl, float* __restrict__ part, int I, int S, long long nkb_total,
                long long kb_per_split, int nPB, int b_pre) {
  using L = StreamSmem<NT, SPLIT>;
  constexpr int STAGES = L::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * L::STAGE_BYTES);
  uint64_t* conv = full + STAGES;
  uint64_t* empty = conv + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mtile = blockIdx.x;
  const long long split = blockIdx.y;
  const long long kb0 = split * kb_per_split;
  long long kb1 = kb0 + kb_per_split;
  if (kb1 > nkb_total) kb1 = nkb_total;
  const int nkb = (int)(kb1 - kb0);
  constexpr int NCOLS = NT <= 32 ? 32 : NT <= 64 ? 64 : NT <= 128 ? 128 : 256;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmX);
    tc::tma_prefetch(&tmM);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&conv[s], 4);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(tmem_full, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<NCOLS>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    const int i0 = mtile * 128;
    for (int it = 0; it < nkb; ++it) {
      const int s = it % STAGES;
      const uint32_t ph = (it / STAGES) & 1;
      tc::mbar_wait(&empty[s], ph ^ 1);
      tc::mbar_expect_tx(&full[s], L::TMA_BYTES + ((SPLIT && b_pre) ? L::B_BYTES : 0));
      const long long kb = kb0 + it;
      uint8_t* a = smem + s * L::STAGE_BYTES;
      uint8_t* b = a + A_BYTES;
      if (AMN) {
        const int q0 = (int)(kb * BK);
#pragma unroll
        for (int c = 0; c < 4; ++c) tc::tma_load_2d(a + c * 4096, &tmX, &full[s], i0 + 32 * c, q0);
        tc::tma_load_2d(b, &tmM, &full[s], q0, 0);
        if (SPLIT && b_pre) tc::tma_load_2d(b + L::TMA_BYTES, &tmMl, &full[s], q0, 0);
      } else {
        const int pb = (int)(kb % nPB) * BK;
        const int q = (int)(kb / nPB);
        tc::tma_load_3d(a, &tmX, &full[s], pb, i0, q);
        tc::tma_load_3d(b, &tmM, &full[s], pb, q, 0);
        if (SPLIT && b_pre) tc::tma_load_3d(b + L::TMA_BYTES, &tmMl, &full[s], pb, q, 0);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer
    constexpr uint32_t idesc = tc::idesc_tf32(128, NT, AMN, false);
    for (int it = 0; it < nkb; ++it) {
      const int s = it % STAGES;
      const uint32_t ph = (it / STAGES) & 1;
      tc::mbar_wait(&conv[s], ph);
      tc::fence_after_sync();
      const uint32_t a = tc::smem_u32(smem + s * L::STAGE_BYTES);
      const uint32_t b = a + A_BYTES;
      const uint32_t lo = L::TMA_BYTES;  // lo tiles follow the hi tiles
#pragma unroll
      for (int kk = 0; kk < BK / 8; ++kk) {
        const uint64_t ad = AMN ? tc::sdesc(a + kk * 1024, 4096, 512, 1) : tc::sdesc(a + kk * 32, 16, 1024);
        const uint64_t bd = tc::sdesc(b + kk * 32, 16, 1024);
        if (SPLIT) {
          const uint64_t adl = AMN ? tc::sdesc(a + lo + kk * 1024, 4096, 512, 1) : tc::sdesc(a + lo + kk * 32, 16, 1024);
          const uint64_t bdl = tc::sdesc(b + lo + kk * 32, 16, 1024);
          tc::mma_tf32(tmem, adl, bd, idesc, (it | kk) != 0);
          tc::mma_tf32(tmem, ad, bdl, idesc, 1);
        }
        tc::mma_tf32(tmem, ad, bd, idesc, SPLIT || (it | kk) != 0);
      }
      tc::mma_commit(&empty[s]);
    }
    tc::mma_commit(tmem_full);
  } else if (warp >= 2) {
    // ---------------- operand rounding / 3xTF32 split, then the epilogue
    const int ct = threadIdx.x - 64;
    for (int it = 0; it < nkb; ++it) {
      const int s = it % STAGES;
      tc::mbar_wait(&full[s], (it / STAGES) & 1);
      uint8_t* a = smem + s * L::STAGE_BYTES;
      // a pre-split B (hi/lo from HBM) leaves only the X tile to convert
      tc::tf32_split_tile<SPLIT>(a, a + L::TMA_BYTES, (b_pre ? A_BYTES : L::TMA_BYTES) / 4, ct, 128);
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&conv[s]);
    }
    tc::mbar_wait(tmem_full, 0);
    tc::fence_after_sync();
    const int q = warp & 3;
    const int row = 32 * q + lane;
    const long long i = (long long)mtile * 128 + row;
    float* out = part + split * (long long)I * S;
#pragma unroll 1
    for (int c0 = 0; c0 < NT; c0 += 16) {
      float v[16];
      tc::tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + c0, v);
      if (i < I) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int s = c0 + j;
          if (s < S) out[i + (long long)I * s] = v[j];
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc<NCOLS>(tmem);
  }
}

// ---------------------------------------------------------------------------
// 3xTF32 variant with the X operand split into TENSOR MEMORY.
//
// The split kernel above is shared-memory-bandwidth bound: per 16 KB X stage
// the converters read the tile and write hi + lo back (48 KB), and the three
// MMAs re-read A three times.  Here the converter warps read the landed X
// tile once, round hi = rn(x), lo = rn(x - hi) and store both rows straight
// into TMEM (tcgen05.st, one row per thread: lane = row), and the MMAs take A
// from TMEM (kind::tf32, A K-major in TMEM whatever X's layout in smem):
//     D[:, 0:2NT]  = A_hi x [B_hi | B_lo]     (one N = 2NT instruction)
//     D[:, 0:NT]  += A_lo x B_hi
// so shared memory only carries the TMA writes, one converter read of X and
// the B reads.  The epilogue sums D[:, c] + D[:, NT + c].
// TMEM: accumulator 2NT columns + per stage 64 columns (32 hi, 32 lo).
template <int NT>
struct TsSmem {
  static constexpr int B_BYTES = NT * BK * 4;
  static constexpr int STAGE_BYTES = A_BYTES + 2 * B_BYTES;  // [X raw | B hi | B lo]
  static constexpr int ACC = 2 * NT;
  static constexpr int S_SMEM = (200 * 1024) / STAGE_BYTES > 6 ? 6 : (200 * 1024) / STAGE_BYTES;
  static constexpr int S_TMEM = (512 - ACC) / 64;
  static constexpr int STAGES = S_SMEM < S_TMEM ? S_SMEM : S_TMEM;
  static constexpr int TOTAL = STAGES * STAGE_BYTES + 1024 + 256;
};

constexpr int TS_CONV_WARPS = 8;
constexpr int TS_THREADS = 64 + 32 * TS_CONV_WARPS;

template <int NT, bool AMN>
__global__ void __launch_bounds__(TS_THREADS, 1)
    k_stream_ts(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmM,
                const __grid_constant__ CUtensorMap tmMl, float* __restrict__ part, int I, int S, long long nkb_total,
                long long kb_per_split, int nPB, int b_pre, int x3d, int rows_b) {
  using L = TsSmem<NT>;
  constexpr int STAGES = L::STAGES;
  static_assert(STAGES >= 2, "stage ring");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * L::STAGE_BYTES);
  uint64_t* conv = full + STAGES;
  uint64_t* empty = conv + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mtile = blockIdx.x;
  const long long split = blockIdx.y;
  const long long kb0 = split * kb_per_split;
  long long kb1 = kb0 + kb_per_split;
  if (kb1 > nkb_total) kb1 = nkb_total;
  const int nkb = (int)(kb1 - kb0);

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmX);
    tc::tma_prefetch(&tmM);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&conv[s], TS_CONV_WARPS);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(tmem_full, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    const int i0 = mtile * 128;
    const uint32_t tx = A_BYTES + L::B_BYTES * (b_pre ? 2 : 1);
    for (int it = 0; it < nkb; ++it) {
      const int s = it % STAGES;
      const uint32_t ph = (it / STAGES) & 1;
      tc::mbar_wait(&empty[s], ph ^ 1);
      tc::mbar_expect_tx(&full[s], tx);
      const long long kb = kb0 + it;
      uint8_t* a = smem + s * L::STAGE_BYTES;
      uint8_t* b = a + A_BYTES;
      if (AMN) {
        const int q0 = (int)(kb * BK);
        if (rows_b) {  // batched [32, Q, rows_b/32, batch] view (tiles never straddle a batch)
          tc::tma_load_4d(a, &tmX, &full[s], 0, q0, (i0 % rows_b) / 32, i0 / rows_b);
        } else if (x3d) {  // [32, Q, I/32] view: the four 32-row boxes in one TMA
          tc::tma_load_3d(a, &tmX, &full[s], 0, q0, i0 / 32);
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) tc::tma_load_2d(a + c * 4096, &tmX, &full[s], i0 + 32 * c, q0);
        }
        tc::tma_load_2d(b, &tmM, &full[s], q0, 0);
        if (b_pre) tc::tma_load_2d(b + L::B_BYTES, &tmMl, &full[s], q0, 0);
      } else {
        const int pb = (int)(kb % nPB) * BK;
        const int q = (int)(kb / nPB);
        tc::tma_load_3d(a, &tmX, &full[s], pb, i0, q);
        tc::tma_load_3d(b, &tmM, &full[s], pb, q, 0);
        if (b_pre) tc::tma_load_3d(b + L::B_BYTES, &tmMl, &full[s], pb, q, 0);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer
    constexpr uint32_t idesc2 = tc::idesc_tf32(128, 2 * NT, false, false);
    constexpr uint32_t idesc1 = tc::idesc_tf32(128, NT, false, false);
    for (int it = 0; it < nkb; ++it) {
      const int s = it % STAGES;
      const uint32_t ph = (it / STAGES) & 1;
      tc::mbar_wait(&conv[s], ph);
      tc::fence_after_sync();
      const uint32_t b = tc::smem_u32(smem + s * L::STAGE_BYTES) + A_BYTES;
      const uint32_t ahi = tmem + L::ACC + 64 * s, alo = ahi + 32;
#pragma unroll
      for (int kk = 0; kk < BK / 8; ++kk) {
        const uint64_t bd = tc::sdesc(b + kk * 32, 16, 1024);  // rows 0..2NT-1 = [B hi | B lo]
        tc::mma_tf32_ts(tmem, ahi + 8 * kk, bd, idesc2, (it | kk) != 0);
        tc::mma_tf32_ts(tmem, alo + 8 * kk, bd, idesc1, 1);
      }
      tc::mma_commit(&empty[s]);
    }
    tc::mma_commit(tmem_full);
  } else if (warp >= 2) {
    // ---------------- X split into TMEM (+ B split in smem when not pre-split), then the epilogue
    // two warps per TMEM lane quadrant, each owning 16 of the stage's 32 K columns
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int hf = (warp - 2) >> 2;
    const int row = 32 * q + lane;
    const int ct = threadIdx.x - 64;
    for (int it = 0; it < nkb; ++it) {
      const int s = it % STAGES;
      tc::mbar_wait(&full[s], (it / STAGES) & 1);
      const uint8_t* a = smem + s * L::STAGE_BYTES;
      float x[16];
      if (AMN) {
        // four 32-row boxes; K row kq holds 32 consecutive rows, 32-B atoms XOR (kq & 3)
        const float* box = reinterpret_cast<const float*>(a + (row >> 5) * 4096);
        const int i = row & 31;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int kq = 16 * hf + j;
          x[j] = box[kq * 32 + ((((i >> 3) ^ (kq & 3))) << 3) + (i & 7)];
        }
      } else {
        // K-major SW128: row r, 16-B chunk c stored at chunk (c ^ (r & 7))
        const float4* r4 = reinterpret_cast<const float4*>(a + row * 128);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 v = r4[(4 * hf + c) ^ (row & 7)];
          x[4 * c] = v.x;
          x[4 * c + 1] = v.y;
          x[4 * c + 2] = v.z;
          x[4 * c + 3] = v.w;
        }
      }
      float lo[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float h = tc::tf32_rn_int(x[j]);
        lo[j] = tc::tf32_rn_int(x[j] - h);
        x[j] = h;
      }
      const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + L::ACC + 64 * s + 16 * hf;
      tc::tmem_st16(ta, x);
      tc::tmem_st16(ta + 32, lo);
      if (!b_pre) {
        uint8_t* b = smem + s * L::STAGE_BYTES + A_BYTES;
        tc::tf32_split_tile<true>(b, b + L::B_BYTES, L::B_BYTES / 4, ct, 32 * TS_CONV_WARPS);
        tc::fence_proxy_async_smem();
      }
      tc::tmem_wait_st();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&conv[s]);
    }
    tc::mbar_wait(tmem_full, 0);
    tc::fence_after_sync();
    const long long i = (long long)mtile * 128 + row;
    float* out = part + split * (long long)I * S;
#pragma unroll 1
    for (int c0 = 16 * hf; c0 < NT; c0 += 32) {
      float v[16], w[16];
      tc::tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + c0, v);
      tc::tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + NT + c0, w);
      if (i < I) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int s = c0 + j;
          if (s < S) out[i + (long long)I * s] = v[j] + w[j];
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
}

// Swapped-role form for short modes (I <= 64 < S <= 128, X tile K-major; c5's
// 48 x 81 products): the bond rows s of the M_k tile are the MMA's M side
// (A, split into TMEM by the converters) and the X rows the N side (B, split
// in place in shared memory, the low half written into the tile's unused rows
// NI..2NI-1 so [X hi | X lo] is one N-doubled operand).  The MMA then spends
// 128 x 3NI instead of 128 x 3S' per K step with only 48 of its 128 rows live
// (ncu, k_stream_ts at c5: tensor pipe 58 % with I = 48).  Partials are
// written in the same [split][i + I s] layout.
template <int NT, int NI>
struct TswSmem {
  static constexpr int X_BYTES = A_BYTES;         // 128 X rows (TMA box), hi in 0..NI-1, lo in NI..2NI-1
  static constexpr int M_BYTES = NT * BK * 4;     // NT bond rows
  static constexpr int STAGE_BYTES = X_BYTES + M_BYTES;
  static constexpr int ACC = 2 * NI;
  static constexpr int S_SMEM = (200 * 1024) / STAGE_BYTES > 6 ? 6 : (200 * 1024) / STAGE_BYTES;
  static constexpr int S_TMEM = (512 - ACC) / 64 > 6 ? 6 : (512 - ACC) / 64;
  static constexpr int STAGES = S_SMEM < S_TMEM ? S_SMEM : S_TMEM;
  static constexpr int TOTAL = STAGES * STAGE_BYTES + 1024 + 256;
};

template <int NT, int NI>
__global__ void __launch_bounds__(TS_THREADS, 1)
    k_stream_tsw(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmM,
                 float* __restrict__ part, int I, int S, long long nkb_total, long long kb_per_split, int nPB) {
  using L = TswSmem<NT, NI>;
  constexpr int STAGES = L::STAGES;
  static_assert(STAGES >= 2 && NI % 16 == 0 && 2 * NI <= 128, "tsw shape");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * L::STAGE_BYTES);
  uint64_t* conv = full + STAGES;
  uint64_t* empty = conv + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long split = blockIdx.y;
  const long long kb0 = split * kb_per_split;
  long long kb1 = kb0 + kb_per_split;
  if (kb1 > nkb_total) kb1 = nkb_total;
  const int nkb = (int)(kb1 - kb0);

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmX);
    tc::tma_prefetch(&tmM);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&conv[s], TS_CONV_WARPS);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(tmem_full, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer: X tile [128 i rows x 32 p] + M tile [NT s rows x 32 p]
    for (int it = 0; it < nkb; ++it) {
      const int s = it % STAGES;
      tc::mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
      tc::mbar_expect_tx(&full[s], L::X_BYTES + L::M_BYTES);
      const long long kb = kb0 + it;
      uint8_t* a = smem + s * L::STAGE_BYTES;
      const int pb = (int)(kb % nPB) * BK;
      const int q = (int)(kb / nPB);
      tc::tma_load_3d(a, &tmX, &full[s], pb, 0, q);
      tc::tma_load_3d(a + L::X_BYTES, &tmM, &full[s], pb, q, 0);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer: D[s, 0:2NI] = A_hi [X_hi | X_lo]^T, D[s, 0:NI] += A_lo X_hi^T
    constexpr uint32_t idesc2 = tc::idesc_tf32(128, 2 * NI, false, false);
    constexpr uint32_t idesc1 = tc::idesc_tf32(128, NI, false, false);
    for (int it = 0; it < nkb; ++it) {
      const int s = it % STAGES;
      tc::mbar_wait(&conv[s], (it / STAGES) & 1);
      tc::fence_after_sync();
      const uint32_t x = tc::smem_u32(smem + s * L::STAGE_BYTES);
      const uint32_t ahi = tmem + L::ACC + 64 * s, alo = ahi + 32;
#pragma unroll
      for (int kk = 0; kk < BK / 8; ++kk) {
        const uint64_t bd = tc::sdesc(x + kk * 32, 16, 1024);  // rows 0..2NI-1 = [X hi | X lo]
        tc::mma_tf32_ts(tmem, ahi + 8 * kk, bd, idesc2, (it | kk) != 0);
        tc::mma_tf32_ts(tmem, alo + 8 * kk, bd, idesc1, 1);
      }
      tc::mma_commit(&empty[s]);
    }
    tc::mma_commit(tmem_full);
  } else if (warp >= 2) {
    // ---------------- M tile split into TMEM (lane = s), X rows split in place
    const int q = warp & 3;
    const int hf = (warp - 2) >> 2;
    const int row = 32 * q + lane;   // bond row s
    const int ct = threadIdx.x - 64;  // 0..255
    for (int it = 0; it < nkb; ++it) {
      const int s = it % STAGES;
      tc::mbar_wait(&full[s], (it / STAGES) & 1);
      uint8_t* a = smem + s * L::STAGE_BYTES;
      if (32 * q < NT) {  // quadrants past the M tile hold no bond row (D rows never stored)
        float x[16];
        const uint8_t* mrow = a + L::X_BYTES + (row < NT ? row : 0) * 128;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 v = tc::lds128(tc::smem_u32(mrow) + 16u * (uint32_t)((4 * hf + c) ^ (row & 7)));
          x[4 * c] = v.x;
          x[4 * c + 1] = v.y;
          x[4 * c + 2] = v.z;
          x[4 * c + 3] = v.w;
        }
        float lo[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float h = tc::tf32_rn_int(x[j]);
          lo[j] = tc::tf32_rn_int(x[j] - h);
          x[j] = h;
        }
        const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + L::ACC + 64 * s + 16 * hf;
        tc::tmem_st16(ta, x);
        tc::tmem_st16(ta + 32, lo);
      }
      // X rows 0..NI-1: hi in place, lo into row + NI (same swizzle phase: NI % 8 == 0)
      const uint32_t xs = tc::smem_u32(a);
      for (int e = ct; e < NI * 8; e += 32 * TS_CONV_WARPS) {
        const int r = e >> 3, c = e & 7;
        const uint32_t off = (uint32_t)(r * 128) + 16u * (uint32_t)(c ^ (r & 7));
        const float4 v = tc::lds128(xs + off);
        const float4 h = make_float4(tc::tf32_rn_int(v.x), tc::tf32_rn_int(v.y), tc::tf32_rn_int(v.z), tc::tf32_rn_int(v.w));
        tc::sts128(xs + off, h);
        tc::sts128(xs + off + (uint32_t)(NI * 128), make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w));
      }
      tc::fence_proxy_async_smem();
      tc::tmem_wait_st();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&conv[s]);
    }
    tc::mbar_wait(tmem_full, 0);
    tc::fence_after_sync();
    float* out = part + split * (long long)I * S;
    if (32 * q < NT) {
#pragma unroll 1
      for (int c0 = 16 * hf; c0 < NI; c0 += 32) {
        float v[16], w[16];
        tc::tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + c0, v);
        tc::tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + NI + c0, w);
        if (row < S) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int i = c0 + j;
            if (i < I) out[i + (long long)I * row] = v[j] + w[j];
          }
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
}

// Persistent form of k_stream_ts for unsplit products with many row tiles
// (the Z_j passes): one CTA per SM walks its row tiles with one continuous
// operand pipeline.  NACC = 1 (default): one TMEM accumulator, which leaves
// TMEM for a 6-stage operand ring instead of 4 (NT = 64); the epilogue warps
// pull a finished tile's rows into registers, hand the accumulator straight
// back to the MMA and only then store, so the MMA stalls for a TMEM read per
// tile (~1 us of 30) while the ring keeps filling.  Measured at c4: 230 ->
// 217 us per Z pass.  NACC = 2 (FCTN_ZPASS_ACC2=1): two accumulators, the
// epilogue of tile j overlaps the MMAs of tile j + 1, 4 stages.
constexpr int TSP_EPI_WARPS = 4;
constexpr int TSP_THREADS = 64 + 32 * (TS_CONV_WARPS + TSP_EPI_WARPS);
template <int NT, int NACC>
struct TspSmem {
  static constexpr int B_BYTES = NT * BK * 4;
  static constexpr int STAGE_BYTES = A_BYTES + 2 * B_BYTES;
  static constexpr int ACC = 2 * NT;  // one accumulator: [hi x (B hi | B lo)]
  static constexpr int S_SMEM = (200 * 1024) / STAGE_BYTES > 6 ? 6 : (200 * 1024) / STAGE_BYTES;
  static constexpr int S_TMEM = (512 - NACC * ACC) / 64;
  static constexpr int STAGES = S_SMEM < S_TMEM ? S_SMEM : S_TMEM;
  static constexpr int TOTAL = STAGES * STAGE_BYTES + 1024 + 256;
};

template <int NT, bool AMN, int NACC>
__global__ void __launch_bounds__(TSP_THREADS, 1)
    k_stream_tsp(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmM,
                 const __grid_constant__ CUtensorMap tmMl, float* __restrict__ out, int I, int S, int nkb,
                 int n_tiles, int nPB, int b_pre, int x3d, int rows_b) {
  using L = TspSmem<NT, NACC>;
  constexpr int STAGES = L::STAGES;
  static_assert(STAGES >= 2, "stage ring");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * L::STAGE_BYTES);
  uint64_t* conv = full + STAGES;
  uint64_t* empty = conv + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int EPI0 = 2 + TS_CONV_WARPS;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmX);
    tc::tma_prefetch(&tmM);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&conv[s], TS_CONV_WARPS);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < NACC; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], TSP_EPI_WARPS);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    const uint32_t tx = A_BYTES + L::B_BYTES * (b_pre ? 2 : 1);
    int g = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const int i0 = t * 128;
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int s = g % STAGES;
        tc::mbar_wait(&empty[s], ((g / STAGES) & 1) ^ 1);
        tc::mbar_expect_tx(&full[s], tx);
        uint8_t* a = smem + s * L::STAGE_BYTES;
        uint8_t* b = a + A_BYTES;
        if (AMN) {
          const int q0 = kb * BK;
          if (rows_b) {
            tc::tma_load_4d(a, &tmX, &full[s], 0, q0, (i0 % rows_b) / 32, i0 / rows_b);
          } else if (x3d) {
            tc::tma_load_3d(a, &tmX, &full[s], 0, q0, i0 / 32);
          } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) tc::tma_load_2d(a + c * 4096, &tmX, &full[s], i0 + 32 * c, q0);
          }
          tc::tma_load_2d(b, &tmM, &full[s], q0, 0);
          if (b_pre) tc::tma_load_2d(b + L::B_BYTES, &tmMl, &full[s], q0, 0);
        } else {
          const int pb = (kb % nPB) * BK;
          const int q = kb / nPB;
          tc::tma_load_3d(a, &tmX, &full[s], pb, i0, q);
          tc::tma_load_3d(b, &tmM, &full[s], pb, q, 0);
          if (b_pre) tc::tma_load_3d(b + L::B_BYTES, &tmMl, &full[s], pb, q, 0);
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer.  This one thread's instruction stream is on
    // the critical path (a run-time switch of two branches per K step cost
    // 12 % of the kernel), so the ring slot / phase are running counters and a
    // stage's B descriptors are the slot-0 descriptor plus an address offset
    // (only the 14-bit start-address field changes; shared memory < 256 KB).
    constexpr uint32_t idesc2 = tc::idesc_tf32(128, 2 * NT, false, false);
    constexpr uint32_t idesc1 = tc::idesc_tf32(128, NT, false, false);
    const uint64_t bd0 = tc::sdesc(tc::smem_u32(smem) + A_BYTES, 16, 1024);
    int s = 0, j = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++j) {
      const int acc = j % NACC;
      tc::mbar_wait(&tempty[acc], ((j / NACC) & 1) ^ 1);
      tc::fence_after_sync();
      const uint32_t d = tmem + acc * L::ACC;
      for (int kb = 0; kb < nkb; ++kb) {
        tc::mbar_wait(&conv[s], ph);
        tc::fence_after_sync();
        const uint64_t bds = bd0 + (uint64_t)((uint32_t)(s * L::STAGE_BYTES) >> 4);
        const uint32_t ahi = tmem + NACC * L::ACC + 64 * s, alo = ahi + 32;
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          const uint64_t bd = bds + (uint64_t)(2 * kk);  // + 32 bytes
          tc::mma_tf32_ts(d, ahi + 8 * kk, bd, idesc2, (kb | kk) != 0);
          tc::mma_tf32_ts(d, alo + 8 * kk, bd, idesc1, 1);
        }
        tc::mma_commit(&empty[s]);
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
      tc::mma_commit(&tfull[acc]);
    }
  } else if (warp >= 2 && warp < EPI0) {
    // ---------------- X split into TMEM (+ B split in smem when not pre-split)
    const int q = warp & 3;
    const int hf = (warp - 2) >> 2;
    const int row = 32 * q + lane;
    const int ct = threadIdx.x - 64;
    int g = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int s = g % STAGES;
        tc::mbar_wait(&full[s], (g / STAGES) & 1);
        const uint8_t* a = smem + s * L::STAGE_BYTES;
        float x[16];
        if (AMN) {
          const float* box = reinterpret_cast<const float*>(a + (row >> 5) * 4096);
          const int i = row & 31;
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const int kq = 16 * hf + jj;
            x[jj] = box[kq * 32 + ((((i >> 3) ^ (kq & 3))) << 3) + (i & 7)];
          }
        } else {
          const float4* r4 = reinterpret_cast<const float4*>(a + row * 128);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float4 v = r4[(4 * hf + c) ^ (row & 7)];
            x[4 * c] = v.x;
            x[4 * c + 1] = v.y;
            x[4 * c + 2] = v.z;
            x[4 * c + 3] = v.w;
          }
        }
        float lo[16];
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const float h = tc::tf32_rn_int(x[jj]);
          lo[jj] = tc::tf32_rn_int(x[jj] - h);
          x[jj] = h;
        }
        const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + NACC * L::ACC + 64 * s + 16 * hf;
        tc::tmem_st16(ta, x);
        tc::tmem_st16(ta + 32, lo);
        if (!b_pre) {
          uint8_t* b = smem + s * L::STAGE_BYTES + A_BYTES;
          tc::tf32_split_tile<true>(b, b + L::B_BYTES, L::B_BYTES / 4, ct, 32 * TS_CONV_WARPS);
          tc::fence_proxy_async_smem();
        }
        tc::tmem_wait_st();
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&conv[s]);
      }
    }
  } else if (warp >= EPI0) {
    // ---------------- epilogue: accumulator j & 1 -> out rows, then release it
    const int q = warp & 3;
    const int row = 32 * q + lane;
    int j = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++j) {
      const int acc = j % NACC;
      tc::mbar_wait(&tfull[acc], (j / NACC) & 1);
      tc::fence_after_sync();
      const long long i = (long long)t * 128 + row;
      const uint32_t base = tmem + ((uint32_t)(32 * q) << 16) + acc * L::ACC;
      if (NACC == 1) {
        // one accumulator: pull the whole row into registers, hand the
        // accumulator back to the MMA, then store
        float v[NT];
#pragma unroll
        for (int c0 = 0; c0 < NT; c0 += 16) {
          float w[16];
          tc::tmem_ld16(base + c0, v + c0);
          tc::tmem_ld16(base + NT + c0, w);
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) v[c0 + jj] += w[jj];
        }
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&tempty[acc]);
        if (i < I) {
#pragma unroll
          for (int sc = 0; sc < NT; ++sc)
            if (sc < S) out[i + (long long)I * sc] = v[sc];
        }
        continue;
      }
#pragma unroll 1
      for (int c0 = 0; c0 < NT; c0 += 16) {
        float v[16], w[16];
        tc::tmem_ld16(base + c0, v);
        tc::tmem_ld16(base + NT + c0, w);
        if (i < I) {
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const int sc = c0 + jj;
            if (sc < S) out[i + (long long)I * sc] = v[jj] + w[jj];
          }
        }
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p)
      throw std::runtime_error("cuTensorMapEncodeTiled is unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

CUtensorMap make_map(const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                     const uint32_t* box, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B,
                     CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32) {
  CUtensorMap m;
  uint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = encode_fn()(&m, dt, (cuuint32_t)rank, const_cast<void*>(base),
                           (const cuuint64_t*)dims, (const cuuint64_t*)strides_bytes, (const cuuint32_t*)box,
                           (const cuuint32_t*)es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

template <int NT, bool AMN, bool SPLIT>
void go3(const CUtensorMap& mx, const CUtensorMap& mm, const CUtensorMap& mml, bool b_pre, float* part, int64_t I,
         int64_t S, const TcStreamPlan& tp, cudaStream_t st) {
  const int smem = StreamSmem<NT, SPLIT>::TOTAL;
  auto fn = k_stream_tc<NT, AMN, SPLIT>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) throw std::runtime_error(std::string("stream_tc smem: ") + cudaGetErrorString(e));
  dim3 grid((unsigned)tp.n_mtiles, (unsigned)tp.nsplit);
  fn<<<grid, 192, smem, st>>>(mx, mm, mml, part, (int)I, (int)S, tp.nkb, tp.kb_per_split, (int)tp.npb,
                              b_pre ? 1 : 0);
  e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("stream_tc: ") + cudaGetErrorString(e));
}

int sm_count() {
  static const int v = [] {
    int d = 0, n = 148;
    if (cudaGetDevice(&d) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    return n;
  }();
  return v;
}

// SMs kept free of the persistent kernels (the context reserves one while the
// side-stream eigendecomposition runs concurrently, eigh.cu)
int g_reserved_sms = 0;

template <int NT, bool AMN>
void go_ts(const CUtensorMap& mx, const CUtensorMap& mm, const CUtensorMap& mml, bool b_pre, bool x3d, float* part,
           int64_t I, int64_t S, const TcStreamPlan& tp, cudaStream_t st, int rows_b = 0) {
  static const bool no_persist = getenv("FCTN_STREAM_NO_PERSIST") != nullptr;
  if constexpr (NT <= 64) {
    if (tp.nsplit == 1 && tp.n_mtiles > sm_count() && !no_persist && tp.nkb < (1LL << 31)) {
      static const bool acc2 = getenv("FCTN_ZPASS_ACC2") != nullptr;  // the older double-buffered accumulator
      const int smem = acc2 ? TspSmem<NT, 2>::TOTAL : TspSmem<NT, 1>::TOTAL;
      auto fn = acc2 ? k_stream_tsp<NT, AMN, 2> : k_stream_tsp<NT, AMN, 1>;
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) throw std::runtime_error(std::string("stream_tsp smem: ") + cudaGetErrorString(e));
      const int grid = (int)std::min<int64_t>(tp.n_mtiles, std::max(1, sm_count() - g_reserved_sms));
      fn<<<grid, TSP_THREADS, smem, st>>>(mx, mm, mml, part, (int)I, (int)S, (int)tp.nkb, (int)tp.n_mtiles,
                                          (int)tp.npb, b_pre ? 1 : 0, x3d ? 1 : 0, rows_b);
      e = cudaGetLastError();
      if (e != cudaSuccess) throw std::runtime_error(std::string("stream_tsp: ") + cudaGetErrorString(e));
      return;
    }
  }
  const int smem = TsSmem<NT>::TOTAL;
  auto fn = k_stream_ts<NT, AMN>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) throw std::runtime_error(std::string("stream_ts smem: ") + cudaGetErrorString(e));
  dim3 grid((unsigned)tp.n_mtiles, (unsigned)tp.nsplit);
  fn<<<grid, TS_THREADS, smem, st>>>(mx, mm, mml, part, (int)I, (int)S, tp.nkb, tp.kb_per_split, (int)tp.npb,
                                     b_pre ? 1 : 0, x3d ? 1 : 0, rows_b);
  e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("stream_ts: ") + cudaGetErrorString(e));
}

bool use_ts() {
  static const int v = [] {
    const char* e = getenv("FCTN_STREAM_SMEM_SPLIT");  // 1: the older smem-split 3xTF32 kernel
    return (e && e[0] == '1') ? 0 : 1;
  }();
  return v != 0;
}

template <int NT, bool AMN>
void go(const CUtensorMap& mx, const CUtensorMap& mx3, const CUtensorMap& mm, const CUtensorMap& mml, bool b_pre,
        bool x3d, float* part, int64_t I, int64_t S, const TcStreamPlan& tp, cudaStream_t st) {
  if (tp.split3 && use_ts())
    go_ts<NT, AMN>(x3d ? mx3 : mx, mm, mml, b_pre, x3d, part, I, S, tp, st);
  else if (tp.split3)
    go3<NT, AMN, true>(mx, mm, mml, b_pre, part, I, S, tp, st);
  else
    go3<NT, AMN, false>(mx, mm, mml, b_pre, part, I, S, tp, st);
}

}  // namespace

void tc_reserve_sms(int n) { g_reserved_sms = n; }

CUtensorMap tc_make_map_f32(const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                            const uint32_t* box, bool mn32) {
  return make_map(base, rank, dims, strides_bytes, box,
                  mn32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B);
}

CUtensorMap tc_make_map_f32_plain(const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                                  const uint32_t* box) {
  return make_map(base, rank, dims, strides_bytes, box, CU_TENSOR_MAP_SWIZZLE_NONE);
}

CUtensorMap tc_make_map_u32_plain(const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                                  const uint32_t* box) {
  return make_map(base, rank, dims, strides_bytes, box, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_DATA_TYPE_UINT32);
}

bool tc_stream_supported(int64_t I, int64_t P, int64_t Q, int64_t S) {
  if (S > 128) return false;
  if (I > (1LL << 31) || Q > (1LL << 31) || P > (1LL << 31)) return false;
  if (P == 1) return (I % 4 == 0) && (Q % 4 == 0);
  return P % 4 == 0;
}

TcStreamPlan plan_stream_tc(int64_t I, int64_t P, int64_t Q, int64_t S, int n_sm, bool split3) {
  TcStreamPlan tp;
  tp.split3 = split3;
  tp.nt = S <= 32 ? 32 : S <= 64 ? 64 : S <= 96 ? 96 : 128;
  tp.n_mtiles = (I + 127) / 128;
  tp.npb = P == 1 ? 1 : (P + BK - 1) / BK;
  tp.nkb = P == 1 ? (Q + BK - 1) / BK : tp.npb * Q;
  int64_t want = n_sm / tp.n_mtiles;
  if (want < 1) want = 1;
  if (want > tp.nkb) want = tp.nkb;
  tp.kb_per_split = (tp.nkb + want - 1) / want;
  tp.nsplit = (tp.nkb + tp.kb_per_split - 1) / tp.kb_per_split;
  return tp;
}

template <int NT, int NI>
static void go_tsw(const CUtensorMap& mx, const CUtensorMap& mm, float* part, int64_t I, int64_t S,
                   const TcStreamPlan& tp, cudaStream_t st) {
  const int smem = TswSmem<NT, NI>::TOTAL;
  auto fn = k_stream_tsw<NT, NI>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) throw std::runtime_error(std::string("stream_tsw smem: ") + cudaGetErrorString(e));
  fn<<<dim3(1u, (unsigned)tp.nsplit), TS_THREADS, smem, st>>>(mx, mm, part, (int)I, (int)S, tp.nkb, tp.kb_per_split,
                                                              (int)tp.npb);
  e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("stream_tsw: ") + cudaGetErrorString(e));
}

void launch_stream_tc(const float* X, const float* M, float* part, int64_t I, int64_t P, int64_t Q, int64_t S,
                      const TcStreamPlan& tp, cudaStream_t st, const float* Mlo) {
  CUtensorMap mx, mx3, mm, mml;
  const bool b_pre = Mlo != nullptr && tp.split3;
  const bool x3d = P == 1 && I % 32 == 0;
  if (P == 1) {
    uint64_t dx[2] = {(uint64_t)I, (uint64_t)Q}, sx[1] = {(uint64_t)I * 4};
    uint32_t bx[2] = {32, 32};
    mx = make_map(X, 2, dx, sx, bx, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);  // MN-major tf32: 32-B atoms
    mx3 = mx;
    if (x3d) {
      uint64_t d3[3] = {32, (uint64_t)Q, (uint64_t)(I / 32)}, s3[2] = {(uint64_t)I * 4, 128};
      uint32_t b3[3] = {32, 32, 4};
      mx3 = make_map(X, 3, d3, s3, b3, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    }
    uint64_t dm[2] = {(uint64_t)Q, (uint64_t)S}, sm[1] = {(uint64_t)Q * 4};
    uint32_t bm[2] = {32, (uint32_t)tp.nt};
    mm = make_map(M, 2, dm, sm, bm);
    mml = b_pre ? make_map(Mlo, 2, dm, sm, bm) : mm;
  } else {
    uint64_t dx[3] = {(uint64_t)P, (uint64_t)I, (uint64_t)Q}, sx[2] = {(uint64_t)P * 4, (uint64_t)P * I * 4};
    uint32_t bx[3] = {32, 128, 1};
    mx = make_map(X, 3, dx, sx, bx);
    mx3 = mx;
    uint64_t dm[3] = {(uint64_t)P, (uint64_t)Q, (uint64_t)S}, sm[2] = {(uint64_t)P * 4, (uint64_t)P * Q * 4};
    uint32_t bm[3] = {32, 1, (uint32_t)tp.nt};
    mm = make_map(M, 3, dm, sm, bm);
    mml = b_pre ? make_map(Mlo, 3, dm, sm, bm) : mm;
  }
  const bool amn = P == 1;
  // short mode (I <= 64) against many bond columns: the swapped-role kernel
  static const bool no_tsw = getenv("FCTN_NO_TSW") != nullptr;
  if (!amn && !b_pre && tp.split3 && !no_tsw && I <= 64 && S > I && tp.nt >= 96 && tp.n_mtiles == 1) {
    const int ni = I <= 32 ? 32 : I <= 48 ? 48 : 64;
    if (tp.nt == 96) {
      if (ni == 32) go_tsw<96, 32>(mx, mm, part, I, S, tp, st);
      else if (ni == 48) go_tsw<96, 48>(mx, mm, part, I, S, tp, st);
      else go_tsw<96, 64>(mx, mm, part, I, S, tp, st);
    } else {
      if (ni == 32) go_tsw<128, 32>(mx, mm, part, I, S, tp, st);
      else if (ni == 48) go_tsw<128, 48>(mx, mm, part, I, S, tp, st);
      else go_tsw<128, 64>(mx, mm, part, I, S, tp, st);
    }
    return;
  }
  switch (tp.nt) {
    case 32: amn ? go<32, true>(mx, mx3, mm, mml, b_pre, x3d, part, I, S, tp, st) : go<32, false>(mx, mx3, mm, mml, b_pre, x3d, part, I, S, tp, st); break;
    case 64: amn ? go<64, true>(mx, mx3, mm, mml, b_pre, x3d, part, I, S, tp, st) : go<64, false>(mx, mx3, mm, mml, b_pre, x3d, part, I, S, tp, st); break;
    case 96: amn ? go<96, true>(mx, mx3, mm, mml, b_pre, x3d, part, I, S, tp, st) : go<96, false>(mx, mx3, mm, mml, b_pre, x3d, part, I, S, tp, st); break;
    default: amn ? go<128, true>(mx, mx3, mm, mml, b_pre, x3d, part, I, S, tp, st) : go<128, false>(mx, mx3, mm, mml, b_pre, x3d, part, I, S, tp, st); break;
  }
}

// Z_j for a middle mode: out[(r, b), s] = sum_q X[r, q, b] B[q, s] with X
// [R, Q, NB] (r fastest), a batch of NB MN-major products (3xTF32, TMEM split;
// B pre-split hi / lo).  R % 128 == 0 so no 128-row tile straddles a batch.
bool tc_stream_batched_supported(int64_t R, int64_t Q, int64_t NB, int64_t S) {
  return R % 128 == 0 && Q % 4 == 0 && S <= 128 && R * Q * NB < (1LL << 40) && NB < (1LL << 31) && use_ts();
}
void launch_stream_tc_batched(const float* X, const float* Bh, const float* Bl, float* out, int64_t R, int64_t Q,
                              int64_t NB, int64_t S, int n_sm, cudaStream_t st) {
  TcStreamPlan tp = plan_stream_tc(R * NB, 1, Q, S, n_sm, true);
  tp.kb_per_split = tp.nkb;
  tp.nsplit = 1;
  uint64_t d4[4] = {32, (uint64_t)Q, (uint64_t)(R / 32), (uint64_t)NB};
  uint64_t s4[3] = {(uint64_t)R * 4, 128, (uint64_t)(R * Q * 4)};
  uint32_t b4[4] = {32, 32, 4, 1};
  CUtensorMap mx = make_map(X, 4, d4, s4, b4, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  uint64_t dm[2] = {(uint64_t)Q, (uint64_t)S}, sm[1] = {(uint64_t)Q * 4};
  uint32_t bm[2] = {32, (uint32_t)tp.nt};
  CUtensorMap mm = make_map(Bh, 2, dm, sm, bm);
  CUtensorMap mml = make_map(Bl, 2, dm, sm, bm);
  const int64_t I = R * NB;
  const int rb = (int)R;
  switch (tp.nt) {
    case 32: go_ts<32, true>(mx, mm, mml, true, true, out, I, S, tp, st, rb); break;
    case 64: go_ts<64, true>(mx, mm, mml, true, true, out, I, S, tp, st, rb); break;
    case 96: go_ts<96, true>(mx, mm, mml, true, true, out, I, S, tp, st, rb); break;
    default: go_ts<128, true>(mx, mm, mml, true, true, out, I, S, tp, st, rb); break;
  }
}

}  // namespace fctn
