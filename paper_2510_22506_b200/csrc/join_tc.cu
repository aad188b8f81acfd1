// K1 join on the B200 tensor cores (fp32 data): the large-output merges that
// write M_k (network.py:478-498 over tensor.py:156-200), as
//   D[m, n] = sum_k P[m, k] Q[n, k]   (tcgen05 kind::tf32, 3xTF32, fp32 TMEM)
// where P is the LONGER operand (M side, 128-row tiles) and Q the shorter (N
// side, one N-tile of <= 256 rows resident at a time).  The output element
// (m, n) goes to offM[m] + offN[n] (label descriptor, kernels.cuh); K <= 128.
//
// Why tensor cores here: the FP32 SIMT join (join.cu) is shared-memory bound
// (ncu: 16 wavefronts per warp k-step, FMA pipe ~40 %) at ~3-10x the HBM time
// of the output it writes; the MMA makes the operand reuse free and leaves the
// M_k store as the only real cost.
//
// Warp roles (416 threads):
//   warps 0-7  epilogue (two per TMEM lane quadrant, alternate 16-column
//              chunks): tcgen05.ld 32 lanes x 16 columns, global stores —
//              coalesced across lanes when P holds the output's fastest label,
//              128-bit per thread along n when Q does (vec_n)
//   warps 8-11 loaders: gather P rows (lane = row; unit stride by the
//              physical-modes-first partial layout, plan.cpp) and the Q tile,
//              round/split to TF32 hi/lo, write the SWIZZLE_128B K-major
//              layout UMMA reads; one 32-wide K block of a P tile per stage
//   warp 12    TMEM allocation + single-thread MMA issue
// Tiles: CTA b owns a contiguous range of (nt-major, mt-minor) tiles so the
// resident Q tile changes rarely; two TMEM accumulators overlap the epilogue
// of tile j with the MMAs of tile j+1.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace fctn {

namespace {

constexpr int JK = 32;           // fp32 per K block (one 128-byte row)
constexpr int P_TILE = 128 * JK * 4;  // 16 KB (hi or lo)
constexpr int NTHR = 416;  // 8 epilogue + 4 loader + 1 MMA warps
constexpr int EPI = 256;   // epilogue threads

struct TcJoinArgs {
  ContractDesc d;   // rows/cols as in kernels.cuh
  bool p_is_rows;   // P = the rows operand (else the cols operand)
  int nkb;          // K blocks (K <= 32 * nkb)
  int ntile;        // UMMA N (multiple of 16, <= 256)
  int pstages;
  int64_t n_mt, n_nt, ntiles, chunk;
  int vec_n;        // 4 (8): 4 (8) consecutive n are consecutive, 16-B (32-B) aligned output entries; else 0
};

struct Side {  // offsets of one operand group: index -> (operand offset, output offset)
  int n;
  const int64_t *ext, *so, *sc;
};

__device__ __forceinline__ void md2(uint32_t idx, const Side& s, int64_t& o1, int64_t& o2) {
  o1 = 0;
  o2 = 0;
  for (int q = 0; q < s.n; ++q) {
    const uint32_t e = (uint32_t)s.ext[q];
    const uint32_t dg = idx % e;
    idx /= e;
    o1 += (int64_t)dg * s.so[q];
    o2 += (int64_t)dg * s.sc[q];
  }
}

// byte offset of (row r, fp32 column c) in a K-major SWIZZLE_128B tile
__device__ __forceinline__ uint32_t swz(int r, int c4) { return (uint32_t)(r * 128 + (((c4 ^ (r & 7)) & 7) << 4)); }

__device__ __forceinline__ void split4(const float* x, float4& h, float4& l) {
  h.x = tc::tf32_rn_int(x[0]);
  h.y = tc::tf32_rn_int(x[1]);
  h.z = tc::tf32_rn_int(x[2]);
  h.w = tc::tf32_rn_int(x[3]);
  l = make_float4(x[0] - h.x, x[1] - h.y, x[2] - h.z, x[3] - h.w);
}

__device__ __forceinline__ void sts128(uint8_t* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

// 32 lanes x 16 columns, no wait (the caller waits with tmem_wait_ld)
__device__ __forceinline__ void tmem_ld16_async(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// PMN: the P tile is MN-major (SWIZZLE_128B with 32-byte atoms, the layout a
// TMA SWIZZLE_128B_ATOM_32B box writes: 32-row boxes of 4 KB, K row kq holds
// 32 consecutive rows, 8-float atoms XOR (kq & 3)) so 4 consecutive rows of
// one K index are one 16-byte cp.async; else K-major SW128 with 4-byte gathers.
template <int NCOL, bool PMN>
__global__ void __launch_bounds__(NTHR, 1)
    k_join_tc(const float* __restrict__ Pg, const float* __restrict__ Qg, float* __restrict__ C, const TcJoinArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const ContractDesc& d = a.d;
  const int S = a.pstages, nkb = a.nkb, NT = a.ntile;
  // [P stages: hi | lo][Q: nkb x (hi | lo) x NT rows][koffP | koffQ][offN][barriers]
  uint8_t* pst = smem;
  uint8_t* qt = pst + (size_t)S * 2 * P_TILE;
  const size_t q_block = (size_t)NT * 128;  // one K block of Q, hi or lo
  int64_t* koffP = reinterpret_cast<int64_t*>(qt + (size_t)nkb * 2 * q_block);
  int64_t* koffQ = koffP + 32 * nkb;
  int32_t* offN = reinterpret_cast<int32_t*>(koffQ + 32 * nkb);  // [NT] output offsets of the N tile (epilogue)
  uint64_t* bars = reinterpret_cast<uint64_t*>(offN + 256);
  uint64_t* pfull = bars;
  uint64_t* pempty = pfull + S;
  uint64_t* qfull = pempty + S;
  uint64_t* qempty = qfull + 1;
  uint64_t* tfull = qempty + 1;   // [2]
  uint64_t* tempty = tfull + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // P / Q label groups (operand offsets, output offsets)
  const Side rowsS{d.nr, d.r_ext, d.r_sa, d.r_sc}, colsS{d.nc, d.c_ext, d.c_sb, d.c_sc};
  const Side& PS = a.p_is_rows ? rowsS : colsS;
  const Side& QS = a.p_is_rows ? colsS : rowsS;
  const int64_t Pn = a.p_is_rows ? d.rows : d.cols, Qn = a.p_is_rows ? d.cols : d.rows;
  const int K = (int)d.K;

  for (int k = threadIdx.x; k < 32 * nkb; k += NTHR) {
    int64_t ka = -1, kb = -1;
    if (k < K) {
      ka = 0;
      kb = 0;
      uint32_t idx = (uint32_t)k;
      for (int q = 0; q < d.nk; ++q) {
        const uint32_t e = (uint32_t)d.k_ext[q];
        const uint32_t dg = idx % e;
        idx /= e;
        ka += (int64_t)dg * d.k_sa[q];
        kb += (int64_t)dg * d.k_sb[q];
      }
    }
    koffP[k] = a.p_is_rows ? ka : kb;  // k_sa: rows operand, k_sb: cols operand
    koffQ[k] = a.p_is_rows ? kb : ka;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&pfull[s], 4);
      tc::mbar_init(&pempty[s], 1);
    }
    tc::mbar_init(qfull, 4);
    tc::mbar_init(qempty, 1);
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], EPI / 32);
    }
    tc::fence_barrier_init();
  }
  if (warp == 12) tc::tmem_alloc<2 * NCOL>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  const int64_t t0 = (int64_t)blockIdx.x * a.chunk;
  int64_t t1 = t0 + a.chunk;
  if (t1 > a.ntiles) t1 = a.ntiles;
  auto tile_mn = [&](int64_t t, int64_t& mt, int64_t& nt) {
    nt = t / a.n_mt;
    mt = t - nt * a.n_mt;
  };

  if (warp >= 8 && warp < 12) {
    // ------------------------------------------------ loaders
    // P stages: cp.async gathers of this thread's row straight into the
    // swizzled hi tile, up to PD stages in flight; when a stage has landed it
    // is split in place (hi) and into the lo tile, then published.
    const int lt = threadIdx.x - EPI;  // 0..127 = row of the P tile
    const int PD = S - 1 < 4 ? S - 1 : 4;
    const int n_st = (int)(t1 - t0) * nkb;  // stages this CTA consumes
    int64_t cur_nt = -1;
    int qphase = 0;
    int issued = 0;
    int64_t iss_op = -1;  // row offset of the tile being issued
    int64_t iss_t = -1;
    int64_t p_m0 = 0;
    auto issue = [&](int i) {  // gathers of stage i (tile t0 + i / nkb, K block i % nkb)
      const int s = i % S;
      tc::mbar_wait(&pempty[s], ((i / S) & 1) ^ 1);
      const int64_t t = t0 + i / nkb;
      const int kb = i % nkb;
      if (t != iss_t) {
        iss_t = t;
        int64_t mt, nt;
        tile_mn(t, mt, nt);
        p_m0 = mt * 128;
        const int64_t m = PMN ? p_m0 + 4 * (lt & 31) : p_m0 + lt;
        int64_t oc;
        iss_op = -1;
        if (m < Pn) md2((uint32_t)m, PS, iss_op, oc);
      }
      uint8_t* hi = pst + (size_t)s * 2 * P_TILE;
      if (PMN) {
        const int mn4 = lt & 31, kq0 = lt >> 5;
        const int i = (4 * mn4) & 31;
        uint8_t* box = hi + (mn4 >> 3) * 4096;
        const int64_t m0 = p_m0 + 4 * mn4;
        const bool full4 = m0 + 3 < Pn;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int k = kq0 + 4 * j;
          const int64_t ko = koffP[kb * 32 + k];
          const uint32_t dst = tc::smem_u32(box + (k * 32 + (((i >> 3) ^ (k & 3)) << 3) + (i & 7)) * 4);
          if (full4 || m0 >= Pn) {
            const bool ok = full4 && ko >= 0;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst),
                         "l"(Pg + (ok ? iss_op + ko : 0)), "r"(ok ? 16 : 0));
          } else {  // ragged end of P: rows one by one
            for (int e = 0; e < 4; ++e) {
              int64_t o1 = -1, oc;
              if (m0 + e < Pn) md2((uint32_t)(m0 + e), PS, o1, oc);
              const bool ok = o1 >= 0 && ko >= 0;
              asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst + 4 * e),
                           "l"(Pg + (ok ? o1 + ko : 0)), "r"(ok ? 4 : 0));
            }
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int64_t ko = koffP[kb * 32 + k];
          const bool ok = iss_op >= 0 && ko >= 0;
          const uint32_t dst = tc::smem_u32(hi + swz(lt, k >> 2) + (k & 3) * 4);
          // no memory clobber: the offset loads may be scheduled ahead; the
          // wait_group below orders the smem reads
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst),
                       "l"(Pg + (ok ? iss_op + ko : 0)), "r"(ok ? 4 : 0));
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int i = 0; i < n_st; ++i) {
      const int64_t t = t0 + i / nkb;
      if (i % nkb == 0) {
        int64_t mt, nt;
        tile_mn(t, mt, nt);
        if (nt != cur_nt) {  // (re)load the Q tile: NT rows x nkb K blocks
          if (cur_nt >= 0) {
            tc::mbar_wait(qempty, qphase);
            qphase ^= 1;
          }
          cur_nt = nt;
          for (int r = lt; r < NT; r += 128) {
            const int64_t n = nt * NT + r;
            int64_t oq = -1, oc;
            if (n < Qn) md2((uint32_t)n, QS, oq, oc);
            for (int kb = 0; kb < nkb; ++kb) {
              uint8_t* hi = qt + (size_t)kb * 2 * q_block;
              uint8_t* lo = hi + q_block;
#pragma unroll
              for (int c4 = 0; c4 < 8; ++c4) {
                float x[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const int64_t ko = koffQ[kb * 32 + c4 * 4 + j];
                  x[j] = (oq >= 0 && ko >= 0) ? __ldg(Qg + oq + ko) : 0.f;
                }
                float4 h, l;
                split4(x, h, l);
                sts128(hi + swz(r, c4), h);
                sts128(lo + swz(r, c4), l);
              }
            }
          }
          tc::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(qfull);
        }
      }
      // keep PD stages of gathers in flight
      while (issued < n_st && issued < i + PD) issue(issued++);
      // stage i has landed when at most (issued - i - 1) younger groups are pending
      const int younger = issued - i - 1;
      if (younger >= 3) asm volatile("cp.async.wait_group 3;" ::: "memory");
      else if (younger == 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
      else if (younger == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
      else asm volatile("cp.async.wait_group 0;" ::: "memory");
      const int s = i % S;
      uint8_t* hi = pst + (size_t)s * 2 * P_TILE;
      uint8_t* lo = hi + P_TILE;
      if (PMN) {  // the 8 chunks this thread gathered
        const int mn4 = lt & 31, kq0 = lt >> 5, ii = (4 * mn4) & 31;
        const uint32_t bo = (mn4 >> 3) * 4096;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int k = kq0 + 4 * j;
          const uint32_t off = bo + (k * 32 + (((ii >> 3) ^ (k & 3)) << 3) + (ii & 7)) * 4;
          const float4 v = *reinterpret_cast<const float4*>(hi + off);
          const float x[4] = {v.x, v.y, v.z, v.w};
          float4 h, l;
          split4(x, h, l);
          sts128(hi + off, h);
          sts128(lo + off, l);
        }
      } else {
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4) {
        const float4 v = *reinterpret_cast<const float4*>(hi + swz(lt, c4));
        const float x[4] = {v.x, v.y, v.z, v.w};
        float4 h, l;
        split4(x, h, l);
        sts128(hi + swz(lt, c4), h);
        sts128(lo + swz(lt, c4), l);
      }
      }
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&pfull[s]);
    }
  } else if (warp == 12) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_tf32(128, NT, PMN, false);
      int64_t cur_nt = -1;
      int qphase = 0;
      int it = 0;
      int j = 0;
      for (int64_t t = t0; t < t1; ++t, ++j) {
        int64_t mt, nt;
        tile_mn(t, mt, nt);
        if (nt != cur_nt) {
          tc::mbar_wait(qfull, qphase);
          qphase ^= 1;
          cur_nt = nt;
        }
        const int b = j & 1;
        tc::mbar_wait(&tempty[b], ((j >> 1) & 1) ^ 1);
        tc::fence_after_sync();
        const uint32_t acc = tmem + b * NCOL;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % S;
          tc::mbar_wait(&pfull[s], (it / S) & 1);
          tc::fence_after_sync();
          const uint32_t ph = tc::smem_u32(pst + (size_t)s * 2 * P_TILE), pl = ph + P_TILE;
          const uint32_t qh = tc::smem_u32(qt + (size_t)kb * 2 * q_block), ql = qh + (uint32_t)q_block;
#pragma unroll
          for (int kk = 0; kk < JK / 8; ++kk) {
            const uint64_t ad = PMN ? tc::sdesc(ph + kk * 1024, 4096, 512, 1) : tc::sdesc(ph + kk * 32, 16, 1024);
            const uint64_t adl = PMN ? tc::sdesc(pl + kk * 1024, 4096, 512, 1) : tc::sdesc(pl + kk * 32, 16, 1024);
            const uint64_t bd = tc::sdesc(qh + kk * 32, 16, 1024), bdl = tc::sdesc(ql + kk * 32, 16, 1024);
            tc::mma_tf32(acc, adl, bd, idesc, (kb | kk) != 0);
            tc::mma_tf32(acc, ad, bdl, idesc, 1);
            tc::mma_tf32(acc, ad, bd, idesc, 1);
          }
          tc::mma_commit(&pempty[s]);
        }
        tc::mma_commit(&tfull[b]);
        int64_t mt2, nt2;
        if (t + 1 < t1) tile_mn(t + 1, mt2, nt2);
        if (t + 1 < t1 && nt2 != nt) tc::mma_commit(qempty);  // Q may be overwritten once these MMAs retire
      }
    }
  } else {
    // ------------------------------------------------ epilogue: warps w and w + 4 share TMEM lane
    // quadrant w & 3 and take alternate 16-column chunks
    const int q = warp & 3, half = warp >> 2;  // lanes 32q .. 32q+31
    int64_t cur_nt = -1;
    bool nfull = false;  // every column of the N tile exists
    int j = 0;
    for (int64_t t = t0; t < t1; ++t, ++j) {
      int64_t mt, nt;
      tile_mn(t, mt, nt);
      if (nt != cur_nt) {
        tc::named_bar(1, EPI);  // previous tile's readers of offN are done
        for (int r = threadIdx.x; r < NT; r += EPI) {
          const int64_t n = nt * NT + r;
          int64_t oq, o = -1;
          if (n < Qn) md2((uint32_t)n, QS, oq, o);
          offN[r] = (int32_t)o;  // M_k < 2^31 entries (tc_join_applicable)
        }
        tc::named_bar(1, EPI);
        cur_nt = nt;
        nfull = (nt + 1) * NT <= Qn;
      }
      const int64_t m = mt * 128 + q * 32 + lane;
      int64_t op, om = -1;
      if (m < Pn) md2((uint32_t)m, PS, op, om);
      const int b = j & 1;
      tc::mbar_wait(&tfull[b], (j >> 1) & 1);
      tc::fence_after_sync();
      const uint32_t acc = tmem + b * NCOL + ((uint32_t)(q * 32) << 16);
      // the next 16 columns are read from TMEM while this block is stored; the
      // block's 16 output offsets come from shared memory in 4 vector loads
      // issued ahead of the stores
      const uint32_t offN_s = tc::smem_u32(offN);
      float* Cm = C + (om >= 0 ? om : 0);
      uint32_t r0[16], r1[16];
      const int nch = NT / 16;
      if (half < nch) {
        tmem_ld16_async(acc + 16 * half, r0);
        tmem_wait_ld();
      }
      for (int c = half; c < nch; c += 2) {
        const int n0 = 16 * c;
        if (c + 2 < nch) tmem_ld16_async(acc + n0 + 32, r1);
        int o[16];
#pragma unroll
        for (int j4 = 0; j4 < 4; ++j4)
          asm("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
              : "=r"(o[4 * j4]), "=r"(o[4 * j4 + 1]), "=r"(o[4 * j4 + 2]), "=r"(o[4 * j4 + 3])
              : "r"(offN_s + 4 * (n0 + 4 * j4)));
        if (om >= 0) {
          if (a.vec_n == 8) {
            // one full 32-byte sector per store: the 128-bit form left the SM
            // as two half-sector writes per sector (ncu: 3.44 GB of L1 -> L2
            // write traffic for the 1.72 GB M_k, 798 us against 484 us for
            // the lane-coalesced form)
#pragma unroll
            for (int j8 = 0; j8 < 2; ++j8) {
              if (nfull || o[8 * j8 + 7] >= 0) {
                asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(Cm + o[8 * j8]),
                             "f"(__uint_as_float(r0[8 * j8])), "f"(__uint_as_float(r0[8 * j8 + 1])),
                             "f"(__uint_as_float(r0[8 * j8 + 2])), "f"(__uint_as_float(r0[8 * j8 + 3])),
                             "f"(__uint_as_float(r0[8 * j8 + 4])), "f"(__uint_as_float(r0[8 * j8 + 5])),
                             "f"(__uint_as_float(r0[8 * j8 + 6])), "f"(__uint_as_float(r0[8 * j8 + 7]))
                             : "memory");
              } else {
#pragma unroll
                for (int e = 0; e < 8; ++e)
                  if (o[8 * j8 + e] >= 0) Cm[o[8 * j8 + e]] = __uint_as_float(r0[8 * j8 + e]);
              }
            }
          } else if (a.vec_n) {
#pragma unroll
            for (int j4 = 0; j4 < 4; ++j4) {
              if (nfull || o[4 * j4 + 3] >= 0) {
                *reinterpret_cast<float4*>(Cm + o[4 * j4]) =
                    make_float4(__uint_as_float(r0[4 * j4]), __uint_as_float(r0[4 * j4 + 1]),
                                __uint_as_float(r0[4 * j4 + 2]), __uint_as_float(r0[4 * j4 + 3]));
              } else {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  if (o[4 * j4 + e] >= 0) Cm[o[4 * j4 + e]] = __uint_as_float(r0[4 * j4 + e]);
              }
            }
          } else if (nfull) {
#pragma unroll
            for (int e = 0; e < 16; ++e) Cm[o[e]] = __uint_as_float(r0[e]);
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (o[e] >= 0) Cm[o[e]] = __uint_as_float(r0[e]);
          }
        }
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e) r0[e] = r1[e];
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[b]);
    }
  }
  __syncthreads();
  if (warp == 12) tc::tmem_dealloc<2 * NCOL>(tmem);
}

size_t tcj_smem(int nkb, int ntile, int pstages) {
  return 1024 + (size_t)pstages * 2 * P_TILE + (size_t)nkb * 2 * ntile * 128 + 2 * 32 * nkb * 8 + 256 * 4 + 256;
}

}  // namespace

bool tc_join_applicable(const ContractDesc& d) {
  if (getenv("FCTN_NO_TC_JOIN")) return false;
  if (d.K < 1 || d.K > 128) return false;
  const int64_t lo = std::min(d.rows, d.cols), hi = std::max(d.rows, d.cols);
  if (lo < 16 || hi < 128) return false;
  if (hi >= ((int64_t)1 << 31) || d.rows * d.cols >= ((int64_t)1 << 31)) return false;
  static const int64_t min_out =
      getenv("FCTN_JOIN_MIN_OUT") ? atoll(getenv("FCTN_JOIN_MIN_OUT")) : ((int64_t)1 << 20);
  return d.rows * d.cols >= min_out;
}

void launch_join_tc(const float* A, const float* B, float* C, const ContractDesc& d, int n_sm, cudaStream_t st) {
  TcJoinArgs a;
  a.d = d;
  a.p_is_rows = d.rows >= d.cols;
  const int64_t Pn = a.p_is_rows ? d.rows : d.cols, Qn = a.p_is_rows ? d.cols : d.rows;
  a.nkb = (int)((d.K + JK - 1) / JK);
  // N tile: the whole short side when it fits 256 columns, else 128/256
  int64_t nt = Qn <= 256 ? Qn : (a.nkb >= 3 ? 128 : 256);
  a.ntile = (int)((nt + 15) / 16 * 16);
  a.n_mt = (Pn + 127) / 128;
  a.n_nt = (Qn + a.ntile - 1) / a.ntile;
  a.ntiles = a.n_mt * a.n_nt;
  const size_t budget = 220 * 1024;
  a.pstages = 6;
  while (a.pstages > 2 && tcj_smem(a.nkb, a.ntile, a.pstages) > budget) --a.pstages;
  const size_t smem = tcj_smem(a.nkb, a.ntile, a.pstages);
  if (smem > budget) throw std::runtime_error("join_tc: tile does not fit shared memory");
  const int64_t grid = std::min<int64_t>(a.ntiles, n_sm);
  a.chunk = (a.ntiles + grid - 1) / grid;
  // n runs along the output's fastest label with unit stride (Q holds it)
  int vec_n = 0;
  for (int w : {8, 4}) {
    const int n = a.p_is_rows ? d.nc : d.nr;
    const int64_t* ext = a.p_is_rows ? d.c_ext : d.r_ext;
    const int64_t* sc = a.p_is_rows ? d.c_sc : d.r_sc;
    bool ok = n >= 1 && sc[0] == 1 && ext[0] % w == 0 && a.ntile % w == 0 &&
              reinterpret_cast<uintptr_t>(C) % (4 * w) == 0;
    for (int q = 1; q < n && ok; ++q) ok = sc[q] % w == 0;
    const int np = a.p_is_rows ? d.nr : d.nc;
    const int64_t* scp = a.p_is_rows ? d.r_sc : d.c_sc;
    for (int q = 0; q < np && ok; ++q) ok = scp[q] % w == 0;
    if (ok && !(w == 8 && getenv("FCTN_JOIN_NO_V8"))) {
      vec_n = w;
      break;
    }
  }
  a.vec_n = vec_n;
  const float* P = a.p_is_rows ? A : B;
  // P rows: 4 consecutive indices = 4 consecutive, 16-byte aligned operand entries
  bool vec_p = reinterpret_cast<uintptr_t>(P) % 16 == 0 && !getenv("FCTN_TC_JOIN_KMAJOR");
  {
    const int n = a.p_is_rows ? d.nr : d.nc;
    const int64_t* ext = a.p_is_rows ? d.r_ext : d.c_ext;
    const int64_t* so = a.p_is_rows ? d.r_sa : d.c_sb;
    const int64_t* ko = a.p_is_rows ? d.k_sa : d.k_sb;
    vec_p = vec_p && n >= 1 && so[0] == 1 && ext[0] % 4 == 0;
    for (int q = 1; q < n && vec_p; ++q) vec_p = so[q] % 4 == 0;
    for (int q = 0; q < d.nk && vec_p; ++q) vec_p = ko[q] % 4 == 0;
  }
  const float* Q = a.p_is_rows ? B : A;
  if (getenv("FCTN_JOIN_TRACE")) {
    fprintf(stderr, "join_tc rows=%lld cols=%lld K=%lld p_rows=%d vec_n=%d vec_p=%d ntile=%d nkb=%d |",
            (long long)d.rows, (long long)d.cols, (long long)d.K, (int)a.p_is_rows, (int)a.vec_n, (int)vec_p,
            a.ntile, a.nkb);
    for (int q = 0; q < d.nr; ++q) fprintf(stderr, " r(%lld,%lld,%lld)", (long long)d.r_ext[q], (long long)d.r_sa[q], (long long)d.r_sc[q]);
    for (int q = 0; q < d.nc; ++q) fprintf(stderr, " c(%lld,%lld,%lld)", (long long)d.c_ext[q], (long long)d.c_sb[q], (long long)d.c_sc[q]);
    fprintf(stderr, " C=%p\n", (void*)C);
  }
  auto go = [&](auto kern) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) throw std::runtime_error(std::string("join_tc smem: ") + cudaGetErrorString(e));
    kern<<<(unsigned)((a.ntiles + a.chunk - 1) / a.chunk), NTHR, smem, st>>>(P, Q, C, a);
    e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("join_tc: ") + cudaGetErrorString(e));
  };
  if (vec_p) {
    if (a.ntile <= 64) go(k_join_tc<64, true>);
    else if (a.ntile <= 128) go(k_join_tc<128, true>);
    else go(k_join_tc<256, true>);
  } else {
    if (a.ntile <= 64) go(k_join_tc<64, false>);
    else if (a.ntile <= 128) go(k_join_tc<128, false>);
    else go(k_join_tc<256, false>);
  }
}

}  // namespace fctn
