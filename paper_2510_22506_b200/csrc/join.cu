// K1 "join": the large-output labeled contractions of the merge — the final
// join of the left and right partials that writes M_k (network.py:478-498
// over tensor.py:156-200), and the other partials whose output is large
// relative to their operands.  Shapes at the BASELINE configs (rows x K x
// cols, rows = the operand holding M_k's fastest label): c5 2985984x27x144,
// 144x27x2985984, 20736x81x20736; c3 633600x25x250.  The output (up to 430 M
// entries, 1.7 GB fp32) dominates the traffic: HBM-bound at K <= ~30 with
// FP32 FMAs, FMA-bound above.
//
// Design: persistent CTAs walk (row tile x col tile) output tiles; the full
// K extent of both operand tiles is staged in shared memory by 4/8-byte
// cp.async gathers (the operands are arbitrary label permutations, so no
// TMA box describes them) into a two-stage ring, so the next tile's gathers
// overlap this tile's FMAs and stores.  A warp covers 32*RT rows x 4 column
// slots (8 x 4 lanes) so each k step costs it one shared wavefront per
// operand fragment (ncu: the 16 x 2-lane layout was shared-bandwidth bound);
// a thread owns RT groups of 4 consecutive rows x CT columns in registers,
// reads them with 128-bit shared loads (ping-pong fragment buffers), and
// stores 4 consecutive rows of one column as one 128-bit (fp32) or two
// 128-bit (fp64) stores — the output's fastest label runs along the rows by
// construction of the descriptor.
// All offsets come from the descriptor on device (32-bit digit extraction).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "kernels.cuh"

namespace fctn {

namespace {

__device__ __forceinline__ void md_off32(uint32_t idx, int nd, const int64_t* ext, const int64_t* s1,
                                         const int64_t* s2, int64_t& o1, int64_t& o2) {
  o1 = 0;
  o2 = 0;
  for (int q = 0; q < nd; ++q) {
    const uint32_t e = (uint32_t)ext[q];
    const uint32_t d = idx % e;
    idx /= e;
    o1 += (int64_t)d * s1[q];
    o2 += (int64_t)d * s2[q];
  }
}

template <int BYTES>
__device__ __forceinline__ void cp_async_zfill(void* smem, const void* gmem, bool valid) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  const int src = valid ? BYTES : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(s), "l"(gmem), "n"(BYTES), "r"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <typename T>
struct Vec4 {
  T v[4];
};
template <typename T>
__device__ __forceinline__ Vec4<T> lds4(const T* p);
template <>
__device__ __forceinline__ Vec4<float> lds4<float>(const float* p) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  return {{a.x, a.y, a.z, a.w}};
}
template <>
__device__ __forceinline__ Vec4<double> lds4<double>(const double* p) {
  const double2 a = *reinterpret_cast<const double2*>(p);
  const double2 b = *reinterpret_cast<const double2*>(p + 2);
  return {{a.x, a.y, b.x, b.y}};
}
template <typename T>
__device__ __forceinline__ void stg4(T* p, const T* v);
template <>
__device__ __forceinline__ void stg4<float>(float* p, const float* v) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
template <>
__device__ __forceinline__ void stg4<double>(double* p, const double* v) {
  reinterpret_cast<double2*>(p)[0] = make_double2(v[0], v[1]);
  reinterpret_cast<double2*>(p)[1] = make_double2(v[2], v[3]);
}

constexpr int JT = 256;  // threads: 8 warps = 2 (rows) x 4 (cols); lanes = 8 (row quads) x 4 (col slots)
constexpr int JX = 16;   // row quads per CTA per row group (2 warps x 8 lanes)
constexpr int JY = 16;   // column slots per CTA (4 warps x 4 lanes), CT columns each
constexpr int BP = JY * 4;  // padded B row: every slot 4 wide (one 128-bit shared load)

struct JoinArgs {
  ContractDesc d;
  int64_t n_rt, n_ct, ntiles;
  int fix;         // 0: both operands streamed; 1: the CTA's row tile is fixed (A resident); 2: col tile fixed
  int64_t n_fix;   // tiles of the fixed side
  bool vec;        // 4 consecutive rows are 4 consecutive output entries
  bool vec_a;      // 4 consecutive rows are 4 consecutive, 16-byte aligned A entries
  bool vec_b;      // same for B along cols
};

// Shared-memory plan: A tiles [K][BR], B tiles [K][BP] (column slot i holds
// columns i*CT .. i*CT+CT-1 in 4 padded entries), one stage for a fixed
// operand, two for a streamed one.
template <typename T, int RT, int CT>
struct JoinTile {
  static constexpr int BR = JX * 4 * RT;
  static constexpr int BC = JY * CT;
};

template <typename T, int RT, int CT>
__global__ void __launch_bounds__(JT) k_join(const T* __restrict__ A, const T* __restrict__ B, T* __restrict__ C,
                                              const JoinArgs p) {
  constexpr int BR = JoinTile<T, RT, CT>::BR, BC = JoinTile<T, RT, CT>::BC;
  const ContractDesc& d = p.d;
  const int K = (int)d.K;
  const int sa = p.fix == 1 ? 1 : 2, sb = p.fix == 2 ? 1 : 2;  // stages
  extern __shared__ __align__(16) unsigned char smraw[];
  T* As = reinterpret_cast<T*>(smraw);                         // [sa][K][BR]
  T* Bs = As + (size_t)sa * K * BR;                            // [sb][K][BP]
  int64_t* sRA = reinterpret_cast<int64_t*>(Bs + (size_t)sb * K * BP);  // [2][BR]
  int64_t* sRC = sRA + 2 * BR;                                 // [2][BR]
  int64_t* sCB = sRC + 2 * BR;                                 // [2][BP]
  int64_t* sCC = sCB + 2 * BP;                                 // [2][BP]
  int64_t* sKA = sCC + 2 * BP;                                 // [K]
  int64_t* sKB = sKA + K;                                      // [K]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row0 = (warp & 1) * (32 * RT) + (lane & 7) * 4;   // first row of the thread's group 0
  const int slot = (warp >> 1) * 4 + (lane >> 3);             // column slot

  for (int k = tid; k < K; k += JT) {
    int64_t a, b;
    md_off32((uint32_t)k, d.nk, d.k_ext, d.k_sa, d.k_sb, a, b);
    sKA[k] = a;
    sKB[k] = b;
  }
  // work item w -> (row tile, col tile)
  int64_t n_items, step;
  if (p.fix == 1) {
    n_items = p.n_ct;
    step = gridDim.x / p.n_fix;
  } else if (p.fix == 2) {
    n_items = p.n_rt;
    step = gridDim.x / p.n_fix;
  } else {
    n_items = p.ntiles;
    step = gridDim.x;
  }
  const int64_t fixed_tile = p.fix ? blockIdx.x % p.n_fix : 0;
  const int64_t first = p.fix ? blockIdx.x / p.n_fix : blockIdx.x;
  auto tile_rc = [&](int64_t w, int64_t& rt, int64_t& ct) {
    if (p.fix == 1) {
      rt = fixed_tile;
      ct = w;
    } else if (p.fix == 2) {
      ct = fixed_tile;
      rt = w;
    } else if (p.n_rt <= p.n_ct) {
      rt = w % p.n_rt;
      ct = w / p.n_rt;
    } else {
      ct = w % p.n_ct;
      rt = w / p.n_ct;
    }
  };
  auto rows_in = [&](int64_t rt, int st) {  // offsets, then gathers of A's row tile into stage st
    const int64_t r0 = rt * BR;
    for (int i = tid; i < BR; i += JT) {
      int64_t oa = -1, oc = 0;
      if (r0 + i < d.rows) md_off32((uint32_t)(r0 + i), d.nr, d.r_ext, d.r_sa, d.r_sc, oa, oc);
      sRA[st * BR + i] = oa;
      sRC[st * BR + i] = oc;
    }
    __syncthreads();
    T* as = As + (size_t)(sa == 1 ? 0 : st) * K * BR;
    if (p.vec_a) {
      for (int e = tid; e < K * (BR / 4); e += JT) {
        const int k = e / (BR / 4), r = 4 * (e - k * (BR / 4));
        const int64_t oa = sRA[st * BR + r + 3] >= 0 ? sRA[st * BR + r] : -1;
        if (oa >= 0 || sRA[st * BR + r] < 0) {
          cp_async_zfill<16>(as + k * BR + r, A + (oa >= 0 ? oa + sKA[k] : 0), oa >= 0);
          if (sizeof(T) == 8) cp_async_zfill<16>(as + k * BR + r + 2, A + (oa >= 0 ? oa + sKA[k] + 2 : 0), oa >= 0);
        } else {  // ragged end of the rows
          for (int q = 0; q < 4; ++q) {
            const int64_t o = sRA[st * BR + r + q];
            cp_async_zfill<sizeof(T)>(as + k * BR + r + q, A + (o >= 0 ? o + sKA[k] : 0), o >= 0);
          }
        }
      }
    } else {
      for (int e = tid; e < K * BR; e += JT) {
        const int k = e / BR, r = e - k * BR;
        const int64_t oa = sRA[st * BR + r];
        cp_async_zfill<sizeof(T)>(as + e, A + (oa >= 0 ? oa + sKA[k] : 0), oa >= 0);
      }
    }
  };
  auto cols_in = [&](int64_t ct, int st) {
    const int64_t c0 = ct * BC;
    for (int i = tid; i < BP; i += JT) {
      const int j = i & 3;
      const int64_t c = c0 + (i >> 2) * CT + j;
      int64_t ob = -1, oc = -1;
      if (j < CT && c < d.cols) md_off32((uint32_t)c, d.nc, d.c_ext, d.c_sb, d.c_sc, ob, oc);
      sCB[st * BP + i] = ob;
      sCC[st * BP + i] = oc;
    }
    __syncthreads();
    T* bs = Bs + (size_t)(sb == 1 ? 0 : st) * K * BP;
    if (CT == 4 && p.vec_b) {
      for (int e = tid; e < K * (BP / 4); e += JT) {
        const int k = e / (BP / 4), c = 4 * (e - k * (BP / 4));
        const int64_t ob = sCB[st * BP + c + 3] >= 0 ? sCB[st * BP + c] : -1;
        if (ob >= 0 || sCB[st * BP + c] < 0) {
          cp_async_zfill<16>(bs + k * BP + c, B + (ob >= 0 ? ob + sKB[k] : 0), ob >= 0);
          if (sizeof(T) == 8) cp_async_zfill<16>(bs + k * BP + c + 2, B + (ob >= 0 ? ob + sKB[k] + 2 : 0), ob >= 0);
        } else {
          for (int q = 0; q < 4; ++q) {
            const int64_t o = sCB[st * BP + c + q];
            cp_async_zfill<sizeof(T)>(bs + k * BP + c + q, B + (o >= 0 ? o + sKB[k] : 0), o >= 0);
          }
        }
      }
    } else {
      for (int e = tid; e < K * BP; e += JT) {
        const int k = e / BP, c = e - k * BP;
        const int64_t ob = sCB[st * BP + c];
        cp_async_zfill<sizeof(T)>(bs + e, B + (ob >= 0 ? ob + sKB[k] : 0), ob >= 0);
      }
    }
  };
  auto stage_in = [&](int64_t w, int st) {
    int64_t rt, ct;
    tile_rc(w, rt, ct);
    if (p.fix != 1) rows_in(rt, st);
    if (p.fix != 2) cols_in(ct, st);
    cp_async_commit();
  };

  __syncthreads();  // sKA / sKB
  int64_t w = first;
  if (w >= n_items) return;
  // the fixed operand: offsets in both table stages, data once
  if (p.fix == 1) {
    rows_in(fixed_tile, 0);
    for (int i = tid; i < BR; i += JT) {
      sRA[BR + i] = sRA[i];
      sRC[BR + i] = sRC[i];
    }
  } else if (p.fix == 2) {
    cols_in(fixed_tile, 0);
    for (int i = tid; i < BP; i += JT) {
      sCB[BP + i] = sCB[i];
      sCC[BP + i] = sCC[i];
    }
  }
  int s = 0;
  stage_in(w, 0);
  for (; w < n_items; w += step, s ^= 1) {
    const int64_t wn = w + step;
    if (wn < n_items) {
      stage_in(wn, s ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const T* as = As + (size_t)(sa == 1 ? 0 : s) * K * BR + row0;
    const T* bs = Bs + (size_t)(sb == 1 ? 0 : s) * K * BP + slot * 4;
    T acc[RT][4][CT];
#pragma unroll
    for (int g = 0; g < RT; ++g)
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int j = 0; j < CT; ++j) acc[g][q][j] = T(0);
    // ping-pong fragments: k + 1 is read from shared memory while k multiplies
    Vec4<T> a0[RT], a1[RT], b0, b1;
    auto frag = [&](int k, Vec4<T>* a, Vec4<T>& b) {
#pragma unroll
      for (int g = 0; g < RT; ++g) a[g] = lds4<T>(as + k * BR + g * 32);
      b = lds4<T>(bs + k * BP);
    };
    auto mac = [&](const Vec4<T>* a, const Vec4<T>& b) {
#pragma unroll
      for (int g = 0; g < RT; ++g)
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int j = 0; j < CT; ++j) acc[g][q][j] += a[g].v[q] * b.v[j];
    };
    frag(0, a0, b0);
    int k = 0;
    for (; k + 2 <= K; k += 2) {
      frag(k + 1, a1, b1);
      mac(a0, b0);
      frag(k + 2 < K ? k + 2 : K - 1, a0, b0);
      mac(a1, b1);
    }
    if (k < K) mac(a0, b0);
    // epilogue: 4 consecutive rows of one column per store
#pragma unroll
    for (int j = 0; j < CT; ++j) {
      const int64_t cc = sCC[s * BP + slot * 4 + j];
      if (cc < 0) continue;
#pragma unroll
      for (int g = 0; g < RT; ++g) {
        const int r = row0 + g * 32;
        if (p.vec && sRA[s * BR + r + 3] >= 0) {
          T v[4] = {acc[g][0][j], acc[g][1][j], acc[g][2][j], acc[g][3][j]};
          stg4<T>(C + sRC[s * BR + r] + cc, v);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (sRA[s * BR + r + q] >= 0) C[sRC[s * BR + r + q] + cc] = acc[g][q][j];
        }
      }
    }
    __syncthreads();  // stage s is refilled by the next iteration's prefetch
  }
}

template <typename T, int RT, int CT>
size_t join_smem(int64_t K, int fix) {
  constexpr int BR = JoinTile<T, RT, CT>::BR, BC = JoinTile<T, RT, CT>::BC;
  const int sa = fix == 1 ? 1 : 2, sb = fix == 2 ? 1 : 2;
  (void)BC;
  return (size_t)K * (sa * BR + sb * BP) * sizeof(T) + (2 * (2 * BR + 2 * BP) + 2 * K) * sizeof(int64_t);
}

// 4 consecutive indices of the group's first label are 4 consecutive,
// 16-byte-aligned entries of the operand (and of the output)
static bool vec_group(int n, const int64_t* ext, const int64_t* s, const void* base, size_t esize) {
  if (n < 1 || s[0] != 1 || ext[0] % 4 != 0) return false;
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0) return false;
  for (int q = 1; q < n; ++q)
    if (s[q] % 4 != 0) return false;
  return esize == 4 || esize == 8;
}

template <typename T, int RT, int CT>
void join_go(const T* A, const T* B, T* C, const ContractDesc& d, int n_sm, cudaStream_t st) {
  constexpr int BR = JoinTile<T, RT, CT>::BR, BC = JoinTile<T, RT, CT>::BC;
  JoinArgs p;
  p.d = d;
  p.n_rt = (d.rows + BR - 1) / BR;
  p.n_ct = (d.cols + BC - 1) / BC;
  p.ntiles = p.n_rt * p.n_ct;
  bool vec = d.nr >= 1 && d.r_sc[0] == 1 && d.r_ext[0] % 4 == 0 &&
             (reinterpret_cast<uintptr_t>(C) % (4 * sizeof(T))) == 0;
  for (int q = 1; q < d.nr && vec; ++q) vec = d.r_sc[q] % 4 == 0;
  for (int q = 0; q < d.nc && vec; ++q) vec = d.c_sc[q] % 4 == 0;
  p.vec = vec;
  // the K offsets must keep 16-byte alignment too
  bool ka4 = true, kb4 = true;
  for (int q = 0; q < d.nk; ++q) {
    ka4 = ka4 && d.k_sa[q] % 4 == 0;
    kb4 = kb4 && d.k_sb[q] % 4 == 0;
  }
  p.vec_a = ka4 && vec_group(d.nr, d.r_ext, d.r_sa, A, sizeof(T));
  p.vec_b = kb4 && vec_group(d.nc, d.c_ext, d.c_sb, B, sizeof(T));
  // a short side of at most 4 tiles stays resident in each CTA
  p.fix = 0;
  p.n_fix = 0;
  if (p.n_rt <= 4 && p.n_ct >= 8 * p.n_rt) {
    p.fix = 1;
    p.n_fix = p.n_rt;
  } else if (p.n_ct <= 4 && p.n_rt >= 8 * p.n_ct) {
    p.fix = 2;
    p.n_fix = p.n_ct;
  }
  const size_t smem = join_smem<T, RT, CT>(d.K, p.fix);
  if (getenv("FCTN_JOIN_TRACE"))
    fprintf(stderr, "join rows=%lld cols=%lld K=%lld RT=%d CT=%d vec=%d vec_a=%d vec_b=%d fix=%d C=%p\n",
            (long long)d.rows, (long long)d.cols, (long long)d.K, RT, CT, (int)p.vec, (int)p.vec_a, (int)p.vec_b, p.fix,
            (void*)C);
  auto fn = k_join<T, RT, CT>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) throw std::runtime_error(std::string("join smem: ") + cudaGetErrorString(e));
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, JT, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = std::min<int64_t>(p.ntiles, (int64_t)n_sm * per_sm);
  if (p.fix) grid = std::max<int64_t>(p.n_fix, grid / p.n_fix * p.n_fix);
  fn<<<(unsigned)grid, JT, smem, st>>>(A, B, C, p);
  e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("join: ") + cudaGetErrorString(e));
}

}  // namespace

bool join_applicable(const ContractDesc& d, size_t esize) {
  if (getenv("FCTN_NO_JOIN")) return false;
  if (d.K < 1 || d.K > 128) return false;
  if (d.rows < 16 || d.cols < 16) return false;
  if (d.rows >= (int64_t)1 << 31 || d.cols >= (int64_t)1 << 31 || d.K >= (int64_t)1 << 31) return false;
  // small outputs stay on the generic kernel (FCTN_JOIN_MIN_OUT: test override)
  static const int64_t min_out = getenv("FCTN_JOIN_MIN_OUT") ? atoll(getenv("FCTN_JOIN_MIN_OUT")) : ((int64_t)1 << 20);
  if (d.rows * d.cols < min_out) return false;
  // the smallest tile (RT = 1, 48 columns, both streamed) must fit the opt-in limit
  return 2 * (size_t)d.K * (64 + 64) * esize + 8 * (2 * (128 + 128) + 2 * d.K) <= 200 * 1024;
}

// padded-work fraction of a (tile, extent) choice
static double tile_eff(int64_t n, int64_t tile) { return (double)n / (double)(((n + tile - 1) / tile) * tile); }

template <typename T>
void launch_join(const T* A, const T* B, T* C, const ContractDesc& d, int n_sm, cudaStream_t st) {
  // columns per thread: 4 (64-wide tiles) or 3 (48-wide) by padding waste;
  // row groups per thread: 2 (128-row tiles) unless that wastes rows or smem
  const int ct = tile_eff(d.cols, 48) > tile_eff(d.cols, 64) + 0.02 ? 3 : 4;
  const bool rt2 = tile_eff(d.rows, 128) >= tile_eff(d.rows, 64) - 0.02 &&
                   2 * (size_t)d.K * (128 + 64) * sizeof(T) <= 100 * 1024;
  if (rt2) {
    if (ct == 3) join_go<T, 2, 3>(A, B, C, d, n_sm, st);
    else join_go<T, 2, 4>(A, B, C, d, n_sm, st);
  } else {
    if (ct == 3) join_go<T, 1, 3>(A, B, C, d, n_sm, st);
    else join_go<T, 1, 4>(A, B, C, d, n_sm, st);
  }
}
template void launch_join<float>(const float*, const float*, float*, const ContractDesc&, int, cudaStream_t);
template void launch_join<double>(const double*, const double*, double*, const ContractDesc&, int, cudaStream_t);

}  // namespace fctn
