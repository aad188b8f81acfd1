// Reconstruction-quality metrics on the device:
// psnr / ssim / rel_err of the reference's metrics.py:33-105, computed where
// X already lives so a per-iteration quality report does not pay a T-sized
// download (1-2 GB at c4/c5).
//
// The first two modes are the image plane, every combination of the
// trailing modes is one slice (metrics.py:19-23); in F order a slice is a
// contiguous run of H*W entries.  Work unit = one warp over one contiguous
// segment of one slice; every sum is fp64 and combined in a fixed order
// (segment partials -> per-slice sums -> slice means), so results are
// deterministic.  Two passes, like the reference's two-pass mean/var/cov
// (metrics.py:59-63):
//   pass 1 per slice: sum e, sum t, sum (e-t)^2, sum t^2, and off the mask
//          sum (e-t)^2, sum t^2, count   (psnr 33-44, rel_err 66-92)
//   pass 2 per slice: sum (e-mu_e)^2, sum (t-mu_t)^2, sum (e-mu_e)(t-mu_t)
// Both passes stream est and truth once: HBM-bound, 2 * (b_e + b_t) * T
// bytes (+ T mask bytes in pass 1).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "kernels.cuh"

namespace fctn {

static constexpr int QP1 = 7;  // pass-1 sums per slice
static constexpr int QP2 = 3;  // pass-2 sums per slice
static constexpr int QWARPS = 8;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One warp per (slice, segment).  part: [slice][seg][QP1].
template <typename TE, typename TT>
__global__ void __launch_bounds__(QWARPS * 32) k_quality_pass1(const TE* __restrict__ est, const TT* __restrict__ truth,
                                                              const uint8_t* __restrict__ mask, int64_t hw,
                                                              int64_t seglen, int nseg, int64_t nslices,
                                                              double* __restrict__ part) {
  const int64_t w = (int64_t)blockIdx.x * QWARPS + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= nslices * nseg) return;
  const int64_t slice = w / nseg, seg = w % nseg;
  const int64_t lo = seg * seglen, hi = lo + seglen < hw ? lo + seglen : hw;
  const int64_t base = slice * hw;
  double se = 0, st = 0, sd = 0, stt = 0, od = 0, ott = 0, on = 0;
  for (int64_t i = lo + lane; i < hi; i += 32) {
    const double e = (double)est[base + i], t = (double)truth[base + i];
    const double d = e - t;
    se += e;
    st += t;
    sd += d * d;
    stt += t * t;
    if (mask && !mask[base + i]) {
      od += d * d;
      ott += t * t;
      on += 1.0;
    }
  }
  double v[QP1] = {se, st, sd, stt, od, ott, on};
#pragma unroll
  for (int q = 0; q < QP1; ++q) v[q] = warp_sum(v[q]);
  if (lane == 0) {
    double* o = part + w * QP1;
#pragma unroll
    for (int q = 0; q < QP1; ++q) o[q] = v[q];
  }
}

template <typename TE, typename TT>
__global__ void __launch_bounds__(QWARPS * 32) k_quality_pass2(const TE* __restrict__ est, const TT* __restrict__ truth,
                                                              const double* __restrict__ sums1, double inv_hw,
                                                              int64_t hw, int64_t seglen, int nseg, int64_t nslices,
                                                              double* __restrict__ part) {
  const int64_t w = (int64_t)blockIdx.x * QWARPS + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= nslices * nseg) return;
  const int64_t slice = w / nseg, seg = w % nseg;
  const int64_t lo = seg * seglen, hi = lo + seglen < hw ? lo + seglen : hw;
  const int64_t base = slice * hw;
  const double mu_e = sums1[slice * QP1 + 0] * inv_hw, mu_t = sums1[slice * QP1 + 1] * inv_hw;
  double vee = 0, vtt = 0, vet = 0;
  for (int64_t i = lo + lane; i < hi; i += 32) {
    const double e = (double)est[base + i] - mu_e, t = (double)truth[base + i] - mu_t;
    vee += e * e;
    vtt += t * t;
    vet += e * t;
  }
  vee = warp_sum(vee);
  vtt = warp_sum(vtt);
  vet = warp_sum(vet);
  if (lane == 0) {
    double* o = part + w * QP2;
    o[0] = vee;
    o[1] = vtt;
    o[2] = vet;
  }
}

// Per-slice sums over the segments, in segment order.
__global__ void k_quality_fold(const double* __restrict__ part, int nseg, int nq, int64_t nslices,
                               double* __restrict__ out) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nslices) return;
  for (int q = 0; q < nq; ++q) {
    double acc = 0;
    for (int g = 0; g < nseg; ++g) acc += part[(s * nseg + g) * nq + q];
    out[s * nq + q] = acc;
  }
}

// One CTA: per-slice PSNR (100 dB cap on zero error, metrics.py:41) and the
// single-window structural index (metrics.py:55-66), averaged over slices,
// plus the global error norms (slice order).  out: [psnr, ssim, num^2,
// den^2, num_off^2, den_off^2, n_off].
__global__ void __launch_bounds__(256) k_quality_final(const double* __restrict__ s1, const double* __restrict__ s2,
                                                       int64_t nslices, double inv_hw, double peak,
                                                       double* __restrict__ out) {
  __shared__ double red[7][256];
  const double c1 = (0.01 * peak) * (0.01 * peak), c2 = (0.03 * peak) * (0.03 * peak);
  double ps = 0, ss = 0, nd = 0, dd = 0, no = 0, dof = 0, cnt = 0;
  for (int64_t s = threadIdx.x; s < nslices; s += blockDim.x) {
    const double* a = s1 + s * QP1;
    const double* b = s2 + s * QP2;
    const double mse = a[2] * inv_hw;
    ps += mse == 0.0 ? 100.0 : 10.0 * log10(peak * peak / mse);
    const double mu_a = a[0] * inv_hw, mu_b = a[1] * inv_hw;
    const double var_a = b[0] * inv_hw, var_b = b[1] * inv_hw, cov = b[2] * inv_hw;
    const double num = (2.0 * mu_a * mu_b + c1) * (2.0 * cov + c2);
    const double den = (mu_a * mu_a + mu_b * mu_b + c1) * (var_a + var_b + c2);
    ss += num / den;
    nd += a[2];
    dd += a[3];
    no += a[4];
    dof += a[5];
    cnt += a[6];
  }
  double v[7] = {ps, ss, nd, dd, no, dof, cnt};
  for (int q = 0; q < 7; ++q) red[q][threadIdx.x] = v[q];
  __syncthreads();
  for (int h = blockDim.x / 2; h > 0; h >>= 1) {
    if ((int)threadIdx.x < h)
      for (int q = 0; q < 7; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double ns = (double)nslices;
    out[0] = red[0][0] / ns;
    out[1] = red[1][0] / ns;
    for (int q = 2; q < 7; ++q) out[q] = red[q][0];
  }
}

QualityPlan quality_plan(int64_t hw, int64_t nslices, int n_sm) {
  QualityPlan p;
  p.hw = hw;
  p.nslices = nslices;
  // segments of >= 2048 entries, enough warps to fill the SMs several times
  const int64_t want_warps = (int64_t)n_sm * 64;
  int64_t nseg = (want_warps + nslices - 1) / nslices;
  const int64_t max_seg = (hw + 2047) / 2048;
  if (nseg > max_seg) nseg = max_seg;
  if (nseg < 1) nseg = 1;
  p.seglen = (hw + nseg - 1) / nseg;
  p.nseg = (int)((hw + p.seglen - 1) / p.seglen);
  p.part_doubles = nslices * p.nseg * QP1;
  p.sums_doubles = nslices * (QP1 + QP2);
  return p;
}

template <typename TE, typename TT>
void launch_quality_pass1(const QualityPlan& p, const TE* est, const TT* truth, const uint8_t* mask, double* part,
                          double* sums1, cudaStream_t st) {
  const int64_t warps = p.nslices * p.nseg;
  const unsigned grid = (unsigned)((warps + QWARPS - 1) / QWARPS);
  k_quality_pass1<TE, TT><<<grid, QWARPS * 32, 0, st>>>(est, truth, mask, p.hw, p.seglen, p.nseg, p.nslices, part);
  k_quality_fold<<<(unsigned)((p.nslices + 255) / 256), 256, 0, st>>>(part, p.nseg, QP1, p.nslices, sums1);
}

template <typename TE, typename TT>
void launch_quality_pass2(const QualityPlan& p, const TE* est, const TT* truth, const double* sums1, double inv_hw,
                          double* part, double* sums2, cudaStream_t st) {
  const int64_t warps = p.nslices * p.nseg;
  const unsigned grid = (unsigned)((warps + QWARPS - 1) / QWARPS);
  k_quality_pass2<TE, TT><<<grid, QWARPS * 32, 0, st>>>(est, truth, sums1, inv_hw, p.hw, p.seglen, p.nseg, p.nslices,
                                                        part);
  k_quality_fold<<<(unsigned)((p.nslices + 255) / 256), 256, 0, st>>>(part, p.nseg, QP2, p.nslices, sums2);
}

void launch_quality_final(const QualityPlan& p, const double* sums1, const double* sums2, double inv_hw, double peak,
                          double* out, cudaStream_t st) {
  k_quality_final<<<1, 256, 0, st>>>(sums1, sums2, p.nslices, inv_hw, peak, out);
}

#define QINST(TE, TT)                                                                                               \
  template void launch_quality_pass1<TE, TT>(const QualityPlan&, const TE*, const TT*, const uint8_t*, double*,     \
                                             double*, cudaStream_t);                                                \
  template void launch_quality_pass2<TE, TT>(const QualityPlan&, const TE*, const TT*, const double*, double,       \
                                             double*, double*, cudaStream_t);
QINST(double, double)
QINST(float, float)
QINST(float, double)
QINST(double, float)
#undef QINST

}  // namespace fctn
