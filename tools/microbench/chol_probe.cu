// Cycle probe of the tiled Cholesky step (copy of k_chol<TL> with clock64 marks).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
template <int TL>
__global__ void __launch_bounds__(256) probe(const double* __restrict__ G, int S, double mu0,
                                             long long* __restrict__ cyc) {
  constexpr int SP = 16 * TL;
  extern __shared__ double sm[];
  double* col = sm + (size_t)S * S;
  double* dinv = col + 2 * SP;
  __shared__ int bad;
  const int tid = threadIdx.x;
  const int ty = tid & 15, tx = tid >> 4;
  if (tid == 0) bad = 0;
  double t[TL][TL];
#pragma unroll
  for (int a = 0; a < TL; ++a)
#pragma unroll
    for (int b = 0; b < TL; ++b) {
      const int i = ty * TL + a, j = tx * TL + b;
      double v = (i == j) ? 1.0 : 0.0;
      if (i < S && j < S) v = G[i + S * j] + (i == j ? mu0 : 0.0);
      t[a][b] = v;
    }
  __syncthreads();
  const unsigned half = 0xFFFFu << (16 * (tx & 1));
  long long c_owner = 0, c_bar = 0, c_upd = 0;
  for (int k = 0; k < SP; ++k) {
    long long t0 = clock64();
    const int kb = k / TL, kk = k - kb * TL;
    double* cb = col + (k & 1) * SP;
    if (tx == kb) {
      double mine = 0.0;
#pragma unroll
      for (int a = 0; a < TL; ++a)
        if (a == kk) mine = t[a][a];
      double pv = __shfl_sync(half, mine, (16 * (tx & 1)) + kb);
      if (!(pv > 0.0) || !isfinite(pv)) { bad = 1; pv = 1.0; }
      const double inv = rsqrt(pv), d = pv * inv;
      if (ty == kb) dinv[k] = inv;
#pragma unroll
      for (int a = 0; a < TL; ++a) {
        const int i = ty * TL + a;
#pragma unroll
        for (int b = 0; b < TL; ++b)
          if (b == kk) {
            if (i == k) t[a][b] = d;
            else if (i > k) t[a][b] *= inv;
            cb[i] = (i > k) ? t[a][b] : 0.0;
          }
      }
    }
    long long t1 = clock64();
    __syncthreads();
    long long t2 = clock64();
    {
      double ci[TL], cj[TL];
#pragma unroll
      for (int a = 0; a < TL; ++a) ci[a] = cb[ty * TL + a];
#pragma unroll
      for (int b = 0; b < TL; ++b) cj[b] = cb[tx * TL + b];
      long long tq = clock64();
      if (tid == 0) cyc[8 + (k & 7)] = tq - t2;   // LDS latency sample
#pragma unroll
      for (int a = 0; a < TL; ++a)
#pragma unroll
        for (int b = 0; b < TL; ++b) t[a][b] = fma(-ci[a], cj[b], t[a][b]);
    }
    long long t3 = clock64();
    c_owner += t1 - t0; c_bar += t2 - t1; c_upd += t3 - t2;
  }
  if (blockIdx.x == 0 && (tid == 0 || tid == 255)) {
    cyc[(tid ? 3 : 0) + 0] = c_owner; cyc[(tid ? 3 : 0) + 1] = c_bar; cyc[(tid ? 3 : 0) + 2] = c_upd;
  }
  if (t[0][0] == 12345.0) cyc[7] = 1;
}
int main() {
  for (int S : {64, 125}) {
    std::vector<double> G(S * S);
    for (int i = 0; i < S; ++i) for (int j = 0; j < S; ++j) G[i + S * j] = (i == j ? S : 0.0) + 1.0 / (1 + i + j);
    double* dG; long long* dc; cudaMalloc(&dG, S * S * 8); cudaMalloc(&dc, 128);
    cudaMemcpy(dG, G.data(), S * S * 8, cudaMemcpyHostToDevice);
    size_t smem = (S * S + 3 * 16 * ((S + 15) / 16)) * 8;
    long long h[16];
    if (S == 64) { cudaFuncSetAttribute(probe<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      for (int r = 0; r < 3; ++r) probe<4><<<1, 256, smem>>>(dG, S, 0.5, dc); }
    else { cudaFuncSetAttribute(probe<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      for (int r = 0; r < 3; ++r) probe<8><<<1, 256, smem>>>(dG, S, 0.5, dc); }
    cudaDeviceSynchronize();
    cudaMemcpy(h, dc, 128, cudaMemcpyDeviceToHost);
    int steps = 16 * ((S + 15) / 16);
    printf("S=%d tid0: owner %lld bar %lld upd %lld cycles/step | tid255: owner %lld bar %lld upd %lld  (%s)\n", S,
           h[0] / steps, h[1] / steps, h[2] / steps, h[3] / steps, h[4] / steps, h[5] / steps,
           cudaGetErrorString(cudaGetLastError()));
    printf("   t2->after-LDS samples: %lld %lld %lld %lld\n", h[8], h[9], h[10], h[11]);
  }
  return 0;
}
