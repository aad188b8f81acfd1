// Measures dependent-chain latency (cycles) of DFMA, FFMA, double rsqrt/sqrt/div,
// and DFMA throughput per SM, on the current GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, int n, double a, double b) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  float y = (float)a;
  for (int i = 0; i < n; ++i) y = fmaf(y, (float)a, (float)b);
  long long t2 = clock64();
  double z = a + 2.0;
  for (int i = 0; i < n; ++i) z = rsqrt(z) + 2.0;
  long long t3 = clock64();
  double u = a + 2.0;
  for (int i = 0; i < n; ++i) u = sqrt(u) + 2.0;
  long long t4 = clock64();
  double v = a + 2.0;
  for (int i = 0; i < n; ++i) v = 1.0 / v + 2.0;
  long long t5 = clock64();
  out[0] = x + y + z + u + v;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
}
__global__ void thr(double* out, int n, double a, double b) {
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 1 << 24); cudaMalloc(&c, 64);
  int n = 10000;
  lat<<<1, 1>>>(d, c, n, 0.999, 0.001);
  long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
  printf("latency cycles: DFMA %.1f  FFMA %.1f  rsqrt(f64)+add %.1f  sqrt(f64)+add %.1f  1/x(f64)+add %.1f\n",
         h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sm; cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  thr<<<sm * 8, 256>>>(d, 1000, 0.999, 0.001);
  cudaEventRecord(e0);
  thr<<<sm * 8, 256>>>(d, 20000, 0.999, 0.001);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 8 * 20000.0 * sm * 8 * 256;
  printf("DFMA throughput: %.2f TFLOP/s (%d SMs)\n", fl / ms / 1e9, sm);
  return 0;
}
