// Effective SM clock during a short single-CTA kernel vs after a warm-up load.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void spin(long long cycles, long long* out) {
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
}
__global__ void burn(float* x, int n) {
  float v = threadIdx.x;
  for (int i = 0; i < n; ++i) v = v * 0.999f + 1.0f;
  x[blockIdx.x * blockDim.x + threadIdx.x] = v;
}
int main() {
  long long* d; float* f; cudaMalloc(&d, 8); cudaMalloc(&f, 148 * 8 * 256 * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int warm = 0; warm < 2; ++warm) {
    if (warm) { burn<<<148 * 8, 256>>>(f, 2000000); }
    cudaEventRecord(a); spin<<<1, 32>>>(1000000, d); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("%s: %lld cycles in %.3f ms -> %.0f MHz\n", warm ? "after burn" : "idle", c, ms, c / ms / 1e3);
  }
  return 0;
}
