// Dump the shared-memory image of a TMA 32x32 fp32 box loaded with
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B (value = linear index), to pin the
// 32-byte-atom swizzle formula used by the stream converter.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void k(const __grid_constant__ CUtensorMap m, float* out) {
  __shared__ alignas(1024) float s[32 * 32];
  __shared__ alignas(8) uint64_t bar;
  uint32_t sb = (uint32_t)__cvta_generic_to_shared(&bar), sd = (uint32_t)__cvta_generic_to_shared(s);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(4096));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(sd),
        "l"((uint64_t)&m), "r"(sb), "r"(0), "r"(0));
    asm volatile(
        "{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}" ::"r"(sb));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = s[i];
}

int main() {
  float h[64 * 64];
  for (int i = 0; i < 64 * 64; ++i) h[i] = (float)i;
  float *d, *o;
  cudaMalloc(&d, sizeof h);
  cudaMalloc(&o, 4096);
  cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
  void* p;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  CUtensorMap m;
  cuuint64_t dims[2] = {64, 64}, str[1] = {64 * 4};
  cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) { printf("encode failed %d\n", (int)r); return 1; }
  k<<<1, 128>>>(m, o);
  float s[1024];
  cudaMemcpy(s, o, 4096, cudaMemcpyDeviceToHost);
  // for each smem row (128 B), print which source column each 32-B atom holds
  for (int row = 0; row < 12; ++row) {
    printf("row %2d:", row);
    for (int a = 0; a < 4; ++a) {
      int v = (int)s[row * 32 + a * 8];
      printf("  atom%d<- (r%d,c%d)", a, v / 64, v % 64);
    }
    printf("\n");
  }
  return 0;
}
