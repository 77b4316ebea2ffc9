#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap pm, unsigned char* out, int bytes, int c0, int c1, int prefetch) {
  __shared__ __align__(1024) unsigned char buf[4096];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (prefetch) asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<unsigned long long>(&pm)) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        :: "r"(smem_addr(buf)), "l"(reinterpret_cast<unsigned long long>(&pm)), "r"(c0), "r"(c1), "r"(smem_addr(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" :: "r"(smem_addr(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) out[i] = buf[i];
}
int main(int argc, char** argv) {
  int mode = atoi(argv[1]);  // 0 int64 32x8, 1 float64 32x8, 2 int32 64x8, 3 uint8 256x8, 4 f32 64x8, 5 int64 + prefetch, 6 bf16 128x8
  CUtensorMapDataType dts[] = {CU_TENSOR_MAP_DATA_TYPE_INT64, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, CU_TENSOR_MAP_DATA_TYPE_INT32, CU_TENSOR_MAP_DATA_TYPE_UINT8, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, CU_TENSOR_MAP_DATA_TYPE_INT64, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16};
  int esz[] = {8, 8, 4, 1, 4, 8, 2};
  const int W = 256, H = 64;
  int e = esz[mode];
  std::vector<unsigned char> h(W * H * 8);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (unsigned char)(i * 7);
  unsigned char *d, *o; cudaMalloc(&d, h.size()); cudaMalloc(&o, 4096);
  cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
  typedef CUresult (*F)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap m;
  int boxc = 256 / e;
  cuuint64_t dims[2] = {(cuuint64_t)(W * 8 / e), (cuuint64_t)H}; cuuint64_t str[1] = {(cuuint64_t)W * 8}; cuuint32_t box[2] = {(cuuint32_t)boxc, 8}, es[2] = {1, 1};
  CUresult r = ((F)fn)(&m, dts[mode], 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  k<<<1, 32>>>(m, o, 2048, 2, 1, mode == 5);
  cudaError_t err = cudaDeviceSynchronize();
  std::vector<unsigned char> ho(2048); cudaMemcpy(ho.data(), o, 2048, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int rr = 0; rr < 8; ++rr) for (int b = 0; b < 256; ++b) { size_t src = (size_t)(1 + rr) * W * 8 + 2 * e + b; if (ho[rr * 256 + b] != h[src]) ++bad; }
  printf("mode %d encode=%d err=%s bad=%d\n", mode, (int)r, cudaGetErrorString(err), bad);
  return 0;
}
