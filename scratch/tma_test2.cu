#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(unsigned long long* bar) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" :: "r"(smem_addr(bar)), "r"(0) : "memory");
}
// MODE 0: 1D bulk copy; 1: tensor map from global memory; 2: tensor map from param (grid_constant)
template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap pm, const CUtensorMap* gm, const long long* src, long long* out, int c0, int c1) {
  __shared__ __align__(128) long long buf[8 * 32];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar)), "r"(MODE == 0 ? 256 : 2048) : "memory");
    if (MODE == 0)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        :: "r"(smem_addr(buf)), "l"(src), "r"(256), "r"(smem_addr(&bar)) : "memory");
    else {
      const CUtensorMap* m = MODE == 1 ? gm : &pm;
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        :: "r"(smem_addr(buf)), "l"(reinterpret_cast<unsigned long long>(m)), "r"(c0), "r"(c1), "r"(smem_addr(&bar)) : "memory");
    }
  }
  wait(&bar);
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = buf[i];
}
int main() {
  int rt, drv; cudaRuntimeGetVersion(&rt); cudaDriverGetVersion(&drv); printf("runtime %d driver %d\n", rt, drv);
  const int W = 100, H = 50;
  std::vector<long long> h(W * H);
  for (int i = 0; i < W * H; ++i) h[i] = i;
  long long *d, *o; cudaMalloc(&d, W * H * 8); cudaMalloc(&o, 256 * 8);
  cudaMemcpy(d, h.data(), W * H * 8, cudaMemcpyHostToDevice);
  typedef CUresult (*F)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaError_t ge = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  printf("entry %d q=%d fn=%p\n", (int)ge, (int)q, fn);
  CUtensorMap m;
  cuuint64_t dims[2] = {W, H}; cuuint64_t str[1] = {W * 8}; cuuint32_t box[2] = {32, 8}, es[2] = {1, 1};
  for (int dt = 0; dt < 2; ++dt) {
  CUresult r = ((F)fn)(&m, dt == 0 ? CU_TENSOR_MAP_DATA_TYPE_INT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("dtype %d encode r=%d\n", dt, (int)r);
  CUtensorMap* gm; cudaMalloc(&gm, sizeof(CUtensorMap)); cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(o, 0xff, 256*8);
    if (mode == 0) k<0><<<1, 32>>>(m, gm, d, o, 3, 2);
    if (mode == 1) k<1><<<1, 32>>>(m, gm, d, o, 3, 2);
    if (mode == 2) k<2><<<1, 32>>>(m, gm, d, o, 3, 2);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<long long> ho(256); cudaMemcpy(ho.data(), o, 256*8, cudaMemcpyDeviceToHost);
    printf("mode %d: err=%s first=%lld %lld\n", mode, cudaGetErrorString(e), ho[0], ho[33]);
    if (e != cudaSuccess) return 1;
  }
  }
  return 0;
}
