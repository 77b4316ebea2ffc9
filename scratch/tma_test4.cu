#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap pm, unsigned char* out, int bytes, int c0, int c1, int soff) {
  __shared__ __align__(1024) unsigned char buf[8192 + 1024];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        :: "r"(smem_addr(buf + soff)), "l"(reinterpret_cast<unsigned long long>(&pm)), "r"(c0), "r"(c1), "r"(smem_addr(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" :: "r"(smem_addr(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) out[i] = buf[soff + i];
}
int main(int argc, char** argv) {
  // args: esize box0 box1 Wbytes soff l2promo c0 c1
  int es = atoi(argv[1]), b0 = atoi(argv[2]), b1 = atoi(argv[3]), wb = atoi(argv[4]), soff = atoi(argv[5]), l2 = atoi(argv[6]);
  int c0 = atoi(argv[7]), c1 = atoi(argv[8]);
  CUtensorMapDataType dt = es == 8 ? CU_TENSOR_MAP_DATA_TYPE_INT64 : es == 4 ? CU_TENSOR_MAP_DATA_TYPE_INT32 : es == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8;
  const int H = 64;
  std::vector<unsigned char> h((size_t)wb * H);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (unsigned char)(i * 7 + 3);
  unsigned char *d, *o; cudaMalloc(&d, h.size()); cudaMalloc(&o, 8192);
  cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
  typedef CUresult (*F)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)(wb / es), (cuuint64_t)H}; cuuint64_t str[1] = {(cuuint64_t)wb}; cuuint32_t box[2] = {(cuuint32_t)b0, (cuuint32_t)b1}, est[2] = {1, 1};
  CUtensorMapL2promotion l2p[] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
  CUresult r = ((F)fn)(&m, dt, 2, d, dims, str, box, est, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, l2p[l2], CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int bytes = b0 * b1 * es;
  k<<<1, 32>>>(m, o, bytes, c0, c1, soff);
  cudaError_t err = cudaDeviceSynchronize();
  std::vector<unsigned char> ho(bytes); cudaMemcpy(ho.data(), o, bytes, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int rr = 0; rr < b1; ++rr) for (int b = 0; b < b0 * es; ++b) {
    long x = (long)c0 * es + b, y = c1 + rr;
    unsigned char want = (x >= 0 && x < wb && y >= 0 && y < H) ? h[(size_t)y * wb + x] : 0;
    if (ho[rr * b0 * es + b] != want) ++bad;
  }
  printf("es=%d box=%dx%d Wb=%d soff=%d l2=%d c=(%d,%d): encode=%d err=%s bad=%d\n", es, b0, b1, wb, soff, l2, c0, c1, (int)r, cudaGetErrorString(err), bad);
  return 0;
}
