#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
struct Maps { CUtensorMap m; };
template <int VARIANT>
__global__ void k(const __grid_constant__ Maps maps, long long* out, int c0, int c1) {
  __shared__ __align__(128) long long buf[8 * 32];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&bar)), "r"(1));
    if (VARIANT & 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar)), "r"(2048) : "memory");
    if (VARIANT & 2)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        :: "r"(smem_addr(buf)), "l"(reinterpret_cast<unsigned long long>(&maps.m)), "r"(c0), "r"(c1), "r"(smem_addr(&bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        :: "r"(smem_addr(buf)), "l"(reinterpret_cast<unsigned long long>(&maps.m)), "r"(c0), "r"(c1), "r"(smem_addr(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" :: "r"(smem_addr(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = buf[i];
}
int main() {
  const int W = 100, H = 50;
  std::vector<long long> h(W * H);
  for (int i = 0; i < W * H; ++i) h[i] = i;
  long long *d, *o; cudaMalloc(&d, W * H * 8); cudaMalloc(&o, 256 * 8);
  cudaMemcpy(d, h.data(), W * H * 8, cudaMemcpyHostToDevice);
  typedef CUresult (*F)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  Maps maps;
  cuuint64_t dims[2] = {W, H}; cuuint64_t str[1] = {W * 8}; cuuint32_t box[2] = {32, 8}, es[2] = {1, 1};
  CUresult r = ((F)fn)(&maps.m, CU_TENSOR_MAP_DATA_TYPE_INT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode r=%d (W*8=%d)\n", (int)r, W*8);
  int coords[3][2] = {{3, 2}, {-5, -3}, {90, 45}};
  for (int v = 0; v < 4; ++v) for (auto& c : coords) {
    cudaMemset(o, 0xff, 256*8);
    if (v == 0) k<0><<<1, 32>>>(maps, o, c[0], c[1]);
    if (v == 1) k<1><<<1, 32>>>(maps, o, c[0], c[1]);
    if (v == 2) k<2><<<1, 32>>>(maps, o, c[0], c[1]);
    if (v == 3) k<3><<<1, 32>>>(maps, o, c[0], c[1]);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<long long> ho(256); cudaMemcpy(ho.data(), o, 256*8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int rr = 0; rr < 8; ++rr) for (int cc = 0; cc < 32; ++cc) {
      int x = c[0] + cc, y = c[1] + rr; long long want = (x >= 0 && x < W && y >= 0 && y < H) ? (long long)y * W + x : 0;
      if (ho[rr * 32 + cc] != want) ++bad;
    }
    printf("variant %d coords (%d,%d): err=%s bad=%d\n", v, c[0], c[1], cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
