// tma_probe.cu -- measures the TMA box-streaming rate that bounds stage 1 of
// the fused ladder (ss_ladder_screen.cu): one producer thread per CTA issues
// NBOX 2-D boxes (BR rows x BW elements) per tile into a STAGES-deep mbarrier
// pipeline, 16 consumer warps read their rows of every box from shared memory
// and release the stage.  Boxes start at random 16-byte aligned columns of an
// L2-resident plane (as stage 1's corner boxes mostly hit L2).  Prints bytes
// per clock per SM and tiles per second for each geometry.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tools/tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
                     smem_addr(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_addr(dst)), "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(smem_addr(bar))
        : "memory");
}

constexpr int CW = 16;  // consumer warps

template <typename T, int BW, int BR, int NBOX, int STAGES, int NPROD = 1, bool ODD = false>
__global__ void __launch_bounds__((CW + 1) * 32, 1)
    probe(const __grid_constant__ CUtensorMap map, int tiles, int cols, int rows, unsigned long long* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) unsigned long long full[STAGES], empty[STAGES];
    constexpr int BOX = BW * BR * (int)sizeof(T);
    constexpr int STAGE = NBOX * BOX;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == CW) {
        if (lane < NPROD) {  // NPROD lanes share each tile's boxes
            unsigned rng = 12345u + blockIdx.x * 7919u + lane * 104729u;
            for (int t = 0; t < tiles; ++t) {
                const int s = t % STAGES;
                mbar_wait(&empty[s], ((t / STAGES) & 1) ^ 1);
                if (lane == 0) mbar_expect_tx(&full[s], STAGE);
                __syncwarp((1u << NPROD) - 1u);
                for (int b = lane; b < NBOX; b += NPROD) {
                    rng = rng * 1664525u + 1013904223u;
                    const int x = ODD ? (int)((rng >> 8) % (unsigned)(cols - BW))  // any element
                                      : (int)((rng >> 8) % (unsigned)(cols - BW)) & ~(16 / (int)sizeof(T) - 1);
                    rng = rng * 1664525u + 1013904223u;
                    const int y = (int)((rng >> 8) % (unsigned)(rows - BR));
                    tma_load_2d(sm + s * STAGE + b * BOX, &map, x, y, &full[s]);
                }
            }
        }
        return;
    }
    unsigned long long acc = 0;
    for (int t = 0; t < tiles; ++t) {
        const int s = t % STAGES;
        mbar_wait(&full[s], (t / STAGES) & 1);
        const T* st = reinterpret_cast<const T*>(sm + s * STAGE);
        // each warp reads its share of every box's elements
        for (int b = 0; b < NBOX; ++b)
            for (int i = warp * 32 + lane; i < BW * BR; i += CW * 32) acc += st[b * BW * BR + i];
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 0x123456789ull) sink[0] = acc;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <typename T, int BW, int BR, int NBOX, int STAGES, int NPROD = 1, bool ODD = false>
void run(const char* name, void* plane, int cols, int rows, int ctas_per_sm) {
    static EncodeFn encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        encode = reinterpret_cast<EncodeFn>(fn);
    }
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)cols * sizeof(T)};
    const cuuint32_t box[2] = {(cuuint32_t)BW, (cuuint32_t)BR};
    const cuuint32_t es[2] = {1, 1};
    if (encode(&map, sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, plane, dims,
               strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("%s: encode failed\n", name);
        return;
    }
    auto k = probe<T, BW, BR, NBOX, STAGES, NPROD, ODD>;
    const int smem = STAGES * NBOX * BW * BR * (int)sizeof(T);
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * ctas_per_sm;
    const int tiles = 3000;
    unsigned long long* sink;
    CK(cudaMalloc(&sink, 8));
    k<<<grid, (CW + 1) * 32, smem>>>(map, 200, cols, rows, sink);  // warm-up
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<grid, (CW + 1) * 32, smem>>>(map, tiles, cols, rows, sink);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);  // kHz
    const double bytes = (double)grid * tiles * NBOX * BW * BR * sizeof(T);
    const double rows_req = (double)grid * tiles * NBOX * BR;
    const double cyc = ms * 1e-3 * 1.965e9;
    printf("%-34s smem %6d B  %7.3f ms  %7.1f GB/s  %6.1f B/clk/SM  %6.2f ns/tile/SM  %5.2f box-rows/clk/SM\n", name, smem,
           ms, bytes / ms / 1e6, bytes / cyc / sms, ms * 1e6 / ((double)tiles * ctas_per_sm), rows_req / cyc / sms);
    cudaFree(sink);
}

int main() {
    // an L2-resident plane: 4096 x 2048 u32 = 32 MB (or 4096 x 4096 u16 = 32 MB)
    void* p;
    CK(cudaMalloc(&p, 64 << 20));
    CK(cudaMemset(p, 1, 64 << 20));
    run<unsigned short, 232, 16, 8, 3, 8>("u16 8 x (16x232) x3 8 lanes [r2]", p, 4096, 4096, 1);
    run<unsigned short, 256, 16, 8, 3, 8>("u16 8 x (16x256) x3 8 lanes aligned", p, 4096, 4096, 1);
    run<unsigned short, 256, 16, 8, 3, 8, true>("u16 8 x (16x256) x3 8 lanes any start", p, 4096, 4096, 1);
    // HBM-resident (1 GB plane): the miss path
    void* q;
    CK(cudaMalloc(&q, 1ull << 30));
    CK(cudaMemset(q, 1, 1ull << 30));
    run<unsigned, 196, 16, 8, 2>("HBM u32 8 x (16x196) x2", q, 16384, 16384, 1);
    return 0;
}
