// tma_gather_probe.cu -- experiment: random label gathers through the TMA
// engine (cp.async.bulk.tensor.2d ... tile::gather4: four arbitrary 16-byte
// rows of a 2-D view of the table per instruction, into shared memory)
// against LSU gathers (ld.global.nc) and both at once.  Decides whether the
// signature passes' gathers, bound at the L1TEX line rate, gain from a second
// path outside the LSU pipeline.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/tma_gather_probe tools/tma_gather_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t lcg(uint64_t& x) {
    x = x * 6364136223846793005ull + 1442695040888963407ull;
    return (uint32_t)(x >> 32);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// LSU: every thread gathers `per_thread` random words
__global__ void lsu_kernel(const uint32_t* __restrict__ tab, uint32_t n, uint32_t per_thread, uint32_t* sink) {
    uint64_t x = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 7;
    uint32_t acc = 0;
    for (uint32_t r = 0; r < per_thread; r += 16) {
        uint32_t v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __ldg(tab + __umulhi(lcg(x), n));
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += v[j];
    }
    if (acc == 0x12345u) sink[0] = acc;
}

// TMA: warp 0..W-1 lane 0 each issue `batches` x G gather4 (4 rows of 16 B)
// into their own shared-memory ring, one mbarrier per stage; the other lanes
// idle.  rows = n / 4.  lsu_per_thread > 0: the remaining warps run LSU
// gathers concurrently.
constexpr int G = 8;       // gather4 per stage
constexpr int STAGES = 4;  // ring depth per issuing warp
constexpr int MAXW = 8;

__global__ void tma_kernel(const __grid_constant__ CUtensorMap map, uint32_t rows, uint32_t batches, int issuers,
                           const uint32_t* __restrict__ tab, uint32_t n, uint32_t lsu_per_thread, uint32_t* sink) {
    __shared__ __align__(128) uint32_t buf[MAXW][STAGES][G * 32];  // 4 rows x 16 B per gather4, 128-byte aligned slots
    __shared__ __align__(8) uint64_t bar[MAXW][STAGES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t x = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 11;
    uint32_t acc = 0;
    if (warp < issuers) {
        if (lane == 0) {
            for (int s = 0; s < STAGES; ++s)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[warp][s])));
            asm volatile("fence.mbarrier_init.release.cluster;");
            uint32_t phase[STAGES] = {};
            for (uint32_t b = 0; b < batches + STAGES; ++b) {
                const int s = b % STAGES;
                if (b >= STAGES) {  // wait for the stage issued STAGES batches ago
                    uint32_t done = 0;
                    while (!done)
                        asm volatile(
                            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                            : "=r"(done)
                            : "r"(smem_u32(&bar[warp][s])), "r"(phase[s]));
                    phase[s] ^= 1;
                    acc += buf[warp][s][lcg(x) & (G * 32 - 1)];
                }
                if (b < batches) {
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[warp][s])),
                                 "r"(G * 64));
                    for (int g = 0; g < G; ++g) {
                        const int32_t r0 = __umulhi(lcg(x), rows), r1 = __umulhi(lcg(x), rows),
                                      r2 = __umulhi(lcg(x), rows), r3 = __umulhi(lcg(x), rows);
                        asm volatile(
                            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(&buf[warp][s][g * 32])),
                            "l"(&map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(&bar[warp][s]))
                            : "memory");
                    }
                }
            }
        }
    } else if (lsu_per_thread) {
        for (uint32_t r = 0; r < lsu_per_thread; r += 16) {
            uint32_t v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = __ldg(tab + __umulhi(lcg(x), n));
#pragma unroll
            for (int j = 0; j < 16; ++j) acc += v[j];
        }
    }
    if (acc == 0x12345u) sink[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const uint32_t n = 5u << 20;  // 5M words = 20 MB (the bench's 16-bit labels of 10M states)
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *tab, *sink;
    cudaMalloc(&tab, (size_t)n * 4);
    cudaMalloc(&sink, 4);
    cudaMemset(tab, 1, (size_t)n * 4);
    EncodeFn encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q);
    if (!encode) {
        printf("no cuTensorMapEncodeTiled\n");
        return 1;
    }
    const uint32_t rows = n / 4;
    CUtensorMap map;
    cuuint64_t dims[2] = {4, rows};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {4, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, tab, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d\n", (int)cr);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timed = [&](auto launch, double gathers, const char* name) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t err = cudaGetLastError();
        printf("%-52s %8.3f ms  %.3g gathers/s  %s\n", name, ms, gathers / (ms / 1e3), cudaGetErrorString(err));
    };
    const uint32_t per = 1024;
    const unsigned lsu_blocks = sms * 8, lsu_threads = 256;
    timed([&] { lsu_kernel<<<lsu_blocks, lsu_threads>>>(tab, n, per, sink); }, (double)lsu_blocks * lsu_threads * per,
          "LSU gathers (ld.global.nc), 8 x 256 threads / SM");
    for (int issuers : {1, 2, 4, 8}) {
        for (int ctas : {1, 2, 4}) {
            const uint32_t batches = 2048;
            char name[96];
            snprintf(name, sizeof name, "TMA gather4: %d CTAs/SM x %d issuing warps", ctas, issuers);
            timed([&] { tma_kernel<<<sms * ctas, 32 * MAXW>>>(map, rows, batches, issuers, tab, n, 0, sink); },
                  (double)sms * ctas * issuers * batches * G * 4, name);
        }
    }
    // both paths: 2 issuing warps + 6 LSU warps per CTA, 4 CTAs / SM
    {
        const uint32_t batches = 2048, lper = 2048;
        const double tma_g = (double)sms * 4 * 2 * batches * G * 4, lsu_g = (double)sms * 4 * 6 * 32 * lper;
        timed([&] { tma_kernel<<<sms * 4, 32 * MAXW>>>(map, rows, batches, 2, tab, n, lper, sink); }, tma_g + lsu_g,
              "both: 4 CTAs/SM, 2 TMA warps + 6 LSU warps");
        printf("  (tma share %.2f of the gathers)\n", tma_g / (tma_g + lsu_g));
    }
    return 0;
}
