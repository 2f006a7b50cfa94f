// dsmem_probe.cu -- experiment: random 32-bit gathers served from the
// (distributed) shared memory of a thread-block cluster, against the same
// gathers from global memory (L2 resident).  Decides whether a label table
// that fits a cluster's shared memory (the 1.25 MB bitmap of a 10M-state
// two-block partition) should be gathered through DSMEM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/dsmem_probe tools/dsmem_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint64_t lcg(uint64_t& x) {
    x = x * 6364136223846793005ull + 1442695040888963407ull;
    return x >> 29;
}

// every CTA of a cluster holds `words` words; a gather picks a random word of
// the cluster-wide table
__global__ void dsmem_kernel(uint32_t words, uint32_t lw, uint32_t rounds, uint32_t* sink) {
    extern __shared__ uint32_t tab[];
    cg::cluster_group cl = cg::this_cluster();
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) tab[i] = i * 2654435761u;
    cl.sync();
    const uint32_t csize = cl.num_blocks();
    const uint64_t total = (uint64_t)words * csize;
    uint64_t x = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 1;
    uint32_t acc = 0;
    for (uint32_t r = 0; r < rounds; ++r) {
        uint32_t v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint32_t g = __umulhi((uint32_t)lcg(x), (uint32_t)total);
            const uint32_t rank = g >> lw, off = g & (words - 1);
            const uint32_t* p = cl.map_shared_rank(tab, rank);
            v[j] = p[off];
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += v[j];
    }
    cl.sync();
    if (acc == 0x12345u) sink[0] = acc;
}

__global__ void local_kernel(uint32_t words, uint32_t rounds, uint32_t* sink) {
    extern __shared__ uint32_t tab[];
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) tab[i] = i * 2654435761u;
    __syncthreads();
    uint64_t x = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 1;
    uint32_t acc = 0;
    for (uint32_t r = 0; r < rounds; ++r) {
        uint32_t v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = tab[__umulhi((uint32_t)lcg(x), words)];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += v[j];
    }
    if (acc == 0x12345u) sink[0] = acc;
}

__global__ void global_kernel(const uint32_t* __restrict__ tab, uint32_t words, uint32_t rounds, uint32_t* sink) {
    uint64_t x = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 1;
    uint32_t acc = 0;
    for (uint32_t r = 0; r < rounds; ++r) {
        uint32_t v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __ldg(tab + __umulhi((uint32_t)lcg(x), words));
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += v[j];
    }
    if (acc == 0x12345u) sink[0] = acc;
}

// load-variant probe: does any PTX load flavour beat one line per SM per clock?
template <int V>
__device__ __forceinline__ uint32_t ldv(const uint32_t* p) {
    uint32_t r;
    if (V == 0) r = __ldg(p);
    else if (V == 1) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(r) : "l"(p));
    else if (V == 2) asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    else if (V == 3) asm volatile("ld.global.nc.L2::64B.u32 %0, [%1];" : "=r"(r) : "l"(p));
    else r = *(volatile const uint32_t*)p;
    return r;
}

template <int V>
__global__ void variant_kernel(const uint32_t* __restrict__ tab, uint32_t words, uint32_t rounds, uint32_t* sink) {
    uint64_t x = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 1;
    uint32_t acc = 0;
    for (uint32_t r = 0; r < rounds; ++r) {
        uint32_t v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = ldv<V>(tab + __umulhi((uint32_t)lcg(x), words));
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += v[j];
    }
    if (acc == 0x12345u) sink[0] = acc;
}

// cp.async 4-byte gathers into shared memory (LDGSTS), 16 per round
__global__ void cpasync_kernel(const uint32_t* __restrict__ tab, uint32_t words, uint32_t rounds, uint32_t* sink) {
    __shared__ uint32_t buf[256 * 16];
    uint64_t x = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 1;
    uint32_t acc = 0;
    for (uint32_t r = 0; r < rounds; ++r) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint32_t* src = tab + __umulhi((uint32_t)lcg(x), words);
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&buf[j * 256 + threadIdx.x]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src));
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += buf[j * 256 + threadIdx.x];
    }
    if (acc == 0x12345u) sink[0] = acc;
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    uint32_t* sink;
    CK(cudaMalloc(&sink, 4));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const uint32_t rounds = 256;
    // global: 1.25 MB, 20 MB, 40 MB tables
    for (uint32_t words : {312500u, 5000000u, 10000000u}) {
        uint32_t* t;
        CK(cudaMalloc(&t, words * 4ull));
        CK(cudaMemset(t, 1, words * 4ull));
        const unsigned grid = sms * 8, threads = 256;
        global_kernel<<<grid, threads>>>(t, words, rounds, sink);
        cudaEventRecord(a);
        global_kernel<<<grid, threads>>>(t, words, rounds, sink);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("global  table %8.2f MB: %.3e gathers/s\n", words * 4e-6, (double)grid * threads * rounds * 16 / (ms * 1e-3));
        cudaFree(t);
    }
    {
        const uint32_t words = 5000000u;
        uint32_t* t;
        CK(cudaMalloc(&t, words * 4ull));
        CK(cudaMemset(t, 1, words * 4ull));
        const unsigned grid = sms * 8, threads = 256;
        const char* names[] = {"ld.global.nc", "ld.global.cg", "ld.nc.L1::no_allocate", "ld.nc.L2::64B", "ld.volatile", "cp.async.ca 4B"};
        for (int v = 0; v < 6; ++v) {
            for (int rep = 0; rep < 2; ++rep) {
                if (rep) cudaEventRecord(a);
                switch (v) {
                    case 0: variant_kernel<0><<<grid, threads>>>(t, words, rounds, sink); break;
                    case 1: variant_kernel<1><<<grid, threads>>>(t, words, rounds, sink); break;
                    case 2: variant_kernel<2><<<grid, threads>>>(t, words, rounds, sink); break;
                    case 3: variant_kernel<3><<<grid, threads>>>(t, words, rounds, sink); break;
                    case 4: variant_kernel<4><<<grid, threads>>>(t, words, rounds, sink); break;
                    case 5: cpasync_kernel<<<grid, threads>>>(t, words, rounds, sink); break;
                }
                if (rep) cudaEventRecord(b);
            }
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("variant %-24s 20 MB: %.3e gathers/s\n", names[v], (double)grid * threads * rounds * 16 / (ms * 1e-3));
        }
        cudaFree(t);
    }
    for (uint32_t kb : {16u, 64u, 160u, 200u}) {
        const uint32_t words = kb * 256;
        CK(cudaFuncSetAttribute(local_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kb * 1024));
        for (unsigned threads : {512u, 1024u}) {
            const unsigned grid = sms;
            local_kernel<<<grid, threads, kb * 1024>>>(words, rounds, sink);
            CK(cudaGetLastError());
            cudaEventRecord(a);
            local_kernel<<<grid, threads, kb * 1024>>>(words, rounds, sink);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("local   %3u KB x %4u thr: %.3e gathers/s\n", kb, threads,
                   (double)grid * threads * rounds * 16 / (ms * 1e-3));
        }
    }
    CK(cudaFuncSetAttribute(dsmem_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (uint32_t kb : {64u, 128u}) {
        CK(cudaFuncSetAttribute(dsmem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kb * 1024));
        for (unsigned cs : {2u, 4u, 8u, 16u}) {
            for (unsigned threads : {512u, 1024u}) {
                const uint32_t words = kb * 256;
                cudaLaunchConfig_t cfg = {};
                int maxc = 0;
                cfg.blockDim = dim3(threads);
                cfg.dynamicSmemBytes = kb * 1024;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = cs;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                cfg.gridDim = dim3(cs);
                if (cudaOccupancyMaxActiveClusters(&maxc, dsmem_kernel, &cfg) != cudaSuccess || maxc == 0) {
                    cudaGetLastError();
                    printf("dsmem cluster %2u: does not fit\n", cs);
                    continue;
                }
                cfg.gridDim = dim3(cs * maxc);
                CK(cudaLaunchKernelEx(&cfg, dsmem_kernel, words, 31 - __builtin_clz(words), rounds, sink));
                cudaEventRecord(a);
                CK(cudaLaunchKernelEx(&cfg, dsmem_kernel, words, 31 - __builtin_clz(words), rounds, sink));
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                printf("dsmem cluster %2u (%3u clusters, %3u KB/CTA = %.2f MB, %4u thr): %.3e gathers/s\n", cs, maxc,
                       kb, cs * kb / 1024.0, threads, (double)cs * maxc * threads * rounds * 16 / (ms * 1e-3));
            }
        }
    }
    return 0;
}
