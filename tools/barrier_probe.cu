// Grid-barrier probe: cooperative-groups grid.sync() against a two-level
// (32 group counters, per-group release flags) barrier, R rounds each, with
// every SM filled at 256-thread CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/barrier_probe tools/barrier_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void cg_kernel(int rounds, unsigned* sink) {
    cg::grid_group g = cg::this_grid();
    unsigned x = 0;
    for (int r = 0; r < rounds; ++r) {
        x += threadIdx.x;
        g.sync();
    }
    if (x == 0xdeadbeef) *sink = x;
}

constexpr int kGroups = 32;
struct Bar {
    unsigned arrive[kGroups * 32];  // one counter per group, 128 bytes apart
    unsigned top[32];
    unsigned gen[kGroups * 32];     // per-group release words, 128 bytes apart
};

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ void two_level_sync(Bar* b, unsigned& epoch) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned G = min(gridDim.x, (unsigned)kGroups);
        const unsigned grp = blockIdx.x % G;
        const unsigned members = gridDim.x / G + (grp < gridDim.x % G ? 1u : 0u);
        ++epoch;
        __threadfence();
        const unsigned a = atomicAdd(&b->arrive[grp * 32], 1u) + 1;
        if (a == members * epoch) {  // last of the group
            const unsigned t = atomicAdd(&b->top[0], 1u) + 1;
            if (t == G * epoch) {  // last group: release every group
                __threadfence();
                for (unsigned j = 0; j < G; ++j) atomicExch(&b->gen[j * 32], epoch);
            }
        }
        while (ld_acq(&b->gen[grp * 32]) < epoch) {
        }
    }
    __syncthreads();
}

__global__ void two_level_kernel(int rounds, Bar* b, unsigned* sink) {
    unsigned epoch = 0, x = 0;
    for (int r = 0; r < rounds; ++r) {
        x += threadIdx.x;
        two_level_sync(b, epoch);
    }
    if (x == 0xdeadbeef) *sink = x;
}

int main() {
    int per_sm = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cg_kernel, 256, 0);
    unsigned* sink;
    Bar* bar;
    cudaMalloc(&sink, 4);
    cudaMalloc(&bar, sizeof(Bar));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int rounds = 20000;
    for (int ctas : {148, 391, 592, 1184, per_sm * sms}) {
        if (ctas > per_sm * sms) continue;
        void* a1[] = {(void*)&rounds, (void*)&sink};
        cudaLaunchCooperativeKernel((void*)cg_kernel, ctas, 256, a1, 0, 0);
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)cg_kernel, ctas, 256, a1, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaMemset(bar, 0, sizeof(Bar));
        void* a2[] = {(void*)&rounds, (void*)&bar, (void*)&sink};
        cudaLaunchCooperativeKernel((void*)two_level_kernel, ctas, 256, a2, 0, 0);
        cudaMemset(bar, 0, sizeof(Bar));
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)two_level_kernel, ctas, 256, a2, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms2 = 0;
        cudaEventElapsedTime(&ms2, e0, e1);
        printf("%5d CTAs: cg grid.sync %.3f us, two-level %.3f us per barrier (%s)\n", ctas, 1000 * ms / rounds,
               1000 * ms2 / rounds, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
