// tex_probe.cu -- experiment: random label gathers through the texture path
// (tex1Dfetch on a linear texture object) against LSU gathers (ld.global.nc),
// and both paths at once.  The signature passes are bound by the L1TEX
// tag-lookup rate of random LSU gathers (~1 line per clock per SM); does the
// texture pipeline look lines up at a different rate?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bin/tex_probe tools/tex_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t lcg(uint64_t& x) {
    x = x * 6364136223846793005ull + 1442695040888963407ull;
    return (uint32_t)(x >> 32);
}

template <typename T>
__global__ void lsu_kernel(const T* __restrict__ tab, uint32_t n, uint32_t per_thread, uint32_t* sink) {
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

template <typename T>
__global__ void tex_kernel(cudaTextureObject_t tex, uint32_t n, uint32_t per_thread, uint32_t* sink) {
    uint64_t x = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 11;
    uint32_t acc = 0;
    for (uint32_t r = 0; r < per_thread; r += 16) {
        uint32_t v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = tex1Dfetch<T>(tex, (int)__umulhi(lcg(x), n));
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += v[j];
    }
    if (acc == 0x12345u) sink[0] = acc;
}

// half the warps on each path
template <typename T>
__global__ void mixed_kernel(const T* __restrict__ tab, cudaTextureObject_t tex, uint32_t n, uint32_t per_thread,
                             uint32_t* sink) {
    uint64_t x = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 13;
    uint32_t acc = 0;
    const bool use_tex = (threadIdx.x >> 5) & 1;
    for (uint32_t r = 0; r < per_thread; r += 16) {
        uint32_t v[16];
        if (use_tex) {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = tex1Dfetch<T>(tex, (int)__umulhi(lcg(x), n));
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = __ldg(tab + __umulhi(lcg(x), n));
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += v[j];
    }
    if (acc == 0x12345u) sink[0] = acc;
}

template <typename T>
void run(uint32_t n, int sms) {
    T* tab;
    uint32_t* sink;
    cudaMalloc(&tab, (size_t)n * sizeof(T));
    cudaMalloc(&sink, 4);
    cudaMemset(tab, 1, (size_t)n * sizeof(T));
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = tab;
    rd.res.linear.desc = cudaCreateChannelDesc<T>();
    rd.res.linear.sizeInBytes = (size_t)n * sizeof(T);
    cudaTextureDesc td{};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex = 0;
    cudaError_t e = cudaCreateTextureObject(&tex, &rd, &td, nullptr);
    if (e != cudaSuccess) {
        printf("texture object: %s\n", cudaGetErrorString(e));
        return;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const uint32_t per = 2048;
    auto timed = [&](auto launch, double gathers, const char* name) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%zu-byte table %6.1f MB  %-34s %8.3f ms  %.3g gathers/s  %s\n", sizeof(T), n * sizeof(T) / 1e6, name,
               ms, gathers / (ms / 1e3), cudaGetErrorString(cudaGetLastError()));
    };
    for (int cps : {4, 8}) {
        const unsigned blocks = sms * cps, threads = 256;
        const double g = (double)blocks * threads * per;
        char nm[64];
        snprintf(nm, sizeof nm, "LSU ld.global.nc, %d CTAs/SM", cps);
        timed([&] { lsu_kernel<T><<<blocks, threads>>>(tab, n, per, sink); }, g, nm);
        snprintf(nm, sizeof nm, "texture tex1Dfetch, %d CTAs/SM", cps);
        timed([&] { tex_kernel<T><<<blocks, threads>>>(tex, n, per, sink); }, g, nm);
        snprintf(nm, sizeof nm, "half LSU / half texture, %d CTAs/SM", cps);
        timed([&] { mixed_kernel<T><<<blocks, threads>>>(tab, tex, n, per, sink); }, g, nm);
    }
    cudaDestroyTextureObject(tex);
    cudaFree(tab);
    cudaFree(sink);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<uint16_t>(10u << 20, sms);   // 20 MB: the bench's 16-bit key labels of 10M states
    run<uint32_t>(10u << 20, sms);   // 40 MB
    run<uint16_t>(1u << 20, sms);    // 2 MB
    return 0;
}
