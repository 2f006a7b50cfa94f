// gen.cu -- benchmark inputs generated in place in HBM.
#include "refine.cuh"

namespace dk {

namespace {

// same formula as oracle/oracle.c or_gen_synth
__global__ void synth_kernel(uint32_t n, uint32_t k, uint64_t seed, uint32_t* __restrict__ delta,
                             uint8_t* __restrict__ acc) {
    const uint64_t total = (uint64_t)k * n;
    for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t h = mix64(seed ^ (idx * 0xD1B54A32D192ED03ull));
        delta[idx] = (uint32_t)(((h >> 32) * (uint64_t)n) >> 32);
    }
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n; q += (uint64_t)gridDim.x * blockDim.x)
        acc[q] = (uint8_t)(mix64(~seed ^ (q * 0xD1B54A32D192ED03ull)) >> 63);
}

__global__ void chain_kernel(uint32_t n, uint32_t* __restrict__ delta, uint8_t* __restrict__ acc) {
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        delta[q] = q + 1 < n ? q + 1 : q;
        acc[q] = q + 1 == n;
    }
}

__global__ void permute_kernel(uint32_t n, uint32_t k, uint64_t mul, uint64_t add, const uint32_t* __restrict__ delta,
                               const uint8_t* __restrict__ acc, uint32_t* __restrict__ out_delta,
                               uint8_t* __restrict__ out_acc) {
    const uint64_t total = (uint64_t)k * n;
    for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a = idx / n, q = idx % n;
        const uint64_t pq = (mul * q + add) % n, pt = (mul * delta[idx] + add) % n;
        out_delta[a * n + pq] = (uint32_t)pt;
    }
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n; q += (uint64_t)gridDim.x * blockDim.x)
        out_acc[(mul * q + add) % n] = acc[q];
}

uint64_t gcd64(uint64_t a, uint64_t b) {
    while (b) {
        uint64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

}  // namespace

void gen_synth_device(Ctx* ctx, uint32_t n, uint32_t k, uint64_t seed, uint32_t* delta, uint8_t* acc,
                      cudaStream_t s) {
    DK_LAUNCH(ctx, synth_kernel, grid_for((uint64_t)k * n), kThreads, 0, s, n, k, seed, delta, acc);
}

void gen_chain_device(Ctx* ctx, uint32_t n, uint32_t* delta, uint8_t* acc, cudaStream_t s) {
    DK_LAUNCH(ctx, chain_kernel, grid_for(n), kThreads, 0, s, n, delta, acc);
}

// q -> (mul*q + add) mod n with gcd(mul, n) = 1; returns the image of state 0
uint32_t permute_states_device(Ctx* ctx, uint32_t n, uint32_t k, uint64_t seed, const uint32_t* delta,
                               const uint8_t* acc, uint32_t* out_delta, uint8_t* out_acc, cudaStream_t s) {
    if (n == 0) return 0;
    uint64_t h = mix64(seed);
    uint64_t mul = (h % n) | 1ull;
    while (gcd64(mul, n) != 1) mul = (mul + 2) % n ? (mul + 2) % n : 1;
    const uint64_t add = mix64(h) % n;
    DK_LAUNCH(ctx, permute_kernel, grid_for((uint64_t)k * n), kThreads, 0, s, n, k, mul, add, delta, acc, out_delta,
              out_acc);
    return (uint32_t)(add % n);
}

}  // namespace dk
