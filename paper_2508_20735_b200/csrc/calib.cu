// calib.cu -- measured ceiling for the random block-label gathers.
//
// The signature kernels read lab[delta(q, a)] for every active state and
// letter: for random automata every lane of a warp-wide gather touches a
// different 128-byte line, so their bound is the L1TEX/L2 line rate, not HBM
// bandwidth.  This kernel issues the same access pattern with nothing else
// around it (independent random 32-bit gathers from a table of the label
// array's size, 16 in flight per thread, grid filling every SM) and is timed
// by bench.py beside the real kernels: achieved gathers/s of a signature
// kernel / this rate = its fraction of the gather roofline.
#include "common.cuh"

namespace dk {

namespace {

template <typename T>
__global__ void __launch_bounds__(256) gather_probe_kernel(const T* __restrict__ table, uint64_t mask,
                                                           uint32_t rounds, uint64_t seed, uint32_t* __restrict__ sink) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    uint64_t x = mix64(seed ^ tid);
    for (uint32_t r = 0; r < rounds; ++r) {
        uint32_t idx[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            x = x * 6364136223846793005ull + 1442695040888963407ull;
            idx[j] = (uint32_t)((x >> 29) & mask);
        }
        uint32_t v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = (uint32_t)table[idx[j]];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += v[j];
    }
    if (acc == 0x9e3779b9u) sink[0] = acc;  // keeps the loads alive
}

}  // namespace

double calibrate_gather(Ctx* ctx, uint64_t table_words, uint32_t elem_bytes, uint64_t gathers, cudaStream_t s,
                        float* ms_out) {
    uint64_t words = 1;
    while (words < table_words) words <<= 1;
    DBuf<uint8_t> table(words * elem_bytes, s);
    DK_CUDA(cudaMemsetAsync(table.get(), 1, words * elem_bytes, s));
    DBuf<uint32_t> sink(1, s);
    const unsigned threads = 256, blocks = (unsigned)ctx->num_sms * 8;
    const uint64_t per_round = (uint64_t)threads * blocks * 16;
    const uint32_t rounds = (uint32_t)std::max<uint64_t>(1, gathers / per_round);
    auto launch = [&] {
        if (elem_bytes == 1)
            DK_LAUNCH(ctx, gather_probe_kernel<uint8_t>, blocks, threads, 0, s, table.get(), words - 1, rounds, 7ull,
                      sink.get());
        else if (elem_bytes == 2)
            DK_LAUNCH(ctx, gather_probe_kernel<uint16_t>, blocks, threads, 0, s,
                      reinterpret_cast<const uint16_t*>(table.get()), words - 1, rounds, 7ull, sink.get());
        else
            DK_LAUNCH(ctx, gather_probe_kernel<uint32_t>, blocks, threads, 0, s,
                      reinterpret_cast<const uint32_t*>(table.get()), words - 1, rounds, 7ull, sink.get());
    };
    launch();  // warm-up: table resident in L2 as far as it fits
    cudaEvent_t a, b;
    DK_CUDA(cudaEventCreate(&a));
    DK_CUDA(cudaEventCreate(&b));
    DK_CUDA(cudaEventRecord(a, s));
    launch();
    DK_CUDA(cudaEventRecord(b, s));
    DK_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    DK_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (ms_out) *ms_out = ms;
    return (double)rounds * per_round / (ms * 1e-3);
}

}  // namespace dk
