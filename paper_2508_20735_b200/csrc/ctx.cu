// ctx.cu -- device context, error state and small readbacks.
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace dk {

void note_launch(Ctx* ctx) {
    if (ctx) ++ctx->launches;
}

void prof_begin_launch(Ctx* ctx, cudaStream_t s) {
    if (!ctx || !ctx->profiling) return;
    DK_CUDA(cudaEventCreate(&ctx->pending));
    DK_CUDA(cudaEventRecord(ctx->pending, s));
}

void prof_end_launch(Ctx* ctx, cudaStream_t s, const char* name, double bytes, double units) {
    if (!ctx || !ctx->profiling || !ctx->pending) return;
    cudaEvent_t b;
    DK_CUDA(cudaEventCreate(&b));
    DK_CUDA(cudaEventRecord(b, s));
    ctx->prof.push_back(ProfRec{name, ctx->pending, b, bytes, units, ctx->prof_pass});
    ctx->pending = nullptr;
}

// Per-kernel totals as a JSON array: [{"name", "launches", "ms", "bytes"}].
std::string prof_collect(Ctx* ctx) {
    struct Agg {
        std::string name;
        uint64_t launches = 0;
        double ms = 0, bytes = 0, units = 0;
    };
    std::vector<Agg> aggs, passes;  // per kernel name; per refinement pass ("#pass N")
    // DFAKIT_PROF_TIMELINE=1: every recorded launch with its start offset and
    // duration on stderr (development aid: gaps between launches)
    const bool timeline = getenv("DFAKIT_PROF_TIMELINE") != nullptr;
    for (size_t i = 0; timeline && i < ctx->prof.size(); ++i) {
        auto& r = ctx->prof[i];
        DK_CUDA(cudaEventSynchronize(r.b));
        float t0 = 0, ms = 0;
        DK_CUDA(cudaEventElapsedTime(&t0, ctx->prof[0].a, r.a));
        DK_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
        fprintf(stderr, "timeline %4zu %10.4f ms  %9.4f ms  %s\n", i, t0, ms, r.name);
    }
    for (auto& r : ctx->prof) {
        DK_CUDA(cudaEventSynchronize(r.b));
        float ms = 0;
        DK_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
        Agg* g = nullptr;
        for (auto& x : aggs)
            if (x.name == r.name) g = &x;
        if (!g) {
            aggs.push_back(Agg{r.name});
            g = &aggs.back();
        }
        ++g->launches;
        g->ms += ms;
        g->bytes += r.bytes;
        g->units += r.units;
        if (r.pass) {
            const std::string pn = "#pass " + std::to_string(r.pass);
            Agg* pg = nullptr;
            for (auto& x : passes)
                if (x.name == pn) pg = &x;
            if (!pg) {
                passes.push_back(Agg{pn});
                pg = &passes.back();
            }
            ++pg->launches;
            pg->ms += ms;
            pg->bytes += r.bytes;
            pg->units += r.units;
        }
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    ctx->prof.clear();
    aggs.insert(aggs.end(), passes.begin(), passes.end());
    std::string out = "[";
    char buf[512];
    for (size_t i = 0; i < aggs.size(); ++i) {
        snprintf(buf, sizeof buf, "%s{\"name\":\"%s\",\"launches\":%llu,\"ms\":%.6f,\"bytes\":%.0f,\"units\":%.0f}",
                 i ? "," : "", aggs[i].name.c_str(), (unsigned long long)aggs[i].launches, aggs[i].ms, aggs[i].bytes,
                 aggs[i].units);
        out += buf;
    }
    return out + "]";
}

// One CTA copies the words into pinned host memory and then publishes the
// sequence number; the host spins on it.  A copy-engine readback plus
// cudaStreamSynchronize cost ~10 us more per pass-loop round trip.
__global__ void mailbox_kernel(const uint8_t* __restrict__ src, uint32_t bytes, uint32_t* box, uint32_t seq) {
    volatile uint8_t* dst = reinterpret_cast<volatile uint8_t*>(box + 2);
    for (uint32_t i = threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        *reinterpret_cast<volatile uint32_t*>(box) = seq;
    }
}

void read_words(Ctx* ctx, const void* dsrc, size_t bytes, void* hdst, cudaStream_t s) {
    read_words_end(ctx, read_words_begin(ctx, dsrc, bytes, s), bytes, hdst, s);
}

uint32_t read_words_begin(Ctx* ctx, const void* dsrc, size_t bytes, cudaStream_t s) {
    if (bytes > 56 * sizeof(uint64_t)) throw Error(DFAKIT_E_INVALID, "read_words: too large");
    const uint32_t seq = ++ctx->fast_seq;
    mailbox_kernel<<<1, 128, 0, s>>>(static_cast<const uint8_t*>(dsrc), (uint32_t)bytes, ctx->fastbox, seq);
    DK_CUDA(cudaGetLastError());
    note_launch(ctx);
    return seq;
}

void read_words_end(Ctx* ctx, uint32_t seq, size_t bytes, void* hdst, cudaStream_t s) {
    // spin for short waits (the pass loop's readbacks follow sub-millisecond
    // kernels); past ~200 us block in cudaStreamSynchronize instead of
    // burning a core behind a long kernel
    volatile uint32_t* flag = ctx->fastbox;
    const auto t0 = std::chrono::steady_clock::now();
    for (uint32_t spin = 1;; ++spin) {
        if (*flag == seq) break;
        if ((spin & 1023u) == 0) {
            const cudaError_t e = cudaStreamQuery(s);  // a failed launch never writes the flag
            if (e != cudaSuccess && e != cudaErrorNotReady)
                throw Error(DFAKIT_E_CUDA, std::string("read_words: ") + cudaGetErrorString(e));
            if (e == cudaSuccess || std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(200)) {
                DK_CUDA(cudaStreamSynchronize(s));
                if (*flag != seq) throw Error(DFAKIT_E_CUDA, "read_words: stream completed without the mailbox write");
                break;
            }
        }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    std::memcpy(hdst, const_cast<const uint32_t*>(ctx->fastbox) + 2, bytes);
}

Ctx* ctx_create(int device) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        throw Error(DFAKIT_E_NODEVICE, "no CUDA device available: the B200 library has no CPU fallback");
    }
    if (device < 0 || device >= count) throw Error(DFAKIT_E_INVALID, "device index out of range");
    DK_CUDA(cudaSetDevice(device));
    Ctx* c = new Ctx();
    c->device = device;
    DK_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    DK_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    DK_CUDA(cudaMallocHost(reinterpret_cast<void**>(&c->mailbox), 64 * sizeof(uint64_t)));
    DK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c->fastbox), 128 * sizeof(uint32_t), cudaHostAllocMapped));
    std::memset(c->fastbox, 0, 128 * sizeof(uint32_t));
    DK_CUDA(cudaMalloc(reinterpret_cast<void**>(&c->dmailbox), 64 * sizeof(uint64_t)));
    {  // leader_info_kernel's accumulators (words 0-3) and CTA counter (word 12), re-armed by the kernel
        uint32_t init[128] = {};
        init[0] = init[1] = 0xffffffffu;
        DK_CUDA(cudaMemcpy(c->dmailbox, init, sizeof(init), cudaMemcpyHostToDevice));
    }
    DK_CUDA(cudaEventCreate(&c->ev0));
    DK_CUDA(cudaEventCreate(&c->ev1));
    DK_CUDA(cudaEventCreateWithFlags(&c->info_ev, cudaEventDisableTiming));
    // keep freed pool memory around: repeated calls reuse it without cudaMalloc
    cudaMemPool_t pool;
    DK_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t threshold = ~0ull;
    DK_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    return c;
}

void ctx_destroy(Ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->mailbox) cudaFreeHost(c->mailbox);
    if (c->fastbox) cudaFreeHost(c->fastbox);
    if (c->dmailbox) cudaFree(c->dmailbox);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->info_ev) cudaEventDestroy(c->info_ev);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->stream && c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
}

}  // namespace dk
