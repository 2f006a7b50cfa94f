// common.cuh -- shared device helpers, error plumbing and the context type.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "dfakit_b200.h"

namespace dk {

constexpr uint32_t kNone = 0xffffffffu;
constexpr int kThreads = 256;

// Thrown inside the library, translated to dfakit_status at the C boundary.
struct Error : std::runtime_error {
    dfakit_status status;
    Error(dfakit_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define DK_CUDA(call)                                                                              \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            throw ::dk::Error(DFAKIT_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct Ctx;

// Launch bookkeeping: every kernel launch in the library goes through
// DK_LAUNCH / DK_LAUNCH_B so the context can report how many of its kernels
// ran and, in profiling mode, time each launch with CUDA events on the
// launching stream.  DK_LAUNCH_B annotates the launch with its ALGORITHMIC
// bytes (the minimum the kernel must move), used for the roofline.
void note_launch(Ctx* ctx);
void prof_begin_launch(Ctx* ctx, cudaStream_t s);
void prof_end_launch(Ctx* ctx, cudaStream_t s, const char* name, double bytes, double units);

// DK_LAUNCH_BU also annotates work units (the random label gathers of the
// signature kernels), for the gather roofline.
#define DK_LAUNCH_BU(ctx, bytes, units, kernel, grid, block, smem, stream, ...)                          \
    do {                                                                                                 \
        ::dk::prof_begin_launch(ctx, stream);                                                            \
        kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                                      \
        ::dk::note_launch(ctx);                                                                          \
        cudaError_t e_ = cudaGetLastError();                                                             \
        if (e_ != cudaSuccess)                                                                           \
            throw ::dk::Error(DFAKIT_E_CUDA, std::string(#kernel) + " launch: " + cudaGetErrorString(e_)); \
        ::dk::prof_end_launch(ctx, stream, #kernel, (double)(bytes), (double)(units));                   \
    } while (0)

#define DK_LAUNCH_B(ctx, bytes, kernel, grid, block, smem, stream, ...) \
    DK_LAUNCH_BU(ctx, bytes, 0, kernel, grid, block, smem, stream, __VA_ARGS__)

#define DK_LAUNCH(ctx, kernel, grid, block, smem, stream, ...) \
    DK_LAUNCH_B(ctx, 0, kernel, grid, block, smem, stream, __VA_ARGS__)

struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
    double bytes, units;
    uint32_t pass;  // refinement pass the launch belongs to (0: none)
};

// Device context: one device, one stream, a stream-ordered pool, a pinned
// mailbox for small device->host readbacks.
struct Ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // host->device input streaming (lazily created)
    bool own_stream = true;
    uint64_t* mailbox = nullptr;  // pinned host, 64 words: [0, 56) read_words, [56, 64) deferred reads
    uint64_t* dmailbox = nullptr; // device, 64 words
    uint32_t* fastbox = nullptr;  // pinned host, device-written: [0] sequence number, [2, 2 + 112) payload
    uint32_t fast_seq = 0;
    cudaEvent_t info_ev = nullptr;  // marks a deferred mailbox read (no timing)
    uint64_t launches = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    bool profiling = false;
    uint32_t prof_pass = 0;  // set by the pass loops: launches are tagged with it
    cudaEvent_t pending = nullptr;
    std::vector<ProfRec> prof;
};

// Stream-ordered device buffer (cudaMallocAsync on the context stream).
template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    DBuf() = default;
    DBuf(size_t count, cudaStream_t st) { alloc(count, st); }
    void alloc(size_t count, cudaStream_t st) {
        release();
        s = st;
        n = count;
        if (count) DK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), st));
    }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    ~DBuf() { release(); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            s = o.s;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    T* get() const { return p; }
};

inline unsigned grid_for(uint64_t n, int threads = kThreads, unsigned cap = 148u * 64u) {
    uint64_t g = (n + threads - 1) / threads;
    if (g == 0) g = 1;
    return (unsigned)(g < cap ? g : cap);
}

inline uint32_t bits_for(uint64_t max_value) {  // bits needed to represent 0..max_value
    uint32_t b = 0;
    while (b < 64 && (max_value >> b) != 0) ++b;
    return b;
}

__host__ __device__ inline uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// Read-only streaming load for data touched once (delta rows).
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) { return __ldcs(p); }

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// Warp-aggregated atomic increment: one atomic per warp, returns this lane's slot.
__device__ __forceinline__ uint32_t warp_append(uint32_t* counter, bool pred) {
    unsigned mask = __ballot_sync(__activemask(), pred);
    if (!pred) return kNone;
    unsigned leader = __ffs(mask) - 1;
    uint32_t base = 0;
    if (lane_id() == leader) base = atomicAdd(counter, (uint32_t)__popc(mask));
    base = __shfl_sync(mask, base, leader);
    return base + __popc(mask & ((1u << lane_id()) - 1u));
}

// Synchronous readback of `count` words from device memory through the pinned mailbox.
void read_words(Ctx* ctx, const void* dsrc, size_t bytes, void* hdst, cudaStream_t s);
// the same in two halves: the copy is queued by _begin, _end waits for it --
// work queued in between runs while the host waits
uint32_t read_words_begin(Ctx* ctx, const void* dsrc, size_t bytes, cudaStream_t s);
void read_words_end(Ctx* ctx, uint32_t seq, size_t bytes, void* hdst, cudaStream_t s);

}  // namespace dk
