// trans.cu -- Cai-Haase style pair-graph closure (paper Alg. 1, reference
// src/minimize.cpp:92-206).  Kept only as a small-n comparison point: the
// reachability matrix over Q x Q has n^4 bits.
//
// Per pass (same semantics as the reference, so closure/refining counts
// match exactly):
//   Reach := Reach | Reach . Reach   from the pass-start matrix.  One CTA per
//            row; a row is recomputed only when it reaches a row that grew in
//            the previous pass (exact);
//   Apart := Apart | { s : Reach[s] meets Apart }   one propagation step.
// Rows are bit-packed (64 pair-nodes per word).
#include "prims.cuh"
#include "refine.cuh"

namespace dk {

namespace {

constexpr int kRowThreads = 128;

__global__ void trans_init_kernel(const uint32_t* __restrict__ delta, const uint8_t* __restrict__ acc, uint32_t n,
                                  uint32_t k, uint64_t W, unsigned long long* __restrict__ reach,
                                  unsigned long long* __restrict__ apart) {
    const uint64_t V = (uint64_t)n * n;
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < V; s += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t q = (uint32_t)(s / n), r = (uint32_t)(s % n);
        if (acc[q] != acc[r]) atomicOr(&apart[s >> 6], 1ull << (s & 63));
        for (uint32_t a = 0; a < k; ++a) {
            const uint64_t t = (uint64_t)delta[(uint64_t)a * n + q] * n + delta[(uint64_t)a * n + r];
            atomicOr(&reach[s * W + (t >> 6)], 1ull << (t & 63));
        }
    }
}

// next[s] = reach[s] | OR_{t in reach[s]} reach[t]
__global__ void __launch_bounds__(kRowThreads) trans_square_kernel(const unsigned long long* __restrict__ reach,
                                                                   unsigned long long* __restrict__ next, uint64_t V,
                                                                   uint64_t W,
                                                                   const unsigned long long* __restrict__ changed,
                                                                   unsigned long long* __restrict__ changed_next) {
    extern __shared__ unsigned long long row[];  // 2 * W words: the row, then the accumulator
    unsigned long long* accw = row + W;
    __shared__ int touch, grew;
    for (uint64_t s = blockIdx.x; s < V; s += gridDim.x) {
        if (threadIdx.x == 0) {
            touch = 0;
            grew = 0;
        }
        __syncthreads();
        const unsigned long long* rs = reach + s * W;
        int t_local = 0;
        for (uint64_t w = threadIdx.x; w < W; w += blockDim.x) {
            unsigned long long v = rs[w];
            row[w] = v;
            accw[w] = v;
            t_local |= (v & changed[w]) != 0ull;
        }
        if (t_local) touch = 1;
        __syncthreads();
        if (touch) {
            for (uint64_t w = 0; w < W; ++w) {
                unsigned long long bits = row[w];
                while (bits) {
                    const uint64_t t = (w << 6) + (uint64_t)__ffsll((long long)bits) - 1;
                    bits &= bits - 1;
                    const unsigned long long* rt = reach + t * W;
                    for (uint64_t v = threadIdx.x; v < W; v += blockDim.x) accw[v] |= rt[v];
                }
            }
        }
        __syncthreads();
        int g_local = 0;
        for (uint64_t w = threadIdx.x; w < W; w += blockDim.x) {
            next[s * W + w] = accw[w];
            g_local |= accw[w] != row[w];
        }
        if (g_local) grew = 1;
        __syncthreads();
        if (threadIdx.x == 0 && grew) atomicOr(&changed_next[s >> 6], 1ull << (s & 63));
        __syncthreads();
    }
}

__global__ void trans_apart_kernel(const unsigned long long* __restrict__ reach, uint64_t V, uint64_t W,
                                   const unsigned long long* __restrict__ apart,
                                   unsigned long long* __restrict__ new_apart, uint32_t* __restrict__ any) {
    // one warp per row
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const unsigned lane = threadIdx.x & 31u;
    for (uint64_t s = warp; s < V; s += nwarps) {
        if ((apart[s >> 6] >> (s & 63)) & 1ull) continue;
        int hit = 0;
        for (uint64_t w = lane; w < W && !hit; w += 32) hit = (reach[s * W + w] & apart[w]) != 0ull;
        if (__any_sync(0xffffffffu, hit) && lane == 0) {
            atomicOr(&new_apart[s >> 6], 1ull << (s & 63));
            atomicOr(any, 1u);
        }
    }
}

__global__ void or_into_kernel(unsigned long long* __restrict__ dst, const unsigned long long* __restrict__ src,
                               uint64_t W) {
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < W; w += (uint64_t)gridDim.x * blockDim.x)
        dst[w] |= src[w];
}

__device__ __forceinline__ bool apart_bit(const unsigned long long* apart, uint32_t n, uint32_t q, uint32_t r) {
    if (q == r) return false;
    if (q > r) {
        uint32_t t = q;
        q = r;
        r = t;
    }
    const uint64_t s = (uint64_t)q * n + r;
    return (apart[s >> 6] >> (s & 63)) & 1ull;
}

// partition_from_apart (src/dfa.cpp:424-454): a state joins the first
// representative it is not apart from -- the minimum of its class.
__global__ void apart_labels_kernel(const unsigned long long* __restrict__ apart, uint32_t n,
                                    uint32_t* __restrict__ lab, uint8_t* __restrict__ apart_bytes) {
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        uint32_t r = 0;
        while (r < q && apart_bit(apart, n, r, q)) ++r;
        lab[q] = r;
        if (apart_bytes)
            for (uint32_t c = 0; c < n; ++c) apart_bytes[(uint64_t)q * n + c] = apart_bit(apart, n, q, c) ? 1 : 0;
    }
}

// the complement of apart must be an equivalence (l.442-452 of src/dfa.cpp)
__global__ void apart_check_kernel(const unsigned long long* __restrict__ apart, uint32_t n,
                                   const uint32_t* __restrict__ lab, uint32_t* __restrict__ bad) {
    const uint64_t V = (uint64_t)n * n;
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < V; s += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t q = (uint32_t)(s / n), r = (uint32_t)(s % n);
        if (q >= r) continue;
        if ((lab[q] == lab[r]) == apart_bit(apart, n, q, r)) atomicOr(bad, 1u);
    }
}

}  // namespace

RefineResult trans_minimize_device(Ctx* ctx, const DevDfa& d, uint64_t max_pair_nodes, uint32_t* block_out,
                                   uint8_t* apart_dev, cudaStream_t s) {
    const uint32_t n = d.n;
    const uint64_t V = (uint64_t)n * n;
    if (V > max_pair_nodes) {
        char need[64];
        snprintf(need, sizeof need, "%.1f MiB", (double)V * (double)V / 8.0 / (1 << 20));
        throw Error(DFAKIT_E_RESOURCE, "trans_minimize: " + std::to_string(V) + " pair nodes need " + need +
                                           " of reachability matrix; budget is " + std::to_string(max_pair_nodes) +
                                           " pair nodes");
    }
    RefineResult res;
    if (n == 0) return res;
    const uint64_t W = (V + 63) / 64;
    DBuf<unsigned long long> reach(V * W, s), next(V * W, s), apart(W, s), changed(W, s), changed_next(W, s),
        new_apart(W, s);
    DBuf<uint32_t> any(1, s), lab(n, s), scratch((uint64_t)n + 1, s);
    DK_CUDA(cudaMemsetAsync(reach.get(), 0, V * W * 8, s));
    DK_CUDA(cudaMemsetAsync(apart.get(), 0, W * 8, s));
    DK_CUDA(cudaMemsetAsync(changed.get(), 0xff, W * 8, s));
    DK_LAUNCH(ctx, trans_init_kernel, grid_for(V), kThreads, 0, s, d.delta, d.acc, n, d.k, W, reach.get(), apart.get());
    const size_t smem = 2 * W * sizeof(unsigned long long);
    if (smem > 200 * 1024) throw Error(DFAKIT_E_RESOURCE, "trans_minimize: row does not fit shared memory");
    DK_CUDA(cudaFuncSetAttribute(trans_square_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const unsigned rows_grid = (unsigned)(V < (uint64_t)ctx->num_sms * 16 ? V : (uint64_t)ctx->num_sms * 16);
    unsigned long long *rp = reach.get(), *np = next.get(), *cp = changed.get(), *cnp = changed_next.get();
    for (;;) {
        ++res.closure;
        ++res.passes;
        DK_CUDA(cudaMemsetAsync(cnp, 0, W * 8, s));
        DK_LAUNCH(ctx, trans_square_kernel, rows_grid, kRowThreads, smem, s, rp, np, V, W, cp, cnp);
        std::swap(rp, np);
        std::swap(cp, cnp);
        DK_CUDA(cudaMemsetAsync(new_apart.get(), 0, W * 8, s));
        DK_CUDA(cudaMemsetAsync(any.get(), 0, 4, s));
        DK_LAUNCH(ctx, trans_apart_kernel, grid_for(V * 32), kThreads, 0, s, rp, V, W, apart.get(), new_apart.get(),
                  any.get());
        uint32_t a = 0;
        read_words(ctx, any.get(), 4, &a, s);
        if (!a) break;
        ++res.iters;
        DK_LAUNCH(ctx, or_into_kernel, grid_for(W), kThreads, 0, s, apart.get(), new_apart.get(), W);
    }
    DK_LAUNCH(ctx, apart_labels_kernel, grid_for(n), kThreads, 0, s, apart.get(), n, lab.get(), apart_dev);
    DK_CUDA(cudaMemsetAsync(any.get(), 0, 4, s));
    DK_LAUNCH(ctx, apart_check_kernel, grid_for(V), kThreads, 0, s, apart.get(), n, lab.get(), any.get());
    uint32_t bad = 0;
    read_words(ctx, any.get(), 4, &bad, s);
    if (bad) throw Error(DFAKIT_E_INVALID, "partition_from_apart: complement of apartness is not transitive");
    res.num_blocks = canonical_from_min_labels(ctx, lab.get(), n, block_out, scratch.get(), s);
    return res;
}

}  // namespace dk
