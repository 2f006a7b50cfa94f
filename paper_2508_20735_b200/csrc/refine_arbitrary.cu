// refine_arbitrary.cu -- naive_pr with ElectionPolicy::arbitrary(seed),
// reproducing the reference's winner sequence exactly (src/minimize.cpp:
// 276, 292-305): ONE std::mt19937_64 seeded with the policy seed for the
// whole run; per pass the split list is scanned in state order and, per
// leader slot, the first writer claims it and the c-th writer (c >= 2)
// replaces it when uniform_int_distribution<uint32_t>(0, c - 1) draws 0 --
// reservoir sampling, one engine output per non-first writer (libstdc++'s
// Lemire downscaling; a rejected product draws again).
//
// The sequential stream is made parallel per pass:
//   1. split flags against the pass-start leaders, compacted in state order
//      (the reference's split list);
//   2. a stable LSD radix sort of (leader, position) gives every writer its
//      rank c among its slot's writers (run heads are the first writers);
//   3. an exclusive scan of the non-first flags gives each non-first writer
//      its engine position; one CTA generates that many mt19937_64 outputs
//      (312-word twists in two parallel phases, tempering in parallel) from
//      the state carried across passes;
//   4. writer j draws 0 iff the high word of x_j * c is 0; the slot's winner
//      is its last writer that drew 0 (atomicMax), else its first writer;
//   5. every split state moves to its slot's winner.
// A draw the reference would reject (low word of the product below
// (2^64 - c) mod c: probability < c / 2^64) shifts the stream; the pass is
// then replayed by one thread from the pre-pass engine state (device-side
// branch, never taken in practice but exact when it is).
#include <cooperative_groups.h>

#include <cstdlib>
#include <vector>

#include "prims.cuh"
#include "refine.cuh"

namespace dk {

namespace {

constexpr int kMtN = 312, kMtM = 156;
constexpr uint64_t kMtUpper = 0xFFFFFFFF80000000ull, kMtLower = 0x000000007FFFFFFFull;
constexpr uint64_t kMtMatrix = 0xB5026F5AA96619E9ull;

struct MtState {
    uint64_t mt[kMtN];
    uint32_t idx;
    uint32_t pad;
};

__host__ __device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}

__host__ __device__ __forceinline__ uint64_t mt_mix(uint64_t hi_word, uint64_t lo_word, uint64_t far) {
    const uint64_t x = (hi_word & kMtUpper) | (lo_word & kMtLower);
    return far ^ (x >> 1) ^ ((x & 1u) ? kMtMatrix : 0ull);
}

// sequential engine step (the replay kernel)
__device__ uint64_t mt_next_seq(MtState& g) {
    if (g.idx >= kMtN) {
        for (int i = 0; i < kMtN; ++i) g.mt[i] = mt_mix(g.mt[i], g.mt[(i + 1) % kMtN], g.mt[(i + kMtM) % kMtN]);
        g.idx = 0;
    }
    return mt_temper(g.mt[g.idx++]);
}

// libstdc++ uniform_int_distribution<uint32_t>(0, c - 1) on a 64-bit engine:
// Lemire on the 128-bit product x * c; returns false when the draw would be
// rejected (the caller then needs further outputs)
__device__ __forceinline__ bool lemire_accepts(uint64_t x, uint32_t c, uint32_t* pick) {
    const uint64_t lo = x * (uint64_t)c, hi = __umul64hi(x, (uint64_t)c);
    if (lo < c) {
        const uint64_t threshold = (0ull - (uint64_t)c) % (uint64_t)c;
        if (lo < threshold) return false;
    }
    *pick = (uint32_t)hi;
    return true;
}

// 1. split flags against the pass-start leaders (lab[q] = q's leader)
__global__ void arb_split_flags_kernel(const uint32_t* __restrict__ delta, uint32_t n, uint32_t k,
                                       const uint32_t* __restrict__ lab, uint8_t* __restrict__ flag) {
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        const uint32_t L = lab[q];
        bool split = false;
        if (L != q)
            for (uint32_t a = 0; a < k && !split; ++a) {
                const uint32_t* row = delta + (uint64_t)a * n;
                split = lab[row[q]] != lab[row[L]];
            }
        flag[q] = split;
    }
}

// 2. sort input: (leader, position j) for the j-th split state
__global__ void arb_keys_kernel(const uint32_t* __restrict__ list, const uint32_t* __restrict__ count,
                                const uint32_t* __restrict__ lab, uint64_t* __restrict__ keys,
                                uint32_t* __restrict__ vals, uint32_t* __restrict__ leader_of) {
    const uint32_t m = *count;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
        const uint32_t L = lab[list[j]];
        keys[j] = L;
        vals[j] = j;
        leader_of[j] = L;
    }
}

// run heads of the leader-sorted order: first writer and run start per slot
__global__ void arb_heads_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                                 const uint32_t* __restrict__ count, const uint32_t* __restrict__ list,
                                 uint32_t* __restrict__ run_start, uint32_t* __restrict__ first_q) {
    const uint32_t m = *count;
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < m; p += gridDim.x * blockDim.x) {
        const uint32_t L = (uint32_t)keys[p];
        if (p == 0 || (uint32_t)keys[p - 1] != L) {
            run_start[L] = p;
            first_q[L] = list[vals[p]];
        }
    }
}

// writer rank c (1-based) back in state order; non-first flag for the scan
__global__ void arb_rank_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                                const uint32_t* __restrict__ count, const uint32_t* __restrict__ run_start,
                                uint32_t* __restrict__ rank_of, uint32_t* __restrict__ nonfirst) {
    const uint32_t m = *count;
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < m; p += gridDim.x * blockDim.x) {
        const uint32_t c = p - run_start[(uint32_t)keys[p]] + 1;
        const uint32_t j = vals[p];
        rank_of[j] = c;
        nonfirst[j] = c >= 2;
    }
}

// 3. the next *draws engine outputs, in stream order (one CTA): snapshot the
// pre-pass state for the replay path first
constexpr int kMtThreads = 320;
__global__ void __launch_bounds__(kMtThreads) arb_mt_kernel(MtState* __restrict__ g, MtState* __restrict__ snap,
                                                            const uint32_t* __restrict__ draws,
                                                            uint64_t* __restrict__ out) {
    __shared__ uint64_t mt[kMtN];
    __shared__ uint32_t s_idx;
    const int t = threadIdx.x;
    if (t < kMtN) {
        mt[t] = g->mt[t];
        snap->mt[t] = mt[t];
    }
    if (t == 0) {
        s_idx = g->idx;
        snap->idx = g->idx;
    }
    __syncthreads();
    const uint32_t total = *draws;
    uint32_t idx = s_idx, done = 0;
    while (done < total) {
        if (idx >= kMtN) {
            // twist: words [0, 156) from the old state, then [156, 312) from
            // the new first half (word 311 also reads the new word 0)
            uint64_t v = 0;
            if (t < kMtM) v = mt_mix(mt[t], mt[t + 1], mt[t + kMtM]);
            __syncthreads();
            if (t < kMtM) mt[t] = v;
            __syncthreads();
            if (t >= kMtM && t < kMtN) v = mt_mix(mt[t], mt[(t + 1) % kMtN], mt[t - kMtM]);
            __syncthreads();
            if (t >= kMtM && t < kMtN) mt[t] = v;
            __syncthreads();
            idx = 0;
        }
        const uint32_t take = min(total - done, (uint32_t)kMtN - idx);
        if ((uint32_t)t < take) out[done + t] = mt_temper(mt[idx + t]);
        done += take;
        idx += take;
    }
    __syncthreads();
    if (t < kMtN) g->mt[t] = mt[t];
    if (t == 0) g->idx = idx;
}

// 4. draws: the last writer of each slot that drew 0 (64-bit atomicMax of
// (pass << 32) | (j + 1): no per-pass reset)
__global__ void arb_draw_kernel(const uint32_t* __restrict__ count, const uint32_t* __restrict__ rank_of,
                                const uint32_t* __restrict__ draw_at, const uint64_t* __restrict__ outputs,
                                const uint32_t* __restrict__ leader_of, uint32_t pass,
                                unsigned long long* __restrict__ last_zero, uint32_t* __restrict__ rejected,
                                int force_replay) {
    const uint32_t m = *count;
    if (force_replay && blockIdx.x == 0 && threadIdx.x == 0) atomicOr(rejected, 1u);
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
        const uint32_t c = rank_of[j];
        if (c < 2) continue;
        uint32_t pick;
        if (!lemire_accepts(outputs[draw_at[j]], c, &pick)) {
            atomicOr(rejected, 1u);
            continue;
        }
        if (pick == 0) atomicMax(&last_zero[leader_of[j]], ((unsigned long long)pass << 32) | (j + 1));
    }
}

// 5. every split state moves to its slot's winner (skipped when a draw was
// rejected: the replay kernel does the pass then)
__global__ void arb_move_kernel(const uint32_t* __restrict__ count, const uint32_t* __restrict__ list,
                                const uint32_t* __restrict__ leader_of, const uint32_t* __restrict__ first_q,
                                const unsigned long long* __restrict__ last_zero, uint32_t pass,
                                const uint32_t* __restrict__ rejected, uint32_t* __restrict__ lab) {
    if (*rejected) return;
    const uint32_t m = *count;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
        const uint32_t L = leader_of[j];
        const unsigned long long z = last_zero[L];
        lab[list[j]] = (uint32_t)(z >> 32) == pass && (uint32_t)z ? list[(uint32_t)z - 1] : first_q[L];
    }
}

// the exact sequential pass from the pre-pass engine state (rejections)
__global__ void arb_replay_kernel(const uint32_t* __restrict__ count, const uint32_t* __restrict__ list,
                                  const uint32_t* __restrict__ leader_of, const uint32_t* __restrict__ rank_of,
                                  const MtState* __restrict__ snap, MtState* __restrict__ g,
                                  uint32_t* __restrict__ winner, const uint32_t* __restrict__ rejected,
                                  uint32_t* __restrict__ lab) {
    if (!*rejected || threadIdx.x != 0 || blockIdx.x != 0) return;
    MtState st = *snap;
    const uint32_t m = *count;
    for (uint32_t j = 0; j < m; ++j) {
        const uint32_t c = rank_of[j], L = leader_of[j];
        if (c == 1) {
            winner[L] = list[j];
            continue;
        }
        uint32_t pick;
        while (!lemire_accepts(mt_next_seq(st), c, &pick)) {
        }
        if (pick == 0) winner[L] = list[j];
    }
    for (uint32_t j = 0; j < m; ++j) lab[list[j]] = winner[leader_of[j]];
    *g = st;
}

}  // namespace

// naive_pr(dfa, ElectionPolicy::arbitrary(seed)), exact reference semantics.
RefineResult naive_pr_arbitrary_device(Ctx* ctx, const DevDfa& d, uint64_t seed, uint32_t* block_out,
                                       cudaStream_t s) {
    const uint32_t n = d.n;
    RefineResult res;
    if (n == 0) return res;
    LeaderInfo li = leader_info(ctx, d, s);
    if (li.min_acc == kNone || li.min_rej == kNone) {
        DK_CUDA(cudaMemsetAsync(block_out, 0, (size_t)n * sizeof(uint32_t), s));
        res.num_blocks = 1;
        return res;
    }
    DBuf<uint32_t> lab(n, s), list(n, s), leader_of(n, s), rank_of(n, s), nonfirst(n, s), draw_at(n, s),
        run_start(n, s), first_q(n, s), winner(n, s), vals0(n, s), vals1(n, s), scratch((uint64_t)n + 1, s);
    DBuf<uint32_t> words(4, s);  // {split count, draws, rejected, -}
    DBuf<uint64_t> keys0(n, s), keys1(n, s), outputs(n, s);
    DBuf<uint8_t> flag(n, s);
    DBuf<unsigned long long> last_zero(n, s);
    DBuf<MtState> eng(1, s), snap(1, s);
    DK_CUDA(cudaMemsetAsync(last_zero.get(), 0, (size_t)n * 8, s));
    DK_CUDA(cudaMemsetAsync(words.get(), 0, 16, s));
    {
        // std::mt19937_64(seed): mt[0] = seed, mt[i] = f * (mt[i-1] ^ mt[i-1] >> 62) + i
        MtState h{};
        h.mt[0] = seed;
        for (int i = 1; i < kMtN; ++i) h.mt[i] = 6364136223846793005ull * (h.mt[i - 1] ^ (h.mt[i - 1] >> 62)) + i;
        h.idx = kMtN;
        DK_CUDA(cudaMemcpyAsync(eng.get(), &h, sizeof(h), cudaMemcpyHostToDevice, s));
        DK_CUDA(cudaStreamSynchronize(s));  // h is a stack object
    }
    init_leader_labels(ctx, d, li, lab.get(), s);
    uint32_t* cnt = words.get();
    uint32_t* draws = words.get() + 1;
    uint32_t* rejected = words.get() + 2;
    const unsigned g = grid_for(n);
    // test hook: every pass through the sequential replay kernel (the path a
    // rejected draw takes), which must give the same winners
    const int force_replay = getenv("DFAKIT_TEST_ARB_REPLAY") != nullptr;
    uint32_t bits = 1;
    while (bits < 32 && (1ull << bits) < n) ++bits;
    for (uint32_t pass = 1;; ++pass) {
        ++res.passes;
        DK_LAUNCH(ctx, arb_split_flags_kernel, g, kThreads, 0, s, d.delta, n, d.k, lab.get(), flag.get());
        compact_flags(ctx, nullptr, flag.get(), n, list.get(), cnt, s);
        uint32_t m = 0;
        read_words(ctx, cnt, 4, &m, s);
        if (m == 0) break;
        ++res.iters;
        const unsigned gm = grid_for(m);
        DK_LAUNCH(ctx, arb_keys_kernel, gm, kThreads, 0, s, list.get(), cnt, lab.get(), keys0.get(), vals0.get(),
                  leader_of.get());
        RadixBuffers rb{keys0.get(), vals0.get(), keys1.get(), vals1.get()};
        const bool flipped = radix_sort_pairs(ctx, rb, m, bits, s);  // stable: positions stay increasing per slot
        const uint64_t* sk = flipped ? keys1.get() : keys0.get();
        const uint32_t* sv = flipped ? vals1.get() : vals0.get();
        DK_LAUNCH(ctx, arb_heads_kernel, gm, kThreads, 0, s, sk, sv, cnt, list.get(), run_start.get(), first_q.get());
        DK_LAUNCH(ctx, arb_rank_kernel, gm, kThreads, 0, s, sk, sv, cnt, run_start.get(), rank_of.get(),
                  nonfirst.get());
        exclusive_scan_u32(ctx, nonfirst.get(), draw_at.get(), m, draws, s);
        DK_LAUNCH(ctx, arb_mt_kernel, 1, kMtThreads, 0, s, eng.get(), snap.get(), draws, outputs.get());
        DK_LAUNCH(ctx, arb_draw_kernel, gm, kThreads, 0, s, cnt, rank_of.get(), draw_at.get(), outputs.get(),
                  leader_of.get(), pass, last_zero.get(), rejected, force_replay);
        DK_LAUNCH(ctx, arb_move_kernel, gm, kThreads, 0, s, cnt, list.get(), leader_of.get(), first_q.get(),
                  last_zero.get(), pass, rejected, lab.get());
        DK_LAUNCH(ctx, arb_replay_kernel, 1, 32, 0, s, cnt, list.get(), leader_of.get(), rank_of.get(), snap.get(),
                  eng.get(), winner.get(), rejected, lab.get());
        DK_CUDA(cudaMemsetAsync(rejected, 0, 4, s));
    }
    // arbitrary winners are not block minima: canonical numbering from any labels
    min_state_labels(ctx, lab.get(), n, scratch.get(), s);
    res.num_blocks = canonical_from_min_labels(ctx, lab.get(), n, block_out, scratch.get(), s);
    return res;
}

}  // namespace dk
