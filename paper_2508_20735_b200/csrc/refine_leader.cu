// refine_leader.cu -- leader-election refinement (paper Alg. 2 / Alg. 3,
// reference src/minimize.cpp:214-348) and the partial transitive closure
// (Alg. 5, src/minimize.cpp:425-478), re-designed for B200.
//
// Election slots are 64-bit words  (epoch << 32) | priority  updated with
// atomicMin.  The epoch field is ~pass, so a slot written in an earlier pass
// always compares larger and is overwritten without any reset kernel.  With
// priority = q the winner is the minimum split state of the block -- the
// reference's min_index policy exactly, so pass counts match bit for bit.
// arbitrary(seed) uses a seeded per-pass bijection of q as priority (a
// deterministic model of the CRCW arbitrary winner).
#include "prims.cuh"
#include "refine.cuh"

namespace dk {

namespace {

constexpr uint32_t kPending = 0x80000000u;

// priority of a candidate: identity for min_index, a seeded bijection of
// 32-bit words (xor, odd multiply, xorshift -- each step invertible) for
// arbitrary(seed)
struct Prio {
    uint32_t salt, mul, mul_inv, ident;
    __host__ __device__ uint32_t enc(uint32_t q) const {
        if (ident) return q;
        uint32_t x = (q ^ salt) * mul;
        return x ^ (x >> 16);
    }
    __host__ __device__ uint32_t dec(uint32_t x) const {
        if (ident) return x;
        x ^= x >> 16;
        return (x * mul_inv) ^ salt;
    }
};

uint32_t inverse_odd(uint32_t a) {  // a * inv == 1 (mod 2^32), Newton iteration
    uint32_t x = a;
    for (int i = 0; i < 5; ++i) x *= 2u - a * x;
    return x;
}

Prio make_prio(int policy, uint64_t seed, uint64_t pass) {
    if (policy == DFAKIT_POLICY_MIN_INDEX) return {0u, 1u, 1u, 1u};
    uint64_t h = mix64(seed * 0x9E3779B97F4A7C15ull + pass);
    uint32_t mul = (uint32_t)(h >> 32) | 1u;
    return {(uint32_t)h, mul, inverse_odd(mul), 0u};
}

// Alg. 2 l.9-11: split test against the leader + election.
__global__ void __launch_bounds__(kThreads) elect_kernel(const uint32_t* __restrict__ delta, uint32_t n, uint32_t k,
                                                         const uint32_t* __restrict__ lab,
                                                         unsigned long long* __restrict__ slot, uint32_t epoch, Prio pr,
                                                         uint32_t* __restrict__ split_list,
                                                         uint32_t* __restrict__ split_count) {
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        const uint32_t L = lab[q];
        bool split = false;
        if (L != q) {
            for (uint32_t a = 0; a < k; ++a) {
                const uint32_t* row = delta + (uint64_t)a * n;
                if (lab[ld_stream(row + q)] != lab[row[L]]) {
                    split = true;
                    break;
                }
            }
        }
        if (split) atomicMin(&slot[L], ((unsigned long long)epoch << 32) | pr.enc(q));
        uint32_t at = warp_append(split_count, split);
        if (split) split_list[at] = q;
    }
}

// Alg. 2 l.12-14: every split state follows its block's elected leader.
__global__ void follow_kernel(const uint32_t* __restrict__ split_list, uint32_t cnt, uint32_t* __restrict__ lab,
                              const unsigned long long* __restrict__ slot, Prio pr) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
        const uint32_t q = split_list[i];
        lab[q] = pr.dec((uint32_t)slot[lab[q]]);
    }
}

// Alg. 3: election and reassignment in one pass.  Reads the pass-start
// labels (cur), writes next; a split state records "pending on slot L" and
// the winner is resolved when the label is next read (slots of the previous
// pass are final by then).
__device__ __forceinline__ uint32_t resolve(uint32_t v, const unsigned long long* __restrict__ prev_slot) {
    return (v & kPending) ? (uint32_t)prev_slot[v & ~kPending] : v;
}

__global__ void __launch_bounds__(kThreads) fused_kernel(const uint32_t* __restrict__ delta, uint32_t n, uint32_t k,
                                                         const uint32_t* __restrict__ cur, uint32_t* __restrict__ next,
                                                         const unsigned long long* __restrict__ prev_slot,
                                                         unsigned long long* __restrict__ slot, uint32_t epoch,
                                                         uint32_t* __restrict__ split_count) {
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        const uint32_t L = resolve(cur[q], prev_slot);
        bool split = false;
        if (L != q) {
            for (uint32_t a = 0; a < k; ++a) {
                const uint32_t* row = delta + (uint64_t)a * n;
                if (resolve(cur[ld_stream(row + q)], prev_slot) != resolve(cur[row[L]], prev_slot)) {
                    split = true;
                    break;
                }
            }
        }
        if (split) {
            atomicMin(&slot[L], ((unsigned long long)epoch << 32) | q);
            next[q] = kPending | L;
        } else {
            next[q] = L;
        }
        unsigned sm = __ballot_sync(__activemask(), split);
        if (sm && (threadIdx.x & 31u) == (unsigned)(__ffs(sm) - 1)) atomicAdd(split_count, (uint32_t)__popc(sm));
    }
}

__global__ void resolve_all_kernel(uint32_t* __restrict__ lab, uint32_t n,
                                   const unsigned long long* __restrict__ prev_slot) {
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x)
        lab[q] = resolve(lab[q], prev_slot);
}

// Alg. 5 l.7: delta^T(q, a^(2^i)) = delta^T(delta^T(q, a^(2^(i-1))), a^(2^(i-1)))
__global__ void double_kernel(uint32_t* __restrict__ out, uint32_t n, uint32_t k, uint32_t levels, uint32_t level) {
    const uint64_t total = (uint64_t)k * n;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t a = (uint32_t)(t / n), q = (uint32_t)(t % n);
        const uint32_t* prev = out + ((uint64_t)a * levels + level - 1) * n;
        out[((uint64_t)a * levels + level) * n + q] = prev[prev[q]];
    }
}

RefineResult single_block(Ctx* ctx, uint32_t n, uint32_t* block_out, cudaStream_t s) {
    RefineResult r;
    if (n) DK_CUDA(cudaMemsetAsync(block_out, 0, (size_t)n * sizeof(uint32_t), s));
    r.num_blocks = n ? 1 : 0;
    return r;
}

}  // namespace

uint32_t floor_log2_u32(uint32_t n) {
    uint32_t r = 0;
    if (n <= 1) return 0;
    while (n >>= 1) ++r;
    return r;
}

RefineResult naive_pr_device(Ctx* ctx, const DevDfa& d, int policy, uint64_t seed, uint32_t* block_out,
                             cudaStream_t s) {
    const uint32_t n = d.n;
    if (n == 0) return RefineResult{};
    LeaderInfo li = leader_info(ctx, d, s);
    if (li.min_acc == kNone || li.min_rej == kNone) return single_block(ctx, n, block_out, s);
    RefineResult res;
    DBuf<uint32_t> lab(n, s), split(n, s), scratch((uint64_t)n + 1, s);
    DBuf<unsigned long long> slot(n, s);
    DBuf<uint32_t> cnt(1, s);
    DK_CUDA(cudaMemsetAsync(slot.get(), 0xff, (size_t)n * sizeof(unsigned long long), s));
    init_leader_labels(ctx, d, li, lab.get(), s);
    const unsigned g = grid_for(n);
    for (uint64_t pass = 0;; ++pass) {
        ++res.passes;
        const Prio pr = make_prio(policy, seed, pass);
        const uint32_t epoch = 0xffffffffu - (uint32_t)pass;
        DK_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(uint32_t), s));
        DK_LAUNCH_B(ctx, (8.0 + 8.0 * d.k) * n, elect_kernel, g, kThreads, 0, s, d.delta, n, d.k, lab.get(), slot.get(), epoch, pr, split.get(),
                  cnt.get());
        uint32_t c = 0;
        read_words(ctx, cnt.get(), sizeof(c), &c, s);
        if (c == 0) break;
        ++res.iters;
        DK_LAUNCH(ctx, follow_kernel, grid_for(c), kThreads, 0, s, split.get(), c, lab.get(), slot.get(), pr);
    }
    // min_index leaders are always block minima; arbitrary winners are not
    if (policy != DFAKIT_POLICY_MIN_INDEX) min_state_labels(ctx, lab.get(), n, scratch.get(), s);
    res.num_blocks = canonical_from_min_labels(ctx, lab.get(), n, block_out, scratch.get(), s);
    return res;
}

RefineResult naive_pr_fused_device(Ctx* ctx, const DevDfa& d, uint32_t* block_out, cudaStream_t s) {
    const uint32_t n = d.n;
    if (n == 0) return RefineResult{};
    if (n >= kPending) throw Error(DFAKIT_E_RESOURCE, "naive_pr_fused: at most 2^31-1 states");
    LeaderInfo li = leader_info(ctx, d, s);
    if (li.min_acc == kNone || li.min_rej == kNone) return single_block(ctx, n, block_out, s);
    RefineResult res;
    DBuf<uint32_t> lab0(n, s), lab1(n, s), scratch((uint64_t)n + 1, s);
    DBuf<unsigned long long> slot0(n, s), slot1(n, s);
    DBuf<uint32_t> cnt(1, s);
    DK_CUDA(cudaMemsetAsync(slot0.get(), 0xff, (size_t)n * sizeof(unsigned long long), s));
    DK_CUDA(cudaMemsetAsync(slot1.get(), 0xff, (size_t)n * sizeof(unsigned long long), s));
    init_leader_labels(ctx, d, li, lab0.get(), s);
    uint32_t *cur = lab0.get(), *next = lab1.get();
    unsigned long long *prev_slot = slot1.get(), *slot = slot0.get();
    const unsigned g = grid_for(n);
    for (uint64_t pass = 0;; ++pass) {
        ++res.passes;
        const uint32_t epoch = 0xffffffffu - (uint32_t)pass;
        DK_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(uint32_t), s));
        DK_LAUNCH_B(ctx, (12.0 + 8.0 * d.k) * n, fused_kernel, g, kThreads, 0, s, d.delta, n, d.k, cur, next, prev_slot, slot, epoch, cnt.get());
        uint32_t c = 0;
        read_words(ctx, cnt.get(), sizeof(c), &c, s);
        std::swap(cur, next);
        std::swap(prev_slot, slot);
        if (c == 0) break;
        ++res.iters;
    }
    // the confirming pass wrote no pending labels; resolve defensively
    DK_LAUNCH(ctx, resolve_all_kernel, g, kThreads, 0, s, cur, n, prev_slot);
    res.num_blocks = canonical_from_min_labels(ctx, cur, n, block_out, scratch.get(), s);
    return res;
}

void transitive_alphabet_device(Ctx* ctx, const DevDfa& d, uint32_t* out, cudaStream_t s) {
    const uint32_t n = d.n, k = d.k, levels = floor_log2_u32(n) + 1;
    for (uint32_t a = 0; a < k; ++a)
        DK_CUDA(cudaMemcpyAsync(out + (uint64_t)a * levels * n, d.delta + (uint64_t)a * n, (size_t)n * sizeof(uint32_t),
                                cudaMemcpyDeviceToDevice, s));
    for (uint32_t lv = 1; lv < levels; ++lv)
        DK_LAUNCH_B(ctx, 12.0 * k * n, double_kernel, grid_for((uint64_t)k * n), kThreads, 0, s, out, n, k, levels, lv);
}

RefineResult trans_pr_device(Ctx* ctx, const DevDfa& d, int policy, uint64_t seed, uint64_t max_transitions,
                             uint32_t* block_out, cudaStream_t s) {
    const uint32_t levels = floor_log2_u32(d.n) + 1;
    const uint64_t total = (uint64_t)d.k * levels * d.n;
    if (total > max_transitions)
        throw Error(DFAKIT_E_RESOURCE, "build_transitive_alphabet: doubled alphabet needs " + std::to_string(total) +
                                           " transition entries; budget is " + std::to_string(max_transitions));
    if ((uint64_t)d.k * levels > 0xffffffffull) throw Error(DFAKIT_E_RESOURCE, "doubled alphabet too large");
    DBuf<uint32_t> closed(total, s);
    transitive_alphabet_device(ctx, d, closed.get(), s);
    DevDfa c = d;
    c.k = d.k * levels;
    c.delta = closed.get();
    RefineResult r = naive_pr_device(ctx, c, policy, seed, block_out, s);
    r.closure = floor_log2_u32(d.n);
    return r;
}

}  // namespace dk
