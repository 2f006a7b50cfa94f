// refine_leader.cu -- leader-election refinement (paper Alg. 2 / Alg. 3,
// reference src/minimize.cpp:214-348) and the partial transitive closure
// (Alg. 5, src/minimize.cpp:425-478), re-designed for B200.
//
// Election slots are 64-bit words  (epoch << 32) | priority  updated with
// atomicMin.  The epoch field is ~pass, so a slot written in an earlier pass
// always compares larger and is overwritten without any reset kernel.  With
// priority = q the winner is the minimum split state of the block -- the
// reference's min_index policy exactly, so pass counts match bit for bit.
// ElectionPolicy::arbitrary(seed) does not come here: refine_arbitrary.cu
// reproduces the reference's mt19937_64 winner stream exactly.  The kernels
// keep their priority hook (Prio; identity for min_index): without it the
// persistent kernel measured slower (10M chain trans_pr 8.25 -> 10.8 ms, a
// scheduling effect of the simpler code), so it stays as a generic
// "order the candidates by" parameter.
#include <cooperative_groups.h>

#include "prims.cuh"
#include "refine.cuh"

namespace cg = cooperative_groups;

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

__host__ __device__ uint32_t inverse_odd(uint32_t a) {  // a * inv == 1 (mod 2^32), Newton iteration
    uint32_t x = a;
    for (int i = 0; i < 5; ++i) x *= 2u - a * x;
    return x;
}

__host__ __device__ Prio make_prio(int policy, uint64_t seed, uint64_t pass) {
    if (policy == DFAKIT_POLICY_MIN_INDEX) return {0u, 1u, 1u, 1u};
    uint64_t h = mix64(seed * 0x9E3779B97F4A7C15ull + pass);
    uint32_t mul = (uint32_t)(h >> 32) | 1u;
    return {(uint32_t)h, mul, inverse_odd(mul), 0u};
}

// Alg. 3: election and reassignment in one pass.  Reads the pass-start
// labels (cur), writes next; a split state records "pending on slot L" and
// the winner is resolved when the label is next read (slots of the previous
// pass are final by then).
__device__ __forceinline__ uint32_t resolve(uint32_t v, const unsigned long long* __restrict__ prev_slot) {
    return (v & kPending) ? (uint32_t)prev_slot[v & ~kPending] : v;
}

__global__ void resolve_all_kernel(uint32_t* __restrict__ lab, uint32_t n,
                                   const unsigned long long* __restrict__ prev_slot) {
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x)
        lab[q] = resolve(lab[q], prev_slot);
}

// ---- persistent variants ---------------------------------------------------------
//
// The whole refinement in ONE cooperative launch: every CTA is resident, the
// passes are separated by grid-wide barriers and the split count is read
// from global memory by every thread, so a pass costs two barriers instead
// of a host round trip (memset + launch + readback + launch).  Counters are
// double-buffered by pass parity; the CTA that resets the next pass's counter
// does so while nobody reads it.

struct PersistOut {
    uint32_t passes, iters;
};

// Does q differ from its leader L on some letter?  Loads of a chunk of C
// letters are issued together (delta rows of q and L, then the labels), so
// a thread waits on two memory latencies per chunk, not per letter; the
// early exit is per chunk.  lab_of maps a stored label to the current one.
// STREAM: delta rows are read once per pass with evict-first loads (large
// automata); the single-CTA kernels re-read them every pass from L1 / shared
// memory instead.
template <typename F, bool STREAM = true, int C = 8>
__device__ __forceinline__ bool differs_from_leader(uint32_t q, uint32_t L, const uint32_t* __restrict__ delta,
                                                    uint32_t n, uint32_t k, const uint32_t* lab, F lab_of) {
    for (uint32_t a = 0; a < k; a += C) {
        uint32_t tq[C], tl[C];
#pragma unroll
        for (int j = 0; j < C; ++j)
            if (a + j < k) {
                const uint32_t* row = delta + (uint64_t)(a + j) * n;
                tq[j] = STREAM ? ld_stream(row + q) : row[q];
                tl[j] = row[L];
            }
#pragma unroll
        for (int j = 0; j < C; ++j)
            if (a + j < k) {
                tq[j] = lab[tq[j]];
                tl[j] = lab[tl[j]];
            }
        bool diff = false;
#pragma unroll
        for (int j = 0; j < C; ++j)
            if (a + j < k) diff |= lab_of(tq[j]) != lab_of(tl[j]);
        if (diff) return true;
    }
    return false;
}

// Election write of one warp: split lanes with the same leader L combine
// their priorities (match_any + reduce_min) and one of them issues the
// atomicMin.  On a chain every state of a warp shares its leader, and
// without the combine the whole block's split states hammered one slot
// (same-address atomics serialise at L2).  A plain reduction measured better
// than reading the slot first to skip it (chain 12.6 -> 12.5 ms, 100K x 10
// naive 456 -> 429 ms, fused 294 -> 274 ms).  All 32 lanes must call it.
__device__ __forceinline__ void elect(unsigned long long* __restrict__ slot, uint32_t L, uint32_t epoch, uint32_t prio,
                                      bool split) {
    const unsigned sm = __ballot_sync(0xffffffffu, split);
    if (!split) return;
    const unsigned peers = __match_any_sync(sm, L);
    const uint32_t best = __reduce_min_sync(peers, prio);
    if (lane_id() == (unsigned)(__ffs(peers) - 1)) {
        const unsigned long long v = ((unsigned long long)epoch << 32) | best;
        atomicMin(&slot[L], v);  // result unused: a fire-and-forget reduction
    }
}

// Alg. 2 (naive_pr): elect, barrier, follow, barrier.  Every CTA appends its
// split states to its own segment of split_list (seg entries, shared-memory
// cursor: a global cursor serialised 10^5 -- 10^6 warp atomics per pass on
// large automata) and adds its count to the pass counter once; in the follow
// phase each CTA relabels its own segment.
template <int C>
__global__ void __launch_bounds__(kThreads)
    naive_persistent_kernel(const uint32_t* __restrict__ delta, uint32_t n, uint32_t k, uint32_t* __restrict__ lab,
                            unsigned long long* __restrict__ slot, uint32_t* __restrict__ split_list,
                            uint32_t* __restrict__ cnt, int policy, uint64_t seed, PersistOut* __restrict__ out) {
    __shared__ uint32_t cta_cnt[2];
    __shared__ uint32_t s_total;
    auto sync_all = [] { cg::this_grid().sync(); };
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    const uint32_t seg = (n + stride - 1) / stride * blockDim.x;
    uint32_t* my_list = split_list + (uint64_t)blockIdx.x * seg;
    if (threadIdx.x == 0) cta_cnt[0] = 0;
    __syncthreads();
    uint64_t pass = 0;
    for (;; ++pass) {
        const Prio pr = make_prio(policy, seed, pass);
        const uint32_t epoch = 0xffffffffu - (uint32_t)pass;
        uint32_t* c = cnt + (pass & 1);
        uint32_t* cc = cta_cnt + (pass & 1);
        if (threadIdx.x == 0) cta_cnt[(pass + 1) & 1] = 0;
        for (uint32_t q0 = blockIdx.x * blockDim.x; q0 < n; q0 += stride) {
            const uint32_t q = q0 + threadIdx.x;
            const uint32_t L = q < n ? lab[q] : q;
            auto ident = [](uint32_t v) { return v; };
            const bool split =
                L != q && differs_from_leader<decltype(ident), true, C>(q, L, delta, n, k, lab, ident);
            elect(slot, L, epoch, split ? pr.enc(q) : 0u, split);
            const uint32_t at = warp_append(cc, split);
            if (split) my_list[at] = q;
        }
        __syncthreads();
        const uint32_t mine = *(volatile uint32_t*)cc;
        if (threadIdx.x == 0 && mine) atomicAdd(c, mine);
        sync_all();
        // one read per CTA, shared through shared memory: every thread
        // reading the counter put thousands of warp requests on one L2 slice
        if (threadIdx.x == 0) s_total = *(volatile uint32_t*)c;
        __syncthreads();
        const uint32_t total = s_total;
        if (total == 0) break;
        if (tid == 0) cnt[(pass + 1) & 1] = 0;
        for (uint32_t i = threadIdx.x; i < mine; i += blockDim.x) {
            const uint32_t q = my_list[i];
            lab[q] = pr.dec((uint32_t)slot[lab[q]]);
        }
        sync_all();
    }
    if (tid == 0) *out = PersistOut{(uint32_t)(pass + 1), (uint32_t)pass};
}

// Alg. 3 (naive_pr_fused): one barrier per pass; labels ping-pong.  cnt: 3 words.
// Two letters per load chunk, as the persistent naive kernel (100K x 10:
// 320 -> 293 ms against 8).
constexpr int kFusedChunk = 2;
__global__ void __launch_bounds__(kThreads) fused_persistent_kernel(const uint32_t* __restrict__ delta, uint32_t n,
                                                                    uint32_t k, uint32_t* __restrict__ lab0,
                                                                    uint32_t* __restrict__ lab1,
                                                                    unsigned long long* __restrict__ slot0,
                                                                    unsigned long long* __restrict__ slot1,
                                                                    uint32_t* __restrict__ cnt,
                                                                    PersistOut* __restrict__ out) {
    __shared__ uint32_t red[kThreads / 32];
    __shared__ uint32_t s_total;
    cg::grid_group grid = cg::this_grid();
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    uint64_t pass = 0;
    for (;; ++pass) {
        const uint32_t* cur = (pass & 1) ? lab1 : lab0;
        uint32_t* next = (pass & 1) ? lab0 : lab1;
        const unsigned long long* prev_slot = (pass & 1) ? slot0 : slot1;
        unsigned long long* slot = (pass & 1) ? slot1 : slot0;
        const uint32_t epoch = 0xffffffffu - (uint32_t)pass;
        // three counters: the one of pass p - 1 may still be read by threads
        // leaving barrier p - 1; the one of pass p - 2 is free
        uint32_t* c = cnt + (pass % 3);
        if (tid == 0) cnt[(pass + 1) % 3] = 0;
        uint32_t splits = 0;
        for (uint32_t q0 = blockIdx.x * blockDim.x; q0 < n; q0 += stride) {
            const uint32_t q = q0 + threadIdx.x;
            const uint32_t L = q < n ? resolve(cur[q], prev_slot) : q;
            auto lab_of = [&](uint32_t v) { return resolve(v, prev_slot); };
            const bool split =
                L != q && differs_from_leader<decltype(lab_of), true, kFusedChunk>(q, L, delta, n, k, cur, lab_of);
            elect(slot, L, epoch, q, split);
            if (q < n) next[q] = split ? (kPending | L) : L;
            splits += split;
        }
        // one counter atomic per CTA
        splits = __reduce_add_sync(0xffffffffu, splits);
        if (lane_id() == 0) red[threadIdx.x >> 5] = splits;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t t = 0;
            for (int w = 0; w < kThreads / 32; ++w) t += red[w];
            if (t) atomicAdd(c, t);
        }
        grid.sync();
        if (threadIdx.x == 0) s_total = *(volatile uint32_t*)c;  // one read per CTA
        __syncthreads();
        if (s_total == 0) break;
    }
    if (tid == 0) *out = PersistOut{(uint32_t)(pass + 1), (uint32_t)pass};
}

// ---- single-CTA variants ---------------------------------------------------------
//
// Small automata with many passes (the Fibonacci family: one split per pass)
// spend a persistent kernel's time in grid barriers (~2 us each).  When the
// pass state fits one SM's shared memory and a pass is little work
// (n * k <= kOneWork), one CTA of 1024 threads runs every pass with
// __syncthreads between phases: labels, election slots and the split list
// live in shared memory, delta too when it fits (else L1-cached loads).

constexpr int kOneThreads = 1024;
constexpr uint64_t kOneWork = 1u << 16;     // n * k per pass
constexpr size_t kOneSmem = 227 * 1024;     // opt-in shared memory per CTA
constexpr size_t kOneMisc = 64 * sizeof(uint32_t);

__device__ __forceinline__ const uint32_t* stage_delta(const uint32_t* delta_g, uint32_t n, uint32_t k,
                                                       uint32_t* smem_delta) {
    if (!smem_delta) return delta_g;
    const uint64_t total = (uint64_t)n * k;
    for (uint64_t i = threadIdx.x; i < total; i += blockDim.x) smem_delta[i] = __ldg(delta_g + i);
    return smem_delta;
}

// Split test of R states per thread at once (the single-CTA kernels: few
// states per thread, every load a dependent shared-memory / L1 round trip,
// so the R chains are interleaved instead of run one after another; all k
// letters are compared, n * k is small there).  Bit r of the result: state
// qs[r] (< n) differs from its leader Ls[r] on some letter.
template <int R, typename F>
__device__ __forceinline__ uint32_t batch_differs(const uint32_t (&qs)[R], const uint32_t (&Ls)[R],
                                                  const uint32_t* delta, uint32_t n, uint32_t k, const uint32_t* lab,
                                                  F lab_of) {
    uint32_t dif = 0;
    for (uint32_t a = 0; a < k; ++a) {
        const uint32_t* row = delta + (uint64_t)a * n;
        uint32_t tq[R], tl[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t q = min(qs[r], n - 1), L = min(Ls[r], n - 1);
            tq[r] = row[q];
            tl[r] = row[L];
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            tq[r] = lab[tq[r]];
            tl[r] = lab[tl[r]];
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (lab_of(tq[r]) != lab_of(tl[r])) dif |= 1u << r;
    }
    return dif;
}

constexpr int kOneBatch = 8;  // states per thread per batch

// Alg. 2 in one CTA.  Shared layout: slot[n] (u64), lab[n], split_list[n],
// misc[64] (counters, append scratch), then delta[k * n] when SMEM_DELTA.
template <bool SMEM_DELTA>
__global__ void __launch_bounds__(kOneThreads, 1) naive_one_kernel(const uint32_t* __restrict__ delta_g, uint32_t n,
                                                                   uint32_t k, uint32_t* __restrict__ lab_g,
                                                                   int policy, uint64_t seed,
                                                                   PersistOut* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char one_raw[];
    unsigned long long* slot = reinterpret_cast<unsigned long long*>(one_raw);
    uint32_t* lab = reinterpret_cast<uint32_t*>(slot + n);
    uint32_t* split_list = lab + n;
    uint32_t* misc = split_list + n;  // [0, 1] split counters
    const uint32_t* delta = stage_delta(delta_g, n, k, SMEM_DELTA ? misc + 64 : nullptr);
    for (uint32_t q = threadIdx.x; q < n; q += blockDim.x) {
        slot[q] = ~0ull;
        lab[q] = lab_g[q];
    }
    if (threadIdx.x < 2) misc[threadIdx.x] = 0;
    __syncthreads();
    uint64_t pass = 0;
    for (;; ++pass) {
        const Prio pr = make_prio(policy, seed, pass);
        const uint32_t epoch = 0xffffffffu - (uint32_t)pass;
        uint32_t* c = misc + (pass & 1);
        for (uint32_t q0 = 0; q0 < n; q0 += blockDim.x * kOneBatch) {
            uint32_t qs[kOneBatch], Ls[kOneBatch];
#pragma unroll
            for (int r = 0; r < kOneBatch; ++r) {
                qs[r] = q0 + r * blockDim.x + threadIdx.x;
                Ls[r] = qs[r] < n ? lab[qs[r]] : qs[r];
            }
            const uint32_t dif = batch_differs(qs, Ls, delta, n, k, lab, [](uint32_t v) { return v; });
#pragma unroll
            for (int r = 0; r < kOneBatch; ++r) {
                const bool split = Ls[r] != qs[r] && ((dif >> r) & 1u);
                if (!__any_sync(0xffffffffu, split)) continue;
                elect(slot, Ls[r], epoch, split ? pr.enc(qs[r]) : 0u, split);
                const uint32_t at = warp_append(c, split);
                if (split) split_list[at] = qs[r];
            }
        }
        __syncthreads();
        const uint32_t total = *(volatile uint32_t*)c;
        if (total == 0) break;
        if (threadIdx.x == 0) misc[(pass + 1) & 1] = 0;
        for (uint32_t i = threadIdx.x; i < total; i += blockDim.x) {
            const uint32_t q = split_list[i];
            lab[q] = pr.dec((uint32_t)slot[lab[q]]);
        }
        __syncthreads();
    }
    for (uint32_t q = threadIdx.x; q < n; q += blockDim.x) lab_g[q] = lab[q];
    if (threadIdx.x == 0) *out = PersistOut{(uint32_t)(pass + 1), (uint32_t)pass};
}

// Alg. 3 in one CTA.  Shared layout: slot0[n], slot1[n] (u64), lab0[n],
// lab1[n], misc[64], then delta when SMEM_DELTA.  The final labels are
// resolved in shared memory and written to lab_g.
template <bool SMEM_DELTA>
__global__ void __launch_bounds__(kOneThreads, 1) fused_one_kernel(const uint32_t* __restrict__ delta_g, uint32_t n,
                                                                   uint32_t k, uint32_t* __restrict__ lab_g,
                                                                   PersistOut* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char one_raw[];
    unsigned long long* slot0 = reinterpret_cast<unsigned long long*>(one_raw);
    unsigned long long* slot1 = slot0 + n;
    uint32_t* lab0 = reinterpret_cast<uint32_t*>(slot1 + n);
    uint32_t* lab1 = lab0 + n;
    uint32_t* misc = lab1 + n;
    const uint32_t* delta = stage_delta(delta_g, n, k, SMEM_DELTA ? misc + 64 : nullptr);
    for (uint32_t q = threadIdx.x; q < n; q += blockDim.x) {
        slot0[q] = ~0ull;
        slot1[q] = ~0ull;
        lab0[q] = lab_g[q];
    }
    if (threadIdx.x < 3) misc[threadIdx.x] = 0;
    __syncthreads();
    uint64_t pass = 0;
    for (;; ++pass) {
        const uint32_t* cur = (pass & 1) ? lab1 : lab0;
        uint32_t* next = (pass & 1) ? lab0 : lab1;
        const unsigned long long* prev_slot = (pass & 1) ? slot0 : slot1;
        unsigned long long* slot = (pass & 1) ? slot1 : slot0;
        const uint32_t epoch = 0xffffffffu - (uint32_t)pass;
        uint32_t* c = misc + (pass % 3);
        if (threadIdx.x == 0) misc[(pass + 1) % 3] = 0;
        uint32_t splits = 0;
        auto lab_of = [&](uint32_t v) { return resolve(v, prev_slot); };
        for (uint32_t q0 = 0; q0 < n; q0 += blockDim.x * kOneBatch) {
            uint32_t qs[kOneBatch], Ls[kOneBatch];
#pragma unroll
            for (int r = 0; r < kOneBatch; ++r) {
                qs[r] = q0 + r * blockDim.x + threadIdx.x;
                Ls[r] = qs[r] < n ? resolve(cur[qs[r]], prev_slot) : qs[r];
            }
            const uint32_t dif = batch_differs(qs, Ls, delta, n, k, cur, lab_of);
#pragma unroll
            for (int r = 0; r < kOneBatch; ++r) {
                const bool split = Ls[r] != qs[r] && ((dif >> r) & 1u);
                if (__any_sync(0xffffffffu, split)) elect(slot, Ls[r], epoch, qs[r], split);
                if (qs[r] < n) next[qs[r]] = split ? (kPending | Ls[r]) : Ls[r];
                splits += split;
            }
        }
        splits = __reduce_add_sync(0xffffffffu, splits);
        if (lane_id() == 0 && splits) atomicAdd(c, splits);
        __syncthreads();
        if (*(volatile uint32_t*)c == 0) break;
    }
    // pass p wrote labels (p & 1) ? lab0 : lab1 resolved through slots of pass p
    const uint32_t* fin = (pass & 1) ? lab0 : lab1;
    const unsigned long long* fslot = (pass & 1) ? slot1 : slot0;
    for (uint32_t q = threadIdx.x; q < n; q += blockDim.x) lab_g[q] = resolve(fin[q], fslot);
    if (threadIdx.x == 0) *out = PersistOut{(uint32_t)(pass + 1), (uint32_t)pass};
}

// Single-CTA plan: mode 0 = not applicable, 1 = delta from global (L1),
// 2 = delta in shared memory.  bytes_per_state: the kernel's shared arrays
// per state.  threads: kOneBatch states per thread (fewer threads for small
// n -- idle batch slots still cost shared-memory wavefronts every pass).
struct OnePlan {
    int mode;
    size_t smem;
    unsigned threads;
};
OnePlan one_plan(uint32_t n, uint32_t k, size_t bytes_per_state) {
    if ((uint64_t)n * k > kOneWork) return {0, 0, 0};
    const size_t base = bytes_per_state * n + kOneMisc;
    if (base > kOneSmem) return {0, 0, 0};
    const unsigned threads =
        (unsigned)std::min<uint64_t>(kOneThreads, std::max<uint64_t>(32, ((uint64_t)n + 8 * 32 - 1) / (8 * 32) * 32));
    const size_t with_delta = base + (size_t)4 * n * k;
    if (with_delta <= kOneSmem) return {2, with_delta, threads};
    return {1, base, threads};
}

unsigned coop_grid(Ctx* ctx, const void* kernel, uint32_t n) {
    int per_sm = 0;
    DK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0));
    if (per_sm < 1) throw Error(DFAKIT_E_RESOURCE, "cooperative kernel does not fit an SM");
    // every resident CTA up to one state per thread: a pass is latency-bound
    // (dependent label / delta loads per state), so resident threads beat
    // the cheaper barrier of a smaller grid (100K x 10 naive: 427 ms with one
    // CTA per SM, 336 ms with every SM full)
    const uint64_t need = ((uint64_t)n + kThreads - 1) / kThreads;
    const uint64_t cap = (uint64_t)per_sm * ctx->num_sms;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(need, cap));
}

// Alg. 5 l.7: delta^T(q, a^(2^i)) = delta^T(delta^T(q, a^(2^(i-1))), a^(2^(i-1)))
// (blockIdx.y = letter; no per-element division)
__global__ void double_kernel(uint32_t* __restrict__ out, uint32_t n, uint32_t levels, uint32_t level, uint32_t a0) {
    const uint32_t a = a0 + blockIdx.y;
    const uint32_t* __restrict__ prev = out + ((uint64_t)a * levels + level - 1) * n;
    uint32_t* __restrict__ dst = out + ((uint64_t)a * levels + level) * n;
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x)
        __stcs(dst + q, __ldg(prev + __ldcs(prev + q)));
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
    // arbitrary(seed): the reference's mt19937_64 reservoir sampling, exactly
    // (refine_arbitrary.cu)
    if (policy != DFAKIT_POLICY_MIN_INDEX) return naive_pr_arbitrary_device(ctx, d, seed, block_out, s);
    LeaderInfo li = leader_info(ctx, d, s);
    if (li.min_acc == kNone || li.min_rej == kNone) return single_block(ctx, n, block_out, s);
    RefineResult res;
    DBuf<uint32_t> lab(n, s), split, scratch((uint64_t)n + 1, s);
    DBuf<unsigned long long> slot(n, s);
    DBuf<uint32_t> cnt(2, s);
    DBuf<PersistOut> out(1, s);
    DK_CUDA(cudaMemsetAsync(slot.get(), 0xff, (size_t)n * sizeof(unsigned long long), s));
    DK_CUDA(cudaMemsetAsync(cnt.get(), 0, 2 * sizeof(uint32_t), s));
    init_leader_labels(ctx, d, li, lab.get(), s);
    if (const OnePlan op = one_plan(n, d.k, 16); op.mode) {
        DK_CUDA(cudaFuncSetAttribute(op.mode == 2 ? naive_one_kernel<true> : naive_one_kernel<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)op.smem));
        if (op.mode == 2)
            DK_LAUNCH(ctx, naive_one_kernel<true>, 1, op.threads, op.smem, s, d.delta, n, d.k, lab.get(), policy,
                      seed, out.get());
        else
            DK_LAUNCH(ctx, naive_one_kernel<false>, 1, op.threads, op.smem, s, d.delta, n, d.k, lab.get(), policy,
                      seed, out.get());
        PersistOut o{};
        read_words(ctx, out.get(), sizeof(o), &o, s);
        res.passes = o.passes;
        res.iters = o.iters;
    } else {
        // The persistent kernels test two letters per load chunk (more loads
        // in flight per thread against a later early exit and fewer resident
        // threads; measured on the 10M chain, trans_pr with 24 closure
        // letters: 1 / 2 / 4 / 8 / 16 / 32 letters -> 12.6 / 11.6 / 13.8 /
        // 14.2 / 20.4 / 41.2 ms; 2 letters: 32 registers, full occupancy).
        const void* kern = (const void*)naive_persistent_kernel<2>;
        const unsigned g = coop_grid(ctx, kern, n);
        split.alloc((uint64_t)n + (uint64_t)g * kThreads, s);  // one segment per CTA
        const uint32_t* delta = d.delta;
        uint32_t k = d.k;
        uint32_t* labp = lab.get();
        unsigned long long* slotp = slot.get();
        uint32_t* splitp = split.get();
        uint32_t* cntp = cnt.get();
        PersistOut* outp = out.get();
        uint32_t nn = n;
        void* args[] = {(void*)&delta, (void*)&nn, (void*)&k, (void*)&labp, (void*)&slotp, (void*)&splitp,
                        (void*)&cntp, (void*)&policy, (void*)&seed, (void*)&outp};
        prof_begin_launch(ctx, s);
        DK_CUDA(cudaLaunchCooperativeKernel(kern, g, kThreads, args, 0, s));
        note_launch(ctx);
        prof_end_launch(ctx, s, "naive_persistent_kernel", 0, 0);
        PersistOut o{};
        read_words(ctx, out.get(), sizeof(o), &o, s);
        res.passes = o.passes;
        res.iters = o.iters;
    }
    // min_index leaders are always block minima
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
    DBuf<uint32_t> cnt(3, s);
    DBuf<PersistOut> out(1, s);
    DK_CUDA(cudaMemsetAsync(slot0.get(), 0xff, (size_t)n * sizeof(unsigned long long), s));
    DK_CUDA(cudaMemsetAsync(slot1.get(), 0xff, (size_t)n * sizeof(unsigned long long), s));
    DK_CUDA(cudaMemsetAsync(cnt.get(), 0, 3 * sizeof(uint32_t), s));
    init_leader_labels(ctx, d, li, lab0.get(), s);
    PersistOut o{};
    if (const OnePlan op = one_plan(n, d.k, 24); op.mode) {
        DK_CUDA(cudaFuncSetAttribute(op.mode == 2 ? fused_one_kernel<true> : fused_one_kernel<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)op.smem));
        if (op.mode == 2)
            DK_LAUNCH(ctx, fused_one_kernel<true>, 1, op.threads, op.smem, s, d.delta, n, d.k, lab0.get(), out.get());
        else
            DK_LAUNCH(ctx, fused_one_kernel<false>, 1, op.threads, op.smem, s, d.delta, n, d.k, lab0.get(),
                      out.get());
        read_words(ctx, out.get(), sizeof(o), &o, s);
        res.passes = o.passes;
        res.iters = o.iters;
        res.num_blocks = canonical_from_min_labels(ctx, lab0.get(), n, block_out, scratch.get(), s);
        return res;
    }
    {
        const unsigned g = coop_grid(ctx, (const void*)fused_persistent_kernel, n);
        const uint32_t* delta = d.delta;
        uint32_t k = d.k, nn = n;
        uint32_t *l0 = lab0.get(), *l1 = lab1.get(), *cntp = cnt.get();
        unsigned long long *s0 = slot0.get(), *s1 = slot1.get();
        PersistOut* outp = out.get();
        void* args[] = {(void*)&delta, (void*)&nn, (void*)&k, (void*)&l0, (void*)&l1, (void*)&s0, (void*)&s1,
                        (void*)&cntp, (void*)&outp};
        prof_begin_launch(ctx, s);
        DK_CUDA(cudaLaunchCooperativeKernel((const void*)fused_persistent_kernel, g, kThreads, args, 0, s));
        note_launch(ctx);
        prof_end_launch(ctx, s, "fused_persistent_kernel", 0, 0);
        read_words(ctx, out.get(), sizeof(o), &o, s);
        res.passes = o.passes;
        res.iters = o.iters;
    }
    // pass p read (lab, slot) index p & 1 and wrote index (p + 1) & 1; the
    // last pass is o.passes - 1
    uint32_t* cur = ((o.passes - 1) & 1) ? lab0.get() : lab1.get();
    unsigned long long* prev_slot = ((o.passes - 1) & 1) ? slot1.get() : slot0.get();
    // the confirming pass wrote no pending labels; resolve defensively
    DK_LAUNCH(ctx, resolve_all_kernel, grid_for(n), kThreads, 0, s, cur, n, prev_slot);
    res.num_blocks = canonical_from_min_labels(ctx, cur, n, block_out, scratch.get(), s);
    return res;
}

void transitive_alphabet_device(Ctx* ctx, const DevDfa& d, uint32_t* out, cudaStream_t s) {
    const uint32_t n = d.n, k = d.k, levels = floor_log2_u32(n) + 1;
    for (uint32_t a = 0; a < k; ++a)
        DK_CUDA(cudaMemcpyAsync(out + (uint64_t)a * levels * n, d.delta + (uint64_t)a * n, (size_t)n * sizeof(uint32_t),
                                cudaMemcpyDeviceToDevice, s));
    for (uint32_t lv = 1; lv < levels; ++lv)
        for (uint32_t a0 = 0; a0 < k; a0 += 65535u) {
            const uint32_t ka = std::min(k - a0, 65535u);
            DK_LAUNCH_B(ctx, 12.0 * ka * n, double_kernel, dim3(grid_for(n, kThreads, 148u * 16u), ka), kThreads, 0, s,
                        out, n, levels, lv, a0);
        }
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
