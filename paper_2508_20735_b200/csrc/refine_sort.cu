// refine_sort.cu -- sortPR (reference src/minimize.cpp:354-419, paper Alg. 4)
// re-designed for B200.
//
// Block labels are min-state ids (every block is named by its smallest
// member), so the canonical first-occurrence numbering of the reference's
// Partition::from_labels is one flag+scan away at any time, and a block's
// label never changes unless the block splits.
//
// Only states in non-singleton blocks ("active" states) take part in a pass;
// singleton runs leave the active list for good.  A pass computes, for every
// active state, the key of its (block, signature) tuple -- the block label
// followed by the labels of its successors, letter by letter -- packed into
// 64 bits exactly when the fields fit, otherwise as a 64-bit fingerprint
// whose equal-key runs are verified tuple by tuple (exactness never rests on
// the hash; a verified collision re-runs the pass with a new salt and then
// falls back to exact letter-chunked keys).  States are then grouped by key
// with one of three strategies:
//
//   table      packed keys of <= 20 bits: the signature kernel aggregates a
//              counting table (shared memory when <= 13 bits) -- a one-digit
//              counting sort without the scatter;
//   segmented  wider keys: a stable MSD radix pass over the top 16 key bits
//              in HBM, then one CTA per group of consecutive buckets loads
//              its <= 4096 keys into shared memory, finishes a stable LSD
//              radix sort there, and in the same kernel marks run boundaries
//              (the reference's ARE_NEQ), labels every run with its first
//              (= minimum) state, verifies fingerprint runs, and appends the
//              surviving non-singleton runs to the next active list;
//   global     fallback when a bucket group overflows shared memory: LSD radix
//              sort of the whole key in HBM + boundary / scan / apply kernels.
//
// The fixed-point test of l.19 is the block count: B' = B - A + R where A is
// the number of active blocks and R the number of runs found.
#include <algorithm>

#include "prims.cuh"
#include "refine.cuh"

namespace dk {

namespace {

constexpr uint32_t kTableBits = 20;
constexpr uint32_t kSmemTableBits = 13;
constexpr uint32_t kPrefixBits = 16;

struct IterCounters {
    uint32_t runs;
    uint32_t active_blocks;
    uint32_t active_states;
    uint32_t collision;
    uint32_t max_group;
    uint32_t pad[3];
};

__global__ void leader_info_kernel(const uint8_t* __restrict__ acc, uint32_t n, uint32_t* __restrict__ info) {
    uint32_t mina = kNone, minr = kNone, ca = 0, cr = 0;
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        if (acc[q]) {
            mina = min(mina, q);
            ++ca;
        } else {
            minr = min(minr, q);
            ++cr;
        }
    }
    mina = __reduce_min_sync(0xffffffffu, mina);
    minr = __reduce_min_sync(0xffffffffu, minr);
    ca = __reduce_add_sync(0xffffffffu, ca);
    cr = __reduce_add_sync(0xffffffffu, cr);
    if ((threadIdx.x & 31u) == 0) {
        if (mina != kNone) atomicMin(&info[0], mina);
        if (minr != kNone) atomicMin(&info[1], minr);
        if (ca) atomicAdd(&info[2], ca);
        if (cr) atomicAdd(&info[3], cr);
    }
}

__global__ void init_labels_kernel(const uint8_t* __restrict__ acc, uint32_t n, uint32_t la, uint32_t lr,
                                   uint32_t* __restrict__ lab) {
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x)
        lab[q] = acc[q] ? la : lr;
}

// active = states whose initial block has >= 2 members
__global__ void init_active_flags_kernel(const uint8_t* __restrict__ acc, uint32_t n, uint8_t keep_acc,
                                         uint8_t keep_rej, uint8_t* __restrict__ flag) {
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x)
        flag[q] = acc[q] ? keep_acc : keep_rej;
}

enum : uint32_t { kKeyPacked = 0, kKeyFingerprint = 1 };

struct SigParams {
    uint32_t kind;        // kKeyPacked / kKeyFingerprint
    uint32_t a0, a1;      // letter range of this chunk
    uint32_t field_bits;  // packed: bits per successor field
    uint64_t salt;        // fingerprint salt
    uint64_t fp_mask;     // fingerprint mask (testing hook)
};

__device__ __forceinline__ uint64_t fp_step(uint64_t h, uint32_t x) {
    return mix64(h ^ ((uint64_t)x * 0xD6E8FEB86659FD93ull));
}

__device__ __forceinline__ uint64_t tuple_key(uint32_t q, uint64_t lead, const uint32_t* __restrict__ delta,
                                              uint32_t n, const uint32_t* __restrict__ lab, const SigParams& p) {
    if (p.kind == kKeyPacked) {
        uint64_t key = lead;
        for (uint32_t a = p.a0; a < p.a1; ++a) key = (key << p.field_bits) | lab[ld_stream(delta + (uint64_t)a * n + q)];
        return key;
    }
    uint64_t h = fp_step(p.salt, (uint32_t)lead);
    for (uint32_t a = p.a0; a < p.a1; ++a) h = fp_step(h + a, lab[ld_stream(delta + (uint64_t)a * n + q)]);
    return h & p.fp_mask;
}

// One thread per active state; delta rows are streamed (coalesced when the
// active list is the identity), block labels are gathered (the label array
// stays L2-resident for n <= ~25M).
__global__ void __launch_bounds__(kThreads) signature_kernel(const uint32_t* __restrict__ list, uint64_t m,
                                                             const uint32_t* __restrict__ delta, uint32_t n,
                                                             const uint32_t* __restrict__ lab,
                                                             const uint32_t* __restrict__ head, SigParams p,
                                                             uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t q = list ? list[i] : (uint32_t)i;
        keys[i] = tuple_key(q, head ? head[i] : lab[q], delta, n, lab, p);
        vals[i] = q;
    }
}

// table strategy, step 1: signature + counting table (count, minimum state)
__global__ void __launch_bounds__(512) sig_table_kernel(const uint32_t* __restrict__ list, uint64_t m,
                                                        const uint32_t* __restrict__ delta, uint32_t n,
                                                        const uint32_t* __restrict__ lab, SigParams p, uint32_t nbits,
                                                        uint32_t* __restrict__ keys32, uint32_t* __restrict__ tmin,
                                                        uint32_t* __restrict__ tcnt) {
    extern __shared__ uint32_t st[];  // [tsize] minima, then [tsize] counts (smem mode only)
    const bool local = nbits <= kSmemTableBits;
    const uint32_t tsize = 1u << nbits;
    uint32_t* smin = st;
    uint32_t* scnt = st + tsize;
    if (local) {
        for (uint32_t e = threadIdx.x; e < tsize; e += blockDim.x) {
            smin[e] = kNone;
            scnt[e] = 0;
        }
        __syncthreads();
    }
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t q = list ? list[i] : (uint32_t)i;
        const uint32_t key = (uint32_t)tuple_key(q, lab[q], delta, n, lab, p);
        keys32[i] = key;
        if (local) {
            atomicMin(&smin[key], q);
            atomicAdd(&scnt[key], 1u);
        } else {
            atomicMin(&tmin[key], q);
            atomicAdd(&tcnt[key], 1u);
        }
    }
    if (local) {
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < tsize; e += blockDim.x)
            if (scnt[e]) {
                atomicAdd(&tcnt[e], scnt[e]);
                atomicMin(&tmin[e], smin[e]);
            }
    }
}

// table strategy, step 2: new labels, survivor flags, counters
__global__ void table_apply_kernel(const uint32_t* __restrict__ list, const uint32_t* __restrict__ keys32, uint64_t m,
                                   const uint32_t* __restrict__ tmin, const uint32_t* __restrict__ tcnt,
                                   uint32_t* __restrict__ lab, uint8_t* __restrict__ keep,
                                   IterCounters* __restrict__ ctr) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t key = keys32[i];
        const uint32_t q = list ? list[i] : (uint32_t)i;
        const uint32_t rep = tmin[key];
        const bool multi = tcnt[key] >= 2;
        lab[q] = rep;
        keep[i] = multi;
        const bool head = rep == q;
        unsigned hm = __ballot_sync(__activemask(), head);
        unsigned am = __ballot_sync(__activemask(), head && multi);
        unsigned mm = __ballot_sync(__activemask(), multi);
        if ((threadIdx.x & 31u) == (unsigned)(__ffs(__activemask()) - 1)) {
            if (hm) atomicAdd(&ctr->runs, (uint32_t)__popc(hm));
            if (am) atomicAdd(&ctr->active_blocks, (uint32_t)__popc(am));
            if (mm) atomicAdd(&ctr->active_states, (uint32_t)__popc(mm));
        }
    }
}

// ---- segmented strategy -------------------------------------------------------

constexpr int kSegThreads = 256;
constexpr int kSegWarps = kSegThreads / 32;
constexpr int kSegCap = 4096;
constexpr int kSegPerThread = kSegCap / kSegThreads;   // 16
constexpr int kSegChunks = kSegCap / (kSegWarps * 32);  // 16 chunks of 32 per warp

struct SegSmem {
    unsigned long long k[2][kSegCap];
    uint32_t v[2][kSegCap];
    union {
        uint32_t whist[kSegWarps][256];
        uint32_t run_start[kSegCap + 1];
    } u;
    uint32_t dstart[256];
    uint32_t ws[kSegWarps];
    uint32_t skip;
    uint32_t base;
    uint32_t ablocks;
};

__global__ void prefix_count_kernel(const unsigned long long* __restrict__ keys, uint64_t m, uint32_t shift,
                                    uint32_t* __restrict__ counts) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t b = (uint32_t)(keys[i] >> shift);
        const unsigned peers = __match_any_sync(__activemask(), b);
        if ((threadIdx.x & 31u) == (unsigned)(__ffs(peers) - 1)) atomicAdd(&counts[b], (uint32_t)__popc(peers));
    }
}

__global__ void group_bounds_kernel(const uint32_t* __restrict__ bucket_start, uint32_t buckets, uint32_t per_group,
                                    uint32_t groups, uint64_t m, uint32_t* __restrict__ gstart,
                                    IterCounters* __restrict__ ctr) {
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += gridDim.x * blockDim.x) {
        const uint64_t b0 = (uint64_t)g * per_group, b1 = b0 + per_group;
        const uint32_t s = bucket_start[b0];
        const uint32_t e = b1 >= buckets ? (uint32_t)m : bucket_start[b1];
        gstart[g] = s;
        if (g == groups - 1) gstart[groups] = (uint32_t)m;
        atomicMax(&ctr->max_group, e - s);
    }
}

__device__ __forceinline__ bool same_tuple(uint32_t q, uint32_t r, const uint32_t* __restrict__ delta, uint32_t n,
                                           uint32_t k, const uint32_t* __restrict__ lab) {
    if (lab[q] != lab[r]) return false;
    for (uint32_t a = 0; a < k; ++a) {
        const uint32_t* row = delta + (uint64_t)a * n;
        if (lab[row[q]] != lab[row[r]]) return false;
    }
    return true;
}

__global__ void __launch_bounds__(kSegThreads) segment_refine_kernel(
    const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ vals, const uint32_t* __restrict__ gstart,
    uint32_t low_bits, const uint32_t* __restrict__ delta, uint32_t n, uint32_t k, int fingerprint,
    const uint32_t* __restrict__ lab_in, uint32_t* __restrict__ lab_out, uint32_t* __restrict__ new_list,
    IterCounters* __restrict__ ctr) {
    extern __shared__ __align__(16) unsigned char seg_raw[];
    SegSmem& sm = *reinterpret_cast<SegSmem*>(seg_raw);
    const unsigned tid = threadIdx.x, lane = tid & 31u, wid = tid >> 5;
    const uint32_t s0 = gstart[blockIdx.x];
    const uint32_t len = gstart[blockIdx.x + 1] - s0;
    if (len == 0) return;
    for (uint32_t i = tid; i < len; i += kSegThreads) {
        sm.k[0][i] = __ldcs(keys + s0 + i);
        sm.v[0][i] = __ldcs(vals + s0 + i);
    }
    if (tid == 0) sm.ablocks = 0;
    __syncthreads();

    // stable LSD radix sort of bits [0, low_bits) in shared memory
    int cur = 0;
    const uint32_t span = ((len + kSegWarps * 32 - 1) / (kSegWarps * 32)) * 32;
    const uint32_t nch = span / 32;
    const unsigned lt_mask = (1u << lane) - 1u;
    for (uint32_t shift = 0; shift < low_bits; shift += 8) {
        for (uint32_t i = tid; i < kSegWarps * 256; i += kSegThreads) (&sm.u.whist[0][0])[i] = 0;
        if (tid == 0) sm.skip = 0;
        __syncthreads();
        uint32_t rank[kSegChunks];
#pragma unroll
        for (int c = 0; c < kSegChunks; ++c) {
            rank[c] = 0;
            if ((uint32_t)c < nch) {
                const uint32_t i = wid * span + c * 32 + lane;
                const bool valid = i < len;
                const unsigned vmask = __ballot_sync(0xffffffffu, valid);
                const uint32_t d = valid ? (uint32_t)(sm.k[cur][i] >> shift) & 255u : 0u;
                unsigned peers = 0;
                if (valid) {
                    peers = __match_any_sync(vmask, d);
                    rank[c] = sm.u.whist[wid][d] + (uint32_t)__popc(peers & lt_mask);
                }
                __syncwarp();
                if (valid && lane == (unsigned)(__ffs(peers) - 1)) sm.u.whist[wid][d] += (uint32_t)__popc(peers);
                __syncwarp();
            }
        }
        __syncthreads();
        {
            const uint32_t d = tid;  // kSegThreads == 256 digits
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < kSegWarps; ++w) {
                const uint32_t c = sm.u.whist[w][d];
                sm.u.whist[w][d] = run;
                run += c;
            }
            if (run == len) sm.skip = 1;  // every key has this digit: the pass is the identity
            uint32_t tot;
            sm.dstart[d] = block_exclusive_scan<kSegThreads>(run, &tot, sm.ws);
        }
        __syncthreads();
        if (!sm.skip) {
#pragma unroll
            for (int c = 0; c < kSegChunks; ++c) {
                if ((uint32_t)c < nch) {
                    const uint32_t i = wid * span + c * 32 + lane;
                    if (i < len) {
                        const unsigned long long key = sm.k[cur][i];
                        const uint32_t d = (uint32_t)(key >> shift) & 255u;
                        const uint32_t p = sm.dstart[d] + sm.u.whist[wid][d] + rank[c];
                        sm.k[cur ^ 1][p] = key;
                        sm.v[cur ^ 1][p] = sm.v[cur][i];
                    }
                }
            }
            __syncthreads();
            cur ^= 1;
        }
        __syncthreads();
    }

    // run boundaries, run minima (first element: the sort is stable and the
    // input is increasing within each block), labels, survivors
    const unsigned long long* K = sm.k[cur];
    const uint32_t* V = sm.v[cur];
    const uint32_t b = tid * kSegPerThread;
    uint32_t nheads = 0;
#pragma unroll
    for (int j = 0; j < kSegPerThread; ++j) {
        const uint32_t i = b + j;
        if (i < len && (i == 0 || K[i] != K[i - 1])) ++nheads;
    }
    uint32_t R;
    const uint32_t rbase = block_exclusive_scan<kSegThreads>(nheads, &R, sm.ws);
    {
        uint32_t r = rbase;
#pragma unroll
        for (int j = 0; j < kSegPerThread; ++j) {
            const uint32_t i = b + j;
            if (i < len && (i == 0 || K[i] != K[i - 1])) sm.u.run_start[r++] = i;
        }
        if (tid == 0) sm.u.run_start[R] = len;
    }
    __syncthreads();
    uint32_t survivors = 0, ablk = 0;
    bool clash = false;
    {
        uint32_t r = rbase - 1;  // run of the element before b (if b is not a head)
#pragma unroll
        for (int j = 0; j < kSegPerThread; ++j) {
            const uint32_t i = b + j;
            if (i < len) {
                const bool head = i == 0 || K[i] != K[i - 1];
                if (head) ++r;
                const uint32_t s = sm.u.run_start[r], e = sm.u.run_start[r + 1];
                const bool multi = e - s >= 2;
                lab_out[V[i]] = V[s];
                survivors += multi;
                ablk += head && multi;
                if (fingerprint && !head && !same_tuple(V[i], V[i - 1], delta, n, k, lab_in)) clash = true;
            }
        }
    }
    if (clash) atomicOr(&ctr->collision, 1u);
    if (ablk) atomicAdd(&sm.ablocks, ablk);
    uint32_t stot;
    const uint32_t sbase = block_exclusive_scan<kSegThreads>(survivors, &stot, sm.ws);
    if (tid == 0) {
        sm.base = stot ? atomicAdd(&ctr->active_states, stot) : 0u;
        atomicAdd(&ctr->runs, R);
        if (sm.ablocks) atomicAdd(&ctr->active_blocks, sm.ablocks);
    }
    __syncthreads();
    if (survivors) {
        uint32_t out = sm.base + sbase;
        uint32_t r = rbase - 1;
        for (int j = 0; j < kSegPerThread; ++j) {
            const uint32_t i = b + j;
            if (i >= len) break;
            if (i == 0 || K[i] != K[i - 1]) ++r;
            if (sm.u.run_start[r + 1] - sm.u.run_start[r] >= 2) new_list[out++] = V[i];
        }
    }
}

// ---- warp-per-bucket variant (buckets of <= 256 keys) --------------------------------
//
// Same algorithm as segment_refine_kernel, one warp per MSD bucket, with a
// private 6.6 KB shared-memory slice: no block-wide barriers, 32 warps per
// SM.  Survivors are written inside the bucket's own index range and the
// per-bucket counts are scanned afterwards (no contended atomics).

constexpr int kWarpCap = 256;
constexpr int kWarpChunks = kWarpCap / 32;
constexpr int kWarpsPerCta = 8;

struct WarpSlice {
    unsigned long long k[2][kWarpCap];
    uint32_t v[2][kWarpCap];
    uint32_t hist[256];
    uint32_t run_start[kWarpCap + 1];
};

__global__ void __launch_bounds__(kWarpsPerCta * 32) bucket_refine_kernel(
    const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ vals,
    const uint32_t* __restrict__ bucket_start, uint32_t buckets, uint64_t m, uint32_t low_bits,
    const uint32_t* __restrict__ delta, uint32_t n, uint32_t k, int fingerprint, const uint32_t* __restrict__ lab_in,
    uint32_t* __restrict__ lab_out, uint32_t* __restrict__ tmp_list, uint32_t* __restrict__ surv_count,
    IterCounters* __restrict__ ctr) {
    extern __shared__ __align__(16) unsigned char warp_raw[];
    const unsigned lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    WarpSlice& ws = reinterpret_cast<WarpSlice*>(warp_raw)[wid];
    const unsigned lt_mask = (1u << lane) - 1u;
    bool clash = false;
    uint32_t runs_total = 0, ablk_total = 0;
    for (uint32_t bkt = blockIdx.x * kWarpsPerCta + wid; bkt < buckets; bkt += gridDim.x * kWarpsPerCta) {
        const uint32_t s0 = bucket_start[bkt];
        const uint32_t len = (bkt + 1 < buckets ? bucket_start[bkt + 1] : (uint32_t)m) - s0;
        if (len == 0) {
            if (lane == 0) surv_count[bkt] = 0;
            continue;
        }
        const uint32_t nch = (len + 31) / 32;
#pragma unroll
        for (int c = 0; c < kWarpChunks; ++c) {
            const uint32_t i = c * 32 + lane;
            if (i < len) {
                ws.k[0][i] = __ldcs(keys + s0 + i);
                ws.v[0][i] = __ldcs(vals + s0 + i);
            }
        }
        __syncwarp();
        int cur = 0;
        for (uint32_t shift = 0; shift < low_bits; shift += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) ws.hist[lane * 8 + j] = 0;
            __syncwarp();
            uint32_t rank[kWarpChunks];
#pragma unroll
            for (int c = 0; c < kWarpChunks; ++c) {
                rank[c] = 0;
                if ((uint32_t)c < nch) {
                    const uint32_t i = c * 32 + lane;
                    const bool valid = i < len;
                    const unsigned vmask = __ballot_sync(0xffffffffu, valid);
                    const uint32_t d = valid ? (uint32_t)(ws.k[cur][i] >> shift) & 255u : 0u;
                    unsigned peers = 0;
                    if (valid) {
                        peers = __match_any_sync(vmask, d);
                        rank[c] = ws.hist[d] + (uint32_t)__popc(peers & lt_mask);
                    }
                    __syncwarp();
                    if (valid && lane == (unsigned)(__ffs(peers) - 1)) ws.hist[d] += (uint32_t)__popc(peers);
                    __syncwarp();
                }
            }
            // exclusive scan of the 256 digit counts: 8 consecutive digits per lane
            uint32_t cnt[8], local = 0;
            bool all_one = false;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                cnt[j] = ws.hist[lane * 8 + j];
                all_one |= cnt[j] == len;
                local += cnt[j];
            }
            uint32_t incl = local;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= (unsigned)o) incl += y;
            }
            uint32_t start = incl - local;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                ws.hist[lane * 8 + j] = start;
                start += cnt[j];
            }
            const bool skip = __any_sync(0xffffffffu, all_one);  // one digit holds every key
            __syncwarp();
            if (!skip) {
#pragma unroll
                for (int c = 0; c < kWarpChunks; ++c) {
                    const uint32_t i = c * 32 + lane;
                    if ((uint32_t)c < nch && i < len) {
                        const unsigned long long key = ws.k[cur][i];
                        const uint32_t p = ws.hist[(uint32_t)(key >> shift) & 255u] + rank[c];
                        ws.k[cur ^ 1][p] = key;
                        ws.v[cur ^ 1][p] = ws.v[cur][i];
                    }
                }
                __syncwarp();
                cur ^= 1;
            }
        }
        const unsigned long long* K = ws.k[cur];
        const uint32_t* V = ws.v[cur];
        // runs
        uint32_t R = 0;
        for (uint32_t c = 0; c < nch; ++c) {
            const uint32_t i = c * 32 + lane;
            const bool head = i < len && (i == 0 || K[i] != K[i - 1]);
            const unsigned hm = __ballot_sync(0xffffffffu, head);
            if (head) ws.run_start[R + __popc(hm & lt_mask)] = i;
            R += __popc(hm);
        }
        if (lane == 0) ws.run_start[R] = len;
        __syncwarp();
        uint32_t r = 0, surv = 0, ablk = 0;
        for (uint32_t c = 0; c < nch; ++c) {
            const uint32_t i = c * 32 + lane;
            const bool valid = i < len;
            const bool head = valid && (i == 0 || K[i] != K[i - 1]);
            // run index of element i: heads at or before i
            const unsigned hm = __ballot_sync(0xffffffffu, head);
            const uint32_t ri = r + __popc(hm & (lt_mask | (1u << lane))) - 1;
            r += __popc(hm);
            bool multi = false;
            if (valid) {
                const uint32_t s = ws.run_start[ri], e = ws.run_start[ri + 1];
                multi = e - s >= 2;
                lab_out[V[i]] = V[s];
                if (fingerprint && !head && !same_tuple(V[i], V[i - 1], delta, n, k, lab_in)) clash = true;
            }
            const unsigned mm = __ballot_sync(0xffffffffu, multi);
            if (multi) tmp_list[s0 + surv + __popc(mm & lt_mask)] = V[i];
            surv += __popc(mm);
            ablk += __popc(__ballot_sync(0xffffffffu, multi && head));
        }
        if (lane == 0) surv_count[bkt] = surv;
        runs_total += R;
        ablk_total += ablk;
        __syncwarp();
    }
    if (__any_sync(0xffffffffu, clash) && lane == 0) atomicOr(&ctr->collision, 1u);
    // one atomic per warp and counter (lane 0 holds the warp's totals)
    if (lane == 0) {
        if (runs_total) atomicAdd(&ctr->runs, runs_total);
        if (ablk_total) atomicAdd(&ctr->active_blocks, ablk_total);
    }
}

// move every bucket's survivors (stored at the bucket's own range) to the
// compacted active list; one warp per bucket, coalesced
__global__ void bucket_gather_kernel(const uint32_t* __restrict__ tmp_list, const uint32_t* __restrict__ bucket_start,
                                     const uint32_t* __restrict__ surv_count, const uint32_t* __restrict__ surv_off,
                                     uint32_t buckets, uint32_t* __restrict__ new_list) {
    const unsigned lane = threadIdx.x & 31u;
    for (uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < buckets; b += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t cnt = surv_count[b], src = bucket_start[b], dst = surv_off[b];
        for (uint32_t i = lane; i < cnt; i += 32) new_list[dst + i] = tmp_list[src + i];
    }
}

// ---- global strategy kernels ---------------------------------------------------------

__global__ void run_heads_kernel(const uint64_t* __restrict__ keys, uint64_t m, uint32_t* __restrict__ heads) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        heads[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}

// Exactness check of fingerprint runs: neighbours with equal keys must have
// identical (block, signature) tuples.
__global__ void verify_runs_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, uint64_t m,
                                   const uint32_t* __restrict__ delta, uint32_t n, uint32_t k,
                                   const uint32_t* __restrict__ lab, IterCounters* __restrict__ ctr) {
    for (uint64_t i = 1 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (keys[i] != keys[i - 1]) continue;
        if (!same_tuple(vals[i], vals[i - 1], delta, n, k, lab)) atomicOr(&ctr->collision, 1u);
    }
}

__global__ void run_starts_kernel(const uint32_t* __restrict__ heads, const uint32_t* __restrict__ pos, uint64_t m,
                                  uint32_t* __restrict__ run_start) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        if (heads[i]) run_start[pos[i]] = (uint32_t)i;
        if (i == m - 1) run_start[pos[i] + heads[i]] = (uint32_t)m;
    }
}

__global__ void run_apply_kernel(const uint32_t* __restrict__ heads, const uint32_t* __restrict__ pos,
                                 const uint32_t* __restrict__ vals, uint64_t m, const uint32_t* __restrict__ run_start,
                                 uint32_t* __restrict__ lab, uint8_t* __restrict__ keep,
                                 IterCounters* __restrict__ ctr) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = pos[i] + heads[i] - 1;
        const uint32_t s = run_start[r], e = run_start[r + 1];
        const bool multi = (e - s) >= 2;
        lab[vals[i]] = vals[s];
        keep[i] = multi;
        unsigned am = __ballot_sync(__activemask(), multi && heads[i]);
        unsigned mm = __ballot_sync(__activemask(), multi);
        if ((threadIdx.x & 31u) == (unsigned)(__ffs(__activemask()) - 1)) {
            if (am) atomicAdd(&ctr->active_blocks, (uint32_t)__popc(am));
            if (mm) atomicAdd(&ctr->active_states, (uint32_t)__popc(mm));
        }
    }
}

// chunked exact refinement: run index of every sorted element becomes the
// leading field of the next chunk's key
__global__ void run_index_kernel(const uint32_t* __restrict__ heads, const uint32_t* __restrict__ pos, uint64_t m,
                                 uint32_t* __restrict__ cur) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        cur[i] = pos[i] + heads[i] - 1;
}

__global__ void gather_dense_kernel(const uint32_t* __restrict__ list, uint64_t m, const uint32_t* __restrict__ dense,
                                    uint32_t* __restrict__ cur) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        cur[i] = dense[list ? list[i] : (uint32_t)i];
}

struct Workspace {
    DBuf<uint32_t> lab, lab2, list0, list1, vals0, vals1, heads, pos, run_start, scratch, dense, cur, tmin, tcnt;
    DBuf<uint32_t> buckets, gstart, surv_off;
    DBuf<uint32_t> stats;  // per-bucket survivor counts
    DBuf<uint64_t> keys0, keys1;
    DBuf<uint8_t> keep;
    DBuf<IterCounters> ctr;
};

}  // namespace

LeaderInfo leader_info(Ctx* ctx, const DevDfa& d, cudaStream_t s) {
    uint32_t* info = reinterpret_cast<uint32_t*>(ctx->dmailbox);
    const uint32_t init[4] = {kNone, kNone, 0, 0};
    DK_CUDA(cudaMemcpyAsync(info, init, sizeof(init), cudaMemcpyHostToDevice, s));
    DK_LAUNCH(ctx, leader_info_kernel, grid_for(d.n, kThreads, (unsigned)ctx->num_sms * 8u), kThreads, 0, s, d.acc,
              d.n, info);
    LeaderInfo li;
    read_words(ctx, info, sizeof(li), &li, s);
    return li;
}

void init_leader_labels(Ctx* ctx, const DevDfa& d, const LeaderInfo& li, uint32_t* lab, cudaStream_t s) {
    DK_LAUNCH(ctx, init_labels_kernel, grid_for(d.n), kThreads, 0, s, d.acc, d.n, li.min_acc, li.min_rej, lab);
}

RefineResult sort_pr_device(Ctx* ctx, const DevDfa& d, const SortOptions& o, uint32_t* block_out, cudaStream_t s) {
    RefineResult res;
    const uint32_t n = d.n, k = d.k;
    if (n == 0) return res;
    Workspace w;
    w.lab.alloc(n, s);
    w.lab2.alloc(n, s);
    w.list0.alloc(n, s);
    w.list1.alloc(n, s);
    w.vals0.alloc(n, s);
    w.vals1.alloc(n, s);
    w.keys0.alloc(n, s);
    w.keys1.alloc(n, s);
    w.heads.alloc((uint64_t)n + 1, s);
    w.pos.alloc((uint64_t)n + 1, s);
    w.run_start.alloc((uint64_t)n + 2, s);
    w.scratch.alloc((uint64_t)n + 1, s);
    w.keep.alloc(n, s);
    w.ctr.alloc(1, s);
    DK_CUDA(cudaFuncSetAttribute(segment_refine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(SegSmem)));
    DK_CUDA(cudaFuncSetAttribute(sig_table_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(2u << kSmemTableBits) * 4));
    DK_CUDA(cudaFuncSetAttribute(bucket_refine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(kWarpsPerCta * sizeof(WarpSlice))));

    // initial partition {F, Q\F} with min-state labels
    LeaderInfo li = leader_info(ctx, d, s);
    init_leader_labels(ctx, d, li, w.lab.get(), s);
    uint32_t B = (li.min_acc != kNone) + (li.min_rej != kNone);
    uint32_t A = (li.cnt_acc >= 2) + (li.cnt_rej >= 2);
    uint64_t m = (li.cnt_acc >= 2 ? li.cnt_acc : 0) + (li.cnt_rej >= 2 ? li.cnt_rej : 0);
    const uint32_t* list = nullptr;  // nullptr = identity (all states active)
    uint32_t* list_buf = w.list0.get();
    uint32_t* list_alt = w.list1.get();
    if (m != n && m != 0) {
        DBuf<uint8_t> f(n, s);
        DK_LAUNCH(ctx, init_active_flags_kernel, grid_for(n), kThreads, 0, s, d.acc, n, (uint8_t)(li.cnt_acc >= 2),
                  (uint8_t)(li.cnt_rej >= 2), f.get());
        m = compact_u32(ctx, nullptr, f.get(), n, list_buf, w.scratch.get(), s);
        list = list_buf;
    }

    const uint32_t label_bits = bits_for(n - 1);
    uint64_t salt = 0x5eed5eed5eedull;
    const uint64_t fp_mask = o.fingerprint_bits >= 64 ? ~0ull : ((1ull << o.fingerprint_bits) - 1ull);
    uint32_t collisions_this_pass = 0;

    while (m > 0) {
        ++res.passes;
        const uint32_t dense_bits = bits_for(B ? B - 1 : 0);
        bool need_dense = false, fingerprint = false, chunked = false;
        uint32_t field_bits = 0;
        if ((uint64_t)(k + 1) * label_bits <= 64) {
            field_bits = label_bits;
        } else if ((uint64_t)(k + 1) * dense_bits <= 64) {
            field_bits = dense_bits;
            need_dense = true;
        } else if (!o.force_exact && collisions_this_pass < 3) {
            fingerprint = true;
        } else {
            chunked = true;
            need_dense = true;
            field_bits = dense_bits;
        }
        const uint32_t* keylab = w.lab.get();
        if (need_dense) {
            if (!w.dense.get()) w.dense.alloc(n, s);
            canonical_from_min_labels(ctx, w.lab.get(), n, w.dense.get(), w.scratch.get(), s);
            keylab = w.dense.get();
        }
        DK_CUDA(cudaMemsetAsync(w.ctr.get(), 0, sizeof(IterCounters), s));
        const unsigned g = grid_for(m);
        RadixBuffers rb{w.keys0.get(), w.vals0.get(), w.keys1.get(), w.vals1.get()};
        uint64_t* skeys = w.keys0.get();
        uint32_t* svals = w.vals0.get();
        IterCounters c{};
        enum { kTable, kGlobal } strategy = kGlobal;
        const uint32_t nbits = fingerprint ? 64u : (k + 1) * field_bits;
        SigParams p{};
        p.kind = fingerprint ? kKeyFingerprint : kKeyPacked;
        p.a0 = 0;
        p.a1 = k;
        p.field_bits = field_bits;
        p.salt = salt;
        p.fp_mask = fp_mask;

        if (!chunked && nbits <= kTableBits) {
            // ---- table strategy
            strategy = kTable;
            const uint64_t tsize = 1ull << nbits;
            if (w.tmin.n < tsize) {
                w.tmin.alloc(tsize, s);
                w.tcnt.alloc(tsize, s);
            }
            DK_CUDA(cudaMemsetAsync(w.tmin.get(), 0xff, tsize * sizeof(uint32_t), s));
            DK_CUDA(cudaMemsetAsync(w.tcnt.get(), 0, tsize * sizeof(uint32_t), s));
            const bool local = nbits <= kSmemTableBits;
            const size_t smem = local ? (size_t)(2u << nbits) * 4 : 0;
            const unsigned tg = (unsigned)std::min<uint64_t>((m + 511) / 512, (uint64_t)ctx->num_sms * 2);
            // algorithmic HBM bytes: delta rows + key out (+ list), the label array once
            DK_LAUNCH_B(ctx, (double)m * (4.0 + 4.0 * k + (list ? 4.0 : 0.0)) + 4.0 * n, sig_table_kernel, tg, 512,
                        smem, s,
                        list, m, d.delta, n, keylab, p, nbits, w.heads.get(), w.tmin.get(), w.tcnt.get());
            DK_LAUNCH_B(ctx, (double)m * (9.0 + (list ? 4.0 : 0.0)), table_apply_kernel, g, kThreads, 0, s, list,
                        w.heads.get(), m, w.tmin.get(),
                        w.tcnt.get(), w.lab.get(), w.keep.get(), w.ctr.get());
            read_words(ctx, w.ctr.get(), sizeof(c), &c, s);
        } else if (!chunked) {
            // algorithmic HBM bytes: delta rows + (key, state) out (+ list), the label array once
            DK_LAUNCH_B(ctx, (double)m * (12.0 + 4.0 * k + (list ? 4.0 : 0.0)) + 4.0 * n, signature_kernel, g,
                        kThreads, 0, s,
                        list, m, d.delta, n, keylab, nullptr, p, w.keys0.get(), w.vals0.get());
            // ---- segmented strategy: MSD pass over the top 16 bits, then shared-memory groups
            uint32_t groups = 1, low_bits = nbits;
            bool fits = true;
            if (m > (uint64_t)kSegCap) {
                const uint32_t shift = nbits - kPrefixBits;
                if (radix_sort_pairs_range(ctx, rb, m, shift, nbits, s)) {
                    skeys = w.keys1.get();
                    svals = w.vals1.get();
                }
                const uint32_t nb = 1u << kPrefixBits;
                if (!w.buckets.get()) w.buckets.alloc(nb + 1, s);
                DK_CUDA(cudaMemsetAsync(w.buckets.get(), 0, (nb + 1) * sizeof(uint32_t), s));
                DK_LAUNCH(ctx, prefix_count_kernel, g, kThreads, 0, s, (const unsigned long long*)skeys, m, shift,
                          w.buckets.get());
                exclusive_scan_u32(ctx, w.buckets.get(), w.buckets.get(), nb, nullptr, s);
                // largest bucket: warp-per-bucket refinement when every bucket fits a warp slice
                if (w.gstart.n < (uint64_t)nb + 1) w.gstart.alloc((uint64_t)nb + 1, s);
                DK_LAUNCH(ctx, group_bounds_kernel, grid_for(nb), kThreads, 0, s, w.buckets.get(), nb, 1u, nb, m,
                          w.gstart.get(), w.ctr.get());
                read_words(ctx, w.ctr.get(), sizeof(c), &c, s);
                if (c.max_group <= (uint32_t)kWarpCap) {
                    if (w.stats.n < nb) {
                        w.stats.alloc(nb, s);
                        w.surv_off.alloc(nb, s);
                    }
                    uint32_t* dst = (list == list_buf) ? list_alt : list_buf;
                    DK_CUDA(cudaMemcpyAsync(w.lab2.get(), w.lab.get(), (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
                    const unsigned bg =
                        (unsigned)std::min<uint64_t>((nb + kWarpsPerCta - 1) / kWarpsPerCta, (uint64_t)ctx->num_sms * 12);
                    DK_LAUNCH_B(ctx, 16.0 * m, bucket_refine_kernel, bg, kWarpsPerCta * 32,
                                kWarpsPerCta * sizeof(WarpSlice), s, (const unsigned long long*)skeys, svals,
                                w.buckets.get(), nb, m, shift, d.delta, n, k, (int)fingerprint, w.lab.get(),
                                w.lab2.get(), w.pos.get(), w.stats.get(), w.ctr.get());
                    exclusive_scan_u32(ctx, w.stats.get(), w.surv_off.get(), nb, &w.ctr.get()->active_states, s);
                    DK_LAUNCH(ctx, bucket_gather_kernel, grid_for((uint64_t)nb * 32), kThreads, 0, s, w.pos.get(),
                              w.buckets.get(), w.stats.get(), w.surv_off.get(), nb, dst);
                    res.sorted += m;
                    read_words(ctx, w.ctr.get(), sizeof(c), &c, s);
                    if (fingerprint && c.collision) {
                        ++res.collisions;
                        ++collisions_this_pass;
                        --res.passes;
                        salt = mix64(salt + 0x1234567ull);
                        continue;
                    }
                    collisions_this_pass = 0;
                    const uint32_t newB = B - A + c.runs;
                    if (newB == B) break;  // fixed point (reference l.411)
                    ++res.iters;
                    B = newB;
                    A = c.active_blocks;
                    std::swap(w.lab, w.lab2);
                    m = c.active_states;
                    list = dst;
                    if (dst == list_alt) std::swap(list_buf, list_alt);
                    continue;
                }
                DK_CUDA(cudaMemsetAsync(&w.ctr.get()->max_group, 0, sizeof(uint32_t), s));
                const uint64_t mean = m / nb;
                const uint32_t per_group = (uint32_t)std::max<uint64_t>(
                    1, std::min<uint64_t>(nb, (kSegCap / 2) / std::max<uint64_t>(mean, 1)));
                groups = (nb + per_group - 1) / per_group;
                if (w.gstart.n < (uint64_t)groups + 1) w.gstart.alloc((uint64_t)groups + 1, s);
                DK_LAUNCH(ctx, group_bounds_kernel, grid_for(groups), kThreads, 0, s, w.buckets.get(), nb, per_group,
                          groups, m, w.gstart.get(), w.ctr.get());
                read_words(ctx, w.ctr.get(), sizeof(c), &c, s);
                fits = c.max_group <= (uint32_t)kSegCap;
                low_bits = shift;
            } else {
                if (w.gstart.n < 2) w.gstart.alloc(2, s);
                const uint32_t bounds[2] = {0u, (uint32_t)m};
                DK_CUDA(cudaMemcpyAsync(w.gstart.get(), bounds, sizeof(bounds), cudaMemcpyHostToDevice, s));
            }
            if (fits) {
                uint32_t* dst = (list == list_buf) ? list_alt : list_buf;
                DK_CUDA(cudaMemcpyAsync(w.lab2.get(), w.lab.get(), (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
                // algorithmic HBM bytes: (key, state) in, new label out
                DK_LAUNCH_B(ctx, 16.0 * m, segment_refine_kernel, groups, kSegThreads, sizeof(SegSmem), s,
                            (const unsigned long long*)skeys,
                            svals, w.gstart.get(), low_bits, d.delta, n, k, (int)fingerprint, w.lab.get(), w.lab2.get(),
                            dst, w.ctr.get());
                res.sorted += m;
                read_words(ctx, w.ctr.get(), sizeof(c), &c, s);
                if (fingerprint && c.collision) {
                    // verified fingerprint collision: the new labels went to
                    // lab2 only; re-run the pass with a new salt
                    ++res.collisions;
                    ++collisions_this_pass;
                    --res.passes;
                    salt = mix64(salt + 0x1234567ull);
                    continue;
                }
                collisions_this_pass = 0;
                const uint32_t newB = B - A + c.runs;
                if (newB == B) break;  // fixed point (reference l.411)
                ++res.iters;
                B = newB;
                A = c.active_blocks;
                std::swap(w.lab, w.lab2);
                m = c.active_states;
                list = dst;
                if (dst == list_alt) std::swap(list_buf, list_alt);
                continue;
            }
            // ---- global strategy (bucket groups overflow shared memory)
            uint64_t* okeys = skeys == w.keys0.get() ? w.keys1.get() : w.keys0.get();
            uint32_t* ovals = svals == w.vals0.get() ? w.vals1.get() : w.vals0.get();
            if (radix_sort_pairs_range(ctx, RadixBuffers{skeys, svals, okeys, ovals}, m, 0, nbits, s)) {
                skeys = okeys;
                svals = ovals;
            }
            res.sorted += m;
            if (fingerprint) {
                DK_LAUNCH(ctx, verify_runs_kernel, g, kThreads, 0, s, skeys, svals, m, d.delta, n, k, w.lab.get(),
                          w.ctr.get());
                read_words(ctx, w.ctr.get(), sizeof(c), &c, s);
                if (c.collision) {
                    ++res.collisions;
                    ++collisions_this_pass;
                    --res.passes;
                    salt = mix64(salt + 0x1234567ull);
                    continue;
                }
            }
        } else {
            // ---- exact refinement letter-chunk by letter-chunk; the run index
            // of the previous chunk leads the next key
            if (!w.cur.get()) w.cur.alloc(n, s);
            DK_LAUNCH(ctx, gather_dense_kernel, g, kThreads, 0, s, list, m, keylab, w.cur.get());
            uint32_t cur_bits = field_bits;
            const uint32_t* elist = list;
            uint32_t a = 0;
            for (;;) {
                uint32_t c_letters = field_bits ? (64u - cur_bits) / field_bits : k;
                if (c_letters < 1) c_letters = 1;
                if (c_letters > k - a) c_letters = k - a;
                SigParams pc{};
                pc.kind = kKeyPacked;
                pc.a0 = a;
                pc.a1 = a + c_letters;
                pc.field_bits = field_bits;
                DK_LAUNCH_B(ctx, (double)m * (24.0 + 8.0 * c_letters), signature_kernel, g, kThreads, 0, s, elist, m,
                            d.delta, n, keylab, w.cur.get(), pc, w.keys0.get(), w.vals0.get());
                const bool flip = radix_sort_pairs(ctx, rb, m, cur_bits + c_letters * field_bits, s);
                res.sorted += m;
                skeys = flip ? w.keys1.get() : w.keys0.get();
                svals = flip ? w.vals1.get() : w.vals0.get();
                a += c_letters;
                if (a >= k) break;
                DK_LAUNCH(ctx, run_heads_kernel, g, kThreads, 0, s, skeys, m, w.heads.get());
                exclusive_scan_u32(ctx, w.heads.get(), w.pos.get(), m, nullptr, s);
                DK_LAUNCH(ctx, run_index_kernel, g, kThreads, 0, s, w.heads.get(), w.pos.get(), m, w.cur.get());
                DK_CUDA(cudaMemcpyAsync(list_alt, svals, m * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
                elist = list_alt;
                cur_bits = bits_for(m - 1);
            }
        }

        if (strategy == kGlobal) {
            DK_LAUNCH(ctx, run_heads_kernel, g, kThreads, 0, s, skeys, m, w.heads.get());
            exclusive_scan_u32(ctx, w.heads.get(), w.pos.get(), m, w.scratch.get() + n, s);
            DK_LAUNCH(ctx, run_starts_kernel, g, kThreads, 0, s, w.heads.get(), w.pos.get(), m, w.run_start.get());
            DK_LAUNCH_B(ctx, 25.0 * m, run_apply_kernel, g, kThreads, 0, s, w.heads.get(), w.pos.get(), svals, m,
                        w.run_start.get(), w.lab.get(), w.keep.get(), w.ctr.get());
            read_words(ctx, w.ctr.get(), sizeof(c), &c, s);
            uint32_t runs = 0;
            read_words(ctx, w.scratch.get() + n, sizeof(uint32_t), &runs, s);
            c.runs = runs;
        }

        collisions_this_pass = 0;
        const uint32_t newB = B - A + c.runs;
        if (newB == B) break;  // fixed point: no block split (reference l.411)
        ++res.iters;
        B = newB;
        A = c.active_blocks;
        // surviving active states, order preserved: the table strategy keeps
        // the list order, the global strategy the sorted order (runs grouped,
        // increasing state order inside each run)
        const uint32_t* src = strategy == kTable ? list : svals;
        uint32_t* dst = (list == list_buf) ? list_alt : list_buf;
        if (c.active_states == 0) {
            m = 0;
        } else {
            m = compact_u32(ctx, src, w.keep.get(), m, dst, w.scratch.get(), s);
            list = dst;
            if (dst == list_alt) std::swap(list_buf, list_alt);
        }
    }
    res.num_blocks = canonical_from_min_labels(ctx, w.lab.get(), n, block_out, w.scratch.get(), s);
    return res;
}

}  // namespace dk
