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
// 64 bits exactly when the fields fit (min-state labels, or dense block ids
// stored as uint8/uint16 when they are narrower), otherwise as a 64-bit
// fingerprint whose groups are verified tuple by tuple (exactness never rests
// on the hash; a verified collision re-runs the pass with a new salt and
// after three strikes falls back to exact letter-chunked keys).  States are
// then grouped by key -- the reference's sort + ARE_NEQ + inclusive scan,
// whose only observable output is "same tuple <=> same new block" -- with
// one of these strategies:
//
//   table   packed keys of <= 20 bits: the signature kernel aggregates a
//           (minimum state) table, in shared memory when <= 13 bits -- a
//           one-digit counting sort without the scatter;
//   bucket  wider keys: the signature kernel hashes each key (a bijection
//           for packed keys, the fingerprint itself otherwise) and appends
//           (hkey, state) to one of 2^D radix buckets chosen by the top D
//           hash bits (fixed-capacity bucket slots, warp-aggregated cursor
//           atomics with __match_any_sync): the MSD radix partition of the
//           keys fused into the pass that produces them.  One CTA per bucket
//           then groups its <= 2048 keys in a shared-memory hash table:
//           atomicMin elects the run minimum (the new block label), a second
//           sweep marks runs with >= 2 members (survivors), counters are
//           block-reduced;
//   ghash   buckets that overflow their slots (heavy key duplication) are
//           grouped through a global open-addressing table instead;
//   radix   SortOptions::grouping = radix_sort, and the exact chunked path:
//           the literal Alg. 4 -- LSD radix sort of (key, state) pairs with
//           warp-match histograms (prims.cu), adjacent difference, scan.
//
// The fixed-point test of l.19 is the block count: B' = B - A + R where A is
// the number of active blocks and R the number of runs found.
#include <cooperative_groups.h>

#include <algorithm>

#include <functional>
#include <type_traits>

#include "prims.cuh"
#include "refine.cuh"

namespace dk {

namespace {

constexpr uint32_t kTableBits = 20;
constexpr uint32_t kSmemTableBits = 13;

// layout of one bucket-strategy pass (see bucket_layout in sort_pr_device)
struct BucketLayout {
    uint32_t nb = 0;
    uint64_t bspace = 0, espace = 0;
    bool state_order = false, defer = false, direct = false;
};
// automata from this size on queue their second pass speculatively
constexpr uint32_t kSpecMinStates = 1u << 22;


struct IterCounters {
    uint32_t runs;
    uint32_t active_blocks;
    uint32_t active_states;
    uint32_t collision;
    uint32_t overflow;       // elements appended past their bucket's slots
    uint32_t listed;         // compaction count
    uint32_t pad[2];
};

// Minimum accepting / rejecting state and class sizes.  Byte loads left the
// kernel latency-bound (one 32-byte sector per warp request); 16-byte aligned
// inputs are read 16 flags per load.
// dense2 (optional): also writes the initial partition's dense block ids,
// dense2[q] = (acc[q] != 0) ^ (acc[0] != 0), from the same loads.
__device__ __forceinline__ uint32_t flags4(uint32_t w, uint32_t a0) {  // byte j -> (byte j != 0) ^ a0
    return (__vcmpne4(w, 0u) & 0x01010101u) ^ (a0 * 0x01010101u);
}

// info: accumulators {min acc, min rej, #acc, #rej} at words 0-3 and a CTA
// counter at word 12, armed at context creation; the last CTA copies the
// totals to `out` (device memory or mapped pinned host memory) and re-arms
// them -- no memsets before and no copy-engine readback after the kernel.
__global__ void __launch_bounds__(kThreads) leader_info_kernel(const uint8_t* __restrict__ acc, uint32_t n,
                                                               uint32_t* __restrict__ info,
                                                               uint8_t* __restrict__ dense2, uint32_t* out) {
    __shared__ uint32_t red[4][kThreads / 32];
    uint32_t mina = kNone, minr = kNone, ca = 0, cr = 0;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    const bool vec = ((uintptr_t)acc & 15u) == 0 && ((uintptr_t)dense2 & 15u) == 0;
    const uint32_t nv = vec ? n / 16 : 0;
    const uint32_t a0 = n ? acc[0] != 0 : 0u;
    constexpr int kU = 4;  // loads in flight per thread before any is used
    for (uint32_t v0 = tid; v0 < nv; v0 += kU * stride) {
        uint4 wv[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t v = v0 + u * stride;
            wv[u] = v < nv ? __ldcs(reinterpret_cast<const uint4*>(acc) + v) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t v = v0 + u * stride;
            if (v >= nv) break;
            const uint4 w = wv[u];
            if (dense2)
                reinterpret_cast<uint4*>(dense2)[v] =
                    make_uint4(flags4(w.x, a0), flags4(w.y, a0), flags4(w.z, a0), flags4(w.w, a0));
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {  // four flags per byte-SIMD compare
                const uint32_t nz = __vcmpne4(ws[j], 0u), q0 = v * 16 + 4 * j;
                const uint32_t c = __popc(nz) >> 3;
                ca += c;
                cr += 4 - c;
                if (nz) mina = min(mina, q0 + ((__ffs(nz) - 1) >> 3));
                if (~nz) minr = min(minr, q0 + ((__ffs(~nz) - 1) >> 3));
            }
        }
    }
    for (uint32_t q = nv * 16 + tid; q < n; q += stride) {
        if (dense2) dense2[q] = (acc[q] != 0) ^ a0;
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
    const unsigned lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    if (lane == 0) {
        red[0][wid] = mina;
        red[1][wid] = minr;
        red[2][wid] = ca;
        red[3][wid] = cr;
    }
    __syncthreads();
    if (wid == 0) {  // one atomic per CTA and counter
        const bool ok = lane < kThreads / 32;
        mina = __reduce_min_sync(0xffffffffu, ok ? red[0][lane] : kNone);
        minr = __reduce_min_sync(0xffffffffu, ok ? red[1][lane] : kNone);
        ca = __reduce_add_sync(0xffffffffu, ok ? red[2][lane] : 0u);
        cr = __reduce_add_sync(0xffffffffu, ok ? red[3][lane] : 0u);
        if (lane == 0) {
            if (mina != kNone) atomicMin(&info[0], mina);
            if (minr != kNone) atomicMin(&info[1], minr);
            if (ca) atomicAdd(&info[2], ca);
            if (cr) atomicAdd(&info[3], cr);
        }
    }
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&info[12], 1u) == gridDim.x - 1) {  // last CTA: publish and re-arm
            __threadfence();
            volatile uint32_t* vi = info;
            volatile uint32_t* o = out;
            const uint32_t r0 = vi[0], r1 = vi[1], r2 = vi[2], r3 = vi[3];
            o[0] = r0;
            o[1] = r1;
            o[2] = r2;
            o[3] = r3;
            vi[0] = kNone;
            vi[1] = kNone;
            vi[2] = 0;
            vi[3] = 0;
            vi[12] = 0;
            // (no system fence: the host reads `out` after the event recorded
            // behind this kernel completes)
        }
    }
}

// lab[q] = la / lr by class; four flags per load when acc is 4-byte aligned
__global__ void init_labels_kernel(const uint8_t* __restrict__ acc, uint32_t n, uint32_t la, uint32_t lr,
                                   uint32_t* __restrict__ lab) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    const bool vec = ((uintptr_t)acc & 3u) == 0 && ((uintptr_t)lab & 15u) == 0;
    const uint32_t nv = vec ? n / 4 : 0;
    for (uint32_t v = tid; v < nv; v += stride) {
        const uint32_t w = __ldcs(reinterpret_cast<const uint32_t*>(acc) + v);
        __stcs(reinterpret_cast<uint4*>(lab) + v, make_uint4(w & 0xffu ? la : lr, (w >> 8) & 0xffu ? la : lr,
                                                            (w >> 16) & 0xffu ? la : lr, w >> 24 ? la : lr));
    }
    for (uint32_t q = nv * 4 + tid; q < n; q += stride) lab[q] = acc[q] ? la : lr;
}

// Key labels of the initial partition straight from the flags: dense ids
// (block of state 0 = 0) as bytes, or one bit per state
__global__ void acc_dense2_kernel(const uint8_t* __restrict__ acc, uint32_t n, uint8_t* __restrict__ out) {
    const uint32_t a0 = acc[0] != 0;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    const bool vec = ((uintptr_t)acc & 15u) == 0 && ((uintptr_t)out & 15u) == 0;
    const uint32_t nv = vec ? n / 16 : 0;
    for (uint32_t v = tid; v < nv; v += stride) {
        const uint4 w = __ldcs(reinterpret_cast<const uint4*>(acc) + v);
        reinterpret_cast<uint4*>(out)[v] = make_uint4(flags4(w.x, a0), flags4(w.y, a0), flags4(w.z, a0), flags4(w.w, a0));
    }
    for (uint32_t q = nv * 16 + tid; q < n; q += stride) out[q] = (acc[q] != 0) ^ a0;
}

__global__ void acc_dense2_bits_kernel(const uint8_t* __restrict__ acc, uint32_t n, uint32_t* __restrict__ out) {
    const uint32_t a0 = acc[0] != 0;
    const uint32_t words = (n + 31) / 32;
    for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < words; w += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t q = w * 32 + (threadIdx.x & 31u);
        const unsigned b = __ballot_sync(0xffffffffu, q < n && ((acc[q] != 0) ^ a0));
        if ((threadIdx.x & 31u) == 0) out[w] = b;
    }
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
    uint32_t q0;          // list == nullptr: the active states are q0, q0 + 1, ...
};

#ifndef DFAKIT_SIGB_THREADS
#define DFAKIT_SIGB_THREADS 256
#endif
#ifndef DFAKIT_SIGB_GRID
#define DFAKIT_SIGB_GRID 8
#endif
constexpr int kSigbThreads = DFAKIT_SIGB_THREADS;
#ifndef DFAKIT_SIGB_MINB
#define DFAKIT_SIGB_MINB 5
#endif
#ifndef DFAKIT_SIGT_CH
#define DFAKIT_SIGT_CH 8
#endif
#ifndef DFAKIT_SIGB_CH
#define DFAKIT_SIGB_CH 16
#endif
// Key-label readers: a dense / min-state label array of T, or one bit per
// state (a two-block partition: the initial {F, Q \ F} of every run -- a
// 10M-state automaton's bitmap is 1.25 MB and stays L2-resident where a byte
// array of a 100M-state one does not).
// kBits: the reader's label width (fingerprints pack 64 / kBits labels per
// hashed word).
template <typename T>
struct ArrLab {
    static constexpr int kBits = 8 * (int)sizeof(T);
    const T* p;
    __device__ __forceinline__ uint32_t operator[](uint32_t i) const { return (uint32_t)__ldg(p + i); }
};
// Labels rewritten inside the same launch (the persistent small-m engine):
// plain coherent loads, ordered by grid.sync().  __ldg's non-coherent path is
// only defined for data that stays read-only for the whole kernel.
struct CohLab {
    static constexpr int kBits = 32;
    const uint32_t* p;
    __device__ __forceinline__ uint32_t operator[](uint32_t i) const { return p[i]; }
};
struct BitLab {
    static constexpr int kBits = 1;
    const uint32_t* w;
    __device__ __forceinline__ uint32_t operator[](uint32_t i) const { return (__ldg(w + (i >> 5)) >> (i & 31u)) & 1u; }
};
// 12-bit labels, five per 64-bit word (1.6 bytes per state, no field spans
// two words): the raw table keys of a first pass whose second pass is sliced
// -- 100M states' labels are 160 MB instead of 200, two L2-friendlier slices
struct Pack12Lab {
    static constexpr int kBits = 12;
    const unsigned long long* w;
    __device__ __forceinline__ uint32_t operator[](uint32_t i) const {
        const uint32_t word = i / 5u, slot = i - word * 5u;
        return (uint32_t)(__ldg(w + word) >> (12u * slot)) & 0xFFFu;
    }
};

// 11-bit labels packed back to back (1.375 bytes per state; a field that
// crosses a 64-bit word boundary -- 10 of every 64 -- takes a second load)
struct Pack11Lab {
    static constexpr int kBits = 11;
    const unsigned long long* w;
    __device__ __forceinline__ uint32_t operator[](uint32_t i) const {
        const uint64_t bit = (uint64_t)i * 11u;
        const uint64_t word = bit >> 6;
        const uint32_t sh = (uint32_t)(bit & 63u);
        unsigned long long v = __ldg(w + word) >> sh;
        if (sh > 53) v |= __ldg(w + word + 1) << (64u - sh);
        return (uint32_t)v & 0x7FFu;
    }
};

// word wi of the 11-bit packing: the fields overlapping bits [64 wi, 64 wi + 64)
__global__ void pack11_kernel(const uint16_t* __restrict__ keys16, uint32_t n, unsigned long long* __restrict__ out,
                              uint64_t words) {
    for (uint64_t wi = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; wi < words;
         wi += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b0 = wi * 64u;
        uint64_t i = b0 / 11u;
        unsigned long long v = 0;
        for (; i * 11u < b0 + 64u && i < n; ++i) {
            const unsigned long long f = (unsigned long long)(__ldg(keys16 + i) & 0x7FFu);
            const int64_t off = (int64_t)(i * 11u) - (int64_t)b0;  // field start relative to the word
            v |= off >= 0 ? f << off : f >> (-off);
        }
        out[wi] = v;
    }
}

__global__ void pack12_kernel(const uint16_t* __restrict__ keys16, uint32_t n, unsigned long long* __restrict__ out) {
    const uint32_t words = (n + 4) / 5;
    for (uint32_t wi = blockIdx.x * blockDim.x + threadIdx.x; wi < words; wi += gridDim.x * blockDim.x) {
        unsigned long long v = 0;
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const uint32_t q = wi * 5u + j;
            if (q < n) v |= (unsigned long long)(__ldcs(keys16 + q) & 0xFFFu) << (12 * j);
        }
        out[wi] = v;
    }
}

// Key of q's (block, signature) tuple.  CLAMP: successor ids are clamped to
// n - 1 -- streamed host-buffer calls validate delta while pass 1 already
// consumes it (the range-check flag is read after the pass and the call
// fails), so an out-of-range target must not fault meanwhile.  Letters are processed in chunks of
// 16: all delta loads of a chunk are issued before the first label gather,
// and all gathers before the first use, so a thread keeps up to 16
// independent loads in flight (the loop-carried version serialised two
// memory latencies per letter).
constexpr int kLetterChunk = 16;  // default; the counting-table kernel runs best with 8

// Keys are built additively from one term per tuple position, so a pass can
// gather its labels in several sweeps over slices of the label array (each
// sweep L2-resident) and add the partial keys:
//   packed keys   -- position p's field at its bit offset, ORed in (exact);
//   fingerprints  -- fp_term(salt, p, label) summed mod 2^64, then mixed
//                    (terms are a bijection of (p, label); collisions are
//                    verified tuple by tuple like every fingerprint).
// Position 0 is the lead (the state's own block), position a + 1 letter a.
__device__ __forceinline__ uint64_t fp_term(uint64_t salt, uint32_t pos, uint32_t x) {
    return mix64(salt ^ (((uint64_t)x << 24) | pos));
}
__device__ __forceinline__ uint64_t packed_field(uint64_t v, uint32_t shift) { return shift < 64 ? v << shift : 0ull; }

// FILTER: only successors in [lo, hi) contribute (one slice of the labels)
template <typename LR, int CH = kLetterChunk, bool CLAMP = false, bool FILTER = false>
__device__ __forceinline__ uint64_t tuple_part(uint32_t q, uint32_t lead, bool with_lead,
                                               const uint32_t* __restrict__ delta, uint32_t n, LR lab,
                                               const SigParams& p, uint32_t lo = 0, uint32_t hi = 0) {
    const bool packed = p.kind == kKeyPacked;
    const uint32_t nl = p.a1 - p.a0;
    uint64_t acc = 0;
    if (with_lead) acc = packed ? packed_field(lead, p.field_bits * nl) : fp_term(p.salt, 0, lead);
    for (uint32_t a = p.a0; a < p.a1; a += CH) {
        uint32_t t[CH];
        bool in[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (a + j < p.a1) {
                t[j] = ld_stream(delta + (uint64_t)(a + j) * n + q);
                if (CLAMP) t[j] = min(t[j], n - 1);
                in[j] = !FILTER || (t[j] >= lo && t[j] < hi);
            }
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (a + j < p.a1 && in[j]) t[j] = lab[t[j]];
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (a + j < p.a1 && in[j]) {
                const uint32_t r = a + j - p.a0;
                if (packed) acc |= packed_field(t[j], p.field_bits * (nl - 1 - r));
                else acc += fp_term(p.salt, r + 1, t[j]);
            }
    }
    return acc;
}

__device__ __forceinline__ uint64_t key_of_part(const SigParams& p, uint64_t acc) {
    return p.kind == kKeyPacked ? acc : mix64(acc) & p.fp_mask;
}

// one fingerprint round over a 64-bit word of packed labels
__device__ __forceinline__ uint64_t fp_word(uint64_t h, uint64_t w) { return mix64(h ^ w); }

// Key of a whole tuple in one sweep.  Fingerprints: the labels are packed
// LR::kBits apiece into 64-bit words (an injective layout: every tuple of a
// pass has k + 1 labels) and each full word is hashed in -- ceil((k + 1) /
// (64 / kBits)) mix rounds instead of one per letter, and few live registers
// (the signature kernels run at 48).  A sliced pass uses the additive terms
// of tuple_part instead; a pass is either sliced or not, on every rank.
template <typename LR, int CH = kLetterChunk, bool CLAMP = false>
__device__ __forceinline__ uint64_t tuple_key(uint32_t q, uint32_t lead, const uint32_t* __restrict__ delta,
                                              uint32_t n, LR lab, const SigParams& p) {
    constexpr int W = LR::kBits >= 64 ? 32 : LR::kBits;
    constexpr uint32_t PER = 64u / (uint32_t)W;
    const bool packed = p.kind == kKeyPacked;
    uint64_t key = lead, h = p.salt;
    for (uint32_t a = p.a0; a < p.a1; a += CH) {
        uint32_t t[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (a + j < p.a1) {
                t[j] = ld_stream(delta + (uint64_t)(a + j) * n + q);
                if (CLAMP) t[j] = min(t[j], n - 1);
            }
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (a + j < p.a1) t[j] = lab[t[j]];
#pragma unroll
        for (int j = 0; j < CH; ++j)
            if (a + j < p.a1) {
                if (packed) {
                    key = (key << p.field_bits) | t[j];
                } else {
                    key = (key << W) | t[j];
                    if (((a + j + 1) & (PER - 1)) == PER - 1) {  // label a+j+1 of the tuple fills the word
                        h = fp_word(h, key);
                        key = 0;
                    }
                }
            }
    }
    return packed ? key : fp_word(h, key) & p.fp_mask;
}

// Identity-list sweep, four consecutive states per thread: 16-byte delta
// loads keep four times the bytes in flight (a sweep streams all of delta
// for a slice's worth of gathers, so it is bound by the stream's latency).
// Requires n % 4 == 0 (16-byte aligned rows) and q0 % 4 == 0.
template <typename LR>
__global__ void __launch_bounds__(kThreads, DFAKIT_SIGB_MINB) sig_part_vec_kernel(
    uint64_t m, const uint32_t* __restrict__ delta, uint32_t n, LR lab, SigParams p, uint32_t lo, uint32_t hi,
    int first, uint64_t* __restrict__ part) {
    const bool packed = p.kind == kKeyPacked;
    const uint32_t nl = p.a1 - p.a0;
    constexpr int CH = 4;
    for (uint64_t i4 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i4 * 4 < m;
         i4 += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = i4 * 4;
        const uint32_t q = p.q0 + (uint32_t)i;
        const uint32_t cnt = m - i < 4 ? (uint32_t)(m - i) : 4u;
        uint64_t acc[4] = {0, 0, 0, 0};
        if (first)
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if ((uint32_t)e < cnt) {
                    const uint32_t lead = lab[q + e];
                    acc[e] = packed ? packed_field(lead, p.field_bits * nl) : fp_term(p.salt, 0, lead);
                }
        for (uint32_t a = p.a0; a < p.a1; a += CH) {
            uint4 t[CH];
#pragma unroll
            for (int j = 0; j < CH; ++j)
                if (a + j < p.a1) t[j] = __ldcs(reinterpret_cast<const uint4*>(delta + (uint64_t)(a + j) * n + q));
#pragma unroll
            for (int j = 0; j < CH; ++j)
                if (a + j < p.a1) {
                    const uint32_t r = a + j - p.a0;
                    const uint32_t tt[4] = {t[j].x, t[j].y, t[j].z, t[j].w};
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if ((uint32_t)e < cnt && tt[e] >= lo && tt[e] < hi) {
                            const uint32_t l = lab[tt[e]];
                            if (packed) acc[e] |= packed_field(l, p.field_bits * (nl - 1 - r));
                            else acc[e] += fp_term(p.salt, r + 1, l);
                        }
                }
        }
        // the four partial keys move as one 32-byte access (a warp's accesses
        // cover 1 KB contiguously; four 8-byte accesses per thread touched 32
        // sectors each)
        if (cnt == 4) {
            uint64_t* dst = part + i;
            if (!first) {
                uint64_t p0, p1, p2, p3;
                asm volatile("ld.global.cs.v4.u64 {%0, %1, %2, %3}, [%4];"
                             : "=l"(p0), "=l"(p1), "=l"(p2), "=l"(p3)
                             : "l"(dst));
                acc[0] = packed ? acc[0] | p0 : acc[0] + p0;
                acc[1] = packed ? acc[1] | p1 : acc[1] + p1;
                acc[2] = packed ? acc[2] | p2 : acc[2] + p2;
                acc[3] = packed ? acc[3] | p3 : acc[3] + p3;
            }
            asm volatile("st.global.cs.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "l"(acc[0]), "l"(acc[1]),
                         "l"(acc[2]), "l"(acc[3])
                         : "memory");
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if ((uint32_t)e < cnt) {
                    if (first) {
                        __stcs(part + i + e, acc[e]);
                    } else {
                        const uint64_t prev = __ldcs(part + i + e);
                        __stcs(part + i + e, packed ? prev | acc[e] : prev + acc[e]);
                    }
                }
        }
    }
}

// One sweep over every state (identity range), S states per thread, the
// key kind fixed at compile time: the delta loads of all (up to 16) letters
// are issued before any label is gathered and every in-slice gather before
// any term is formed -- one HBM round trip and one L2 round trip per S
// states (the chunked vec kernel paid both per 4 letters).
#ifndef DFAKIT_PART_MINB
#define DFAKIT_PART_MINB 4
#endif

// C: letters per load chunk, the smallest of 8 / 10 / 12 / 16 covering the
// alphabet (predicated-off letters still cost registers and issue slots:
// 1B transitions, k = 10: C = 16 7.56 ms of sweeps, C = 10 6.07, C = 8 --
// two chunks -- 8.93)
template <typename LR, bool FP, int S, int C = 16>
__global__ void __launch_bounds__(kThreads, DFAKIT_PART_MINB) sig_part_all_kernel(
    uint64_t m, const uint32_t* __restrict__ delta, uint32_t n, LR lab, SigParams p, uint32_t lo, uint32_t hi,
    int first, uint64_t* __restrict__ part) {
    const uint32_t nl = p.a1 - p.a0;
    for (uint64_t iS = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; iS * S < m;
         iS += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = iS * S;
        const uint32_t q = p.q0 + (uint32_t)i;
        const bool full = i + S <= m;
        uint64_t acc[S];
#pragma unroll
        for (int e = 0; e < S; ++e) acc[e] = 0;
        if (first)
#pragma unroll
            for (int e = 0; e < S; ++e)
                if (full || i + e < m) {
                    const uint32_t lead = lab[q + e];
                    acc[e] = FP ? fp_term(p.salt, 0, lead) : packed_field(lead, p.field_bits * nl);
                }
        for (uint32_t a = p.a0; a < p.a1; a += C) {
            uint32_t t[C][S];
#pragma unroll
            for (int j = 0; j < C; ++j)
                if (a + j < p.a1) {
                    const uint32_t* row = delta + (uint64_t)(a + j) * n + q;
                    if (S == 2 && full) {
                        const uint2 v = __ldcs(reinterpret_cast<const uint2*>(row));
                        t[j][0] = v.x;
                        t[j][S - 1] = v.y;
                    } else {
#pragma unroll
                        for (int e = 0; e < S; ++e) t[j][e] = (full || i + e < m) ? __ldcs(row + e) : lo - 1;
                    }
                }
            uint32_t in = 0;  // bit j * S + e: successor in the slice
#pragma unroll
            for (int j = 0; j < C; ++j)
                if (a + j < p.a1)
#pragma unroll
                    for (int e = 0; e < S; ++e)
                        if (t[j][e] - lo < hi - lo) {
                            in |= 1u << (j * S + e);
                            t[j][e] = lab[t[j][e]];
                        }
#pragma unroll
            for (int j = 0; j < C; ++j)
                if (a + j < p.a1) {
                    const uint32_t r = a + j - p.a0;
#pragma unroll
                    for (int e = 0; e < S; ++e)
                        if ((in >> (j * S + e)) & 1u) {
                            if (FP) acc[e] += fp_term(p.salt, r + 1, t[j][e]);
                            else acc[e] |= packed_field(t[j][e], p.field_bits * (nl - 1 - r));
                        }
                }
        }
        // streaming accesses: the partial keys must not push the slice's labels out of the L2
        if (S == 2 && full) {
            ulonglong2* dst = reinterpret_cast<ulonglong2*>(part + i);
            if (!first) {
                const ulonglong2 pv = __ldcs(dst);
                acc[0] = FP ? acc[0] + pv.x : acc[0] | pv.x;
                acc[S - 1] = FP ? acc[S - 1] + pv.y : acc[S - 1] | pv.y;
            }
            __stcs(dst, make_ulonglong2(acc[0], acc[S - 1]));
        } else {
#pragma unroll
            for (int e = 0; e < S; ++e)
                if (full || i + e < m) {
                    if (first) {
                        __stcs(part + i + e, acc[e]);
                    } else {
                        const uint64_t prev = __ldcs(part + i + e);
                        __stcs(part + i + e, FP ? prev + acc[e] : prev | acc[e]);
                    }
                }
        }
    }
}

// One sweep of a sliced signature pass: the partial keys of the active
// states over successors in [lo, hi) (the lead in the first sweep), added
// into part[] (written by the first sweep).
template <typename LR>
__global__ void __launch_bounds__(kThreads, DFAKIT_SIGB_MINB) sig_part_kernel(const uint32_t* __restrict__ list, uint64_t m,
                                                            const uint32_t* __restrict__ delta, uint32_t n, LR lab,
                                                            SigParams p, uint32_t lo, uint32_t hi, int first,
                                                            uint64_t* __restrict__ part) {
    const bool packed = p.kind == kKeyPacked;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t q = list ? list[i] : p.q0 + (uint32_t)i;
        const uint64_t acc = tuple_part<LR, 8, false, true>(q, first ? lab[q] : 0u, first != 0, delta, n, lab, p, lo, hi);
        // streaming accesses: the partial keys must not push the slice's labels out of the L2
        if (first) {
            __stcs(part + i, acc);
        } else {
            const uint64_t prev = __ldcs(part + i);
            __stcs(part + i, packed ? prev | acc : prev + acc);
        }
    }
}

// Plain signature kernel (radix-sort grouping and the exact chunked path):
// one thread per active state, (key, state) written in list order.
// FP: fingerprint keys known at compile time (1) or the kind read from p (0)
// 512-thread CTAs, three per SM (the radix-sort grouping's signature passes
// 0.41 -> 0.39 ms at 10M; 1024 x 2 spills, no minimum let ptxas take ~90
// registers and ran at 0.48 -- 0.72 ms)
#ifndef DFAKIT_SIG_THREADS
#define DFAKIT_SIG_THREADS 512
#endif
#ifndef DFAKIT_SIG_MINB
#define DFAKIT_SIG_MINB 3
#endif
constexpr int kSigThreads = DFAKIT_SIG_THREADS, kSigCtas = DFAKIT_SIG_MINB;
template <typename LR, int FP = 0>
__global__ void __launch_bounds__(kSigThreads, kSigCtas) signature_kernel(const uint32_t* __restrict__ list, uint64_t m,
                                                             const uint32_t* __restrict__ delta, uint32_t n,
                                                             LR lab,
                                                             const uint32_t* __restrict__ head, SigParams p,
                                                             uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    if (FP) p.kind = kKeyFingerprint;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t q = list ? list[i] : p.q0 + (uint32_t)i;
        keys[i] = tuple_key<LR>(q, head ? head[i] : lab[q], delta, n, lab, p);
        vals[i] = q;
    }
}

// ---- table strategy -----------------------------------------------------------------

// step 1: signature + table of (run minimum, run size), in shared memory
// when <= 13 bits; equal keys of a warp are combined first (match_any).
// 1024-thread CTAs, two per SM (32 registers, no spills): 0.400 -> 0.387 ms
// on the bench pass, 3.92 -> 3.80 ms at 1B (512 x 3 / 4, 256 x 6, 768 x 2,
// 1024 x 1 measured: 0.393 -- 0.408 ms)
#ifndef DFAKIT_SIGT_THREADS
#define DFAKIT_SIGT_THREADS 1024
#endif
#ifndef DFAKIT_SIGT_MINB
#define DFAKIT_SIGT_MINB 2
#endif
constexpr int kSigtThreads = DFAKIT_SIGT_THREADS;
constexpr int kSigtCtas = DFAKIT_SIGT_MINB;
template <typename LR, bool CLAMP = false>
__global__ void __launch_bounds__(kSigtThreads, kSigtCtas) sig_table_kernel(const uint32_t* __restrict__ list, uint64_t m,
                                                        const uint32_t* __restrict__ delta, uint32_t n,
                                                        LR lab, SigParams p, uint32_t nbits,
                                                        uint32_t* __restrict__ keys32, uint32_t* __restrict__ tmin,
                                                        uint32_t* __restrict__ tcnt, int inc,
                                                        uint16_t* __restrict__ keys16 = nullptr) {
    extern __shared__ uint32_t st[];  // [tsize] minima, then [tsize] counts (shared mode only)
    p.kind = kKeyPacked;  // table keys are packed: the compiler drops the fingerprint paths
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
        const uint32_t q = list ? list[i] : p.q0 + (uint32_t)i;
        const uint32_t key = (uint32_t)tuple_key<LR, DFAKIT_SIGT_CH, CLAMP>(q, lab[q], delta, n, lab, p);
        keys32[i] = key;
        if (keys16) keys16[i] = (uint16_t)key;  // the raw keys as the next pass's labels (lazy apply)
        const unsigned peers = __match_any_sync(__activemask(), key);
        // inc: states increase with the lane (identity / increasing list), so
        // the lowest peer lane -- the one that updates the table -- holds the
        // minimum (the masked reduction compiles to a loop)
        const uint32_t mq = inc ? q : __reduce_min_sync(peers, q);
        if ((threadIdx.x & 31u) == (unsigned)(__ffs(peers) - 1)) {
            if (local) {
                atomicMin(&smin[key], mq);
                atomicAdd(&scnt[key], (uint32_t)__popc(peers));
            } else {
                atomicMin(&tmin[key], mq);
                atomicAdd(&tcnt[key], (uint32_t)__popc(peers));
            }
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

// block-wide sums of three counters, one atomic each per CTA
template <int THREADS>
__device__ __forceinline__ void flush_counters(uint32_t a, uint32_t b, uint32_t c, uint32_t* ga, uint32_t* gb,
                                               uint32_t* gc) {
    __shared__ uint32_t red[3][THREADS / 32];
    a = __reduce_add_sync(0xffffffffu, a);
    b = __reduce_add_sync(0xffffffffu, b);
    c = __reduce_add_sync(0xffffffffu, c);
    const unsigned lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    if (lane == 0) {
        red[0][wid] = a;
        red[1][wid] = b;
        red[2][wid] = c;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        uint32_t x = lane < THREADS / 32 ? red[0][lane] : 0u;
        uint32_t y = lane < THREADS / 32 ? red[1][lane] : 0u;
        uint32_t z = lane < THREADS / 32 ? red[2][lane] : 0u;
        x = __reduce_add_sync(0xffffffffu, x);
        y = __reduce_add_sync(0xffffffffu, y);
        z = __reduce_add_sync(0xffffffffu, z);
        if (lane == 0) {
            if (x) atomicAdd(ga, x);
            if (y) atomicAdd(gb, y);
            if (z) atomicAdd(gc, z);
        }
    }
}

// step 3: new labels, survivor flags, counters
__global__ void __launch_bounds__(kThreads) table_apply_kernel(const uint32_t* __restrict__ list,
                                                               const uint32_t* __restrict__ keys32, uint64_t m,
                                                               const uint32_t* __restrict__ tmin,
                                                               const uint32_t* __restrict__ tcnt,
                                                               uint32_t* __restrict__ lab, uint8_t* __restrict__ keep,
                                                               uint8_t* __restrict__ act,
                                                               const uint32_t* __restrict__ rank,
                                                               uint16_t* __restrict__ next16,
                                                               uint32_t* __restrict__ next32, uint32_t q0,
                                                               IterCounters* __restrict__ ctr) {
    uint32_t heads = 0, ablk = 0, surv = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t key = keys32[i];
        const uint32_t q = list ? list[i] : q0 + (uint32_t)i;
        const uint32_t rep = tmin[key];
        const bool multi = tcnt[key] >= 2;
        lab[q] = rep;
        if (next16) next16[q] = (uint16_t)rank[key];
        if (next32) next32[q] = rank[key];
        if (keep) keep[i] = multi;
        if (act && multi) act[q] = 1;  // act zeroed by the caller
        heads += rep == q;
        ablk += (rep == q) && multi;
        surv += multi;
    }
    flush_counters<kThreads>(heads, ablk, surv, &ctr->runs, &ctr->active_blocks, &ctr->active_states);
}

// Same over the identity list (states 0 .. m-1), four states per thread
// with 16-byte key / label loads and stores (the scalar kernel sat at
// ~2.4 TB/s: one 4-byte access per thread in flight).  Requires 16-byte
// aligned keys32 / lab, 8-byte next16, 4-byte keep / next32.
// STAGE: tables of <= kApplyStageMax entries are copied into shared memory
// first (the three table lookups per state were L1 gathers over 128-byte
// lines); tsize is the table size then.
constexpr uint32_t kApplyStageMax = 2048;

template <bool STAGE>
__global__ void __launch_bounds__(kThreads) table_apply_vec_kernel(const uint32_t* __restrict__ keys32, uint64_t m,
                                                                   const uint32_t* __restrict__ tmin_g,
                                                                   const uint32_t* __restrict__ tcnt_g,
                                                                   uint32_t* __restrict__ lab,
                                                                   uint8_t* __restrict__ keep,
                                                                   const uint32_t* __restrict__ rank_g,
                                                                   uint16_t* __restrict__ next16,
                                                                   uint32_t* __restrict__ next32,
                                                                   IterCounters* __restrict__ ctr, uint32_t tsize,
                                                                   uint8_t* __restrict__ act = nullptr,
                                                                   uint32_t q0 = 0) {
    __shared__ uint32_t s_min[STAGE ? kApplyStageMax : 1], s_cnt[STAGE ? kApplyStageMax : 1],
        s_rank[STAGE ? kApplyStageMax : 1];
    const uint32_t* tmin = tmin_g;
    const uint32_t* tcnt = tcnt_g;
    const uint32_t* rank = rank_g;
    if (STAGE) {
        for (uint32_t i = threadIdx.x; i < tsize; i += blockDim.x) {
            s_min[i] = tmin_g[i];
            s_cnt[i] = tcnt_g[i];
        }
        __syncthreads();
        tmin = s_min;
        tcnt = s_cnt;
        if (rank_g) {  // the ranks of the occupied entries, computed here (no rank kernel)
            __shared__ uint32_t ws[kThreads / 32];
            constexpr uint32_t per = kApplyStageMax / kThreads;  // entries per thread
            const uint32_t e0 = threadIdx.x * per;
            uint32_t c = 0;
#pragma unroll
            for (uint32_t j = 0; j < per; ++j) c += e0 + j < tsize && s_cnt[e0 + j] != 0;
            uint32_t tot;
            uint32_t r = block_exclusive_scan<kThreads>(c, &tot, ws);
#pragma unroll
            for (uint32_t j = 0; j < per; ++j)
                if (e0 + j < tsize) {
                    s_rank[e0 + j] = r;
                    r += s_cnt[e0 + j] != 0;
                }
            __syncthreads();
            rank = s_rank;
        }
    }
    uint32_t heads = 0, ablk = 0, surv = 0;
    const uint64_t nv = m / 4;
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = tid; v < nv + (m & 3); v += stride) {
        if (v < nv) {
            const uint4 kv = __ldcs(reinterpret_cast<const uint4*>(keys32) + v);
            const uint32_t key[4] = {kv.x, kv.y, kv.z, kv.w};
            uint32_t rep[4], rk[4], kp = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t q = q0 + (uint32_t)(4 * v + j);
                rep[j] = tmin[key[j]];
                const bool multi = tcnt[key[j]] >= 2;
                if (rank) rk[j] = rank[key[j]];
                kp |= (uint32_t)multi << (8 * j);
                heads += rep[j] == q;
                ablk += (rep[j] == q) && multi;
                surv += multi;
            }
            __stcs(reinterpret_cast<uint4*>(lab) + v, make_uint4(rep[0], rep[1], rep[2], rep[3]));
            if (keep) reinterpret_cast<uint32_t*>(keep)[v] = kp;
            if (act) reinterpret_cast<uint32_t*>(act)[v] = kp;  // survivor flags of a state range
            if (next16)
                reinterpret_cast<uint2*>(next16)[v] = make_uint2((rk[0] & 0xffffu) | (rk[1] << 16),
                                                                 (rk[2] & 0xffffu) | (rk[3] << 16));
            if (next32) reinterpret_cast<uint4*>(next32)[v] = make_uint4(rk[0], rk[1], rk[2], rk[3]);
        } else {  // tail: m % 4 states, one per thread
            const uint64_t i = 4 * nv + (v - nv);
            const uint32_t key = keys32[i], q = q0 + (uint32_t)i;
            const uint32_t rep = tmin[key];
            const bool multi = tcnt[key] >= 2;
            lab[i] = rep;
            if (next16) next16[i] = (uint16_t)rank[key];
            if (next32) next32[i] = rank[key];
            if (act) act[i] = multi;
            if (keep) keep[i] = multi;
            heads += rep == q;
            ablk += (rep == q) && multi;
            surv += multi;
        }
    }
    flush_counters<kThreads>(heads, ablk, surv, &ctr->runs, &ctr->active_blocks, &ctr->active_states);
}

// ranks of the occupied table entries in one CTA (tables of <= 2^14
// entries: the counting tables of two-block-derived keys): rank[e] = number
// of occupied entries before e
__global__ void __launch_bounds__(1024) table_rank_one_kernel(const uint32_t* __restrict__ tcnt, uint32_t tsize,
                                                              uint32_t* __restrict__ rank) {
    __shared__ uint32_t ws[32];
    uint32_t carry = 0;
    for (uint32_t b = 0; b < tsize; b += 1024 * 4) {
        const uint32_t e0 = b + threadIdx.x * 4;
        uint32_t f[4], c = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            f[j] = e0 + j < tsize && tcnt[e0 + j] ? 1u : 0u;
            c += f[j];
        }
        uint32_t tot;
        uint32_t o = carry + block_exclusive_scan<1024>(c, &tot, ws);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (e0 + j < tsize) {
                rank[e0 + j] = o;
                o += f[j];
            }
        carry += tot;
    }
}

// counters of a counting-table pass over every state, from the table alone
// (runs = occupied keys, active blocks = keys counted twice or more, active
// states = their counts): what the apply kernel would sum per state
__global__ void __launch_bounds__(1024) table_counts_kernel(const uint32_t* __restrict__ tcnt, uint32_t tsize,
                                                            IterCounters* __restrict__ ctr) {
    uint32_t runs = 0, ablk = 0, surv = 0;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < tsize; e += gridDim.x * blockDim.x) {
        const uint32_t c = tcnt[e];
        runs += c != 0;
        ablk += c >= 2;
        surv += c >= 2 ? c : 0u;
    }
    flush_counters<1024>(runs, ablk, surv, &ctr->runs, &ctr->active_blocks, &ctr->active_states);
}

__global__ void table_occupied_kernel(const uint32_t* __restrict__ tcnt, uint32_t tsize, uint32_t* __restrict__ occ) {
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < tsize; e += gridDim.x * blockDim.x)
        occ[e] = tcnt[e] ? 1u : 0u;
}

// dense ids of a two-block partition: the block of state 0 is block 0
__global__ void dense2_kernel(const uint32_t* __restrict__ lab, uint32_t n, uint8_t* __restrict__ out) {
    const uint32_t l0 = lab[0];
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x)
        out[q] = lab[q] != l0;
}

// delta targets of states [q0, q1) must be < n (reference dfa.cpp validation)
// (letter a0 + blockIdx.y; 16-byte loads where the row segment allows: a
// 64-bit division per element made the check of a streamed chunk cost more
// than the chunk's signature pass)
__global__ void range_check_rows_kernel(const uint32_t* __restrict__ delta, uint32_t n, uint32_t a0, uint32_t q0,
                                        uint32_t q1, uint32_t* __restrict__ bad) {
    const uint32_t* row = delta + (uint64_t)(a0 + blockIdx.y) * n;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    uint32_t lo = q0;
    bool b = false;
    // scalar head up to a 16-byte boundary, then four per load
    const uint32_t head = min(q1 - q0, (uint32_t)((4u - ((uintptr_t)(row + q0) >> 2)) & 3u));
    for (uint32_t q = q0 + tid; q < q0 + head; q += stride) b |= __ldcs(row + q) >= n;
    lo = q0 + head;
    const uint32_t nv = (q1 - lo) / 4;
    const uint4* v4 = reinterpret_cast<const uint4*>(row + lo);
    for (uint32_t v = tid; v < nv; v += stride) {
        const uint4 x = __ldcs(v4 + v);
        b |= (x.x >= n) | (x.y >= n) | (x.z >= n) | (x.w >= n);
    }
    for (uint32_t q = lo + 4 * nv + tid; q < q1; q += stride) b |= __ldcs(row + q) >= n;
    if (__syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1u);
}

void range_check_rows(Ctx* ctx, const uint32_t* delta, uint32_t n, uint32_t k, uint32_t q0, uint32_t q1, uint32_t* bad,
                      cudaStream_t s) {
    if (q1 <= q0) return;
    const unsigned gx = grid_for((uint64_t)(q1 - q0) / 4 + 1, kThreads, 148u * 4u);
    for (uint32_t a0 = 0; a0 < k; a0 += 65535u)
        DK_LAUNCH_B(ctx, 4.0 * (q1 - q0) * std::min(k - a0, 65535u), range_check_rows_kernel,
                    dim3(gx, std::min(k - a0, 65535u)), kThreads, 0, s, delta, n, a0, q0, q1, bad);
}

// bitmap of a two-block partition: bit q = (lab[q] != lab[0]); one warp per word
__global__ void dense2_bits_kernel(const uint32_t* __restrict__ lab, uint32_t n, uint32_t* __restrict__ out) {
    const uint32_t l0 = lab[0];
    const uint32_t words = (n + 31) / 32;
    for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < words; w += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t q = w * 32 + (threadIdx.x & 31u);
        const unsigned b = __ballot_sync(0xffffffffu, q < n && lab[q] != l0);
        if ((threadIdx.x & 31u) == 0) out[w] = b;
    }
}

// ---- bucket strategy -----------------------------------------------------------------

#ifndef DFAKIT_GRP_THREADS
#define DFAKIT_GRP_THREADS 256
#endif
#ifndef DFAKIT_GRP_MINB
#define DFAKIT_GRP_MINB 4
#endif
constexpr int kGrpThreads = DFAKIT_GRP_THREADS;
constexpr unsigned kGrpCtasPerSm = DFAKIT_GRP_MINB;
constexpr int kGrpItems = 2048 / kGrpThreads;
constexpr uint32_t kGrpCap = kGrpThreads * kGrpItems;  // bucket capacity (slots per bucket)
constexpr uint32_t kGrpSlots = 2 * kGrpCap;            // shared hash table (load <= 1/2)
constexpr unsigned long long kEmptyKey = ~0ull;         // a real ~0 key takes the extra slot
constexpr uint32_t kBucketShift = 20;                   // bucket = hkey bits [20, 20 + D): slots use the low
                                                        // bits, the sharded engine's owner rank the top 32

// Bucket cursors are kCntStride words apart (one per 32-byte sector): the
// cursor atomics of a pass are spread over nb sectors instead of nb / 8 --
// L2 serialises atomics per sector, and packed cursors made the appends wait.
#ifndef DFAKIT_CNT_STRIDE
#define DFAKIT_CNT_STRIDE 8
#endif
constexpr uint32_t kCntStride = DFAKIT_CNT_STRIDE;

// q and r have the same (block, signature) tuple under any injective block
// labelling `lab` (min-state labels, or the pass's key labels)
template <typename LR>
__device__ __forceinline__ bool same_tuple(uint32_t q, uint32_t r, const uint32_t* __restrict__ delta, uint32_t n,
                                           uint32_t k, LR lab) {
    if (lab[q] != lab[r]) return false;
    for (uint32_t a = 0; a < k; ++a) {
        const uint32_t* row = delta + (uint64_t)a * n;
        if (lab[row[q]] != lab[row[r]]) return false;
    }
    return true;
}

// Bucket entries are 16 bytes {hkey lo, hkey hi, state, 0}: one vector
// store per append (a scattered 8 + 4 byte pair costs two L1 wavefronts).
__device__ __forceinline__ void st_entry(uint4* p, unsigned long long hk, uint32_t q, uint32_t idx) {
    *p = make_uint4((uint32_t)hk, (uint32_t)(hk >> 32), q, idx);
}
__device__ __forceinline__ unsigned long long entry_key(const uint4& e) {
    return ((unsigned long long)e.y << 32) | e.x;
}

// Appends {hk, q, idx} to bucket (hk >> kBucketShift) & (nb - 1): lanes of a
// warp hitting the same bucket share one cursor atomic.  Past the bucket's
// kGrpCap slots the entry goes to the overflow region at nb * kGrpCap.
__device__ __forceinline__ void bucket_append(unsigned long long hk, uint32_t q, uint32_t idx, uint32_t nb,
                                              uint32_t* __restrict__ bcnt, uint4* __restrict__ bent,
                                              IterCounters* __restrict__ ctr) {
    const unsigned lane = threadIdx.x & 31u;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t b = (uint32_t)(hk >> kBucketShift) & (nb - 1);
    const unsigned act = __activemask();
    const unsigned peers = __match_any_sync(act, b);
    const unsigned leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(&bcnt[b * kCntStride], (uint32_t)__popc(peers));
    base = __shfl_sync(act, base, leader);
    const uint32_t pos = base + (uint32_t)__popc(peers & lt);
    uint64_t slot;
    const bool over = pos >= kGrpCap;
    const unsigned om = __ballot_sync(act, over);
    if (over) {
        const unsigned ol = __ffs(om) - 1;
        uint32_t obase = 0;
        if (lane == ol) obase = atomicAdd(&ctr->overflow, (uint32_t)__popc(om));
        obase = __shfl_sync(om, obase, ol);
        slot = (uint64_t)nb * kGrpCap + obase + (uint32_t)__popc(om & lt);
    } else {
        slot = (uint64_t)b * kGrpCap + pos;
    }
    st_entry(bent + slot, hk, q, idx);
}

// Signature + fused radix partition: (hkey, state) appended to bucket
// hkey >> shift.  Slots b*cap .. b*cap+cap-1; the excess goes to the
// overflow region at nb*cap (counted in ctr->overflow).
// MODE (compile time): 0 any key kind, 1 fingerprints, 2 finishing the
// partial keys of a sliced pass
// The append split in two for software pipelining: issue (bucket, warp
// peers, the leader's cursor atomic) and finish (position, overflow, store).
// Every lane of the warp takes part in both (invalid lanes carry no entry).
struct PendingAppend {
    unsigned long long hk;
    uint32_t q, b, base, rank, leader;
    bool valid;
};

__device__ __forceinline__ PendingAppend append_issue(bool valid, unsigned long long hk, uint32_t q, uint32_t nb,
                                                      uint32_t* __restrict__ bcnt) {
    const unsigned lane = threadIdx.x & 31u;
    PendingAppend a;
    a.hk = hk;
    a.q = q;
    a.valid = valid;
    a.b = valid ? (uint32_t)(hk >> kBucketShift) & (nb - 1) : 0xffffffffu;  // no valid bucket matches
    const unsigned peers = __match_any_sync(0xffffffffu, a.b);
    a.leader = __ffs(peers) - 1;
    a.rank = (uint32_t)__popc(peers & ((1u << lane) - 1u));
    a.base = 0;
    if (valid && lane == a.leader) a.base = atomicAdd(&bcnt[a.b * kCntStride], (uint32_t)__popc(peers));
    return a;
}

__device__ __forceinline__ void append_finish(const PendingAppend& a, uint32_t nb, uint4* __restrict__ bent,
                                              IterCounters* __restrict__ ctr) {
    const unsigned lane = threadIdx.x & 31u, lt = (1u << lane) - 1u;
    const uint32_t pos = __shfl_sync(0xffffffffu, a.base, a.leader) + a.rank;
    const bool over = a.valid && pos >= kGrpCap;
    const unsigned om = __ballot_sync(0xffffffffu, over);
    uint64_t slot = (uint64_t)a.b * kGrpCap + pos;
    if (om) {
        const unsigned ol = __ffs(om) - 1;
        uint32_t obase = 0;
        if (lane == ol) obase = atomicAdd(&ctr->overflow, (uint32_t)__popc(om));
        obase = __shfl_sync(0xffffffffu, obase, ol);
        if (over) slot = (uint64_t)nb * kGrpCap + obase + (uint32_t)__popc(om & lt);
    }
    if (a.valid) st_entry(bent + slot, a.hk, a.q, 0u);
}


template <typename LR, int MODE>
__global__ void __launch_bounds__(kSigbThreads, DFAKIT_SIGB_MINB) sig_bucket_kernel(const uint32_t* __restrict__ list, uint64_t m,
                                                              const uint32_t* __restrict__ delta, uint32_t n,
                                                              LR lab, SigParams p,
                                                              uint32_t nb, uint32_t* __restrict__ bcnt,
                                                              uint4* __restrict__ bent,
                                                              IterCounters* __restrict__ ctr,
                                                              const uint64_t* __restrict__ part) {
    if (MODE == 1) p.kind = kKeyFingerprint;  // lets the compiler drop the packed-key paths
    if constexpr (MODE == 2) {
    // finishing the partial keys of a sliced pass (no gathers left): warp-
    // uniform trips, the cursor atomic of one state in flight while the next
    // state's partial key is read, its entry stored after that (1B: 2.88 ->
    // 2.56 ms; the gathering modes lose by it, 0.485 -> 0.512 ms at 10M)
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + (threadIdx.x & ~31u);
    const unsigned lane = threadIdx.x & 31u;
    PendingAppend pend;
    bool have = false;
    for (uint64_t w = i0; w < m; w += stride) {
        const uint64_t i = w + lane;
        const bool valid = i < m;
        unsigned long long hk = 0;
        uint32_t q = 0;
        if (valid) {
            q = list ? list[i] : p.q0 + (uint32_t)i;
            const uint64_t key = MODE == 2 ? key_of_part(p, __ldcs(part + i))
                                           : tuple_key<LR, DFAKIT_SIGB_CH>(q, lab[q], delta, n, lab, p);
            hk = p.kind == kKeyPacked ? mix64(key) : key;
        }
        if (have) append_finish(pend, nb, bent, ctr);
        pend = append_issue(valid, hk, q, nb, bcnt);
        have = true;
    }
    if (have) append_finish(pend, nb, bent, ctr);
    } else {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t q = list ? list[i] : p.q0 + (uint32_t)i;
        // part: the keys were gathered by a sliced pass (sig_part_kernel sweeps)
        const uint64_t key = MODE == 2 ? key_of_part(p, __ldcs(part + i))
                                       : tuple_key<LR, DFAKIT_SIGB_CH>(q, lab[q], delta, n, lab, p);
        const unsigned long long hk = p.kind == kKeyPacked ? mix64(key) : key;
        bucket_append(hk, q, 0u, nb, bcnt, bent, ctr);
    }
    }
}

struct GroupSmem {  // slot kGrpSlots: the ~0 key's own slot
    alignas(16) unsigned long long key[kGrpSlots + 2];
    alignas(16) uint32_t rep[kGrpSlots + 4];
    alignas(16) uint8_t multi[kGrpSlots + 16];
};

__device__ __forceinline__ uint32_t pow2_at_least(uint32_t x) { return x <= 1 ? 1u : 1u << (32 - __clz(x - 1)); }

// Group outputs of one element (shared by the bucket and ghash kernels).
struct GroupOut {
    int direct;        // exact keys: write labels in place now
    int state_order;   // survivors flagged per state (act) instead of per slot
    uint32_t* lab;     // direct: new labels
    uint8_t* act;      // state_order: survivor flag per state
    uint32_t* rep_slot;
    uint8_t* keep_slot;
    uint32_t* res;     // sharded engine: res[entry index] = rep | multi << 31
    uint2* rec;        // deferred: rec[slot] = {state, rep | multi << 31}, applied once verified
    int rec_index;     // rec[slot].x = the entry index instead of the state (sharded owners)
    uint8_t* bsingle;  // EM 1: per bucket, 1 = every key distinct (no records written: the
                       // bucket's states keep their own ids)
};

__device__ __forceinline__ void emit(const GroupOut& o, uint64_t slot, uint32_t q, uint32_t r, bool multi,
                                     uint32_t idx) {
    if (o.res) {
        o.res[idx] = r | (multi ? 0x80000000u : 0u);
    } else if (o.rec) {
        o.rec[slot] = make_uint2(o.rec_index ? idx : q, r | (multi ? 0x80000000u : 0u));
    } else if (o.direct) {
        o.lab[q] = r;
        if (o.state_order) {
            if (multi) o.act[q] = 1;  // act was zeroed: only survivors are written
        } else {
            o.keep_slot[slot] = multi;
        }
    } else {
        o.rep_slot[slot] = r;
        o.keep_slot[slot] = multi;
    }
}

// Emit with the output mode fixed at compile time (EM 1: deferred records by
// state, EM 2: per-entry results; 0: decided at run time from o)
template <int EM>
__device__ __forceinline__ void emit_as(const GroupOut& o, uint64_t slot, uint32_t q, uint32_t r, bool multi,
                                        uint32_t idx) {
    if (EM == 1) o.rec[slot] = make_uint2(q, r | (multi ? 0x80000000u : 0u));
    else if (EM == 2) o.res[idx] = r | (multi ? 0x80000000u : 0u);
    else emit(o, slot, q, r, multi, idx);
}

// Bucket sources of the grouping kernel.  OneSrc: the single-GPU layout --
// bucket b's entries at bent + b * kGrpCap, its count at bcnt[b * stride].
// MultiSrc (sharded owners): bucket b is the concatenation of one sub-bucket
// per sender s (capacity cs, count cnt[s][b]); a count above cs on any
// sender sends the whole bucket to the ghash fallback.  The view of a bucket
// loads its idx-th entry and names the output index of that entry.
struct OneSrc {
    const uint32_t* __restrict__ bcnt;
    const uint4* __restrict__ bent;
    struct View {
        const uint4* base;
        __device__ __forceinline__ uint4 load(uint32_t idx) const { return __ldcs(base + idx); }
        // what the entry keeps for its output index, and the index
        __device__ __forceinline__ uint32_t keep(const uint4& e) const { return e.w; }
        __device__ __forceinline__ uint32_t index(uint32_t, uint32_t kept) const { return kept; }
    };
    __device__ __forceinline__ void init() const {}
    __device__ __forceinline__ uint32_t count(uint32_t b) const { return bcnt[b * kCntStride]; }
    __device__ __forceinline__ View view(uint32_t b) const { return View{bent + (uint64_t)b * kGrpCap}; }
    __device__ __forceinline__ uint64_t slot0(uint32_t b) const { return (uint64_t)b * kGrpCap; }
    __device__ __forceinline__ void prefetch(uint32_t b, uint32_t len, unsigned tid, unsigned nt) const {
        const uint32_t lines = (min(len, kGrpCap) * 16u + 127u) / 128u;
        const char* base = reinterpret_cast<const char*>(bent + (uint64_t)b * kGrpCap);
        for (uint32_t l = tid; l < lines; l += nt) asm volatile("prefetch.global.L2 [%0];" ::"l"(base + 128ull * l));
    }
};

constexpr int kMaxSrc = 8;
struct MultiSrc {
    const uint4* base[kMaxSrc];     // sender s's sub-buckets for this owner: nb * cs slots
    const uint32_t* cnt[kMaxSrc];   // sender s's counts (nb words, unclamped)
    uint32_t nsrc, nb, cs;
    // per-bucket view in shared memory (the CTA's current bucket): prefix of
    // the senders' clamped counts and each sender's chunk pointer -- runtime
    // indices into shared memory, not register arrays (which go to local
    // memory); the per-sender pointers are staged in shared memory once per
    // CTA too (hoisted into registers they crowded out the grouping's state)
    struct View {
        const uint32_t* pre;       // kMaxSrc + 1 prefix sums
        const uint4* const* ptr;   // kMaxSrc chunk bases
        uint32_t nsrc, b, nb, cs;
        // the last sender whose prefix is <= idx: a binary search over the 8
        // prefixes (those of absent senders equal the total, never <= idx)
        __device__ __forceinline__ uint32_t source(uint32_t idx) const {
            static_assert(kMaxSrc == 8, "three halving steps");
            if (nsrc == 1) return 0;
            uint32_t s = idx >= pre[4] ? 4u : 0u;
            s += idx >= pre[s + 2] ? 2u : 0u;
            s += idx >= pre[s + 1] ? 1u : 0u;
            return s;
        }
        __device__ __forceinline__ uint4 load(uint32_t idx) const {
            const uint32_t s = source(idx);
            return __ldcs(ptr[s] + (idx - pre[s]));
        }
        // output index: sender s's padded slot, in the layout the results
        // travel back in (recomputed at output time: nothing kept per item)
        __device__ __forceinline__ uint32_t keep(const uint4&) const { return 0; }
        __device__ __forceinline__ uint32_t index(uint32_t idx, uint32_t) const {
            const uint32_t s = source(idx);
            return (s * nb + b) * cs + (idx - pre[s]);
        }
    };
    struct Shared {
        const uint4* base[kMaxSrc];
        const uint32_t* cnt[kMaxSrc];
        const uint4* ptr[kMaxSrc];
        uint32_t pre[kMaxSrc + 1];
    };
    __device__ __forceinline__ Shared& sh() const {
        __shared__ Shared s_multi;
        return s_multi;
    }
    __device__ __forceinline__ void init() const {
        if (threadIdx.x < kMaxSrc) {
            sh().base[threadIdx.x] = threadIdx.x < nsrc ? base[threadIdx.x] : nullptr;
            sh().cnt[threadIdx.x] = threadIdx.x < nsrc ? cnt[threadIdx.x] : nullptr;
        }
        __syncthreads();
    }
    __device__ __forceinline__ uint32_t count(uint32_t b) const {
        const Shared& m = sh();
        uint32_t t = 0;
        bool over = false;
        for (uint32_t s = 0; s < nsrc; ++s) {
            const uint32_t c = m.cnt[s][b];
            over |= c > cs;
            t += c;
        }
        return over ? kGrpCap + 1 : t;
    }
    // every thread computes (and stores) the same values: the writes are
    // identical, and the grouping kernel's end-of-bucket barrier orders them
    // after the previous bucket's reads
    __device__ __forceinline__ View view(uint32_t b) const {
        Shared& m = sh();
        uint32_t t = 0;
        for (uint32_t s = 0; s < kMaxSrc; ++s) {
            m.pre[s] = t;
            if (s < nsrc) {
                m.ptr[s] = m.base[s] + (uint64_t)b * cs;
                t += min(m.cnt[s][b], cs);
            }
        }
        m.pre[kMaxSrc] = t;
        return View{m.pre, m.ptr, nsrc, b, nb, cs};
    }
    __device__ __forceinline__ uint64_t slot0(uint32_t b) const { return (uint64_t)b * kGrpCap; }
    __device__ __forceinline__ void prefetch(uint32_t b, uint32_t, unsigned tid, unsigned nt) const {
        const Shared& m = sh();
        for (uint32_t s = 0; s < nsrc; ++s) {
            const uint32_t lines = (min(m.cnt[s][b], cs) * 16u + 127u) / 128u;
            const char* p = reinterpret_cast<const char*>(m.base[s] + (uint64_t)b * cs);
            for (uint32_t l = tid; l < lines; l += nt) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + 128ull * l));
        }
    }
};

// One CTA per bucket (persistent over buckets).  Buckets whose count
// exceeds the capacity are left to the ghash fallback.
// EM: the output mode at compile time (see emit_as); EM 1 implies fingerprints.
template <typename LR, typename Src = OneSrc, int EM = 0>
__global__ void __launch_bounds__(kGrpThreads, DFAKIT_GRP_MINB) bucket_group_kernel(
    const __grid_constant__ Src src, uint32_t nb, int fingerprint_rt, const uint32_t* __restrict__ delta, uint32_t n,
    uint32_t k, LR lab_in,
    GroupOut o, IterCounters* __restrict__ ctr) {
    const int fingerprint = EM == 1 ? 1 : fingerprint_rt;
    extern __shared__ __align__(16) unsigned char grp_raw[];
    GroupSmem& sm = *reinterpret_cast<GroupSmem*>(grp_raw);
    const unsigned tid = threadIdx.x;
    uint32_t heads = 0, ablk = 0, surv = 0;
    bool clash = false;
    src.init();
    uint32_t len_next = blockIdx.x < nb ? src.count(blockIdx.x) : 0u;
    for (uint32_t b = blockIdx.x; b < nb; b += gridDim.x) {
        const uint32_t len = len_next;
        // the next bucket's length now, its entries into L2 while this one
        // is grouped (one prefetch per 128-byte line)
        const uint32_t bn = b + gridDim.x;
        if (bn < nb) {
            len_next = src.count(bn);
            src.prefetch(bn, len_next, tid, kGrpThreads);
        }
        if (len == 0 || len > kGrpCap) {  // uniform across the CTA
            if ((EM == 1 || EM == 2) && o.bsingle && tid == 0) o.bsingle[b] = 0;
            continue;
        }
        const uint32_t T = max(64u, pow2_at_least(2 * len));
        // rep needs no reset: every claimed slot's rep is written by its
        // claimer; keys and flags are reset with 16-byte stores (T >= 64)
        for (uint32_t e = tid; e < T / 2; e += kGrpThreads)
            reinterpret_cast<ulonglong2*>(sm.key)[e] = make_ulonglong2(kEmptyKey, kEmptyKey);
        for (uint32_t e = tid; e < T / 16; e += kGrpThreads)
            reinterpret_cast<uint4*>(sm.multi)[e] = make_uint4(0, 0, 0, 0);
        if (tid == 0) {
            sm.key[kGrpSlots] = kEmptyKey;
            sm.multi[kGrpSlots] = 0;
        }
        __syncthreads();
        const uint64_t s0 = src.slot0(b);
        const auto view = src.view(b);
        unsigned long long hk[kGrpItems];
        uint32_t q[kGrpItems], slot[kGrpItems], ix[kGrpItems];
#pragma unroll
        for (int j = 0; j < kGrpItems; ++j) {
            const uint32_t idx = j * kGrpThreads + tid;
            if (idx < len) {
                const uint4 e = view.load(idx);
                hk[j] = entry_key(e);
                q[j] = e.z;
                ix[j] = view.keep(e);
            }
        }
        // claim: the member whose CAS takes the empty slot writes the run's
        // rep with a plain store; a member that finds its key already there
        // makes the run multi-member and joins the minimum after the barrier
        // (one shared atomic per entry instead of two when keys are distinct).
        // The ~0 key takes its own slot, where the first claimer writes 0.
        unsigned dup = 0;
#pragma unroll
        for (int j = 0; j < kGrpItems; ++j) {
            const uint32_t idx = j * kGrpThreads + tid;
            if (idx < len) {
                const unsigned long long want = hk[j] == kEmptyKey ? 0ull : hk[j];
                uint32_t s = hk[j] == kEmptyKey ? kGrpSlots : (uint32_t)hk[j] & (T - 1);
                unsigned long long o = atomicCAS(&sm.key[s], kEmptyKey, want);
                while (o != kEmptyKey && o != want) {
                    s = (s + 1) & (T - 1);
                    o = atomicCAS(&sm.key[s], kEmptyKey, want);
                }
                slot[j] = s;
                if (o == kEmptyKey) {
                    sm.rep[s] = q[j];
                } else {
                    sm.multi[s] = 1;
                    dup |= 1u << j;
                }
            }
        }
        const bool any_dup = __syncthreads_or(dup != 0);
        if (EM == 1 || (EM == 2 && o.bsingle)) {
            if (tid == 0) o.bsingle[b] = any_dup ? 0 : 1;
            if (!any_dup) {
                // every key distinct: all singletons, nothing to verify and no
                // records / results (rec_apply_kernel, owner_scatter_kernel
                // read the states from the entries)
#pragma unroll
                for (int j = 0; j < kGrpItems; ++j) heads += j * kGrpThreads + tid < len;
                __syncthreads();
                continue;
            }
        }
        if (any_dup) {
#pragma unroll
            for (int j = 0; j < kGrpItems; ++j)
                if (dup & (1u << j)) atomicMin(&sm.rep[slot[j]], q[j]);
            __syncthreads();
        }
#pragma unroll
        for (int j = 0; j < kGrpItems; ++j) {
            const uint32_t idx = j * kGrpThreads + tid;
            if (idx < len) {
                const uint32_t r = sm.rep[slot[j]];
                const bool multi = sm.multi[slot[j]] != 0;
                const bool head = r == q[j];
                heads += head;
                ablk += head && multi;
                surv += multi;
                if (fingerprint && !head && !same_tuple(q[j], r, delta, n, k, lab_in)) clash = true;
                emit_as<EM>(o, s0 + idx, q[j], r, multi, view.index(idx, ix[j]));
            }
        }
        __syncthreads();
    }
    if (__syncthreads_or(clash) && tid == 0) atomicOr(&ctr->collision, 1u);
    flush_counters<kGrpThreads>(heads, ablk, surv, &ctr->runs, &ctr->active_blocks, &ctr->active_states);
}

// ---- ghash fallback: elements of overflowed buckets + the overflow region ----------

__device__ __forceinline__ bool fallback_elem(uint64_t e, const uint32_t* __restrict__ bcnt, uint32_t nb,
                                              uint32_t ovf) {
    const uint64_t bspace = (uint64_t)nb * kGrpCap;
    if (e >= bspace) return e - bspace < ovf;
    return bcnt[(e / kGrpCap) * kCntStride] > kGrpCap;
}

__global__ void ghash_insert_kernel(const uint32_t* __restrict__ bcnt, uint32_t nb, uint32_t ovf,
                                    const uint4* __restrict__ bent, uint64_t T, unsigned long long* __restrict__ gkey, uint32_t* __restrict__ grep,
                                    uint32_t* __restrict__ gslot) {
    const uint64_t total = (uint64_t)nb * kGrpCap + ovf;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        if (!fallback_elem(e, bcnt, nb, ovf)) continue;
        const uint4 ent = bent[e];
        const unsigned long long hk = entry_key(ent);
        const uint32_t q = ent.z;
        uint64_t s;
        if (hk == kEmptyKey) {
            s = T;
        } else {
            s = mix64(hk) & (T - 1);
            for (;;) {
                const unsigned long long old = atomicCAS(&gkey[s], kEmptyKey, hk);
                if (old == kEmptyKey || old == hk) break;
                s = (s + 1) & (T - 1);
            }
        }
        gslot[e] = (uint32_t)s;
        // equal keys of one warp elect their minimum before the global atomic
        const unsigned peers = __match_any_sync(__activemask(), (unsigned long long)s);
        const uint32_t mq = __reduce_min_sync(peers, q);
        if ((threadIdx.x & 31u) == (unsigned)(__ffs(peers) - 1)) atomicMin(&grep[s], mq);
    }
}

__global__ void ghash_multi_kernel(const uint32_t* __restrict__ bcnt, uint32_t nb, uint32_t ovf,
                                   const uint4* __restrict__ bent, const uint32_t* __restrict__ grep,
                                   const uint32_t* __restrict__ gslot, uint8_t* __restrict__ gmul) {
    const uint64_t total = (uint64_t)nb * kGrpCap + ovf;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        if (!fallback_elem(e, bcnt, nb, ovf)) continue;
        const uint32_t s = gslot[e];
        if (grep[s] != bent[e].z && !gmul[s]) gmul[s] = 1;
    }
}

template <typename LR>
__global__ void __launch_bounds__(kThreads) ghash_out_kernel(
    const uint32_t* __restrict__ bcnt, uint32_t nb, uint32_t ovf, const uint4* __restrict__ bent,
    const uint32_t* __restrict__ grep, const uint32_t* __restrict__ gslot, const uint8_t* __restrict__ gmul,
    int fingerprint, const uint32_t* __restrict__ delta, uint32_t n, uint32_t k, LR lab_in,
    GroupOut o, IterCounters* __restrict__ ctr) {
    const uint64_t total = (uint64_t)nb * kGrpCap + ovf;
    uint32_t heads = 0, ablk = 0, surv = 0;
    bool clash = false;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        if (!fallback_elem(e, bcnt, nb, ovf)) continue;
        const uint4 ent = bent[e];
        const uint32_t s = gslot[e], q = ent.z;
        const uint32_t r = grep[s];
        const bool multi = gmul[s] != 0, head = r == q;
        heads += head;
        ablk += head && multi;
        surv += multi;
        if (fingerprint && !head && !same_tuple(q, r, delta, n, k, lab_in)) clash = true;
        emit(o, e, q, r, multi, ent.w);
    }
    if (__syncthreads_or(clash) && threadIdx.x == 0) atomicOr(&ctr->collision, 1u);
    flush_counters<kThreads>(heads, ablk, surv, &ctr->runs, &ctr->active_blocks, &ctr->active_states);
}

// deferred (fingerprint) passes: labels applied once the pass verified clean
__global__ void slot_apply_kernel(const uint32_t* __restrict__ bcnt, uint32_t nb, uint32_t ovf,
                                  const uint4* __restrict__ bent, const uint32_t* __restrict__ rep_slot,
                                  const uint8_t* __restrict__ keep_slot, uint32_t* __restrict__ lab,
                                  uint8_t* __restrict__ act) {
    const uint64_t bspace = (uint64_t)nb * kGrpCap, total = bspace + ovf;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        if (e < bspace && (uint32_t)(e % kGrpCap) >= min(bcnt[(e / kGrpCap) * kCntStride], kGrpCap)) continue;
        const uint32_t q = bent[e].z;
        lab[q] = rep_slot[e];
        if (act) act[q] = keep_slot[e];
    }
}

// deferred big fingerprint passes: the packed per-slot records of a verified
// pass become labels (and survivor flags; act was zeroed) -- skipped when the
// pass left every block a singleton (the numbering is then the identity)
__global__ void rec_apply_kernel(const uint32_t* __restrict__ bcnt, uint32_t nb, uint32_t ovf,
                                 const uint2* __restrict__ rec, uint32_t* __restrict__ lab,
                                 uint8_t* __restrict__ act, const uint8_t* __restrict__ bsingle,
                                 const uint4* __restrict__ bent) {
    const uint64_t bspace = (uint64_t)nb * kGrpCap, total = bspace + ovf;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        if (e < bspace && (uint32_t)(e % kGrpCap) >= min(bcnt[(e / kGrpCap) * kCntStride], kGrpCap)) continue;
        if (e < bspace && bsingle[e / kGrpCap]) {  // a bucket of distinct keys: singletons
            const uint32_t q = __ldcs(bent + e).z;
            lab[q] = q;
            continue;
        }
        const uint2 r = __ldcs(rec + e);
        lab[r.x] = r.y & 0x7fffffffu;
        if (r.y >> 31) act[r.x] = 1;
    }
}

// sharded owners: slot-ordered records -> per-entry results (for the trip
// back to the senders); only when the pass is not the last
__global__ void rec_results_kernel(const uint32_t* __restrict__ bcnt, uint32_t nb, uint32_t ovf,
                                   const uint2* __restrict__ rec, uint32_t* __restrict__ results) {
    const uint64_t bspace = (uint64_t)nb * kGrpCap, total = bspace + ovf;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        if (e < bspace && (uint32_t)(e % kGrpCap) >= min(bcnt[(e / kGrpCap) * kCntStride], kGrpCap)) continue;
        const uint2 r = __ldcs(rec + e);
        results[r.x] = r.y;
    }
}

__global__ void entry_state_kernel(const uint4* __restrict__ bent, const uint8_t* __restrict__ keep, uint64_t total,
                                   uint32_t* __restrict__ out) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x)
        if (keep[e]) out[e] = bent[e].z;
}

// ---- radix-sort grouping (literal Alg. 4) -------------------------------------------

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
        if (!same_tuple(vals[i], vals[i - 1], delta, n, k, ArrLab<uint32_t>{lab})) atomicOr(&ctr->collision, 1u);
    }
}

__global__ void run_starts_kernel(const uint32_t* __restrict__ heads, const uint32_t* __restrict__ pos, uint64_t m,
                                  uint32_t* __restrict__ run_start) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        if (heads[i]) run_start[pos[i]] = (uint32_t)i;
        if (i == m - 1) run_start[pos[i] + heads[i]] = (uint32_t)m;
    }
}

// run minimum (lists need not be increasing: bucket passes emit survivors
// in bucket order); consecutive elements of one run elect first per warp
__global__ void run_min_kernel(const uint32_t* __restrict__ heads, const uint32_t* __restrict__ pos,
                               const uint32_t* __restrict__ vals, uint64_t m, uint32_t* __restrict__ rmin) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = pos[i] + heads[i] - 1;
        const unsigned peers = __match_any_sync(__activemask(), r);
        const uint32_t mq = __reduce_min_sync(peers, vals[i]);
        if ((threadIdx.x & 31u) == (unsigned)(__ffs(peers) - 1)) atomicMin(&rmin[r], mq);
    }
}

__global__ void __launch_bounds__(kThreads) run_apply_kernel(const uint32_t* __restrict__ heads,
                                                             const uint32_t* __restrict__ pos,
                                                             const uint32_t* __restrict__ vals, uint64_t m,
                                                             const uint32_t* __restrict__ run_start,
                                                             const uint32_t* __restrict__ rmin,
                                                             uint32_t* __restrict__ lab, uint8_t* __restrict__ keep,
                                                             uint8_t* __restrict__ act,
                                                             IterCounters* __restrict__ ctr) {
    uint32_t ablk = 0, surv = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = pos[i] + heads[i] - 1;
        const uint32_t s = run_start[r], e = run_start[r + 1];
        const bool multi = (e - s) >= 2;
        lab[vals[i]] = rmin[r];
        keep[i] = multi;
        if (act) act[vals[i]] = multi;
        ablk += multi && heads[i];
        surv += multi;
    }
    flush_counters<kThreads>(0u, ablk, surv, &ctr->runs, &ctr->active_blocks, &ctr->active_states);
}

// Run labels in one pass, for a stably sorted (key, state) sequence whose
// states were increasing before the sort (the pass's list was): inside a run
// of equal keys the states are still increasing, so the run minimum -- the
// new min-state label of the run's block -- is the state at the run head.
// Every element takes the state of the nearest head at or before it; the
// elements of a tile that continue a run from earlier tiles get its head
// state by decoupled look-back (a tile with a head publishes the state of its
// last head at once; a tile without one publishes "transparent" and, once
// resolved, the state it carried).  Replaces heads + scan + run starts + run
// minima + apply (8 launches, 5 full passes) of the general path.
constexpr int kRunItems = 8;
constexpr int kRunTile = kThreads * kRunItems;
constexpr unsigned long long kRunAgg = 1ull, kRunPre = 2ull;

__global__ void __launch_bounds__(kThreads) run_label_kernel(const uint64_t* __restrict__ keys,
                                                             const uint32_t* __restrict__ vals, uint64_t m,
                                                             unsigned long long* __restrict__ look,
                                                             uint32_t* __restrict__ tile_ctr,
                                                             uint32_t* __restrict__ lab, uint8_t* __restrict__ keep,
                                                             uint8_t* __restrict__ act,
                                                             IterCounters* __restrict__ ctr, int multi_only) {
    __shared__ uint32_t s_tile, s_carry;
    __shared__ uint32_t s_has[kThreads / 32], s_val[kThreads / 32];
    const unsigned lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t i0 = (uint64_t)tile * kRunTile + (uint64_t)threadIdx.x * kRunItems;
    uint64_t key[kRunItems + 2];  // [0] = element i0 - 1, [kRunItems + 1] = element i0 + kRunItems
    uint32_t val[kRunItems];
    if (i0 + kRunItems <= m) {  // a full run of items: 16-byte loads (i0 is a multiple of 8)
#pragma unroll
        for (int j = 0; j < kRunItems; j += 2) {
            const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2*>(keys + i0 + j));
            key[j + 1] = v.x;
            key[j + 2] = v.y;
        }
#pragma unroll
        for (int j = 0; j < kRunItems; j += 4) {
            const uint4 v = __ldcs(reinterpret_cast<const uint4*>(vals + i0 + j));
            val[j] = v.x;
            val[j + 1] = v.y;
            val[j + 2] = v.z;
            val[j + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < kRunItems; ++j) {
            key[j + 1] = i0 + j < m ? __ldcs(keys + i0 + j) : ~0ull;
            val[j] = i0 + j < m ? __ldcs(vals + i0 + j) : 0u;
        }
    }
    // the neighbours' elements: from the adjacent lanes, loaded at warp edges
    {
        const uint64_t up = __shfl_up_sync(0xffffffffu, key[kRunItems], 1);
        const uint64_t dn = __shfl_down_sync(0xffffffffu, key[1], 1);
        key[0] = lane > 0 ? up : (i0 == 0 ? ~0ull : keys[i0 - 1]);
        key[kRunItems + 1] = lane < 31 && i0 + kRunItems < m ? dn
                             : (i0 + kRunItems < m ? keys[i0 + kRunItems] : ~0ull);
    }
    uint32_t head_mask = 0, multi_mask = 0, has = 0, last = 0;
#pragma unroll
    for (int j = 0; j < kRunItems; ++j) {
        const uint64_t i = i0 + j;
        if (i >= m) break;
        const bool head = i == 0 || key[j + 1] != key[j];
        const bool multi = (i > 0 && key[j] == key[j + 1]) || (i + 1 < m && key[j + 2] == key[j + 1]);
        if (head) {
            head_mask |= 1u << j;
            has = 1;
            last = val[j];
        }
        if (multi) multi_mask |= 1u << j;
    }
    // exclusive "last head before me" over the lanes, then over the warps
    uint32_t c_has = 0, c_val = 0;
    {
        uint32_t h = has, v = last;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t hh = __shfl_up_sync(0xffffffffu, h, o), vv = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= (unsigned)o && !h) {
                h = hh;
                v = vv;
            }
        }
        c_has = __shfl_up_sync(0xffffffffu, h, 1);
        c_val = __shfl_up_sync(0xffffffffu, v, 1);
        if (lane == 0) c_has = 0;
        if (lane == 31) {
            s_has[wid] = h;
            s_val[wid] = v;
        }
    }
    __syncthreads();
    if (!c_has) {
        for (int w = (int)wid - 1; w >= 0; --w)
            if (s_has[w]) {
                c_has = 1;
                c_val = s_val[w];
                break;
            }
    }
    if (threadIdx.x == 0) {
        uint32_t t_has = 0, t_val = 0;
        for (int w = kThreads / 32 - 1; w >= 0; --w)
            if (s_has[w]) {
                t_has = 1;
                t_val = s_val[w];
                break;
            }
        volatile unsigned long long* lk = look;
        if (t_has) lk[tile] = (kRunPre << 32) | t_val;
        else lk[tile] = kRunAgg << 32;
        // the carry into this tile (needed unless the tile starts with a head)
        uint32_t carry = 0;
        if (tile > 0 && (head_mask & 1u) == 0) {
            for (int64_t t = (int64_t)tile - 1; t >= 0;) {
                const unsigned long long v = lk[t];
                const unsigned long long f = v >> 32;
                if (f == 0) continue;  // not published yet
                if (f == kRunPre) {
                    carry = (uint32_t)v;
                    break;
                }
                --t;  // transparent: no head there
            }
            if (!t_has) lk[tile] = (kRunPre << 32) | carry;  // resolved: later tiles stop here
        }
        s_carry = carry;
    }
    __syncthreads();
    uint32_t hv = c_has ? c_val : s_carry;
    uint32_t nh = 0, ab = 0, sv = 0;
#pragma unroll
    for (int j = 0; j < kRunItems; ++j) {
        const uint64_t i = i0 + j;
        if (i >= m) break;
        const bool head = (head_mask >> j) & 1u, multi = (multi_mask >> j) & 1u;
        if (head) hv = val[j];
        if (!multi_only || multi) lab[val[j]] = hv;  // (multi_only: singletons hold their own id already)
        if (keep && i0 + kRunItems > m) keep[i] = multi;
        if (act && multi) act[val[j]] = 1;  // act was zeroed
        nh += head;
        ab += head && multi;
        sv += multi;
    }
    if (keep && i0 + kRunItems <= m) {  // the eight flags in one store
        static_assert(kRunItems == 8, "one 8-byte flag store");
        uint64_t f = 0;
#pragma unroll
        for (int j = 0; j < kRunItems; ++j) f |= (uint64_t)((multi_mask >> j) & 1u) << (8 * j);
        *reinterpret_cast<uint64_t*>(keep + i0) = f;
    }
    flush_counters<kThreads>(nh, ab, sv, &ctr->runs, &ctr->active_blocks, &ctr->active_states);
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
    DBuf<uint32_t> lab, lab2, list0, list1, vals0, vals1, heads, pos, run_start, scratch, cur, tmin, tcnt, trank, next32;
    DBuf<uint16_t> next16;
    DBuf<uint32_t> dense32, bits;
    DBuf<uint8_t> dense8;
    DBuf<uint16_t> dense16;
    DBuf<uint64_t> keys0, keys1;
    DBuf<uint8_t> keep, act;
    // bucket strategy
    DBuf<uint32_t> bcnt, rep_slot, gslot, grep, eval;
    DBuf<uint2> rec;
    DBuf<uint8_t> bsingle;
    DBuf<unsigned long long> pack12;  // packed 12-bit key labels of a sliced speculative pass
    DBuf<uint64_t> part;  // partial keys of a sliced pass
    DBuf<uint4> bent;
    DBuf<unsigned long long> gkey;
    DBuf<uint8_t> keep_slot, gmul;
    DBuf<IterCounters> ctr, ctr2;  // ctr2: the counters of a speculative second pass
};

// Key-label array of one pass: min-state labels, or dense block ids in the
// narrowest type.
struct KeyLab {
    const void* p;
    int bytes;
};

constexpr int kBitLabels = (int)kKeylabBits;  // KeyLab::bytes tag: one bit per state

template <typename F>
void with_lab_type(const KeyLab& kl, F&& f) {
    if (kl.bytes == kBitLabels) f(BitLab{static_cast<const uint32_t*>(kl.p)});
    else if (kl.bytes == 1) f(ArrLab<uint8_t>{static_cast<const uint8_t*>(kl.p)});
    else if (kl.bytes == 2) f(ArrLab<uint16_t>{static_cast<const uint16_t*>(kl.p)});
    else f(ArrLab<uint32_t>{static_cast<const uint32_t*>(kl.p)});
}

constexpr int kPack12Labels = 254;  // KeyLab::bytes tags: Pack12Lab / Pack11Lab (signature passes only)
constexpr int kPack11Labels = 253;

double keylab_bytes_per_state(const KeyLab& kl) {
    return kl.bytes == kBitLabels      ? 0.125
           : kl.bytes == kPack12Labels ? 1.6
           : kl.bytes == kPack11Labels ? 1.375
                                       : (double)kl.bytes;
}

// with_lab_type plus the packed labels (the signature paths of big passes)
template <typename F>
void with_lab_type_p12(const KeyLab& kl, F&& f) {
    if (kl.bytes == kPack12Labels) f(Pack12Lab{static_cast<const unsigned long long*>(kl.p)});
    else if (kl.bytes == kPack11Labels) f(Pack11Lab{static_cast<const unsigned long long*>(kl.p)});
    else with_lab_type(kl, f);
}

// Label arrays past the L2 (100M states' 16-bit key labels are 200 MB against
// 126 MB of L2) make every gather of a signature pass a DRAM sector read.
// Such passes gather in sweeps over slices of at most kSliceBytes of labels
// (each L2-resident while its sweep runs), adding partial keys (tuple_part);
// the bucket kernel then only finishes the keys.  DFAKIT_TEST_SLICE_BYTES
// overrides the slice size (tests force slicing on small automata).
// Measured (16-bit labels, 10 letters, no L2 pin): 80 MB unsliced 4.5 ms vs
// 5.3 in 2 slices; 100 MB 6.6 either way; 120 MB 9.1 vs 8.2; 200 MB 19.1
// unsliced, 15.3 in 2 slices, 16.3 in 3, 18.9 in 4 -- a sweep re-reads all
// of delta, so the fewest slices that still mostly hit the L2 win.
constexpr double kSliceBytes = 100.0 * 1024 * 1024;

uint32_t label_slices(const KeyLab& kl, uint32_t n) {
    double slice = kSliceBytes;
    if (const char* e = getenv("DFAKIT_TEST_SLICE_BYTES")) slice = std::max(1.0, atof(e));
    const double bytes = keylab_bytes_per_state(kl) * n;
    return bytes <= slice ? 1u : (uint32_t)std::min<double>(64.0, std::ceil(bytes / slice));
}

// The sweeps of a sliced pass into part[0, m): nullptr when one slice suffices.
const uint64_t* sliced_parts(Ctx* ctx, const KeyLab& kl, const uint32_t* list, uint64_t m, const DevDfa& d,
                             const SigParams& p, DBuf<uint64_t>& part, cudaStream_t s) {
    const uint32_t slices = label_slices(kl, d.n);
    if (slices <= 1 || m == 0) return nullptr;
    if (part.n < m) part.alloc(m, s);
    // DFAKIT_L2_PIN=1: the slice of labels a sweep gathers is pinned in the
    // L2 (access-policy window, persisting) while delta and the partial keys
    // stream past it -- off by default: no gain at 72 MB slices (8.64 vs 8.68
    // ms for 1B transitions), a loss at 100 MB ones (10.6 vs 7.6 ms)
    bool pin = (kl.bytes == 1 || kl.bytes == 2 || kl.bytes == 4) && getenv("DFAKIT_L2_PIN") &&
               getenv("DFAKIT_L2_PIN")[0] == '1';
    size_t pin_max = 0;
    if (pin) {
        int v = 0;
        pin = cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, ctx->device) == cudaSuccess && v > 0 &&
              cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)v) == cudaSuccess;
        pin_max = pin ? (size_t)v : 0;
        if (!pin) (void)cudaGetLastError();
    }
    for (uint32_t j = 0; j < slices; ++j) {
        const uint32_t lo = (uint32_t)((uint64_t)d.n * j / slices), hi = (uint32_t)((uint64_t)d.n * (j + 1) / slices);
        if (pin && pin_max) {
            cudaStreamAttrValue av{};
            av.accessPolicyWindow.base_ptr = const_cast<char*>(static_cast<const char*>(kl.p) + (size_t)lo * kl.bytes);
            av.accessPolicyWindow.num_bytes = std::min<size_t>((size_t)(hi - lo) * kl.bytes, pin_max);
            av.accessPolicyWindow.hitRatio = 1.0f;
            av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            if (cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &av) != cudaSuccess)
                (void)cudaGetLastError();
        }
        const bool vec = !list && d.n % 4 == 0 && p.q0 % 4 == 0;
        // all-letters kernel, one state per thread (1B transitions: 8.87 -> 8.64 ms
        // for the three sweeps; two states per thread 9.20); DFAKIT_PART_KERNEL=0
        // selects the chunked four-state kernel
        static const int part_kernel = getenv("DFAKIT_PART_KERNEL") ? atoi(getenv("DFAKIT_PART_KERNEL")) : 1;
        const bool all_letters = part_kernel > 0 && !list && d.k <= 16;
        if (kl.bytes == kPack12Labels && !all_letters)
            throw Error(DFAKIT_E_INVALID, "packed 12-bit labels need the all-letters sweep kernel");
        with_lab_type_p12(kl, [&](auto lab) {
            using LR = decltype(lab);
            // algorithmic HBM bytes: delta rows, the slice's labels, the partial keys
            const double bytes = (double)m * (4.0 * d.k + (j ? 16.0 : 8.0)) + keylab_bytes_per_state(kl) * (hi - lo);
            const bool fp = p.kind != kKeyPacked;
            if (all_letters) {
                const unsigned grid = grid_for(m, kThreads, (unsigned)ctx->num_sms * 8u);
                auto sweep = [&](auto fpc, auto cc) {
                    constexpr bool FPV = decltype(fpc)::value;
                    constexpr int CV = decltype(cc)::value;
                    DK_LAUNCH_BU(ctx, bytes, (double)m * d.k / slices, (sig_part_all_kernel<LR, FPV, 1, CV>), grid,
                                 kThreads, 0, s, m, d.delta, d.n, lab, p, lo, hi, j == 0 ? 1 : 0, part.get());
                };
                auto by_c = [&](auto fpc) {
                    if (d.k <= 8) sweep(fpc, std::integral_constant<int, 8>{});
                    else if (d.k <= 10) sweep(fpc, std::integral_constant<int, 10>{});
                    else if (d.k <= 12) sweep(fpc, std::integral_constant<int, 12>{});
                    else sweep(fpc, std::integral_constant<int, 16>{});
                };
                if (fp) by_c(std::true_type{});
                else by_c(std::false_type{});
            } else if (vec)
                DK_LAUNCH_BU(ctx, bytes, (double)m * d.k / slices, sig_part_vec_kernel,
                             grid_for((m + 3) / 4, kThreads, (unsigned)ctx->num_sms * 5u), kThreads, 0, s, m, d.delta,
                             d.n, lab, p, lo, hi, j == 0 ? 1 : 0, part.get());
            else
                DK_LAUNCH_BU(ctx, bytes, (double)m * d.k / slices, sig_part_kernel,
                             grid_for(m, kThreads, (unsigned)ctx->num_sms * 8u), kThreads, 0, s, list, m, d.delta,
                             d.n, lab, p, lo, hi, j == 0 ? 1 : 0, part.get());
        });
    }
    if (pin && pin_max) {  // release the window and the persisting lines
        cudaStreamAttrValue av{};
        av.accessPolicyWindow.num_bytes = 0;
        // give the set-aside L2 back to normal accesses (the kernels after
        // the sweeps lost ~10 % with it reserved)
        if (cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &av) != cudaSuccess ||
            cudaCtxResetPersistingL2Cache() != cudaSuccess ||
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0) != cudaSuccess)
            (void)cudaGetLastError();
    }
    return part.get();
}

// ---- persistent small-m engine ---------------------------------------------------
//
// Once few states are active (and on small automata with many passes --
// Fibonacci: one pass per state), a pass is a few microseconds of work and
// the host round trips dominate.  This cooperative kernel runs the remaining
// passes on the device: per pass, insert every active key into a global
// open-addressing table (L2 resident; atomicMin elects the run minimum,
// atomicAdd sizes the run), count heads / active blocks / survivors and
// verify fingerprint runs, then relabel, append survivors and clear the
// other of two tables for the next pass -- three grid barriers.  A verified collision re-runs the pass with a new salt; after
// three in one pass the kernel hands the pass back to the host engine (which
// falls back to exact letter chunks).  Counters are triple-buffered so a
// slot is reset only after every thread has read it.

namespace cg = cooperative_groups;

struct PersistCtr {
    uint32_t runs, ablk, surv, collision, listed, pad[3];
};

struct SmallState {
    uint32_t B, A;
    uint64_t m;
    uint64_t passes, iters, collisions;
    uint32_t list_sel;  // which list buffer holds the active states on exit
    uint32_t status;    // 0 fixed point / drained, 1 hand back (collisions)
    uint64_t salt;
    uint32_t strikes, pad;
};

struct SmallArgs {
    const uint32_t* delta;
    uint32_t n, k;
    uint32_t* lab;
    uint32_t* list[2];
    uint32_t* slot;  // per active entry
    unsigned long long* tkey;  // two tables of tcap + 1 slots
    uint32_t* trep;
    uint32_t* tcnt;
    uint32_t tcap;  // power of two
    PersistCtr* ctr;  // [3]
    SmallState* st;
    uint32_t field_bits;  // packed keys when nonzero
    uint64_t fp_mask;     // fingerprint mask (testing hook)
};

__global__ void __launch_bounds__(kThreads) small_persistent_kernel(SmallArgs A) {
    cg::grid_group grid = cg::this_grid();
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    SmallState s = *A.st;
    uint32_t sel = s.list_sel;
    uint64_t pass_no = 0;  // counter / table slot index
    const uint32_t T = A.tcap;
    s.status = 0;
    // tables alternate by pass: pass p inserts into table p & 1 while the
    // relabel phase of pass p clears table (p + 1) & 1 for the next pass
    for (uint32_t e = tid; e <= T; e += stride) {
        A.tkey[e] = kEmptyKey;
        A.trep[e] = kNone;
        A.tcnt[e] = 0;
    }
    grid.sync();
    while (s.m > 0) {
        PersistCtr* c = A.ctr + (pass_no % 3);
        if (tid == 0) A.ctr[(pass_no + 1) % 3] = PersistCtr{};
        const uint32_t m = (uint32_t)s.m;
        const uint32_t* list = A.list[sel];
        uint32_t* next = A.list[sel ^ 1];
        const uint32_t tb = (uint32_t)(pass_no & 1) * (T + 1);  // this pass's table
        const uint32_t ob = (T + 1) - tb;                       // the other one
        SigParams p{};
        p.kind = A.field_bits ? kKeyPacked : kKeyFingerprint;
        p.a0 = 0;
        p.a1 = A.k;
        p.field_bits = A.field_bits;
        p.salt = s.salt;
        p.fp_mask = A.fp_mask;
        // keys, insert, elect the run minimum, count the run (slot T: a ~0 key)
        for (uint32_t i = tid; i < m; i += stride) {
            const uint32_t q = list[i];
            const uint64_t key = tuple_key<CohLab, 8>(q, A.lab[q], A.delta, A.n, CohLab{A.lab}, p);
            const unsigned long long hk = p.kind == kKeyPacked ? mix64(key) : key;
            uint32_t sl;
            if (hk == kEmptyKey) {
                sl = T;
            } else {
                sl = (uint32_t)mix64(hk) & (T - 1);
                for (;;) {
                    const unsigned long long old = atomicCAS(&A.tkey[tb + sl], kEmptyKey, hk);
                    if (old == kEmptyKey || old == hk) break;
                    sl = (sl + 1) & (T - 1);
                }
            }
            A.slot[i] = tb + sl;
            atomicMin(&A.trep[tb + sl], q);
            atomicAdd(&A.tcnt[tb + sl], 1u);
        }
        grid.sync();
        // counters + fingerprint verification.  Packed keys need no
        // verification, so their relabel, survivor append and clearing of the
        // other table happen in this sweep too (two barriers per pass instead
        // of three): a fixed-point pass rewrites every label with itself and
        // its appended list is never used.
        const bool fused = A.field_bits != 0;
        uint32_t heads = 0, ablk = 0, surv = 0;
        bool clash = false;
        for (uint32_t i = tid; i < m; i += stride) {
            const uint32_t q = list[i], sl = A.slot[i];
            const uint32_t r = __ldcg(&A.trep[sl]);
            const bool multi = __ldcg(&A.tcnt[sl]) >= 2, head = r == q;
            heads += head;
            ablk += head && multi;
            surv += multi;
            if (fused) {
                A.lab[q] = r;
                const uint32_t at = warp_append(&c->listed, multi);
                if (multi) next[at] = q;
            } else if (!head && !same_tuple(q, r, A.delta, A.n, A.k, CohLab{A.lab})) {
                clash = true;
            }
        }
        if (fused)
            for (uint32_t e = tid; e <= T; e += stride) {
                A.tkey[ob + e] = kEmptyKey;
                A.trep[ob + e] = kNone;
                A.tcnt[ob + e] = 0;
            }
        if (__syncthreads_or(clash) && threadIdx.x == 0) atomicOr(&c->collision, 1u);
        flush_counters<kThreads>(heads, ablk, surv, &c->runs, &c->ablk, &c->surv);
        grid.sync();
        // one read per CTA, shared through shared memory (every thread reading
        // the same counters queued thousands of requests on one L2 slice)
        __shared__ PersistCtr s_cv;
        if (threadIdx.x == 0) {
            s_cv.runs = __ldcg(&c->runs);
            s_cv.ablk = __ldcg(&c->ablk);
            s_cv.surv = __ldcg(&c->surv);
            s_cv.collision = __ldcg(&c->collision);
        }
        __syncthreads();
        const PersistCtr cv = s_cv;
        ++s.passes;
        ++pass_no;
        const uint32_t newB = s.B - s.A + cv.runs;
        const bool retry = cv.collision != 0;
        if (!retry && newB == s.B) break;  // fixed point (reference l.411)
        if (retry && s.strikes + 1 >= 3) {
            ++s.collisions;
            --s.passes;
            s.status = 1;  // three collisions: hand the pass back to the host engine
            break;
        }
        // relabel + append survivors (order is free: keys carry the labels);
        // clear the other table for the next pass
        if (!fused) {
            if (!retry) {
                uint32_t* listed = &c->listed;
                for (uint32_t i = tid; i < m; i += stride) {
                    const uint32_t q = list[i], sl = A.slot[i];
                    A.lab[q] = __ldcg(&A.trep[sl]);
                    const bool multi = __ldcg(&A.tcnt[sl]) >= 2;
                    const uint32_t at = warp_append(listed, multi);
                    if (multi) next[at] = q;
                }
            }
            for (uint32_t e = tid; e <= T; e += stride) {
                A.tkey[ob + e] = kEmptyKey;
                A.trep[ob + e] = kNone;
                A.tcnt[ob + e] = 0;
            }
            grid.sync();
        }
        if (retry) {
            ++s.collisions;
            ++s.strikes;
            --s.passes;
            s.salt = mix64(s.salt + 0x1234567ull);
            continue;
        }
        s.strikes = 0;
        ++s.iters;
        s.B = newB;
        s.A = cv.ablk;
        s.m = cv.surv;
        sel ^= 1;
    }
    if (tid == 0) {
        s.list_sel = sel;
        *A.st = s;
    }
}

}  // namespace

LeaderInfo leader_info(Ctx* ctx, const DevDfa& d, cudaStream_t s) {
    uint32_t* info = reinterpret_cast<uint32_t*>(ctx->dmailbox);
    DK_LAUNCH(ctx, leader_info_kernel, grid_for(d.n / 64 + 1, kThreads, (unsigned)ctx->num_sms * 8u), kThreads, 0, s,
              d.acc, d.n, info, (uint8_t*)nullptr, info + 16);
    LeaderInfo li;
    read_words(ctx, info + 16, sizeof(li), &li, s);
    return li;
}

void leader_info_async(Ctx* ctx, const DevDfa& d, cudaStream_t s, uint8_t* dense2) {
    uint32_t* info = reinterpret_cast<uint32_t*>(ctx->dmailbox);
    // ~4 16-byte loads in flight per thread, ~2 CTAs per SM: one round trip
    // to HBM, and few CTAs in the atomic tail
    DK_LAUNCH(ctx, leader_info_kernel, grid_for(d.n / 64 + 1, kThreads, (unsigned)ctx->num_sms * 8u), kThreads, 0, s,
              d.acc, d.n, info, dense2, ctx->fastbox + 120);  // straight into mapped pinned memory
    DK_CUDA(cudaEventRecord(ctx->info_ev, s));
}

LeaderInfo leader_info_wait(Ctx* ctx) {
    DK_CUDA(cudaEventSynchronize(ctx->info_ev));
    LeaderInfo li;
    const volatile uint32_t* v = ctx->fastbox + 120;
    li.min_acc = v[0];
    li.min_rej = v[1];
    li.cnt_acc = v[2];
    li.cnt_rej = v[3];
    return li;
}

void init_leader_labels(Ctx* ctx, const DevDfa& d, const LeaderInfo& li, uint32_t* lab, cudaStream_t s) {
    DK_LAUNCH(ctx, init_labels_kernel, grid_for(d.n), kThreads, 0, s, d.acc, d.n, li.min_acc, li.min_rej, lab);
}

// Key choice of one pass (shared by the single-GPU and the sharded engine):
// min-state labels when they pack, dense block ids (in the narrowest type)
// when only those pack or when they make the counting table possible on a
// large pass -- the dense relabelling is O(n), so it is avoided on small
// late passes -- else fingerprints (narrow dense gathers on large passes),
// else (force_exact / three collisions in one pass) exact letter chunks.
PassPlan plan_pass(uint32_t n, uint32_t k, uint32_t B, uint64_t m, uint32_t collisions, bool force_exact) {
    PassPlan p;
    const uint32_t label_bits = bits_for(n ? n - 1 : 0);
    const uint32_t dense_bits = bits_for(B ? B - 1 : 0);
    const uint64_t k1 = (uint64_t)k + 1;
    const bool big_pass = m >= (uint64_t)n / 16;
    auto narrow = [](uint32_t bits) { return bits <= 8 ? 1u : bits <= 16 ? 2u : 4u; };
    if (k1 * label_bits <= kTableBits) {
        p.strategy = kPlanTable;
        p.field_bits = label_bits;
    } else if (k1 * dense_bits <= kTableBits && big_pass) {
        p.strategy = kPlanTable;
        p.field_bits = dense_bits;
        p.keylab_bytes = narrow(dense_bits);
    } else if (k1 * label_bits <= 64) {
        p.strategy = kPlanPacked;
        p.field_bits = label_bits;
    } else if (k1 * dense_bits <= 64) {
        p.strategy = k1 * dense_bits <= kTableBits ? kPlanTable : kPlanPacked;
        p.field_bits = dense_bits;
        p.keylab_bytes = narrow(dense_bits);
    } else if (!force_exact && collisions < 3) {
        p.strategy = kPlanFingerprint;
        if (dense_bits <= 16 && big_pass) p.keylab_bytes = narrow(dense_bits);
    } else {
        p.strategy = kPlanChunked;
        p.field_bits = dense_bits;
        p.keylab_bytes = 4;
    }
    p.key_bits = p.strategy == kPlanFingerprint ? 64u : (uint32_t)(k1 * p.field_bits);
    return p;
}

namespace {

constexpr uint64_t kSmallPersistMax = 1u << 17;

struct SmallRun {
    SmallState st;
    const uint32_t* list_out;
};

SmallRun run_small_persistent(Ctx* ctx, const DevDfa& d, uint32_t* lab, uint32_t* list_in, uint32_t* list_other,
                              uint64_t m, uint32_t B, uint32_t A, uint64_t salt, uint64_t fp_mask, cudaStream_t s) {
    const uint32_t n = d.n, k = d.k;
    const uint32_t label_bits = bits_for(n ? n - 1 : 0);
    const uint32_t field_bits = (uint64_t)(k + 1) * label_bits <= 64 ? label_bits : 0;
    uint32_t T = 64;
    while (T < 2 * m) T <<= 1;
    DBuf<uint32_t> slot(m, s), trep(2 * (T + 1), s), tcnt(2 * (T + 1), s);
    DBuf<unsigned long long> tkey(2 * (T + 1), s);
    DBuf<PersistCtr> ctr(3, s);
    DBuf<SmallState> st(1, s);
    DK_CUDA(cudaMemsetAsync(ctr.get(), 0, 3 * sizeof(PersistCtr), s));
    SmallState hs{};
    hs.B = B;
    hs.A = A;
    hs.m = m;
    hs.salt = salt;
    hs.list_sel = 0;
    DK_CUDA(cudaMemcpyAsync(st.get(), &hs, sizeof(hs), cudaMemcpyHostToDevice, s));
    SmallArgs args{d.delta, n, k, lab, {list_in, list_other}, slot.get(), tkey.get(), trep.get(), tcnt.get(), T,
                   ctr.get(), st.get(), field_bits, fp_mask};
    int per_sm = 0;
    DK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, small_persistent_kernel, kThreads, 0));
    if (per_sm < 1) throw Error(DFAKIT_E_RESOURCE, "persistent sort_pr kernel does not fit an SM");
    const uint64_t want = (m + kThreads - 1) / kThreads;
    // one state per thread up to every resident CTA (a pass is a dependent
    // chain per state: more CTAs beat the cheaper barrier of a smaller grid)
    const unsigned grid =
        (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)ctx->num_sms * (uint64_t)per_sm));
    void* kargs[] = {(void*)&args};
    prof_begin_launch(ctx, s);
    DK_CUDA(cudaLaunchCooperativeKernel((const void*)small_persistent_kernel, grid, kThreads, kargs, 0, s));
    note_launch(ctx);
    prof_end_launch(ctx, s, "small_persistent_kernel", 0, 0);
    SmallRun r;
    read_words(ctx, st.get(), sizeof(SmallState), &r.st, s);
    r.list_out = r.st.list_sel ? list_other : list_in;
    return r;
}

}  // namespace

RefineResult sort_pr_device(Ctx* ctx, const DevDfa& d, const SortOptions& o, uint32_t* block_out, cudaStream_t s,
                            const DeltaStream* ds) {
    RefineResult res;
    const uint32_t n = d.n, k = d.k;
    if (n == 0) return res;
    Workspace w;
    w.lab.alloc(n, s);
    w.list0.alloc(n, s);
    w.list1.alloc(n, s);
    w.scratch.alloc((uint64_t)n + 1, s);
    w.keep.alloc(n, s);
    w.ctr.alloc(1, s);
    w.ctr2.alloc(1, s);
    DK_CUDA(cudaFuncSetAttribute(bucket_group_kernel<ArrLab<uint32_t>, OneSrc>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(GroupSmem)));
    DK_CUDA(cudaFuncSetAttribute(bucket_group_kernel<ArrLab<uint32_t>, OneSrc, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(GroupSmem)));
    const int smem_table = (int)(2u << kSmemTableBits) * 4;
    DK_CUDA(cudaFuncSetAttribute(sig_table_kernel<BitLab>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_table));
    DK_CUDA(cudaFuncSetAttribute(sig_table_kernel<ArrLab<uint8_t>>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_table));
    DK_CUDA(cudaFuncSetAttribute(sig_table_kernel<ArrLab<uint16_t>>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_table));
    DK_CUDA(cudaFuncSetAttribute(sig_table_kernel<ArrLab<uint32_t>>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_table));
    IterCounters* dctr = w.ctr.get();

    // initial partition {F, Q\F} with min-state labels.
    // Large automata whose first pass is a counting-table pass with dense key
    // labels (taken from the flags) run that pass over every state without
    // waiting for the class sizes: the pass overwrites every label (the
    // initial min-state labels are never read), and a singleton or empty
    // class only adds its own single-member run, so with A = B (every
    // nonempty class counted active) B - A + runs, the survivors and the pass
    // count are those of the reference's pass over the non-singleton
    // classes.  The class sizes are read after the pass is queued.
    const bool streamed_in = ds && ds->chunks;
    const PassPlan p_full = plan_pass(n, k, 2, n, 0, o.force_exact);
    const bool deferred_info = !streamed_in && (uint64_t)n > kSmallPersistMax && o.grouping != 1 && !o.force_exact &&
                               p_full.strategy == kPlanTable && p_full.keylab_bytes != 0;
    LeaderInfo li{};
    uint32_t B, A;
    uint64_t m;
    bool dense8_ready = false;  // the first pass's byte key labels, written by the class-size kernel
    if (deferred_info) {
        if (n < kBitLabelsMinStates) {
            w.dense8.alloc(n, s);
            dense8_ready = true;
        }
        leader_info_async(ctx, d, s, dense8_ready ? w.dense8.get() : nullptr);
        B = 2;  // the plan's assumption; corrected from the counts after the pass
        A = 2;
        m = n;
    } else {
        li = leader_info(ctx, d, s);
        B = (li.min_acc != kNone) + (li.min_rej != kNone);
        A = (li.cnt_acc >= 2) + (li.cnt_rej >= 2);
        m = (li.cnt_acc >= 2 ? li.cnt_acc : 0) + (li.cnt_rej >= 2 ? li.cnt_rej : 0);
        // a first pass over every state with the counting table and dense key
        // labels overwrites every label: no initial labels then
        const PassPlan p0 = plan_pass(n, k, B, m, 0, o.force_exact);
        const bool small_first = m <= kSmallPersistMax && o.grouping == 0 && !o.force_exact;
        const bool skip_init = m == n && !small_first && o.grouping != 1 && p0.strategy == kPlanTable &&
                               p0.keylab_bytes != 0;
        if (!skip_init) init_leader_labels(ctx, d, li, w.lab.get(), s);
    }
    const uint32_t* list = nullptr;  // nullptr = identity (all states active)
    uint32_t* list_buf = w.list0.get();
    uint32_t* list_alt = w.list1.get();
    if (m != n && m != 0) {
        DBuf<uint8_t> f(n, s);
        DK_LAUNCH(ctx, init_active_flags_kernel, grid_for(n), kThreads, 0, s, d.acc, n, (uint8_t)(li.cnt_acc >= 2),
                  (uint8_t)(li.cnt_rej >= 2), f.get());
        compact_flags(ctx, nullptr, f.get(), n, list_buf, &dctr->listed, s);
        list = list_buf;
    }

    uint64_t salt = 0x5eed5eed5eedull;
    bool next_valid = false;  // next16 / next32 hold compact block ids of the current partition
    uint32_t prev_nbits = 0;
    const uint64_t fp_mask = o.fingerprint_bits >= 64 ? ~0ull : ((1ull << o.fingerprint_bits) - 1ull);
    uint32_t collisions_this_pass = 0;
    bool all_survive = false;
    // the active list is in increasing state order (identity, flag
    // compactions in state order, and order-preserving table compactions);
    // lists in bucket-slot or sorted order clear it
    bool list_inc = true;
    // Speculative second pass: a first pass over every state with a counting
    // table already wrote the next key labels (table ranks) and labels when
    // its counters are still on their way to the host; the second pass -- a
    // fingerprint bucket pass over every state, the plan every wide second
    // pass can take -- is queued right behind it instead of after the
    // readback (one host round trip less between the passes).  It defers its
    // labels (nothing is applied before its counters are read), so a pass-1
    // fixed point or survivors that make it moot just drop it.
    bool spec_launched = false;
    bool iota_out = false;  // block_out holds the identity numbering (queued speculatively)
    // lab_pending: pass 1 (a counting-table pass over every state, every
    // state surviving) skipped its per-state apply -- its labels are
    // tmin[heads[q]], materialised by `materialise` only if something reads
    // them; meanwhile the raw table keys (heads) label the blocks
    bool lab_pending = false;
    std::function<void()> materialise;
    PassPlan spec_plan{};
    KeyLab spec_kl{nullptr, 0};
    // DFAKIT_TEST_SPEC_MIN=<states> lowers the threshold (tests), DFAKIT_NO_SPEC=1 disables it
    const char* spec_min_env = getenv("DFAKIT_TEST_SPEC_MIN");
    const uint64_t spec_min = spec_min_env ? strtoull(spec_min_env, nullptr, 10) : kSpecMinStates;
    const bool spec_ok = !(ds && ds->chunks) && o.grouping == 0 && !o.force_exact && n >= spec_min &&
                         n < 0x80000000u && !getenv("DFAKIT_NO_SPEC");

    // bucket strategy: 2^D buckets of 768..1536 expected keys (Poisson tail
    // well inside the 2048 slots unless keys repeat).  Big passes flag
    // survivors per state (the next list comes out sorted, so its delta
    // reads stay coalesced) and write labels in place (exact keys); big
    // fingerprint passes defer their labels: packed per-slot records
    // (coalesced) applied after verification -- and not at all when every
    // block came out a singleton (the usual last pass: 4-byte label stores to
    // random states cost as much as the rest of the grouping); small passes
    // keep per-slot outputs and apply fingerprint labels afterwards
    auto bucket_layout = [&](bool fingerprint, uint64_t mm) {
        BucketLayout L;
        uint32_t D = 1;
        while (D < 24 && ((uint64_t)1 << D) * (kGrpCap * 3 / 4) < mm) ++D;
        L.nb = 1u << D;
        L.bspace = (uint64_t)L.nb * kGrpCap;
        L.espace = L.bspace + mm;
        L.state_order = mm >= (uint64_t)n / 16;
        L.defer = fingerprint && L.state_order && n < 0x80000000u;
        L.direct = (!fingerprint || L.state_order) && !L.defer;
        return L;
    };
    // allocations, the pass prologue's fills, signature + bucket append,
    // grouping (counters into ctrx)
    auto bucket_launch = [&](const PassPlan& pl, const KeyLab& klx, const SigParams& px, const uint32_t* lst,
                             uint64_t mm, IterCounters* ctrx, Fills& fl, const uint32_t* vlab) {
        const bool fingerprint = pl.strategy == kPlanFingerprint;
        const BucketLayout L = bucket_layout(fingerprint, mm);
        if (w.bcnt.n < (uint64_t)L.nb * kCntStride) w.bcnt.alloc((uint64_t)L.nb * kCntStride, s);
        if (w.bent.n < L.espace) {
            w.bent.alloc(L.espace, s);
            w.keep_slot.alloc(L.espace, s);
        }
        if (!L.direct && !L.defer && w.rep_slot.n < L.espace) w.rep_slot.alloc(L.espace, s);
        if (L.defer && w.rec.n < L.espace) w.rec.alloc(L.espace, s);
        if (L.defer && w.bsingle.n < L.nb) w.bsingle.alloc(L.nb, s);
        if (L.state_order && !w.act.get()) w.act.alloc(n, s);
        if (fingerprint && L.direct) {
            if (!w.lab2.get()) w.lab2.alloc(n, s);
            // a pass over every state writes every label of the copy
            if (lst) DK_CUDA(cudaMemcpyAsync(w.lab2.get(), w.lab.get(), (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
        }
        uint32_t* out_lab = fingerprint && L.direct ? w.lab2.get() : w.lab.get();
        fl.add(w.bcnt.get(), (size_t)L.nb * kCntStride * 4, 0);
        // (deferred passes flag survivors in rec_apply_kernel, which zeroes
        // act itself when it runs -- not at all in the usual all-singleton pass)
        if (L.state_order && !L.defer) fl.add(w.act.get(), n, 0);
        if (!L.state_order) fl.add(w.keep_slot.get(), L.espace, 0);
        fl.flush(ctx, s);
        const double lb = lst ? 4.0 : 0.0;
        const uint64_t* part = sliced_parts(ctx, klx, lst, mm, d, px, w.part, s);
        with_lab_type_p12(klx, [&](auto lab) {
            using LR = decltype(lab);
            // algorithmic HBM bytes: delta rows (+ list), (hkey, state) out, the key-label array once
            // (a sliced pass: the partial keys in, hkey out)
            const double bytes = part ? (double)mm * 24.0
                                      : (double)mm * (4.0 * k + 16.0 + lb) + keylab_bytes_per_state(klx) * n;
            const unsigned grid = grid_for(mm, kSigbThreads, (unsigned)ctx->num_sms * DFAKIT_SIGB_GRID);
            if (part)
                DK_LAUNCH_BU(ctx, bytes, 0.0, (sig_bucket_kernel<LR, 2>), grid, kSigbThreads, 0, s, lst, mm, d.delta, n, lab, px,
                             L.nb, w.bcnt.get(), w.bent.get(), ctrx, part);
            else if (fingerprint)
                DK_LAUNCH_BU(ctx, bytes, (double)mm * k, (sig_bucket_kernel<LR, 1>), grid, kSigbThreads, 0, s, lst, mm, d.delta, n,
                             lab, px, L.nb, w.bcnt.get(), w.bent.get(), ctrx, part);
            else
                DK_LAUNCH_BU(ctx, bytes, (double)mm * k, (sig_bucket_kernel<LR, 0>), grid, kSigbThreads, 0, s, lst, mm, d.delta, n,
                             lab, px, L.nb, w.bcnt.get(), w.bent.get(), ctrx, part);
        });
        GroupOut go{L.direct ? 1 : 0, L.state_order ? 1 : 0, out_lab, w.act.get(),
                    L.direct || L.defer ? nullptr : w.rep_slot.get(), w.keep_slot.get(), nullptr,
                    L.defer ? w.rec.get() : nullptr, 0, w.bsingle.get()};
        const unsigned gg = (unsigned)std::min<uint64_t>(L.nb, (uint64_t)ctx->num_sms * kGrpCtasPerSm);
        // algorithmic HBM bytes: (hkey, state) in, label + survivor flag out
        const double gbytes = (double)mm * (16.0 + 4.0 + 1.0 + (L.direct ? 0.0 : 4.0));
        if (L.defer)  // deferred records (fingerprints): the output mode fixed at compile time
            DK_LAUNCH_B(ctx, gbytes, (bucket_group_kernel<ArrLab<uint32_t>, OneSrc, 1>), gg, kGrpThreads,
                        sizeof(GroupSmem), s, OneSrc{w.bcnt.get(), w.bent.get()}, L.nb, 1, d.delta, n, k,
                        ArrLab<uint32_t>{vlab}, go, ctrx);
        else
            DK_LAUNCH_B(ctx, gbytes, bucket_group_kernel, gg, kGrpThreads, sizeof(GroupSmem), s,
                        OneSrc{w.bcnt.get(), w.bent.get()}, L.nb, fingerprint ? 1 : 0, d.delta, n, k,
                        ArrLab<uint32_t>{vlab}, go, ctrx);
    };

    auto dense_keylab = [&](int bytes) -> KeyLab {
        void* p;
        if (bytes == 1) {
            if (!w.dense8.get()) w.dense8.alloc(n, s);
            p = w.dense8.get();
        } else if (bytes == 2) {
            if (!w.dense16.get()) w.dense16.alloc(n, s);
            p = w.dense16.get();
        } else {
            if (!w.dense32.get()) w.dense32.alloc(n, s);
            p = w.dense32.get();
        }
        dense_labels(ctx, w.lab.get(), n, p, bytes, w.scratch.get(), s);
        return KeyLab{p, bytes};
    };

    // streamed input: which chunks the compute stream has waited for
    uint32_t* bad = reinterpret_cast<uint32_t*>(ctx->dmailbox) + 40;
    bool streamed = ds && ds->chunks;
    auto check_streamed = [&] {
        if (!streamed) return;
        uint32_t b = 0;
        read_words(ctx, bad, 4, &b, s);
        if (b) throw Error(DFAKIT_E_INVALID, "delta: transition target out of range");
        streamed = false;
    };
    // paths other than the chunked pass 1 take the whole input, validated
    // before any kernel reads it
    auto wait_all_chunks = [&] {
        if (!streamed) return;
        for (uint32_t c = 0; c < ds->chunks; ++c) DK_CUDA(cudaStreamWaitEvent(s, ds->ready[c], 0));
        DK_CUDA(cudaMemsetAsync(bad, 0, 4, s));
        range_check_rows(ctx, d.delta, n, k, 0u, n, bad, s);
        check_streamed();
    };
    while (m > 0) {
        // few active states: the remaining passes on the device (no host
        // round trip per pass); a pass with three collisions comes back here
        if (m <= kSmallPersistMax && o.grouping == 0 && !o.force_exact && collisions_this_pass == 0) {
            wait_all_chunks();
            check_streamed();
            const bool identity = list == nullptr;
            if (identity) {  // materialise the identity list
                iota_u32(ctx, list_buf, m, s);
                list = list_buf;
            }
            SmallRun sr = run_small_persistent(ctx, d, w.lab.get(), list == list_buf ? list_buf : list_alt,
                                               list == list_buf ? list_alt : list_buf, m, B, A, salt, fp_mask, s);
            res.passes += sr.st.passes;
            res.iters += sr.st.iters;
            res.collisions += sr.st.collisions;
            B = sr.st.B;
            A = sr.st.A;
            m = sr.st.m;
            salt = sr.st.salt;
            if (sr.st.status == 0) break;  // fixed point reached on the device
            // three collisions: the host engine takes the pass
            list = sr.list_out;
            if (list == list_alt) std::swap(list_buf, list_alt);
            list_inc = false;
            collisions_this_pass = 3;
        }
        ++res.passes;
        ctx->prof_pass = (uint32_t)res.passes;  // profiler: this pass's launches
        // a speculative pass launched behind the previous one is used when
        // that pass left every state active (it then covered exactly this
        // pass's states); otherwise its work is dropped (it applied nothing)
        const bool use_spec = spec_launched && list == nullptr && m == n && collisions_this_pass == 0;
        spec_launched = false;
        const PassPlan plan = use_spec ? spec_plan : plan_pass(n, k, B, m, collisions_this_pass, o.force_exact);
        const bool fingerprint = plan.strategy == kPlanFingerprint, chunked = plan.strategy == kPlanChunked;
        const uint32_t field_bits = plan.field_bits;
        KeyLab kl{w.lab.get(), 4};
        if (use_spec) {
            kl = spec_kl;
        } else if (plan.keylab_bytes) {
            if (next_valid && plan.strategy != kPlanChunked) {
                kl = w.next16.get() && prev_nbits <= 16 ? KeyLab{w.next16.get(), 2} : KeyLab{w.next32.get(), 4};
            } else if (B <= 2 && plan.strategy != kPlanChunked && n >= kBitLabelsMinStates) {
                if (!w.bits.get()) w.bits.alloc((n + 31) / 32, s);
                if (res.iters == 0)  // still the initial partition: from the flags
                    DK_LAUNCH(ctx, acc_dense2_bits_kernel, grid_for((uint64_t)n), kThreads, 0, s, d.acc, n,
                              w.bits.get());
                else
                    DK_LAUNCH(ctx, dense2_bits_kernel, grid_for((uint64_t)n), kThreads, 0, s, w.lab.get(), n,
                              w.bits.get());
                kl = KeyLab{w.bits.get(), kBitLabels};
            } else if (B <= 2 && plan.strategy != kPlanChunked) {
                if (!w.dense8.get()) w.dense8.alloc(n, s);
                if (res.iters != 0)
                    DK_LAUNCH(ctx, dense2_kernel, grid_for(n), kThreads, 0, s, w.lab.get(), n, w.dense8.get());
                else if (!dense8_ready)  // else written with the class sizes
                    DK_LAUNCH(ctx, acc_dense2_kernel, grid_for(n), kThreads, 0, s, d.acc, n, w.dense8.get());
                kl = KeyLab{w.dense8.get(), 1};
            } else {
                kl = dense_keylab(plan.keylab_bytes);
            }
        }
        next_valid = false;
        Fills fills;  // the pass prologue's fills, one launch before its first kernel
        fills.add(dctr, sizeof(IterCounters), 0);
        const unsigned g = grid_for(m);
        const uint32_t nbits = plan.key_bits;
        SigParams p{};
        p.kind = fingerprint ? kKeyFingerprint : kKeyPacked;
        p.a0 = 0;
        p.a1 = k;
        p.field_bits = field_bits;
        p.salt = salt;
        p.fp_mask = fp_mask;
        const double list_b = list ? 4.0 : 0.0;
        IterCounters c{};
        uint32_t* dst = (list == list_buf) ? list_alt : list_buf;

        if (plan.strategy == kPlanTable && o.grouping != 1) {
            // ---- table strategy
            const uint64_t tsize = 1ull << nbits;
            if (w.tmin.n < tsize) {
                w.tmin.alloc(tsize, s);
                w.tcnt.alloc(tsize, s);
            }
            if (!w.heads.get()) w.heads.alloc((uint64_t)n + 1, s);
            fills.add(w.tmin.get(), tsize * sizeof(uint32_t), 0xff);
            fills.add(w.tcnt.get(), tsize * sizeof(uint32_t), 0);
            fills.flush(ctx, s);
            const bool local = nbits <= kSmemTableBits;
            const size_t smem = local ? (size_t)(2u << nbits) * 4 : 0;
            const int inc = list == nullptr || list_inc ? 1 : 0;
            // a table pass over every state sees every block of the next
            // partition as one table key: the ranks of the occupied entries
            // are compact block ids, the next pass's key labels (no O(n) scan)
            const bool full = list == nullptr;
            auto a16 = [](const void* x) { return ((uintptr_t)x & 15u) == 0; };
            if (full) {
                if (nbits <= 16 && !w.next16.get()) w.next16.alloc(n, s);
                if (nbits > 16 && !w.next32.get()) w.next32.alloc(n, s);
            }
            const bool vec = full && a16(w.heads.get()) && a16(w.lab.get()) && a16(w.keep.get()) &&
                             a16(nbits <= 16 ? (void*)w.next16.get() : (void*)w.next32.get());
            const bool staged = vec && tsize <= kApplyStageMax;  // ranks computed by the apply kernel
            // lazy: the second pass is queued speculatively on the raw table
            // keys (every block of the next partition is one key; written as
            // 16-bit labels by the signature kernel), and the per-state apply
            // only runs when its outputs are needed
            const bool lazy = spec_ok && staged && nbits <= 16 && res.passes == 1 && collisions_this_pass == 0 &&
                              !streamed;
            uint16_t* keys16 = lazy ? w.next16.get() : nullptr;
            auto sig_table = [&](uint32_t q0, uint64_t mm, bool clamp) {
                const unsigned tg = (unsigned)std::min<uint64_t>((mm + kSigtThreads - 1) / kSigtThreads,
                                                                 (uint64_t)ctx->num_sms * kSigtCtas);
                SigParams pc = p;
                pc.q0 = q0;
                with_lab_type(kl, [&](auto lab) {
                    using LR = decltype(lab);
                    // algorithmic HBM bytes: delta rows + key out (+ list), the key-label array once
                    const double bytes = (double)mm * (4.0 + 4.0 * k + list_b) + keylab_bytes_per_state(kl) * n;
                    if (clamp) {
                        auto sig_table_clamped_kernel = sig_table_kernel<LR, true>;
                        DK_CUDA(cudaFuncSetAttribute(sig_table_clamped_kernel,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)(2u << kSmemTableBits) * 4));
                        DK_LAUNCH_BU(ctx, bytes, (double)mm * k, sig_table_clamped_kernel, tg, kSigtThreads, smem, s, list,
                                     mm, d.delta, n, lab, pc, nbits, w.heads.get() + q0, w.tmin.get(), w.tcnt.get(),
                                     inc, keys16 ? keys16 + q0 : nullptr);
                    } else {
                        DK_LAUNCH_BU(ctx, bytes, (double)mm * k, sig_table_kernel<LR>, tg, kSigtThreads, smem, s, list, mm,
                                     d.delta, n, lab, pc, nbits, w.heads.get() + q0, w.tmin.get(), w.tcnt.get(),
                                     inc, keys16 ? keys16 + q0 : nullptr);
                    }
                });
            };
            if (streamed && list == nullptr) {
                // pass 1 chunk by chunk as delta arrives
                DK_CUDA(cudaMemsetAsync(bad, 0, 4, s));
                for (uint32_t c = 0; c < ds->chunks; ++c) {
                    const uint32_t q0 = ds->bounds[c], q1 = ds->bounds[c + 1];
                    DK_CUDA(cudaStreamWaitEvent(s, ds->ready[c], 0));
                    if (q1 == q0) continue;
                    range_check_rows(ctx, d.delta, n, k, q0, q1, bad, s);
                    sig_table(q0, q1 - q0, true);
                }
            } else {
                wait_all_chunks();
                sig_table(0, m, false);
            }
            auto apply_table = [&, vec, staged, full, nbits, tsize, g, list, m, list_b]() {
            if (full) {
                if (w.trank.n < tsize) w.trank.alloc(tsize, s);
                if (staged) {
                    // ranks computed inside the apply kernel (w.trank only flags "full")
                } else if (tsize <= (1u << 14)) {
                    DK_LAUNCH(ctx, table_rank_one_kernel, 1, 1024, 0, s, w.tcnt.get(), (uint32_t)tsize, w.trank.get());
                } else {
                    DK_LAUNCH(ctx, table_occupied_kernel, grid_for(tsize), kThreads, 0, s, w.tcnt.get(),
                              (uint32_t)tsize, w.trank.get());
                    exclusive_scan_u32(ctx, w.trank.get(), w.trank.get(), tsize, nullptr, s);
                }
            }
            if (staged)  // identity list, four states per thread, tables in smem
                DK_LAUNCH_B(ctx, (double)m * (9.0 + (nbits <= 16 ? 2.0 : 4.0)), table_apply_vec_kernel<true>,
                            grid_for((m + 3) / 4, kThreads, (unsigned)ctx->num_sms * 4u), kThreads, 0, s,
                            w.heads.get(), m, w.tmin.get(), w.tcnt.get(), w.lab.get(), w.keep.get(), w.trank.get(),
                            nbits <= 16 ? w.next16.get() : nullptr, nbits > 16 ? w.next32.get() : nullptr, dctr,
                            (uint32_t)tsize);
            else if (vec)  // identity list, four states per thread
                DK_LAUNCH_B(ctx, (double)m * (9.0 + (nbits <= 16 ? 2.0 : 4.0)), table_apply_vec_kernel<false>,
                            grid_for((m + 3) / 4), kThreads, 0, s, w.heads.get(), m, w.tmin.get(), w.tcnt.get(),
                            w.lab.get(), w.keep.get(), w.trank.get(), nbits <= 16 ? w.next16.get() : nullptr,
                            nbits > 16 ? w.next32.get() : nullptr, dctr, (uint32_t)tsize);
            else
                DK_LAUNCH_B(ctx, (double)m * (9.0 + 2 * list_b), table_apply_kernel, g, kThreads, 0, s, list,
                            w.heads.get(), m, w.tmin.get(), w.tcnt.get(), w.lab.get(), w.keep.get(), nullptr,
                            full ? w.trank.get() : nullptr, full && nbits <= 16 ? w.next16.get() : nullptr,
                            full && nbits > 16 ? w.next32.get() : nullptr, 0u, dctr);
            };
            if (lazy) {
                DK_LAUNCH(ctx, table_counts_kernel, 1, 1024, 0, s, w.tcnt.get(), (uint32_t)tsize, dctr);
            } else {
                apply_table();
                next_valid = full;
                prev_nbits = nbits;
            }
            if (spec_ok && full && nbits <= 16 && res.passes == 1 && collisions_this_pass == 0) {
                // the second pass, queued before this pass's readback: a
                // fingerprint bucket pass over every state on the table ranks
                // (or the raw table keys when the apply is skipped)
                spec_plan = PassPlan{};
                spec_plan.strategy = kPlanFingerprint;
                spec_plan.key_bits = 64;
                spec_plan.keylab_bytes = 2;
                spec_kl = KeyLab{w.next16.get(), 2};  // the ranks, or the raw keys when the apply is skipped
                // raw keys of at most 12 bits for a big second pass: packed
                // when that keeps its labels L2-friendlier (see pack_choice)
                const int pack = lazy && k <= 16 ? pack_choice(n, nbits) : 0;
                if (pack) {
                    if (w.pack12.n < pack_words(n)) w.pack12.alloc(pack_words(n), s);
                    const uint32_t tag = pack12_labels(ctx, w.next16.get(), n, w.pack12.get(), s, pack == 11);
                    spec_kl = KeyLab{w.pack12.get(), (int)tag};
                }
                SigParams sp{};
                sp.kind = kKeyFingerprint;
                sp.a0 = 0;
                sp.a1 = k;
                sp.salt = salt;
                sp.fp_mask = fp_mask;
                Fills sf;
                sf.add(w.ctr2.get(), sizeof(IterCounters), 0);
                ctx->prof_pass = (uint32_t)res.passes + 1;
                bucket_launch(spec_plan, spec_kl, sp, nullptr, n, w.ctr2.get(), sf, lazy ? w.heads.get() : w.lab.get());
                ctx->prof_pass = (uint32_t)res.passes;
                spec_launched = true;
            }
            // every state survives (the first pass of a random automaton):
            if (deferred_info && res.passes == 1) {  // the class sizes, read while the pass ran
                li = leader_info_wait(ctx);
                B = (li.min_acc != kNone) + (li.min_rej != kNone);
                A = B;
            }
            read_words(ctx, dctr, sizeof(c), &c, s);
            if (lazy) {
                if (!list && c.active_states == m && B - A + c.runs != B) {
                    // every state survives and the pass split: the speculative
                    // second pass on the raw keys is the next pass
                    lab_pending = true;
                    materialise = [apply_table, nbits, &next_valid, &prev_nbits, &lab_pending]() {
                        apply_table();
                        next_valid = true;
                        prev_nbits = nbits;
                        lab_pending = false;
                    };
                } else {
                    apply_table();  // labels, survivor flags and ranks now (counters unchanged)
                    next_valid = full;
                    prev_nbits = nbits;
                }
            }
            // compaction after the readback: when every state survives the
            // identity list stays and nothing is launched (three launches of
            // ~2.4K CTAs that would only exit cost ~25 us)
            if (!list && c.active_states == m) all_survive = true;
            else if (c.active_states && B - A + c.runs != B) compact_flags(ctx, list, w.keep.get(), m, dst, &dctr->listed, s);
        } else if (!chunked && o.grouping != 1) {
            wait_all_chunks();
            // ---- bucket strategy
            const BucketLayout L = bucket_layout(fingerprint, m);
            const uint32_t nb = L.nb;
            const uint64_t bspace = L.bspace, espace = L.espace;
            const bool state_order = L.state_order, defer = L.defer, direct = L.direct;
            IterCounters* pctr = use_spec ? w.ctr2.get() : dctr;  // the counters this pass's kernels wrote
            if (!use_spec) bucket_launch(plan, kl, p, list, m, dctr, fills, w.lab.get());
            // verification labels: any injective labelling of the current blocks
            const uint32_t* vlab = lab_pending ? w.heads.get() : w.lab.get();
            uint32_t* out_lab = fingerprint && direct ? w.lab2.get() : w.lab.get();
            GroupOut go{direct ? 1 : 0, state_order ? 1 : 0, out_lab, w.act.get(),
                        direct || defer ? nullptr : w.rep_slot.get(), w.keep_slot.get(), nullptr,
                        defer ? w.rec.get() : nullptr, 0};
            {
                const uint32_t seq = read_words_begin(ctx, pctr, sizeof(c), s);
                // a deferred pass over every state is usually the last one,
                // leaving every block a singleton: the identity numbering is
                // queued while the host waits for the counters (the final
                // numbering overwrites it otherwise)
                if (defer && m == n && !iota_out) {
                    iota_u32(ctx, block_out, n, s);
                    iota_out = true;
                }
                read_words_end(ctx, seq, sizeof(c), &c, s);
            }
            if (c.overflow) {
                // heavy duplication: overflowed buckets through a global table
                uint64_t T = 2;
                while (T < 2 * (uint64_t)m) T <<= 1;
                if (w.gkey.n < T + 1) {
                    w.gkey.alloc(T + 1, s);
                    w.grep.alloc(T + 1, s);
                    w.gmul.alloc(T + 1, s);
                }
                if (w.gslot.n < espace) w.gslot.alloc(espace, s);
                DK_CUDA(cudaMemsetAsync(w.gkey.get(), 0xff, (T + 1) * 8, s));
                DK_CUDA(cudaMemsetAsync(w.grep.get(), 0xff, (T + 1) * 4, s));
                DK_CUDA(cudaMemsetAsync(w.gmul.get(), 0, T + 1, s));
                const unsigned eg = grid_for(bspace + c.overflow);
                DK_LAUNCH(ctx, ghash_insert_kernel, eg, kThreads, 0, s, w.bcnt.get(), nb, c.overflow, w.bent.get(), T,
                          w.gkey.get(), w.grep.get(), w.gslot.get());
                DK_LAUNCH(ctx, ghash_multi_kernel, eg, kThreads, 0, s, w.bcnt.get(), nb, c.overflow, w.bent.get(),
                          w.grep.get(), w.gslot.get(), w.gmul.get());
                DK_LAUNCH(ctx, ghash_out_kernel, eg, kThreads, 0, s, w.bcnt.get(), nb, c.overflow, w.bent.get(),
                          w.grep.get(), w.gslot.get(), w.gmul.get(), fingerprint ? 1 : 0, d.delta, n, k,
                          ArrLab<uint32_t>{vlab}, go, pctr);
                read_words(ctx, pctr, sizeof(c), &c, s);
            }
            res.sorted += m;
            check_streamed();
            if (fingerprint && c.collision) {
                // verified collision: nothing was written to the labels
                ++res.collisions;
                ++collisions_this_pass;
                --res.passes;
                salt = mix64(salt + 0x1234567ull);
                if (lab_pending) materialise();  // the retry plans on the labels
                continue;
            }
            collisions_this_pass = 0;
            if (B - A + c.runs == B) {  // fixed point (reference l.411)
                if (lab_pending) materialise();
                break;
            }
            if (fingerprint && direct) std::swap(w.lab, w.lab2);
            if (defer) {
                if (B - A + c.runs != n) {
                    // (a pass over every state: every label is rewritten)
                    DK_CUDA(cudaMemsetAsync(w.act.get(), 0, n, s));
                    DK_LAUNCH_B(ctx, (double)m * 12.0, rec_apply_kernel, grid_for(bspace + c.overflow), kThreads, 0,
                                s, w.bcnt.get(), nb, c.overflow, w.rec.get(), w.lab.get(), w.act.get(),
                                w.bsingle.get(), w.bent.get());
                    lab_pending = false;
                }
            } else if (!direct)
                DK_LAUNCH_B(ctx, (double)m * 13.0, slot_apply_kernel, grid_for(bspace + c.overflow), kThreads, 0, s,
                            w.bcnt.get(), nb, c.overflow, w.bent.get(), w.rep_slot.get(), w.keep_slot.get(),
                            w.lab.get(), state_order ? w.act.get() : nullptr);
            list_inc = state_order;
            if (c.active_states) {
                if (state_order) compact_flags(ctx, nullptr, w.act.get(), n, dst, &pctr->listed, s);
                else {
                    // survivors in slot order: states of the slot entries
                    if (w.eval.n < espace) w.eval.alloc(espace, s);
                    DK_LAUNCH(ctx, entry_state_kernel, grid_for(bspace + c.overflow), kThreads, 0, s, w.bent.get(),
                              w.keep_slot.get(), bspace + c.overflow, w.eval.get());
                    compact_flags(ctx, w.eval.get(), w.keep_slot.get(), bspace + c.overflow, dst, &pctr->listed, s);
                }
            }
        } else {
            wait_all_chunks();
            fills.flush(ctx, s);
            // ---- radix-sort grouping: (key, state) pairs, LSD radix sort, runs
            if (!w.keys0.get()) {
                w.keys0.alloc(n, s);
                w.keys1.alloc(n, s);
                w.vals0.alloc(n, s);
                w.vals1.alloc(n, s);
                w.heads.alloc((uint64_t)n + 1, s);
                w.pos.alloc((uint64_t)n + 1, s);
                w.run_start.alloc((uint64_t)n + 2, s);
            }
            RadixBuffers rb{w.keys0.get(), w.vals0.get(), w.keys1.get(), w.vals1.get()};
            uint64_t* skeys = w.keys0.get();
            uint32_t* svals = w.vals0.get();
            uint32_t sort_bits = nbits;
            if (!chunked && fingerprint) {
                // the radix sort orders only the low 2 log2(m) + 8 fingerprint
                // bits (a false merge stays ~2^-8 likely per pass and is caught
                // by verify_runs_kernel): 7 digit passes instead of 8 at 10M
                const uint32_t want = std::min(64u, std::max(32u, 2u * bits_for(m) + 8u));
                const uint32_t have = 64u - (uint32_t)__builtin_clzll(fp_mask | 1ull);
                sort_bits = std::min(want, have);
                if (sort_bits < 64) p.fp_mask = fp_mask & ((1ull << sort_bits) - 1ull);
            }
            if (!chunked) {
                const unsigned gs = grid_for(m, kSigThreads);
                with_lab_type(kl, [&](auto lab) {
                    using LR = decltype(lab);
                    const double bytes = (double)m * (12.0 + 4.0 * k + list_b) + keylab_bytes_per_state(kl) * n;
                    if (fingerprint)
                        DK_LAUNCH_BU(ctx, bytes, (double)m * k, (signature_kernel<LR, 1>), gs, kSigThreads, 0, s, list, m,
                                     d.delta, n, lab, nullptr, p, w.keys0.get(), w.vals0.get());
                    else
                        DK_LAUNCH_BU(ctx, bytes, (double)m * k, signature_kernel, gs, kSigThreads, 0, s, list, m, d.delta,
                                     n, lab, nullptr, p, w.keys0.get(), w.vals0.get());
                });
                if (radix_sort_pairs(ctx, rb, m, sort_bits, s)) {
                    skeys = w.keys1.get();
                    svals = w.vals1.get();
                }
                res.sorted += m;
                if (fingerprint) {
                    DK_LAUNCH(ctx, verify_runs_kernel, g, kThreads, 0, s, skeys, svals, m, d.delta, n, k, w.lab.get(),
                              dctr);
                    read_words(ctx, dctr, sizeof(c), &c, s);
                    if (c.collision) {
                        ++res.collisions;
                        ++collisions_this_pass;
                        --res.passes;
                        salt = mix64(salt + 0x1234567ull);
                        continue;
                    }
                }
            } else {
                // exact refinement letter-chunk by letter-chunk; the run index
                // of the previous chunk leads the next key
                if (!w.cur.get()) w.cur.alloc(n, s);
                DK_LAUNCH(ctx, gather_dense_kernel, g, kThreads, 0, s, list, m,
                          static_cast<const uint32_t*>(kl.p), w.cur.get());
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
                    DK_LAUNCH_B(ctx, (double)m * (24.0 + 8.0 * c_letters), signature_kernel<ArrLab<uint32_t>>, g, kThreads, 0,
                                s, elist, m, d.delta, n, ArrLab<uint32_t>{static_cast<const uint32_t*>(kl.p)}, w.cur.get(), pc,
                                w.keys0.get(), w.vals0.get());
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
            // big passes flag survivors per state so the next list is increasing
            // (coalesced delta rows); small ones keep the sorted order
            const bool state_order = m >= (uint64_t)n / 16;
            if (state_order) {
                if (!w.act.get()) w.act.alloc(n, s);
                DK_CUDA(cudaMemsetAsync(w.act.get(), 0, n, s));
            }
            if (!chunked && list_inc) {
                // states entered the sort increasing: each run's minimum is its head
                const uint64_t tiles = (m + kRunTile - 1) / kRunTile;
                DBuf<unsigned long long> look(tiles + 1, s);  // look-back words + the tile counter
                DK_CUDA(cudaMemsetAsync(look.get(), 0, (tiles + 1) * 8, s));
                // a pass over every state: the identity labels first (one
                // coalesced write), then only the members of multi-state runs
                // are scattered -- none once the partition is all singletons
                const bool multi_only = m == n;
                if (multi_only) iota_u32(ctx, w.lab.get(), n, s);
                DK_LAUNCH_B(ctx, 17.0 * m, run_label_kernel, (unsigned)tiles, kThreads, 0, s, skeys, svals, m,
                            look.get(), reinterpret_cast<uint32_t*>(look.get() + tiles), w.lab.get(),
                            state_order ? nullptr : w.keep.get(), state_order ? w.act.get() : nullptr, dctr,
                            multi_only ? 1 : 0);
            } else {
                DK_LAUNCH(ctx, run_heads_kernel, g, kThreads, 0, s, skeys, m, w.heads.get());
                exclusive_scan_u32(ctx, w.heads.get(), w.pos.get(), m, &dctr->runs, s);
                DK_LAUNCH(ctx, run_starts_kernel, g, kThreads, 0, s, w.heads.get(), w.pos.get(), m,
                          w.run_start.get());
                DK_CUDA(cudaMemsetAsync(w.scratch.get(), 0xff, m * sizeof(uint32_t), s));
                DK_LAUNCH(ctx, run_min_kernel, g, kThreads, 0, s, w.heads.get(), w.pos.get(), svals, m,
                          w.scratch.get());
                DK_LAUNCH_B(ctx, 25.0 * m, run_apply_kernel, g, kThreads, 0, s, w.heads.get(), w.pos.get(), svals, m,
                            w.run_start.get(), w.scratch.get(), w.lab.get(), w.keep.get(),
                            state_order ? w.act.get() : nullptr, dctr);
            }
            list_inc = state_order;
            read_words(ctx, dctr, sizeof(c), &c, s);
            // compaction after the readback: nothing when no state survives
            // or when every state does (the identity list stays)
            if (state_order && c.active_states == n) all_survive = true;
            else if (c.active_states && B - A + c.runs != B) {
                if (state_order) compact_flags(ctx, nullptr, w.act.get(), n, dst, &dctr->listed, s);
                else compact_flags(ctx, svals, w.keep.get(), m, dst, &dctr->listed, s);
            }
        }

        check_streamed();
        collisions_this_pass = 0;
        const uint32_t newB = B - A + c.runs;
        if (newB == B) break;  // fixed point: no block split (reference l.411)
        ++res.iters;
        B = newB;
        A = c.active_blocks;
        m = c.active_states;
        if (all_survive) {  // identity list kept (nothing was compacted)
            all_survive = false;
        } else if (m) {  // every strategy compacted the survivors into dst
            list = dst;
            if (dst == list_alt) std::swap(list_buf, list_alt);
        }
    }
    ctx->prof_pass = 0;
    wait_all_chunks();  // inputs that needed no pass are still validated
    check_streamed();
    if (B == n && iota_out) res.num_blocks = n;  // the identity numbering is in block_out already
    else res.num_blocks = canonical_from_min_labels(ctx, w.lab.get(), n, block_out, w.scratch.get(), s, B);
    return res;
}

// ==========================================================================
// Sharded sortPR primitives (paper_2508_20735_b200/sharded.py drives them).
//
// States are sharded in contiguous ranges; delta and the block-label array
// are replicated (delta read-only, labels allgathered after every pass).  A
// pass on rank r: keys of its active states are partitioned by owner rank
// (top 32 hash bits, multiply-shift), exchanged with one all-to-all, grouped
// at the owner in shared-memory buckets (the owner can verify fingerprint
// tuples of any state: delta and labels are replicated), and the per-entry
// results (new label | survivor bit) travel back by the reverse all-to-all.
// Counting-table passes allreduce the (min, count) table instead.
// ==========================================================================

namespace {

constexpr int kPartThreads = 256;
constexpr int kPartItems = 16;
constexpr int kMaxWorld = 64;

__device__ __forceinline__ uint32_t owner_of(unsigned long long hk, uint32_t world) {
    return (uint32_t)(((hk >> 32) * (unsigned long long)world) >> 32);
}

// entries {hk, state, dest} in list order + per-destination counts
template <typename LR>
__global__ void __launch_bounds__(kThreads) sig_entries_kernel(const uint32_t* __restrict__ list, uint64_t m,
                                                               const uint32_t* __restrict__ delta, uint32_t n,
                                                               LR lab, SigParams p,
                                                               uint32_t world, uint4* __restrict__ tmp,
                                                               uint32_t* __restrict__ counts) {
    __shared__ uint32_t cnt[kMaxWorld];
    for (uint32_t d = threadIdx.x; d < world; d += blockDim.x) cnt[d] = 0;
    __syncthreads();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t q = list ? list[i] : p.q0 + (uint32_t)i;
        const uint64_t key = tuple_key<LR>(q, lab[q], delta, n, lab, p);
        const unsigned long long hk = p.kind == kKeyPacked ? mix64(key) : key;
        const uint32_t d = owner_of(hk, world);
        tmp[i] = make_uint4((uint32_t)hk, (uint32_t)(hk >> 32), q, d);
        const unsigned peers = __match_any_sync(__activemask(), d);
        if ((threadIdx.x & 31u) == (unsigned)(__ffs(peers) - 1)) atomicAdd(&cnt[d], (uint32_t)__popc(peers));
    }
    __syncthreads();
    for (uint32_t d = threadIdx.x; d < world; d += blockDim.x)
        if (cnt[d]) atomicAdd(&counts[d], cnt[d]);
}

__global__ void dest_offsets_kernel(const uint32_t* __restrict__ counts, uint32_t world, uint32_t* __restrict__ cur) {
    if (threadIdx.x == 0) {
        uint32_t o = 0;
        for (uint32_t d = 0; d < world; ++d) {
            cur[d] = o;
            o += counts[d];
        }
    }
}

// tile of 4096 entries -> destination-contiguous send buffer; one global
// cursor atomic per (CTA, destination)
__global__ void __launch_bounds__(kPartThreads) partition_kernel(const uint4* __restrict__ tmp, uint64_t m,
                                                                 uint32_t world, uint32_t* __restrict__ cur,
                                                                 uint4* __restrict__ send) {
    __shared__ uint32_t cnt[kMaxWorld], gbase[kMaxWorld];
    const unsigned lane = threadIdx.x & 31u, lt = (1u << lane) - 1u;
    for (uint32_t d = threadIdx.x; d < world; d += blockDim.x) cnt[d] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)blockIdx.x * kPartThreads * kPartItems;
    uint4 e[kPartItems];
    uint32_t pos[kPartItems];
#pragma unroll
    for (int j = 0; j < kPartItems; ++j) {
        const uint64_t i = base + (uint64_t)j * kPartThreads + threadIdx.x;
        if (i < m) e[j] = __ldcs(tmp + i);
    }
#pragma unroll
    for (int j = 0; j < kPartItems; ++j) {
        const uint64_t i = base + (uint64_t)j * kPartThreads + threadIdx.x;
        const bool ok = i < m;
        const unsigned act = __ballot_sync(0xffffffffu, ok);
        if (ok) {
            const unsigned peers = __match_any_sync(act, e[j].w);
            const unsigned leader = __ffs(peers) - 1;
            uint32_t b = 0;
            if (lane == leader) b = atomicAdd(&cnt[e[j].w], (uint32_t)__popc(peers));
            b = __shfl_sync(act, b, leader);
            pos[j] = b + (uint32_t)__popc(peers & lt);
        }
    }
    __syncthreads();
    for (uint32_t d = threadIdx.x; d < world; d += blockDim.x) gbase[d] = cnt[d] ? atomicAdd(&cur[d], cnt[d]) : 0u;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPartItems; ++j) {
        const uint64_t i = base + (uint64_t)j * kPartThreads + threadIdx.x;
        if (i < m) send[gbase[e[j].w] + pos[j]] = make_uint4(e[j].x, e[j].y, e[j].z, 0u);
    }
}

// received entries -> owner-side buckets; entry index kept in .w
__global__ void entry_bucket_kernel(const uint4* __restrict__ recv, uint64_t count, uint32_t nb,
                                    uint32_t* __restrict__ bcnt, uint4* __restrict__ bent,
                                    IterCounters* __restrict__ ctr) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 e = __ldcs(recv + i);
        bucket_append(entry_key(e), e.z, (uint32_t)i, nb, bcnt, bent, ctr);
    }
}

__global__ void shard_apply_kernel(const uint4* __restrict__ send, const uint32_t* __restrict__ res, uint64_t count,
                                   uint32_t* __restrict__ lab, uint8_t* __restrict__ act) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t q = send[i].z, r = res[i];
        lab[q] = r & 0x7fffffffu;
        if (r >> 31) act[q] = 1;  // act zeroed by the caller
    }
}

__global__ void init_act_range_kernel(const uint8_t* __restrict__ acc, uint32_t lo, uint32_t hi, uint8_t keep_acc,
                                      uint8_t keep_rej, uint8_t* __restrict__ act) {
    for (uint32_t q = lo + blockIdx.x * blockDim.x + threadIdx.x; q < hi; q += gridDim.x * blockDim.x)
        act[q] = acc[q] ? keep_acc : keep_rej;
}

// ---- owner-bucket layout (native driver) --------------------------------------------
//
// The sender's signature kernel appends (hkey, state) straight into
// sub-bucket (owner o, bucket b) of its send regions -- region o holds nb
// sub-buckets of cs slots, b from the same hash bits as the single-GPU
// buckets -- so the owner groups what it receives as is (MultiSrc): no
// staging pass, no partition pass, no re-bucketing at the owner.  Past cs a
// sub-bucket's entries go to an overflow list {hk lo, hk hi, state, owner}.
// four CTAs per SM (64 registers): 0.522 -> 0.480 ms on the 10M x 10 pass
#ifndef DFAKIT_SIGO_MINB
#define DFAKIT_SIGO_MINB 4
#endif
template <typename LR, int MODE>  // as sig_bucket_kernel: 0 any kind, 1 fingerprints, 2 sliced partial keys
__global__ void __launch_bounds__(kThreads, DFAKIT_SIGO_MINB) sig_owner_kernel(
    const uint32_t* __restrict__ list, uint64_t m, const uint32_t* __restrict__ delta, uint32_t n, LR lab, SigParams p,
    uint32_t world, uint32_t nb, uint32_t cs, uint32_t* __restrict__ scur, const __grid_constant__ OwnerDst dst,
    uint4* __restrict__ ovf, uint32_t* __restrict__ ovf_cnt, const uint64_t* __restrict__ part) {
    const unsigned lane = threadIdx.x & 31u, lt = (1u << lane) - 1u;
    if (MODE == 1) p.kind = kKeyFingerprint;
    // the owners' region pointers in shared memory (a runtime-indexed kernel
    // parameter is a local-memory copy per thread)
    __shared__ uint4* s_dst[8];
    if (threadIdx.x < 8) s_dst[threadIdx.x] = threadIdx.x < world ? dst.entries[threadIdx.x] : nullptr;
    __syncthreads();
    if constexpr (MODE == 2) {
        // partial keys of a sliced pass (no gathers): the cursor atomic of one
        // state in flight while the next state's key is read (as sig_bucket)
        const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
        const uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + (threadIdx.x & ~31u);
        bool have = false, pvalid = false;
        unsigned long long phk = 0;
        uint32_t pq = 0, po = 0, pg = 0, pbase = 0, prank = 0, pleader = 0;
        auto finish = [&]() {
            const uint32_t pos = __shfl_sync(0xffffffffu, pbase, pleader) + prank;
            if (!pvalid) return;
            const uint4 e = make_uint4((uint32_t)phk, (uint32_t)(phk >> 32), pq, po);
            if (pos < cs) {
                s_dst[po][(uint64_t)(pg - po * nb) * cs + pos] = e;
            } else {
                ovf[atomicAdd(&ovf_cnt[world], 1u)] = e;
                atomicAdd(&ovf_cnt[po], 1u);
            }
        };
        for (uint64_t w = i0; w < m; w += stride) {
            const uint64_t i = w + lane;
            const bool valid = i < m;
            unsigned long long hk = 0;
            uint32_t q = 0;
            if (valid) {
                q = list ? list[i] : p.q0 + (uint32_t)i;
                const uint64_t key = key_of_part(p, __ldcs(part + i));
                hk = p.kind == kKeyPacked ? mix64(key) : key;
            }
            if (have) finish();
            pvalid = valid;
            phk = hk;
            pq = q;
            po = valid ? owner_of(hk, world) : 0u;
            pg = valid ? po * nb + ((uint32_t)(hk >> kBucketShift) & (nb - 1)) : 0xffffffffu;
            const unsigned peers = __match_any_sync(0xffffffffu, pg);
            pleader = __ffs(peers) - 1;
            prank = (uint32_t)__popc(peers & lt);
            pbase = 0;
            if (valid && lane == pleader) pbase = atomicAdd(&scur[pg * kCntStride], (uint32_t)__popc(peers));
            have = true;
        }
        if (have) finish();
        if (dst.peer) __threadfence_system();  // the stores into other GPUs are complete before the barrier
        return;
    }
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t q = list ? list[i] : p.q0 + (uint32_t)i;
        const uint64_t key = MODE == 2 ? key_of_part(p, __ldcs(part + i))
                                       : tuple_key<LR, DFAKIT_SIGB_CH>(q, lab[q], delta, n, lab, p);
        const unsigned long long hk = p.kind == kKeyPacked ? mix64(key) : key;
        const uint32_t o = owner_of(hk, world);
        const uint32_t g = o * nb + ((uint32_t)(hk >> kBucketShift) & (nb - 1));
        const unsigned act = __activemask();
        const unsigned peers = __match_any_sync(act, g);
        const unsigned leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(&scur[g * kCntStride], (uint32_t)__popc(peers));
        base = __shfl_sync(act, base, leader);
        const uint32_t pos = base + (uint32_t)__popc(peers & lt);
        const uint4 e = make_uint4((uint32_t)hk, (uint32_t)(hk >> 32), q, o);
        if (pos < cs) {
            s_dst[o][(uint64_t)(g - o * nb) * cs + pos] = e;  // (peer mode: a store over NVLink)
        } else {
            ovf[atomicAdd(&ovf_cnt[world], 1u)] = e;
            atomicAdd(&ovf_cnt[o], 1u);
        }
    }
    if (dst.peer) __threadfence_system();  // the stores into other GPUs are complete before the barrier
}

// per owner o: the nb sub-bucket counts then its overflow count (nb + 1 words)
__global__ void owner_counts_kernel(const uint32_t* __restrict__ scur, const uint32_t* __restrict__ ovf_cnt,
                                    uint32_t world, uint32_t nb, const __grid_constant__ OwnerDst dst) {
    const uint64_t total = (uint64_t)world * (nb + 1);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t o = (uint32_t)(i / (nb + 1)), b = (uint32_t)(i % (nb + 1));
        dst.counts[o][b] = b < nb ? scur[((uint64_t)o * nb + b) * kCntStride] : ovf_cnt[o];
    }
    if (dst.peer) __threadfence_system();
}

// peer mode, owner side: region entry e of sender s = e / region gets its
// result written straight into s's label / survivor-flag arrays
__global__ void owner_scatter_kernel(const uint4* __restrict__ recv, const uint32_t* __restrict__ recv_cnt,
                                     uint32_t world, uint32_t nb, uint32_t cs, const uint32_t* __restrict__ results,
                                     const uint8_t* __restrict__ bsingle, const __grid_constant__ PeerLabels out) {
    const uint64_t region = (uint64_t)nb * cs, total = region * world;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = (uint32_t)(e / region), r = (uint32_t)(e % region);
        if (r % cs >= min(recv_cnt[(uint64_t)s * (nb + 1) + r / cs], cs)) continue;
        const uint32_t q = __ldcs(recv + e).z;
        const uint32_t v = bsingle && bsingle[r / cs] ? q : results[e];  // (a bucket of distinct keys: singletons)
        out.lab[s][q] = v & 0x7fffffffu;
        if (v >> 31) out.act[s][q] = 1;  // zeroed by the sender before the pass's counter exchange
    }
    __threadfence_system();  // the label stores into other GPUs are complete before the barrier
}

// received overflow counts of every sender (for the host readback)
__global__ void owner_ovf_gather_kernel(const uint32_t* __restrict__ recv_msg, uint32_t world, uint32_t nb,
                                        uint32_t* __restrict__ out) {
    for (uint32_t s = threadIdx.x; s < world; s += blockDim.x) out[s] = recv_msg[(uint64_t)s * (nb + 1) + nb];
}

// the ghash fallback's elements: every entry of a bucket that overflowed on
// some sender, then every received overflow entry; .w = the output index
__global__ void owner_collect_kernel(MultiSrc src, const uint4* __restrict__ ovf_in, uint32_t ovf_total,
                                     uint4* __restrict__ out, uint32_t* __restrict__ out_count) {
    const uint64_t region = (uint64_t)src.nb * src.cs, total = region * src.nsrc + ovf_total;
    src.init();  // count() reads the shared-memory copy of the pointers
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total; e += (uint64_t)gridDim.x * blockDim.x) {
        uint4 v;
        if (e < region * src.nsrc) {
            const uint32_t sidx = (uint32_t)(e / region), r = (uint32_t)(e % region), b = r / src.cs, off = r % src.cs;
            if (src.count(b) <= kGrpCap || off >= min(src.cnt[sidx][b], src.cs)) continue;
            v = src.base[sidx][(uint64_t)b * src.cs + off];
            v.w = (uint32_t)e;
        } else {
            v = ovf_in[e - region * src.nsrc];
            v.w = (uint32_t)e;
        }
        out[atomicAdd(out_count, 1u)] = v;
    }
}

// sender: results of its sub-bucket entries (padded layout) -> labels
__global__ void owner_apply_kernel(const uint4* __restrict__ send, const uint32_t* __restrict__ scur, uint32_t world,
                                   uint32_t nb, uint32_t cs, uint32_t rank, const uint32_t* __restrict__ own_res,
                                   const uint32_t* __restrict__ back, uint32_t* __restrict__ lab,
                                   uint8_t* __restrict__ act) {
    const uint64_t region = (uint64_t)nb * cs, total = region * world;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t o = (uint32_t)(e / region), r = (uint32_t)(e % region);
        if (r % cs >= min(scur[((uint64_t)o * nb + r / cs) * kCntStride], cs)) continue;
        const uint32_t q = send[e].z;
        const uint32_t v = o == rank ? own_res[r] : back[(uint64_t)(o - (o > rank)) * region + r];
        lab[q] = v & 0x7fffffffu;
        if (v >> 31) act[q] = 1;  // act zeroed by the caller
    }
}

SigParams sig_params(const PassPlan& plan, uint32_t k, uint64_t salt) {
    SigParams p{};
    p.kind = plan.strategy == kPlanFingerprint ? kKeyFingerprint : kKeyPacked;
    p.a0 = 0;
    p.a1 = k;
    p.field_bits = plan.field_bits;
    p.salt = salt;
    p.fp_mask = ~0ull;
    return p;
}

}  // namespace

// lazy: skip the initial labels and survivor flags when the first pass will
// overwrite them -- every state active and a counting-table pass whose key
// labels come from the flags (its apply writes every label and flag of the
// rank's range), as in the single-GPU engine.
ShardInit shard_init(Ctx* ctx, const DevDfa& d, uint32_t lo, uint32_t hi, uint32_t* lab, uint8_t* act,
                     cudaStream_t s, bool lazy) {
    ShardInit r{};
    if (d.n == 0) return r;
    LeaderInfo li = leader_info(ctx, d, s);
    r.num_blocks = (li.min_acc != kNone) + (li.min_rej != kNone);
    r.active_blocks = (li.cnt_acc >= 2) + (li.cnt_rej >= 2);
    r.active_states = (li.cnt_acc >= 2 ? li.cnt_acc : 0) + (li.cnt_rej >= 2 ? li.cnt_rej : 0);
    if (lazy && r.active_states == d.n) {
        const PassPlan p0 = plan_pass(d.n, d.k, r.num_blocks, r.active_states, 0, false);
        if (p0.strategy == kPlanTable && p0.keylab_bytes != 0) return r;
    }
    init_leader_labels(ctx, d, li, lab, s);
    if (hi > lo)
        DK_LAUNCH(ctx, init_act_range_kernel, grid_for(hi - lo), kThreads, 0, s, d.acc, lo, hi,
                  (uint8_t)(li.cnt_acc >= 2), (uint8_t)(li.cnt_rej >= 2), act);
    return r;
}

// initial_acc: the partition is still {F, Q \ F}: two-block key labels come
// straight from the flags (10 MB read instead of 40).
void shard_keylab(Ctx* ctx, const uint32_t* lab, uint32_t n, uint32_t num_blocks, const PassPlan& plan, void* out,
                  uint32_t* scratch, cudaStream_t s, const uint8_t* initial_acc) {
    if (!plan.keylab_bytes) return;
    if (plan.keylab_bytes == kBitLabels) {  // two blocks: a bitmap, no scan
        if (initial_acc)
            DK_LAUNCH(ctx, acc_dense2_bits_kernel, grid_for((uint64_t)n), kThreads, 0, s, initial_acc, n,
                      static_cast<uint32_t*>(out));
        else
            DK_LAUNCH(ctx, dense2_bits_kernel, grid_for((uint64_t)n), kThreads, 0, s, lab, n,
                      static_cast<uint32_t*>(out));
    } else if (num_blocks <= 2 && plan.keylab_bytes == 1) {  // two blocks: no scan
        if (initial_acc)
            DK_LAUNCH(ctx, acc_dense2_kernel, grid_for(n), kThreads, 0, s, initial_acc, n, static_cast<uint8_t*>(out));
        else
            DK_LAUNCH(ctx, dense2_kernel, grid_for(n), kThreads, 0, s, lab, n, static_cast<uint8_t*>(out));
    } else {
        dense_labels(ctx, lab, n, out, (int)plan.keylab_bytes, scratch, s);
    }
}

void shard_table_signature(Ctx* ctx, const DevDfa& d, const void* keylab, const PassPlan& plan, const uint32_t* list,
                           uint32_t list_base, uint64_t m, uint32_t* keys32, uint32_t* tmin, uint32_t* tcnt,
                           cudaStream_t s) {
    const uint32_t nbits = plan.key_bits;
    const uint64_t tsize = 1ull << nbits;
    DK_CUDA(cudaMemsetAsync(tmin, 0xff, tsize * 4, s));
    DK_CUDA(cudaMemsetAsync(tcnt, 0, tsize * 4, s));
    if (m == 0) return;
    const bool local = nbits <= kSmemTableBits;
    const size_t smem = local ? (size_t)(2u << nbits) * 4 : 0;
    const int smem_table = (int)(2u << kSmemTableBits) * 4;
    const unsigned tg = (unsigned)std::min<uint64_t>((m + kSigtThreads - 1) / kSigtThreads, (uint64_t)ctx->num_sms * kSigtCtas);
    SigParams p = sig_params(plan, d.k, 0);
    p.q0 = list_base;
    with_lab_type(KeyLab{keylab, plan.keylab_bytes ? (int)plan.keylab_bytes : 4}, [&](auto lab) {
        using LR = decltype(lab);
        DK_CUDA(cudaFuncSetAttribute(sig_table_kernel<LR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_table));
        DK_LAUNCH_BU(ctx, (double)m * (8.0 + 4.0 * d.k), (double)m * d.k, sig_table_kernel<LR>, tg, kSigtThreads, smem, s, list, m, d.delta,
                    d.n, lab, p, nbits, keys32, tmin, tcnt, 1 /* local lists are compacted in state order */);
    });
}

void shard_table_apply(Ctx* ctx, const PassPlan& plan, const uint32_t* list, uint32_t list_base,
                       const uint32_t* keys32, uint64_t m, const uint32_t* tmin, const uint32_t* tcnt, uint32_t* lab,
                       uint8_t* act, void* next_keylab, uint32_t* counters, cudaStream_t s) {
    DK_CUDA(cudaMemsetAsync(counters, 0, 4 * sizeof(uint32_t), s));
    if (m == 0) return;
    // ranks of the occupied entries of the (allreduced, identical) table:
    // compact block ids of the next partition when the pass covered every state
    DBuf<uint32_t> rank;
    const uint32_t tsize = 1u << plan.key_bits;
    const bool narrow = plan.key_bits <= 16;
    // a state range starting at a multiple of four with a small table: the
    // vectorised apply with the table (and its ranks) staged in shared memory
    auto a16 = [](const void* x) { return ((uintptr_t)x & 15u) == 0; };
    uint32_t* lab_r = lab + list_base;
    void* next_r = next_keylab ? static_cast<char*>(next_keylab) + (size_t)list_base * (narrow ? 2 : 4) : nullptr;
    if (!list && list_base % 4 == 0 && tsize <= kApplyStageMax && a16(keys32) && a16(lab_r) &&
        (!next_r || (narrow ? ((uintptr_t)next_r & 7u) == 0 : a16(next_r)))) {
        DK_LAUNCH_B(ctx, (double)m * 13.0, table_apply_vec_kernel<true>,
                    grid_for((m + 3) / 4, kThreads, (unsigned)ctx->num_sms * 4u), kThreads, 0, s, keys32, m, tmin,
                    tcnt, lab_r, (uint8_t*)nullptr, next_r ? tcnt : nullptr /* ranks: computed in the kernel */,
                    next_r && narrow ? static_cast<uint16_t*>(next_r) : nullptr,
                    next_r && !narrow ? static_cast<uint32_t*>(next_r) : nullptr, reinterpret_cast<IterCounters*>(counters),
                    tsize, act + list_base, list_base);
        return;
    }
    if (next_keylab) {
        rank.alloc(tsize, s);
        DK_LAUNCH(ctx, table_occupied_kernel, grid_for(tsize), kThreads, 0, s, tcnt, tsize, rank.get());
        exclusive_scan_u32(ctx, rank.get(), rank.get(), tsize, nullptr, s);
    }
    DK_LAUNCH_B(ctx, (double)m * 13.0, table_apply_kernel, grid_for(m), kThreads, 0, s, list, keys32, m, tmin, tcnt,
                lab, nullptr, act, rank.get(), next_keylab && narrow ? static_cast<uint16_t*>(next_keylab) : nullptr,
                next_keylab && !narrow ? static_cast<uint32_t*>(next_keylab) : nullptr, list_base,
                reinterpret_cast<IterCounters*>(counters));
}

void shard_sig_partition(Ctx* ctx, const DevDfa& d, const void* keylab, const PassPlan& plan, uint64_t salt,
                         const uint32_t* list, uint32_t list_base, uint64_t m, uint32_t world, uint4* send,
                         uint32_t* send_counts, cudaStream_t s) {
    if (world == 0 || world > (uint32_t)kMaxWorld) throw Error(DFAKIT_E_INVALID, "shard: world size out of range");
    DK_CUDA(cudaMemsetAsync(send_counts, 0, world * 4, s));
    if (m == 0) return;
    DBuf<uint4> tmp(m, s);
    DBuf<uint32_t> cur(world, s);
    SigParams p = sig_params(plan, d.k, salt);
    p.q0 = list_base;
    with_lab_type(KeyLab{keylab, plan.keylab_bytes ? (int)plan.keylab_bytes : 4}, [&](auto lab) {
        DK_LAUNCH_BU(ctx, (double)m * (4.0 * d.k + 20.0), (double)m * d.k, sig_entries_kernel, grid_for(m, kThreads,
                    (unsigned)ctx->num_sms * 8u), kThreads, 0, s, list, m, d.delta, d.n, lab, p, world, tmp.get(),
                    send_counts);
    });
    DK_LAUNCH(ctx, dest_offsets_kernel, 1, 32, 0, s, send_counts, world, cur.get());
    const uint64_t tiles = (m + kPartThreads * kPartItems - 1) / (kPartThreads * kPartItems);
    DK_LAUNCH_B(ctx, 32.0 * m, partition_kernel, (unsigned)tiles, kPartThreads, 0, s, tmp.get(), m, world, cur.get(),
                send);
}

// Owner-side grouping of received entries into the workspace: per-slot
// records {entry index, rep | multi << 31} (coalesced), counters.  The
// per-entry results for the trip back are scattered from the records by
// shard_group_results, which the driver skips after the last pass.
void shard_group_deferred(Ctx* ctx, const DevDfa& d, const void* verify_lab, uint32_t verify_bytes,
                          const PassPlan& plan, const uint4* recv, uint64_t count, ShardGroupWs& ws,
                          uint32_t* counters, cudaStream_t s) {
    IterCounters* dctr = reinterpret_cast<IterCounters*>(ctx->dmailbox) + 4;
    DK_CUDA(cudaMemsetAsync(dctr, 0, sizeof(IterCounters), s));
    ws.count = count;
    ws.ovf = 0;
    if (count) {
        uint32_t D = 1;
        while (D < 24 && ((uint64_t)1 << D) * (kGrpCap * 3 / 4) < count) ++D;
        const uint32_t nb = 1u << D;
        const uint64_t bspace = (uint64_t)nb * kGrpCap, espace = bspace + count;
        ws.nb = nb;
        if (ws.bcnt.n < (uint64_t)nb * kCntStride) ws.bcnt.alloc((uint64_t)nb * kCntStride, s);
        if (ws.bent.n < espace) {
            ws.bent.alloc(espace, s);
            ws.rec.alloc(espace, s);
        }
        DK_CUDA(cudaMemsetAsync(ws.bcnt.get(), 0, (size_t)nb * kCntStride * 4, s));
        DK_LAUNCH_B(ctx, 32.0 * count, entry_bucket_kernel, grid_for(count), kThreads, 0, s, recv, count, nb,
                    ws.bcnt.get(), ws.bent.get(), dctr);
        const int fp = plan.strategy == kPlanFingerprint ? 1 : 0;
        GroupOut go{0, 0, nullptr, nullptr, nullptr, nullptr, nullptr, ws.rec.get(), 1};
        const unsigned gg = (unsigned)std::min<uint64_t>(nb, (uint64_t)ctx->num_sms * kGrpCtasPerSm);
        const KeyLab vl{verify_lab, (int)verify_bytes};
        with_lab_type(vl, [&](auto lab) {
            using LR = decltype(lab);
            DK_CUDA(cudaFuncSetAttribute(bucket_group_kernel<LR, OneSrc>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(GroupSmem)));
            DK_LAUNCH_B(ctx, 24.0 * count, bucket_group_kernel, gg, kGrpThreads, sizeof(GroupSmem), s,
                        OneSrc{ws.bcnt.get(), ws.bent.get()}, nb, fp, d.delta, d.n, d.k, lab, go, dctr);
        });
        IterCounters c{};
        read_words(ctx, dctr, sizeof(c), &c, s);
        if (c.overflow) {
            ws.ovf = c.overflow;
            uint64_t T = 2;
            while (T < 2 * count) T <<= 1;
            DBuf<unsigned long long> gkey(T + 1, s);
            DBuf<uint32_t> grep(T + 1, s), gslot(espace, s);
            DBuf<uint8_t> gmul(T + 1, s);
            DK_CUDA(cudaMemsetAsync(gkey.get(), 0xff, (T + 1) * 8, s));
            DK_CUDA(cudaMemsetAsync(grep.get(), 0xff, (T + 1) * 4, s));
            DK_CUDA(cudaMemsetAsync(gmul.get(), 0, T + 1, s));
            const unsigned eg = grid_for(bspace + c.overflow);
            DK_LAUNCH(ctx, ghash_insert_kernel, eg, kThreads, 0, s, ws.bcnt.get(), nb, c.overflow, ws.bent.get(), T,
                      gkey.get(), grep.get(), gslot.get());
            DK_LAUNCH(ctx, ghash_multi_kernel, eg, kThreads, 0, s, ws.bcnt.get(), nb, c.overflow, ws.bent.get(),
                      grep.get(), gslot.get(), gmul.get());
            with_lab_type(vl, [&](auto lab) {
                DK_LAUNCH(ctx, ghash_out_kernel, eg, kThreads, 0, s, ws.bcnt.get(), nb, c.overflow, ws.bent.get(),
                          grep.get(), gslot.get(), gmul.get(), fp, d.delta, d.n, d.k, lab, go, dctr);
            });
        }
    }
    DK_CUDA(cudaMemcpyAsync(counters, dctr, 4 * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
}

void shard_group_results(Ctx* ctx, const ShardGroupWs& ws, uint32_t* results, cudaStream_t s) {
    if (!ws.count) return;
    const uint64_t total = (uint64_t)ws.nb * kGrpCap + ws.ovf;
    DK_LAUNCH_B(ctx, 12.0 * ws.count, rec_results_kernel, grid_for(total), kThreads, 0, s, ws.bcnt.get(), ws.nb,
                ws.ovf, ws.rec.get(), results);
}

void shard_group(Ctx* ctx, const DevDfa& d, const void* verify_lab, uint32_t verify_bytes, const PassPlan& plan,
                 const uint4* recv, uint64_t count, uint32_t* results, uint32_t* counters, cudaStream_t s) {
    ShardGroupWs ws;
    shard_group_deferred(ctx, d, verify_lab, verify_bytes, plan, recv, count, ws, counters, s);
    shard_group_results(ctx, ws, results, s);
}

void shard_apply(Ctx* ctx, const uint4* send, const uint32_t* results, uint64_t count, uint32_t* lab, uint8_t* act,
                 cudaStream_t s) {
    if (count)
        DK_LAUNCH_B(ctx, 25.0 * count, shard_apply_kernel, grid_for(count), kThreads, 0, s, send, results, count, lab,
                    act);
}

void shard_compact(Ctx* ctx, const uint8_t* act, uint32_t lo, uint32_t hi, uint32_t* list, uint32_t* count_dev,
                   cudaStream_t s) {
    compact_flags(ctx, nullptr, act + lo, hi > lo ? hi - lo : 0, list, count_dev, s, lo);
}

// ---- owner-bucket layout: host side --------------------------------------------------

OwnerPlan owner_plan(uint64_t m_total, uint32_t world) {
    OwnerPlan op;
    op.world = world;
    op.cs = (kGrpCap / world) & ~3u;  // every sender's share of a bucket: merged buckets fit kGrpCap
    // buckets of ~768..1536 expected entries over all senders, as on one GPU
    const uint64_t per_owner = (m_total + world - 1) / world;
    uint32_t D = 1;
    while (D < 22 && ((uint64_t)1 << D) * (kGrpCap * 3 / 4) < per_owner) ++D;
    op.nb = 1u << D;
    return op;
}

uint32_t pack12_labels(Ctx* ctx, const uint16_t* keys16, uint32_t n, unsigned long long* out, cudaStream_t s,
                       bool eleven) {
    if (eleven) {
        const uint64_t words = ((uint64_t)n * 11u + 63u) / 64u + 1;  // + 1: the reader's straddle load stays inside
        DK_LAUNCH_B(ctx, (double)n * 3.4, pack11_kernel, grid_for(words), kThreads, 0, s, keys16, n, out, words);
        return (uint32_t)kPack11Labels;
    }
    DK_LAUNCH_B(ctx, (double)n * 3.6, pack12_kernel, grid_for(((uint64_t)n + 4) / 5), kThreads, 0, s, keys16, n, out);
    return (uint32_t)kPack12Labels;
}

bool pack11_unsliced(uint32_t n) { return label_slices(KeyLab{nullptr, kPack11Labels}, n) == 1; }

// Label layout of a big signature pass over 16-bit labels below 2^bits (0:
// keep 16 bits, 11 / 12: packed).  Measured on random n x 10 automata (wall
// ms, 16-bit / 12-bit / 11-bit): 50M 6.63 / 6.17 / 5.88 (11-bit unsliced
// best), 60M 8.22 / 8.65 / 8.12, 70M 9.37 / 10.01 / 10.07, 80M 10.78 /
// 11.60 / --, 100M 15.45 / 15.00 / 17.3: 16-bit labels win while their
// slices stay under ~90 MiB; packing pays for an unsliced pass just past the
// unsliced limit and for slices the 16-bit layout would make too big.
int pack_choice(uint32_t n, uint32_t bits) {
    const double pack_min = getenv("DFAKIT_PACK12_MIN_MB") ? atof(getenv("DFAKIT_PACK12_MIN_MB")) : 90.0;
    if (getenv("DFAKIT_NO_PACK12") || bits > 12) return 0;
    const double mib = 1048576.0, u16 = 2.0 * n;
    if (u16 <= pack_min * mib) return 0;
    const bool forced = pack_min < 90.0;  // (tests: pack whatever the size)
    if (bits <= 11 && !getenv("DFAKIT_NO_PACK11") && (1.375 * n <= 80.0 * mib || forced) && pack11_unsliced(n))
        return 11;
    const uint32_t slices = label_slices(KeyLab{nullptr, 2}, n);
    if (!forced && u16 / slices <= 90.0 * mib) return 0;
    return 12;
}

uint64_t pack_words(uint32_t n) { return std::max<uint64_t>(((uint64_t)n + 4) / 5, ((uint64_t)n * 11u + 63u) / 64u + 1); }

void shard_sig_owner(Ctx* ctx, const DevDfa& d, const void* keylab, const PassPlan& plan, uint64_t salt,
                     const uint32_t* list, uint32_t list_base, uint64_t m, const OwnerPlan& op, OwnerSend& ws,
                     cudaStream_t s, const OwnerDst* dst_in) {
    const uint32_t W = op.world, nb = op.nb, cs = op.cs;
    const uint64_t slots = (uint64_t)W * nb * cs;
    if (!dst_in && ws.send.n < std::max<uint64_t>(1, slots)) ws.send.alloc(std::max<uint64_t>(1, slots), s);
    if (ws.scur.n < (uint64_t)W * nb * kCntStride) ws.scur.alloc((uint64_t)W * nb * kCntStride, s);
    if (ws.ovf.n < std::max<uint64_t>(1, m)) {
        ws.ovf.alloc(std::max<uint64_t>(1, m), s);
        ws.ovf_sorted.alloc(std::max<uint64_t>(1, m), s);
    }
    if (ws.ovf_cnt.n < (uint64_t)W + 1) {
        ws.ovf_cnt.alloc(W + 1, s);
        ws.ovf_cur.alloc(W, s);
    }
    if (!dst_in && ws.msg.n < (uint64_t)W * (nb + 1)) ws.msg.alloc((uint64_t)W * (nb + 1), s);
    OwnerDst dst{};
    if (dst_in) {
        dst = *dst_in;
    } else {
        for (uint32_t o = 0; o < W; ++o) {
            dst.entries[o] = ws.send.get() + (uint64_t)o * nb * cs;
            dst.counts[o] = ws.msg.get() + (uint64_t)o * (nb + 1);
        }
    }
    Fills f;
    f.add(ws.scur.get(), (size_t)W * nb * kCntStride * 4, 0);
    f.add(ws.ovf_cnt.get(), (size_t)(W + 1) * 4, 0);
    f.flush(ctx, s);
    if (m) {
        SigParams p = sig_params(plan, d.k, salt);
        p.q0 = list_base;
        const KeyLab kl{keylab, plan.keylab_bytes ? (int)plan.keylab_bytes : 4};
        const uint64_t* part = sliced_parts(ctx, kl, list, m, d, p, ws.part, s);
        with_lab_type_p12(kl, [&](auto lab) {
            using LR = decltype(lab);
            const double bytes = part ? (double)m * 24.0 : (double)m * (4.0 * d.k + 16.0);
            const unsigned grid = grid_for(m, kThreads, (unsigned)ctx->num_sms * 8u);
            if (part)
                DK_LAUNCH_BU(ctx, bytes, 0.0, (sig_owner_kernel<LR, 2>), grid, kThreads, 0, s, list, m, d.delta, d.n,
                             lab, p, W, nb, cs, ws.scur.get(), dst, ws.ovf.get(), ws.ovf_cnt.get(), part);
            else if (plan.strategy == kPlanFingerprint)
                DK_LAUNCH_BU(ctx, bytes, (double)m * d.k, (sig_owner_kernel<LR, 1>), grid, kThreads, 0, s, list, m,
                             d.delta, d.n, lab, p, W, nb, cs, ws.scur.get(), dst, ws.ovf.get(),
                             ws.ovf_cnt.get(), part);
            else
                DK_LAUNCH_BU(ctx, bytes, (double)m * d.k, (sig_owner_kernel<LR, 0>), grid, kThreads, 0, s, list, m,
                             d.delta, d.n, lab, p, W, nb, cs, ws.scur.get(), dst, ws.ovf.get(),
                             ws.ovf_cnt.get(), part);
        });
    }
    DK_LAUNCH(ctx, owner_counts_kernel, grid_for((uint64_t)W * (nb + 1)), kThreads, 0, s, ws.scur.get(),
              ws.ovf_cnt.get(), W, nb, dst);
}

void shard_sort_overflow(Ctx* ctx, const OwnerPlan& op, OwnerSend& ws, uint32_t ovf_total, cudaStream_t s) {
    if (!ovf_total) return;
    DK_LAUNCH(ctx, dest_offsets_kernel, 1, 32, 0, s, ws.ovf_cnt.get(), op.world, ws.ovf_cur.get());
    const uint64_t tiles = (ovf_total + kPartThreads * kPartItems - 1) / (kPartThreads * kPartItems);
    DK_LAUNCH(ctx, partition_kernel, (unsigned)tiles, kPartThreads, 0, s, ws.ovf.get(), (uint64_t)ovf_total, op.world,
              ws.ovf_cur.get(), ws.ovf_sorted.get());
}

void shard_owner_ovf_counts(Ctx* ctx, const OwnerPlan& op, const uint32_t* recv_msg, uint32_t* out, cudaStream_t s) {
    DK_LAUNCH(ctx, owner_ovf_gather_kernel, 1, 64, 0, s, recv_msg, op.world, op.nb, out);
}

void shard_group_owner(Ctx* ctx, const DevDfa& d, const void* verify_lab, uint32_t verify_bytes, const PassPlan& plan,
                       const OwnerPlan& op, const OwnerSources& in, const uint4* ovf_in, uint32_t ovf_total,
                       uint32_t* results, uint32_t* counters, cudaStream_t s, uint8_t* bsingle) {
    if (op.world > (uint32_t)kMaxSrc) throw Error(DFAKIT_E_INVALID, "owner buckets: at most 8 ranks");
    IterCounters* dctr = reinterpret_cast<IterCounters*>(ctx->dmailbox) + 4;
    DK_CUDA(cudaMemsetAsync(dctr, 0, sizeof(IterCounters), s));
    MultiSrc src{};
    for (uint32_t r = 0; r < op.world; ++r) {
        src.base[r] = in.base[r];
        src.cnt[r] = in.cnt[r];
    }
    src.nsrc = op.world;
    src.nb = op.nb;
    src.cs = op.cs;
    const int fp = plan.strategy == kPlanFingerprint ? 1 : 0;
    GroupOut go{0, 0, nullptr, nullptr, nullptr, nullptr, results, nullptr, 0, bsingle};
    const unsigned gg = (unsigned)std::min<uint64_t>(op.nb, (uint64_t)ctx->num_sms * kGrpCtasPerSm);
    const KeyLab vl{verify_lab, (int)verify_bytes};
    with_lab_type(vl, [&](auto lab) {
        using LR = decltype(lab);
        DK_CUDA(cudaFuncSetAttribute(bucket_group_kernel<LR, MultiSrc, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(GroupSmem)));
        DK_LAUNCH_B(ctx, 20.0 * (double)op.nb * kGrpCap * 3 / 4, (bucket_group_kernel<LR, MultiSrc, 2>), gg,
                    kGrpThreads, sizeof(GroupSmem), s, src, op.nb, fp, d.delta, d.n, d.k, lab, go, dctr);
    });
    if (ovf_total) {
        // some sub-bucket overflowed: its whole bucket (every sender's part)
        // and the overflow entries through the global table
        const uint64_t cap = (uint64_t)op.world * op.nb * op.cs + ovf_total;
        DBuf<uint4> fl(cap, s);
        DBuf<uint32_t> fc(1, s);
        DK_CUDA(cudaMemsetAsync(fc.get(), 0, 4, s));
        DK_LAUNCH(ctx, owner_collect_kernel, grid_for(cap), kThreads, 0, s, src, ovf_in, ovf_total, fl.get(), fc.get());
        uint32_t count = 0;
        read_words(ctx, fc.get(), 4, &count, s);
        uint64_t T = 2;
        while (T < 2 * (uint64_t)count) T <<= 1;
        DBuf<unsigned long long> gkey(T + 1, s);
        DBuf<uint32_t> grep(T + 1, s), gslot(count ? count : 1, s);
        DBuf<uint8_t> gmul(T + 1, s);
        DK_CUDA(cudaMemsetAsync(gkey.get(), 0xff, (T + 1) * 8, s));
        DK_CUDA(cudaMemsetAsync(grep.get(), 0xff, (T + 1) * 4, s));
        DK_CUDA(cudaMemsetAsync(gmul.get(), 0, T + 1, s));
        const unsigned eg = grid_for(count ? count : 1);
        // a compact element list: no buckets (nb = 0), every element a fallback one
        DK_LAUNCH(ctx, ghash_insert_kernel, eg, kThreads, 0, s, nullptr, 0u, count, fl.get(), T, gkey.get(),
                  grep.get(), gslot.get());
        DK_LAUNCH(ctx, ghash_multi_kernel, eg, kThreads, 0, s, nullptr, 0u, count, fl.get(), grep.get(), gslot.get(),
                  gmul.get());
        with_lab_type(vl, [&](auto lab) {
            DK_LAUNCH(ctx, ghash_out_kernel, eg, kThreads, 0, s, nullptr, 0u, count, fl.get(), grep.get(),
                      gslot.get(), gmul.get(), fp, d.delta, d.n, d.k, lab, go, dctr);
        });
    }
    DK_CUDA(cudaMemcpyAsync(counters, dctr, 4 * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
}

void shard_owner_scatter(Ctx* ctx, const OwnerPlan& op, const uint4* recv, const uint32_t* recv_cnt,
                         const uint32_t* results, const uint8_t* bsingle, const PeerLabels& out, cudaStream_t s) {
    const uint64_t total = (uint64_t)op.world * op.nb * op.cs;
    DK_LAUNCH_B(ctx, 25.0 * total * 3 / 4, owner_scatter_kernel, grid_for(total), kThreads, 0, s, recv, recv_cnt,
                op.world, op.nb, op.cs, results, bsingle, out);
}

void shard_apply_overflow(Ctx* ctx, const OwnerSend& ws, const uint32_t* back_ovf, uint32_t ovf_total, uint32_t* lab,
                          uint8_t* act, cudaStream_t s) {
    if (ovf_total)
        DK_LAUNCH(ctx, shard_apply_kernel, grid_for(ovf_total), kThreads, 0, s, ws.ovf_sorted.get(), back_ovf,
                  (uint64_t)ovf_total, lab, act);
}

void shard_apply_owner(Ctx* ctx, const OwnerPlan& op, const OwnerSend& ws, uint32_t rank, const uint32_t* own_res,
                       const uint32_t* back, const uint32_t* back_ovf, uint32_t ovf_total, uint32_t* lab,
                       uint8_t* act, cudaStream_t s) {
    const uint64_t total = (uint64_t)op.world * op.nb * op.cs;
    DK_LAUNCH_B(ctx, 25.0 * total * 3 / 4, owner_apply_kernel, grid_for(total), kThreads, 0, s, ws.send.get(),
                ws.scur.get(), op.world, op.nb, op.cs, rank, own_res, back, lab, act);
    if (ovf_total)
        DK_LAUNCH(ctx, shard_apply_kernel, grid_for(ovf_total), kThreads, 0, s, ws.ovf_sorted.get(), back_ovf,
                  (uint64_t)ovf_total, lab, act);
}

}  // namespace dk
