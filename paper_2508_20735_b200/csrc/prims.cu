// prims.cu -- scan, compaction and the LSD radix sort.
//
// Radix sort design: see "radix sort (one sweep per digit)" below.
#include <algorithm>

#include "prims.cuh"

namespace dk {

// ---------------------------------------------------------------------------
// block-level scan helpers (256 threads)
// ---------------------------------------------------------------------------


// ---------------------------------------------------------------------------
// exclusive scan
// ---------------------------------------------------------------------------

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const uint32_t* __restrict__ in, uint64_t n,
                                                                   uint32_t* __restrict__ sums) {
    __shared__ uint32_t ws[kScanThreads / 32];
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        uint64_t i = base + (uint64_t)j * kScanThreads + threadIdx.x;
        if (i < n) acc += in[i];
    }
    uint32_t total;
    block_exclusive_scan<kScanThreads>(acc, &total, ws);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads) scan_tile_kernel(const uint32_t* __restrict__ in, uint64_t n,
                                                                 uint32_t* __restrict__ out,
                                                                 const uint32_t* __restrict__ tile_offsets,
                                                                 uint32_t* __restrict__ total_dev) {
    __shared__ uint32_t tile[kScanTile];
    __shared__ uint32_t ws[kScanThreads / 32];
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        uint64_t i = base + (uint64_t)j * kScanThreads + threadIdx.x;
        tile[j * kScanThreads + threadIdx.x] = i < n ? in[i] : 0u;
    }
    __syncthreads();
    uint32_t local[kScanItems];
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        local[j] = tile[threadIdx.x * kScanItems + j];
        acc += local[j];
    }
    uint32_t total;
    uint32_t prefix = block_exclusive_scan<kScanThreads>(acc, &total, ws);
    const uint32_t off = tile_offsets ? tile_offsets[blockIdx.x] : 0u;
    prefix += off;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        tile[threadIdx.x * kScanItems + j] = prefix;
        prefix += local[j];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        uint64_t i = base + (uint64_t)j * kScanThreads + threadIdx.x;
        if (i < n) out[i] = tile[j * kScanThreads + threadIdx.x];
    }
    if (total_dev && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *total_dev = off + total;
}

void exclusive_scan_u32(Ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* total_dev,
                        cudaStream_t s) {
    if (n == 0) {
        if (total_dev) DK_CUDA(cudaMemsetAsync(total_dev, 0, sizeof(uint32_t), s));
        return;
    }
    const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
    if (tiles == 1) {
        DK_LAUNCH(ctx, scan_tile_kernel, 1, kScanThreads, 0, s, in, n, out, nullptr, total_dev);
        return;
    }
    DBuf<uint32_t> sums(tiles, s);
    DK_LAUNCH(ctx, scan_reduce_kernel, (unsigned)tiles, kScanThreads, 0, s, in, n, sums.get());
    exclusive_scan_u32(ctx, sums.get(), sums.get(), tiles, nullptr, s);
    DK_LAUNCH(ctx, scan_tile_kernel, (unsigned)tiles, kScanThreads, 0, s, in, n, out, sums.get(), total_dev);
}

// ---------------------------------------------------------------------------
// fill / iota / compaction
// ---------------------------------------------------------------------------

__global__ void fill_kernel(uint32_t* p, uint64_t n, uint32_t v) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

__global__ void iota_kernel(uint32_t* p, uint64_t n) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t nv = ((uintptr_t)p & 15u) == 0 ? n / 4 : 0;  // four per 16-byte store
    for (uint64_t v = tid; v < nv; v += stride) {
        const uint32_t i = (uint32_t)(4 * v);
        __stcs(reinterpret_cast<uint4*>(p) + v, make_uint4(i, i + 1, i + 2, i + 3));
    }
    for (uint64_t i = 4 * nv + tid; i < n; i += stride) p[i] = (uint32_t)i;
}

struct FillArgs {
    uint8_t* p[4];
    uint64_t bytes[4];
    uint32_t value[4];
};

// blockIdx.y = region; 16-byte stores between a byte head and tail
__global__ void fill_regions_kernel(FillArgs a) {
    uint8_t* p = a.p[blockIdx.y];
    const uint64_t nb = a.bytes[blockIdx.y];
    if (!p || !nb) return;
    const uint32_t v8 = a.value[blockIdx.y] & 0xffu, w = v8 * 0x01010101u;
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t head = (16u - ((uintptr_t)p & 15u)) & 15u;
    if (head > nb) head = nb;
    for (uint64_t i = tid; i < head; i += stride) p[i] = (uint8_t)v8;
    const uint64_t nv = (nb - head) / 16;
    uint4* q = reinterpret_cast<uint4*>(p + head);
    for (uint64_t i = tid; i < nv; i += stride) q[i] = make_uint4(w, w, w, w);
    for (uint64_t i = head + 16 * nv + tid; i < nb; i += stride) p[i] = (uint8_t)v8;
}

void Fills::add(void* ptr, uint64_t nbytes, uint8_t v) {
    if (!ptr || !nbytes) return;
    if (count == 4) throw Error(DFAKIT_E_INVALID, "Fills: more than four regions");
    p[count] = ptr;
    bytes[count] = nbytes;
    value[count] = v;
    ++count;
}

void Fills::flush(Ctx* ctx, cudaStream_t s) {
    if (!count) return;
    FillArgs a{};
    uint64_t most = 0;
    for (int i = 0; i < 4; ++i) {
        a.p[i] = static_cast<uint8_t*>(p[i]);
        a.bytes[i] = i < count ? bytes[i] : 0;
        a.value[i] = value[i];
        most = std::max<uint64_t>(most, bytes[i]);
    }
    const unsigned gx = grid_for(most / 16 + 1, kThreads, (unsigned)ctx->num_sms * 4u);
    DK_LAUNCH(ctx, fill_regions_kernel, dim3(gx, (unsigned)count), kThreads, 0, s, a);
    count = 0;
}

void fill_u32(Ctx* ctx, uint32_t* p, uint64_t n, uint32_t value, cudaStream_t s) {
    if (n) DK_LAUNCH(ctx, fill_kernel, grid_for(n), kThreads, 0, s, p, n, value);
}

void iota_u32(Ctx* ctx, uint32_t* p, uint64_t n, cudaStream_t s) {
    // ~8 16-byte stores per thread: one store per thread made the launch of
    // ~10^4 CTAs the cost of a 40 MB write
    if (n) DK_LAUNCH(ctx, iota_kernel, grid_for(n / 4 + 1, kThreads, (unsigned)ctx->num_sms * 8u), kThreads, 0, s, p, n);
}

// ---------------------------------------------------------------------------
// tiled compaction / head scan: per-tile counts, one-CTA scan of the tile
// counts, then an apply pass that re-reads its tile (coalesced), scans it in
// shared memory and writes coalesced.  Three launches, no inter-CTA spinning.
// ---------------------------------------------------------------------------

constexpr int kCpThreads = 256;
constexpr int kCpItems = 16;
constexpr int kCpTile = kCpThreads * kCpItems;

template <bool HEADS>
__device__ __forceinline__ uint32_t elem_flag(const uint32_t* __restrict__ lab, const uint8_t* __restrict__ flag,
                                              uint64_t i) {
    if (HEADS) return lab[i] == (uint32_t)i ? 1u : 0u;
    return flag[i] != 0 ? 1u : 0u;
}

template <bool HEADS>
__global__ void __launch_bounds__(kCpThreads) tile_count_kernel(const uint32_t* __restrict__ lab,
                                                                const uint8_t* __restrict__ flag, uint64_t n,
                                                                uint32_t* __restrict__ sums,
                                                                const uint32_t* __restrict__ skip) {
    if (skip && *skip == n) return;
    __shared__ uint32_t ws[kCpThreads / 32];
    const uint64_t base = (uint64_t)blockIdx.x * kCpTile;
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < kCpItems; ++j) {
        const uint64_t i = base + (uint64_t)j * kCpThreads + threadIdx.x;
        if (i < n) c += elem_flag<HEADS>(lab, flag, i);
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31u) == 0) ws[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
#pragma unroll
        for (int w = 0; w < kCpThreads / 32; ++w) t += ws[w];
        sums[blockIdx.x] = t;
    }
}

// exclusive scan of `tiles` counts in place by one CTA; total -> *total
__global__ void __launch_bounds__(1024) scan_counts_kernel(uint32_t* __restrict__ sums, uint32_t tiles,
                                                           uint32_t* __restrict__ total,
                                                           const uint32_t* __restrict__ skip, uint64_t n) {
    if (skip && *skip == n) return;
    __shared__ uint32_t ws[32];
    uint32_t carry = 0;
    for (uint32_t b = 0; b < tiles; b += 1024) {
        const uint32_t i = b + threadIdx.x;
        const uint32_t v = i < tiles ? sums[i] : 0u;
        uint32_t tot;
        const uint32_t e = block_exclusive_scan<1024>(v, &tot, ws);
        if (i < tiles) sums[i] = carry + e;
        carry += tot;
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

// Shared staging is skewed by one word per 32 (sk(p) = p + p / 32): the
// coalesced fill writes element j*256 + t, the scan reads 16 consecutive
// elements per thread -- unskewed that read is a 16-way bank conflict.
__device__ __forceinline__ uint32_t sk(uint32_t p) { return p + (p >> 5); }

struct CompactSmem {
    uint32_t v[kCpTile + kCpTile / 32];  // staged values, then selected values / positions
    uint32_t f[kCpTile + kCpTile / 32];  // staged flags
    uint32_t ws[kCpThreads / 32];
};

// HEADS: pos[i] = offset + #heads before i in the tile.  Else: compaction.
template <bool HEADS>
__global__ void __launch_bounds__(kCpThreads) tile_apply_kernel(const uint32_t* __restrict__ lab,
                                                                const uint8_t* __restrict__ flag,
                                                                const uint32_t* __restrict__ in, uint64_t n,
                                                                const uint32_t* __restrict__ offs,
                                                                uint32_t* __restrict__ out, uint32_t id_base,
                                                                const uint32_t* __restrict__ skip) {
    if (skip && *skip == n) return;
    __shared__ CompactSmem sm;
    const unsigned tid = threadIdx.x;
    const uint64_t base = (uint64_t)blockIdx.x * kCpTile;
#pragma unroll
    for (int j = 0; j < kCpItems; ++j) {
        const uint32_t p = j * kCpThreads + tid;
        const uint64_t i = base + p;
        const bool ok = i < n;
        sm.f[sk(p)] = ok ? elem_flag<HEADS>(lab, flag, i) : 0u;
        if (!HEADS) sm.v[sk(p)] = ok ? (in ? __ldcs(in + i) : id_base + (uint32_t)i) : 0u;
    }
    __syncthreads();
    uint32_t c = 0;
    uint32_t f[kCpItems];
    uint32_t v[kCpItems];
#pragma unroll
    for (int j = 0; j < kCpItems; ++j) {
        f[j] = sm.f[sk(tid * kCpItems + j)];
        if (!HEADS) v[j] = sm.v[sk(tid * kCpItems + j)];
        c += f[j];
    }
    uint32_t agg;
    uint32_t o = block_exclusive_scan<kCpThreads>(c, &agg, sm.ws);  // ends with a barrier
    const uint32_t off = offs[blockIdx.x];
    if (HEADS) {
        o += off;
#pragma unroll
        for (int j = 0; j < kCpItems; ++j) {
            sm.v[sk(tid * kCpItems + j)] = o;
            o += f[j];
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kCpItems; ++j) {
            const uint32_t p = j * kCpThreads + tid;
            const uint64_t i = base + p;
            if (i < n) out[i] = sm.v[sk(p)];
        }
    } else {
#pragma unroll
        for (int j = 0; j < kCpItems; ++j)
            if (f[j]) sm.v[sk(o++)] = v[j];
        __syncthreads();
        for (uint32_t i = tid; i < agg; i += kCpThreads) out[(uint64_t)off + i] = sm.v[sk(i)];
    }
}

template <bool HEADS>
void tiled_scan(Ctx* ctx, const uint32_t* lab, const uint8_t* flag, const uint32_t* in, uint64_t n, uint32_t* out,
                uint32_t* total_dev, cudaStream_t s, uint32_t id_base = 0, const uint32_t* skip = nullptr) {
    if (n == 0) {
        DK_CUDA(cudaMemsetAsync(total_dev, 0, sizeof(uint32_t), s));
        return;
    }
    const uint64_t tiles = (n + kCpTile - 1) / kCpTile;
    if (tiles > 0xffffffffull) throw Error(DFAKIT_E_RESOURCE, "scan: too many tiles");
    DBuf<uint32_t> sums(tiles, s);
    const double eb = HEADS ? 4.0 : 1.0;
    DK_LAUNCH_B(ctx, eb * n, tile_count_kernel<HEADS>, (unsigned)tiles, kCpThreads, 0, s, lab, flag, n, sums.get(),
                skip);
    DK_LAUNCH(ctx, scan_counts_kernel, 1, 1024, 0, s, sums.get(), (uint32_t)tiles, total_dev, skip, n);
    DK_LAUNCH_B(ctx, HEADS ? 8.0 * n : (double)n * (1.0 + (in ? 4.0 : 0.0)), tile_apply_kernel<HEADS>,
                (unsigned)tiles, kCpThreads, 0, s, lab, flag, in, n, sums.get(), out, id_base, skip);
}

void compact_flags(Ctx* ctx, const uint32_t* in, const uint8_t* flag, uint64_t n, uint32_t* out,
                   uint32_t* count_dev, cudaStream_t s, uint32_t id_base, const uint32_t* skip_if_all) {
    tiled_scan<false>(ctx, nullptr, flag, in, n, out, count_dev, s, id_base, skip_if_all);
}

void head_scan(Ctx* ctx, const uint32_t* lab, uint64_t n, uint32_t* pos, uint32_t* total_dev, cudaStream_t s) {
    tiled_scan<true>(ctx, lab, nullptr, nullptr, n, pos, total_dev, s);
}

// ---------------------------------------------------------------------------
// canonical renumbering
// ---------------------------------------------------------------------------

__global__ void relabel_kernel(const uint32_t* __restrict__ lab, uint64_t n, const uint32_t* __restrict__ dense,
                               uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = dense[lab[i]];
}

__global__ void label_min_kernel(const uint32_t* __restrict__ lab, uint64_t n, uint32_t* __restrict__ minof) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        atomicMin(&minof[lab[i]], (uint32_t)i);
}

__global__ void to_min_label_kernel(uint32_t* __restrict__ lab, uint64_t n, const uint32_t* __restrict__ minof) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        lab[i] = minof[lab[i]];
}

void min_state_labels(Ctx* ctx, uint32_t* lab, uint64_t n, uint32_t* scratch, cudaStream_t s) {
    if (n == 0) return;
    fill_u32(ctx, scratch, n, kNone, s);
    DK_LAUNCH(ctx, label_min_kernel, grid_for(n), kThreads, 0, s, lab, n, scratch);
    DK_LAUNCH(ctx, to_min_label_kernel, grid_for(n), kThreads, 0, s, lab, n, scratch);
}

template <typename T>
__global__ void relabel_narrow_kernel(const uint32_t* __restrict__ lab, uint64_t n, const uint32_t* __restrict__ dense,
                                      T* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = (T)dense[lab[i]];
}

uint32_t dense_labels(Ctx* ctx, const uint32_t* lab, uint64_t n, void* out, int bytes, uint32_t* scratch,
                      cudaStream_t s) {
    if (n == 0) return 0;
    head_scan(ctx, lab, n, scratch, scratch + n, s);
    if (bytes == 1)
        DK_LAUNCH(ctx, relabel_narrow_kernel<uint8_t>, grid_for(n), kThreads, 0, s, lab, n, scratch,
                  static_cast<uint8_t*>(out));
    else if (bytes == 2)
        DK_LAUNCH(ctx, relabel_narrow_kernel<uint16_t>, grid_for(n), kThreads, 0, s, lab, n, scratch,
                  static_cast<uint16_t*>(out));
    else
        DK_LAUNCH(ctx, relabel_kernel, grid_for(n), kThreads, 0, s, lab, n, scratch, static_cast<uint32_t*>(out));
    uint32_t total = 0;
    read_words(ctx, scratch + n, sizeof(uint32_t), &total, s);
    return total;
}

uint32_t canonical_from_min_labels(Ctx* ctx, const uint32_t* lab, uint64_t n, uint32_t* out, uint32_t* scratch,
                                   cudaStream_t s, uint64_t known_blocks) {
    if (n == 0) return 0;
    if (known_blocks == n) {  // every block a singleton: block q is number q
        iota_u32(ctx, out, n, s);
        return (uint32_t)n;
    }
    head_scan(ctx, lab, n, scratch, scratch + n, s);
    DK_LAUNCH(ctx, relabel_kernel, grid_for(n), kThreads, 0, s, lab, n, scratch, out);
    uint32_t total = 0;
    read_words(ctx, scratch + n, sizeof(uint32_t), &total, s);
    return total;
}

// ---------------------------------------------------------------------------
// radix sort (one sweep per digit)
//
//   1. radix_hist_all_kernel: one read of the keys histograms EVERY digit of
//      the sort (shared-memory counters, one global add per CTA and bin);
//      radix_bins_kernel turns each digit's histogram into bin offsets.
//   2. per digit, radix_onesweep_kernel: tiles are claimed in order from a
//      counter (so every lower tile is resident or done); the tile's digit
//      counts (shared atomics) are published first; each warp then ranks
//      its keys stably (match_any peers + popc of lower lanes + a per-warp
//      running count); thread d looks back over the predecessors' published
//      counts of digit d until it meets an inclusive prefix (decoupled
//      look-back), then publishes its own inclusive prefix; keys are staged digit-sorted in shared memory and
//      written out with consecutive threads on consecutive addresses of a
//      digit's output run.  Keys and values are read once and written once
//      per digit: no separate histogram or scan pass.
// Look-back words are 64-bit {tag:24 | flag:8 | count:32}; the tag is the
// digit pass (+1), so the passes share one array, zeroed once per sort: a
// word left by the previous pass reads as "not yet published".
// ---------------------------------------------------------------------------

constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
#ifndef DFAKIT_SORT_THREADS
#define DFAKIT_SORT_THREADS 256
#endif
constexpr int kSortThreads = DFAKIT_SORT_THREADS;  // >= kRadix: threads d < 256 own digit d in the tile scan
constexpr int kSortWarps = kSortThreads / 32;
#ifndef DFAKIT_SORT_ITEMS
#define DFAKIT_SORT_ITEMS 12
#endif
#ifndef DFAKIT_SORT_MINB
#define DFAKIT_SORT_MINB 3
#endif
constexpr int kSortItems = DFAKIT_SORT_ITEMS;
constexpr int kSortTile = kSortThreads * kSortItems;  // 3072 keys
constexpr int kWarpSpan = 32 * kSortItems;            // keys per warp segment
constexpr int kMaxDigits = 8;
constexpr unsigned long long kFlagAgg = 1ull, kFlagPre = 2ull;
// look-back window (predecessors per round trip): 1 / 4 / 8 measured
// 138 / 135 / 139 us per digit pass on 10M keys -- the ranking, not the
// look-back, bounds the pass once counts are published before it
#ifndef DFAKIT_SORT_LOOKWIN
#define DFAKIT_SORT_LOOKWIN 4
#endif
constexpr int kLookWin = DFAKIT_SORT_LOOKWIN;

__device__ __forceinline__ uint32_t digit_of(uint64_t key, uint32_t shift) {
    return (uint32_t)(key >> shift) & (kRadix - 1);
}

__global__ void __launch_bounds__(kSortThreads) radix_hist_all_kernel(const uint64_t* __restrict__ keys, uint64_t m,
                                                                      uint32_t bit_lo, uint32_t digits,
                                                                      uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[kMaxDigits][kRadix];
    for (int i = threadIdx.x; i < kMaxDigits * kRadix; i += kSortThreads) (&h[0][0])[i] = 0;
    __syncthreads();
    for (uint64_t i = blockIdx.x * (uint64_t)kSortThreads + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * kSortThreads) {
        const uint64_t key = __ldcs(keys + i);
        for (uint32_t p = 0; p < digits; ++p) atomicAdd(&h[p][digit_of(key, bit_lo + p * kRadixBits)], 1u);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < digits * kRadix; i += kSortThreads) {
        const uint32_t v = (&h[0][0])[i];
        if (v) atomicAdd(hist + i, v);
    }
}

// hist[p][d] -> exclusive bin offsets in place (one CTA per digit pass)
__global__ void __launch_bounds__(kRadix) radix_bins_kernel(uint32_t* __restrict__ hist) {
    __shared__ uint32_t ws[kRadix / 32];
    uint32_t* h = hist + (uint64_t)blockIdx.x * kRadix;
    uint32_t tot;
    const uint32_t e = block_exclusive_scan<kRadix>(h[threadIdx.x], &tot, ws);
    h[threadIdx.x] = e;
}

struct OnesweepSmem {
    uint64_t keys[kSortTile];
    uint32_t vals[kSortTile];
    uint32_t warp_hist[kSortWarps][kRadix];
    uint32_t match[kSortWarps][kRadix];  // per-warp digit -> lane mask (atomicOr ranking)
    uint32_t digit_start[kRadix];
    uint32_t global_base[kRadix];
    uint32_t tile_hist[kRadix];
    uint32_t ws[kSortWarps];
    uint32_t tile;
};

template <int W>
__global__ void __launch_bounds__(kSortThreads, DFAKIT_SORT_MINB) radix_onesweep_kernel(
    const uint64_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, uint64_t m, uint32_t shift,
    const uint32_t* __restrict__ bins, unsigned long long* __restrict__ look, uint32_t* __restrict__ tile_ctr,
    uint32_t tag, uint64_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    OnesweepSmem& sm = *reinterpret_cast<OnesweepSmem*>(smem_raw);
    const unsigned lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) sm.tile = atomicAdd(tile_ctr, 1u);
    for (int i = threadIdx.x; i < kSortWarps * kRadix; i += kSortThreads) {
        (&sm.warp_hist[0][0])[i] = 0;
        (&sm.match[0][0])[i] = 0;
    }
    if (threadIdx.x < kRadix) sm.tile_hist[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t tile = sm.tile;
    const uint64_t seg = (uint64_t)tile * kSortTile + (uint64_t)wid * kWarpSpan;
    uint64_t key[kSortItems];
    uint32_t val[kSortItems];
    uint32_t rank[kSortItems];
    const unsigned lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {  // all loads first
        const uint64_t i = seg + (uint64_t)j * 32 + lane;
        key[j] = i < m ? __ldcs(keys_in + i) : 0ull;
        val[j] = i < m ? __ldcs(vals_in + i) : 0u;
    }
    // the tile's digit counts are published before the ranking, so the
    // successors' look-back rarely waits on this tile
#pragma unroll
    for (int j = 0; j < kSortItems; ++j)
        if (seg + (uint64_t)j * 32 + lane < m) atomicAdd(&sm.tile_hist[digit_of(key[j], shift)], 1u);
    __syncthreads();
    volatile unsigned long long* lk = look;
    const unsigned long long hi = (unsigned long long)tag << 40;
    if (threadIdx.x < kRadix) {
        const uint32_t d = threadIdx.x, c = sm.tile_hist[d];
        lk[(uint64_t)tile * kRadix + d] = hi | ((tile == 0 ? kFlagPre : kFlagAgg) << 32) | c;
    }
    // stable warp ranking: the lanes of a digit find each other through a
    // shared lane mask (atomicOr, read back after a warp barrier -- cheaper
    // than match.any, whose latency bound this loop); the lowest lane of the
    // group owns the digit's warp counter for this item, bumps it and clears
    // the mask, and the peers take their offsets from it
    uint32_t* wmatch = sm.match[wid];
    uint32_t* whist = sm.warp_hist[wid];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const uint64_t i = seg + (uint64_t)j * 32 + lane;
        const bool valid = i < m;
        const uint32_t d = digit_of(key[j], shift);
        if (valid) atomicOr(&wmatch[d], 1u << lane);
        __syncwarp();
        const unsigned peers = valid ? wmatch[d] : 0u;
        const unsigned leader = valid ? (unsigned)(__ffs(peers) - 1) : lane;
        uint32_t base = 0;
        __syncwarp();
        if (valid && lane == leader) {
            base = whist[d];
            whist[d] = base + (uint32_t)__popc(peers);
            wmatch[d] = 0;
        }
        __syncwarp();  // the clears land before the next item's atomicOr
        base = __shfl_sync(0xffffffffu, base, leader);
        rank[j] = valid ? base + (uint32_t)__popc(peers & lt_mask) : kNone;
    }
    __syncthreads();
    uint32_t tile_count = 0;
    {
        const int d = threadIdx.x;  // digit d < kRadix; the other threads only join the scan
        uint32_t run = 0;
        if (d < kRadix) {
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            const uint32_t c = sm.warp_hist[w][d];
            sm.warp_hist[w][d] = run;
            run += c;
        }
        // decoupled look-back on digit d: W predecessors per round trip
        if (tile == 0) {
            sm.global_base[d] = bins[d];
        } else {
            uint32_t excl = 0;
            for (int64_t t = (int64_t)tile - 1; t >= 0;) {
                unsigned long long v[W];
#pragma unroll
                for (int j = 0; j < W; ++j)
                    v[j] = t - j >= 0 ? lk[(uint64_t)(t - j) * kRadix + d] : (hi | (kFlagPre << 32));
                int used = 0;
                bool done = false;
#pragma unroll
                for (int j = 0; j < W; ++j) {
                    if (done || used < j || (v[j] >> 40) != tag) continue;  // stop at the first unpublished word
                    excl += (uint32_t)v[j];
                    used = j + 1;
                    done = ((v[j] >> 32) & 0xffull) == kFlagPre;
                }
                if (done) break;
                t -= used;  // re-read from the first unpublished predecessor
            }
            lk[(uint64_t)tile * kRadix + d] = hi | (kFlagPre << 32) | (excl + run);
            sm.global_base[d] = bins[d] + excl;
        }
        }
        const uint32_t ds = block_exclusive_scan<kSortThreads>(run, &tile_count, sm.ws);
        if (d < kRadix) sm.digit_start[d] = ds;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        if (rank[j] != kNone) {
            const uint32_t d = digit_of(key[j], shift);
            const uint32_t p = sm.digit_start[d] + sm.warp_hist[wid][d] + rank[j];
            sm.keys[p] = key[j];
            sm.vals[p] = val[j];
        }
    }
    __syncthreads();
    for (uint32_t p = threadIdx.x; p < tile_count; p += kSortThreads) {
        const uint64_t k = sm.keys[p];
        const uint32_t d = digit_of(k, shift);
        const uint64_t g = (uint64_t)sm.global_base[d] + (p - sm.digit_start[d]);
        __stcs(keys_out + g, k);
        __stcs(vals_out + g, sm.vals[p]);
    }
}

bool radix_sort_pairs_range(Ctx* ctx, RadixBuffers b, uint64_t m, uint32_t bit_lo, uint32_t bit_hi,
                            cudaStream_t s) {
    static_assert(kSortThreads >= kRadix && kSortThreads % 32 == 0, "one thread per digit in the tile scan");
    if (m <= 1 || bit_hi <= bit_lo) return false;
    if (m > 0xffffffffull) throw Error(DFAKIT_E_RESOURCE, "radix sort: more than 2^32 keys");
    DK_CUDA(cudaFuncSetAttribute(radix_onesweep_kernel<kLookWin>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(OnesweepSmem)));
    DK_CUDA(cudaFuncSetAttribute(radix_onesweep_kernel<kLookWin>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    const uint32_t passes = (bit_hi - bit_lo + kRadixBits - 1) / kRadixBits;
    if (passes > kMaxDigits) throw Error(DFAKIT_E_INVALID, "radix sort: more than 64 key bits");
    const uint32_t tiles = (uint32_t)((m + kSortTile - 1) / kSortTile);
    // [hist: passes x 256][tile counters: passes] then the look-back words
    const size_t small = (size_t)passes * kRadix + passes;
    const size_t small_words = (small + 1) / 2 * 2;  // 8-byte alignment of the look-back words
    const size_t bytes = small_words * 4 + (size_t)tiles * kRadix * 8;  // look-back words shared by the passes
    DBuf<unsigned char> scratch(bytes, s);
    DK_CUDA(cudaMemsetAsync(scratch.get(), 0, bytes, s));
    uint32_t* hist = reinterpret_cast<uint32_t*>(scratch.get());
    uint32_t* ctr = hist + (size_t)passes * kRadix;
    unsigned long long* look = reinterpret_cast<unsigned long long*>(scratch.get() + small_words * 4);
    DK_LAUNCH_B(ctx, 8.0 * m, radix_hist_all_kernel, grid_for(m, kSortThreads, 148u * 8u), kSortThreads, 0, s, b.k0,
                m, bit_lo, passes, hist);
    DK_LAUNCH(ctx, radix_bins_kernel, passes, kRadix, 0, s, hist);
    bool flipped = false;
    for (uint32_t p = 0; p < passes; ++p) {
        const uint32_t shift = bit_lo + p * kRadixBits;
        const uint64_t* kin = flipped ? b.k1 : b.k0;
        const uint32_t* vin = flipped ? b.v1 : b.v0;
        uint64_t* kout = flipped ? b.k0 : b.k1;
        uint32_t* vout = flipped ? b.v0 : b.v1;
        DK_LAUNCH_B(ctx, 24.0 * m, radix_onesweep_kernel<kLookWin>, tiles, kSortThreads, sizeof(OnesweepSmem), s, kin, vin, m,
                    shift, hist + (size_t)p * kRadix, look, ctr + p, p + 1, kout, vout);
        flipped = !flipped;
    }
    return flipped;
}

bool radix_sort_pairs(Ctx* ctx, RadixBuffers b, uint64_t m, uint32_t nbits, cudaStream_t s) {
    return radix_sort_pairs_range(ctx, b, m, 0, nbits, s);
}

}  // namespace dk
