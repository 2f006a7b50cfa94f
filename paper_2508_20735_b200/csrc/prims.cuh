// prims.cuh -- device-wide primitives used by every refinement path:
// exclusive scan, stream compaction, and the LSD radix sort of
// (64-bit key, 32-bit value) pairs with warp-match histograms.
#pragma once

#include "common.cuh"

namespace dk {

// Block-wide exclusive scan of one value per thread (THREADS a multiple of
// 32, <= 1024); *total receives the block sum.  warp_sums: THREADS/32 words
// of shared memory.  Contains __syncthreads: call from every thread.
template <int THREADS>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total, uint32_t* warp_sums) {
    constexpr int W = THREADS / 32;
    const unsigned lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (unsigned)o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t s = lane < (unsigned)W ? warp_sums[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= (unsigned)o) s += y;
        }
        if (lane < (unsigned)W) warp_sums[lane] = s;
    }
    __syncthreads();
    uint32_t prefix = wid ? warp_sums[wid - 1] : 0u;
    *total = warp_sums[W - 1];
    __syncthreads();
    return prefix + x - v;
}

// out[i] = sum_{j<i} in[i]; optional *total_dev receives the full sum.
// in and out may alias.  Works for any n (multi-level).
void exclusive_scan_u32(Ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* total_dev,
                        cudaStream_t s);

// LSD radix sort on bits [0, nbits) of 64-bit keys with 32-bit values.
// Stable.  Ping-pongs between (k0,v0) and (k1,v1); returns true when the
// sorted data ended in (k1,v1).
struct RadixBuffers {
    uint64_t* k0;
    uint32_t* v0;
    uint64_t* k1;
    uint32_t* v1;
};
bool radix_sort_pairs(Ctx* ctx, RadixBuffers b, uint64_t m, uint32_t nbits, cudaStream_t s);
// Same, on the bit range [bit_lo, bit_hi) only (8-bit digits from bit_lo up).
bool radix_sort_pairs_range(Ctx* ctx, RadixBuffers b, uint64_t m, uint32_t bit_lo, uint32_t bit_hi,
                            cudaStream_t s);

// Stream compaction (tile counts, one-CTA scan, apply):
// out[j] = in ? in[i] : id_base + i for the j-th i with flag[i] != 0, order
// preserved.
// *count_dev receives the count.  Returns nothing (no host sync).  When
// skip_if_all is given and *skip_if_all == n on the device, every launch
// exits at once (all flags set: the caller keeps the identity list) and
// neither out nor *count_dev is written.
void compact_flags(Ctx* ctx, const uint32_t* in, const uint8_t* flag, uint64_t n, uint32_t* out,
                   uint32_t* count_dev, cudaStream_t s, uint32_t id_base = 0, const uint32_t* skip_if_all = nullptr);

// Dense first-occurrence block ids of min-state labels written in the
// narrowest type that holds them: bytes = 1, 2 or 4 (uint8/uint16/uint32).
// Returns the block count (synchronises).  scratch holds n+1 uint32.
uint32_t dense_labels(Ctx* ctx, const uint32_t* lab, uint64_t n, void* out, int bytes, uint32_t* scratch,
                      cudaStream_t s);

// Up to four byte-fills (cudaMemsetAsync semantics) in one launch: each
// separate memset is its own operation on the stream (~2-3 us of the pass
// prologue each).
struct Fills {
    void* p[4] = {nullptr, nullptr, nullptr, nullptr};
    uint64_t bytes[4] = {0, 0, 0, 0};
    uint32_t value[4] = {0, 0, 0, 0};
    int count = 0;
    void add(void* ptr, uint64_t nbytes, uint8_t v);
    void flush(Ctx* ctx, cudaStream_t s);
};

// Fills [0, n) with value.
void fill_u32(Ctx* ctx, uint32_t* p, uint64_t n, uint32_t value, cudaStream_t s);
void iota_u32(Ctx* ctx, uint32_t* p, uint64_t n, cudaStream_t s);

// Canonical first-occurrence renumbering of min-state labels: every block's
// label is its minimum member, so heads are states with lab[q] == q and the
// dense id of a block is the number of heads before its label.
// out may alias nothing; scratch holds n+1 uint32.  Returns the block count.
// known_blocks == n (the caller's block count says every block is a
// singleton): the numbering is the identity, no scan.
uint32_t canonical_from_min_labels(Ctx* ctx, const uint32_t* lab, uint64_t n, uint32_t* out, uint32_t* scratch,
                                   cudaStream_t s, uint64_t known_blocks = 0);

// Rewrites arbitrary block labels (label values < n) in place so every
// block is labelled by its minimum member.  scratch holds n uint32.
void min_state_labels(Ctx* ctx, uint32_t* lab, uint64_t n, uint32_t* scratch, cudaStream_t s);

}  // namespace dk
