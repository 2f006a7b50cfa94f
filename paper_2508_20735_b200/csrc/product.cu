// product.cu -- Hopcroft-Karp equivalence / inclusion checking (paper Alg. 6,
// reference src/equivalence.cpp:138-215) on B200.
//
// explore_product: level-synchronous BFS over the synchronous product with
// a lock-free open-addressing hash set of packed (qA, qB) pairs.  Each
// 16-byte slot holds the key and a "discoverer" word (parent record << 32 |
// letter); every lane first tries its key's home slot alone, and keys that
// collide continue with tile-cooperative probing: 4 lanes inspect a 4-slot
// (64 B) window per step with ballots for match / empty, and the leader
// claims an empty slot with a 64-bit CAS.  Within a wave every (frontier record,
// letter) item atomicMin's its discoverer into the slot it reached, so the
// minimum (parent, letter) -- the pair's position in the reference's
// sequential insertion order -- wins.  A flag + exclusive scan then emits the
// wave's new records in exactly the reference's record order, which makes
// explored_states, levels and the counterexample word identical to the
// reference's (the first failing record in that order is the one the
// sequential loop stops at).
//
// check_equiv_uf: Hopcroft-Karp proper, with a GPU union-find over
// QA + QB (path-halving CAS finds, union by index); a pair is explored only
// when its union succeeds.
#include <cooperative_groups.h>

#include <cstdlib>
#include <vector>

#include "prims.cuh"
#include "refine.cuh"

namespace cg = cooperative_groups;

namespace dk {

namespace {

constexpr unsigned long long kEmpty = ~0ull;
constexpr int kTile = 4;

struct Slot {
    unsigned long long key;
    unsigned long long disc;
};

// primary slot of first-automaton state pa: the pair's second state and its
// discoverer in one 16-byte record (one sector per pair, not two)
struct PrimSlot {
    uint32_t pb, pad;
    unsigned long long disc;
};

struct Rec {
    unsigned long long* key;
    uint32_t* parent;
    uint32_t* letter;
};

__device__ __forceinline__ uint64_t slot_hash(uint64_t key) { return mix64(key ^ 0x243F6A8885A308D3ull); }

// Find-or-insert of every lane's key.  Probe order is linear from the home
// slot.  Each lane first inspects its home slot on its own (at the table's
// load <= 1/2 that settles almost every key in one round trip, and the lanes'
// round trips overlap); keys whose home slot holds another key continue
// tile-cooperatively: 4 lanes inspect a 4-slot window (home + 1 ...) per step
// with ballots for match / empty, and the leader claims an empty slot with a
// 64-bit CAS.  Slots only go empty -> full, so scanning in one fixed order and
// claiming the first empty slot never inserts a key twice.  Returns the slot
// of this lane's key (kNone when !valid).
__device__ uint32_t tile_find_or_insert(cg::thread_block_tile<kTile> tile, bool valid, unsigned long long key,
                                        Slot* __restrict__ table, uint64_t mask) {
    uint32_t mine = kNone;
    bool open = false;
    if (valid) {
        const uint64_t home = slot_hash(key) & mask;
        unsigned long long e = __ldcg(&table[home].key);
        if (e == kEmpty) e = atomicCAS(&table[home].key, kEmpty, key);
        if (e == kEmpty || e == key)
            mine = (uint32_t)home;
        else
            open = true;
    }
    if (!tile.any(open)) return mine;
    const unsigned lane = tile.thread_rank();
    for (int j = 0; j < kTile; ++j) {
        if (!tile.shfl(open, j)) continue;
        const unsigned long long kj = tile.shfl(key, j);
        uint64_t base = (slot_hash(kj) + 1) & mask;
        uint32_t found = kNone;
        for (;;) {
            const uint64_t sl = (base + lane) & mask;
            const unsigned long long e = __ldcg(&table[sl].key);
            const unsigned match = tile.ballot(e == kj);
            const unsigned empty = tile.ballot(e == kEmpty);
            // the first slot in probe order that holds kj or is empty
            const unsigned hit = match | empty;
            if (hit) {
                const unsigned first = __ffs(hit) - 1;
                if (match & (1u << first)) {
                    found = (uint32_t)((base + first) & mask);
                    break;
                }
                unsigned long long old = 0;
                if (lane == first) old = atomicCAS(&table[(base + first) & mask].key, kEmpty, kj);
                old = tile.shfl(old, first);
                if (old == kEmpty || old == kj) {
                    found = (uint32_t)((base + first) & mask);
                    break;
                }
                continue;  // lost the slot to another key: re-read the window
            }
            base = (base + kTile) & mask;
        }
        if (lane == (unsigned)j) mine = found;
    }
    return mine;
}

// Records into a fresh table, discovered before any current wave.  Primary
// mode (prim): a record takes its first state's primary slot when free (the
// initial pair) or already holds it (keeps its discoverer); the others go
// back into the (grown) hash table, counted as its reservations.
__global__ void reinsert_kernel(const unsigned long long* __restrict__ keys, uint64_t count, Slot* __restrict__ table,
                                uint64_t mask, PrimSlot* __restrict__ prim, unsigned long long* __restrict__ hkeys) {
    auto tile = cg::tiled_partition<kTile>(cg::this_thread_block());
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t first = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t trips = (count + stride - 1) / stride;
    for (uint64_t it = 0; it < trips; ++it) {
        const uint64_t t = first + it * stride;
        const unsigned long long key = t < count ? keys[t] : 0ull;
        bool valid = t < count;
        if (valid && prim) {
            const uint32_t pa = (uint32_t)(key >> 32), pb = (uint32_t)key;
            uint32_t e = prim[pa].pb;
            if (e == kNone) e = atomicCAS(&prim[pa].pb, kNone, pb);
            if (e == kNone) prim[pa].disc = 0ull;
            valid = e != kNone && e != pb;
        }
        const uint32_t s = tile_find_or_insert(tile, valid, key, table, mask);
        if (valid) {
            table[s].disc = 0ull;
            if (hkeys) atomicAdd(hkeys, 1ull);
        }
    }
}

__global__ void walk_word_kernel(Rec rec, uint32_t idx, uint32_t* __restrict__ word, uint32_t cap,
                                 uint32_t* __restrict__ len_out) {
    uint32_t len = 0;
    for (uint32_t i = idx; i != 0; i = rec.parent[i]) ++len;
    uint32_t p = len;
    for (uint32_t i = idx; i != 0; i = rec.parent[i]) {
        --p;
        if (p < cap) word[p] = rec.letter[i];
    }
    *len_out = len;
}

// ---- union-find -------------------------------------------------------------

__device__ __forceinline__ uint32_t uf_find(uint32_t* __restrict__ P, uint32_t x) {
    for (;;) {
        const uint32_t p = __ldcg(P + x);
        if (p == x) return x;
        const uint32_t gp = __ldcg(P + p);
        if (gp != p) atomicCAS(P + x, p, gp);  // path halving
        x = gp;
    }
}

__device__ __forceinline__ bool uf_union(uint32_t* __restrict__ P, uint32_t a, uint32_t b) {
    for (;;) {
        a = uf_find(P, a);
        b = uf_find(P, b);
        if (a == b) return false;
        if (a < b) {
            const uint32_t t = a;
            a = b;
            b = t;
        }
        if (atomicCAS(P + a, a, b) == a) return true;  // link the larger root under the smaller
    }
}

__global__ void uf_init_kernel(uint32_t* P, uint64_t total) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x)
        P[i] = (uint32_t)i;
}

__global__ void uf_seed_kernel(uint32_t* P, uint32_t a, uint32_t b) { uf_union(P, a, b); }

// ---- persistent BFS ------------------------------------------------------------
//
// All levels of the product BFS in one cooperative launch.  Per level:
// expand (find-or-insert + discoverer atomicMin), barrier, winner counts
// over contiguous item chunks (one per CTA), barrier, emit: each CTA's chunk
// in item order at its prefix of the counts (block-scanned tiles), so the
// records land in exactly the order the per-level kernels produce --
// barrier, then every thread reads the level's total and first failure.
// The kernel returns to the host only when the table / record store must
// grow or the exploration ends.

enum : uint32_t { kBfsRunning = 0, kBfsDone = 1, kBfsGrow = 2, kBfsFail = 3, kBfsBudget = 4 };

struct BfsState {
    unsigned long long wb, we;
    unsigned long long first_fail_all;  // FULL mode: first failing record (~0 if none)
    uint32_t levels, status;
    uint32_t fail_rec;                  // failing record (kBfsFail)
    uint32_t need_grow;                 // primary mode: a hash-table insertion found no room (level re-run)
    uint32_t fail[3];                   // per level (mod 3): first failing emit position
    uint32_t pad;
    unsigned long long hkeys;           // primary mode: hash-table reservations (>= keys in it)
};

struct BfsArgs {
    Rec rec;
    uint64_t rec_cap;
    Slot* table;
    uint64_t cap;  // slots (power of two)
    uint32_t* item_slot;
    uint8_t* item_win;  // winner flags of the counting phase, reused by the emit phase
    unsigned long long* item_key;  // each item's pair key (coalesced; spares a random table read)
    uint64_t item_cap;
    uint32_t* cta_cnt;
    const uint32_t *da, *db, *to_b;
    uint32_t na, nb, k;
    const uint8_t *acc_a, *acc_b;
    int mode;
    uint64_t max_visited;
    BfsState* st;
    // primary mode: pair (pa, pb) lives in slot pa of a direct-mapped table
    // (prim: {pb, discoverer} per state of A) unless another pb holds it -- then in the
    // hash table, whose insertions reserve room first
    PrimSlot* prim;
};

constexpr uint32_t kPrim = 0x80000000u;  // item slot: primary slot pa (pa < 2^31)

__device__ __forceinline__ unsigned long long* disc_at(const BfsArgs& A, uint32_t sl) {
    return (sl & kPrim) ? &A.prim[sl & ~kPrim].disc : &A.table[sl].disc;
}

// find-or-insert of every lane's pair: its primary slot when free or its
// own, else the hash table (all lanes of the tile call; a lane whose hash
// insertion finds no reserved room gets kNone and flags the level for a re-run)
__device__ __forceinline__ uint32_t pair_find_or_insert(cg::thread_block_tile<kTile> tile, bool valid,
                                                        unsigned long long key, const BfsArgs& A, uint64_t mask) {
    bool hash = valid;
    uint32_t mine = kNone;
    if (valid && A.prim) {
        const uint32_t pa = (uint32_t)(key >> 32), pb = (uint32_t)key;
        uint32_t e = __ldcg(&A.prim[pa].pb);
        if (e == kNone) e = atomicCAS(&A.prim[pa].pb, kNone, pb);
        if (e == kNone || e == pb) {
            mine = kPrim | pa;
            hash = false;
        } else if (atomicAdd(&A.st->hkeys, 1ull) >= A.cap / 2) {
            atomicExch(&A.st->need_grow, 1u);
            hash = false;
        }
    }
    const uint32_t h = tile_find_or_insert(tile, hash, key, A.table, mask);
    return hash ? h : mine;
}

__device__ __forceinline__ bool item_wins(const BfsArgs& A, uint64_t wb, uint64_t t, uint32_t k) {
    const uint32_t s = A.item_slot[t];
    if (s == kNone) return false;
    const unsigned long long disc = ((unsigned long long)(wb + t / k + 1) << 32) | (uint32_t)(t % k);
    return __ldcg(disc_at(A, s)) == disc;
}

// Levels of at most kSoloItems (frontier records x letters) run on CTA 0
// alone, one after another, with block barriers between the phases; the
// other CTAs wait at ONE grid barrier for the whole run of small levels
// (the ~30 small levels of a 10M-state exploration otherwise paid three grid
// barriers each).  Same table, same winner rule, same record order.
#ifndef DFAKIT_BFS_SOLO
#define DFAKIT_BFS_SOLO 1024
#endif
constexpr uint64_t kSoloItems = DFAKIT_BFS_SOLO;

struct SoloOut {
    uint64_t wb, we;
    unsigned long long first_fail_all;
    uint32_t levels, status;
};

__device__ void solo_levels(const BfsArgs& A, SoloOut& o) {
    auto tile = cg::tiled_partition<kTile>(cg::this_thread_block());
    __shared__ uint32_t ws[kThreads / 32];
    __shared__ uint32_t s_fail;
    BfsState* st = A.st;
    const uint64_t mask = A.cap - 1;
    uint64_t wb = o.wb, we = o.we;
    uint32_t levels = o.levels;
    uint32_t status = kBfsRunning;
    while (wb < we) {
        const uint64_t items = (we - wb) * A.k;
        if (items > kSoloItems) break;  // back to the whole grid
        if (items > A.item_cap || we + items > A.rec_cap || (!A.prim && 2 * (we + items) + 64 > A.cap)) {
            status = kBfsGrow;
            break;
        }
        if (threadIdx.x == 0) s_fail = kNone;
        for (uint64_t base = 0; base < items; base += blockDim.x) {
            const uint64_t t = base + threadIdx.x;
            const bool valid = t < items;
            unsigned long long key = 0, disc = 0;
            if (valid) {
                const uint64_t i = wb + t / A.k;
                const uint32_t la = (uint32_t)(t % A.k);
                const unsigned long long pk = __ldcg(A.rec.key + i);
                const uint32_t pa = A.da[(uint64_t)la * A.na + (uint32_t)(pk >> 32)];
                const uint32_t pb = A.db[(uint64_t)A.to_b[la] * A.nb + (uint32_t)pk];
                key = ((unsigned long long)pa << 32) | pb;
                disc = ((unsigned long long)(i + 1) << 32) | la;
            }
            const uint32_t sl = pair_find_or_insert(tile, valid, key, A, mask);
            if (valid && sl != kNone) {
                const unsigned long long old = atomicMin(disc_at(A, sl), disc);
                // a candidate winner only if the slot is new this level AND no
                // smaller discoverer got there first (a loser needs no re-check;
                // old == disc: this item's own discoverer from an aborted run
                // of the level -- the level is re-run after the table grows)
                A.item_slot[t] = (old >= ((unsigned long long)(wb + 1) << 32) && old >= disc) ? sl : kNone;
                A.item_key[t] = key;
            }
        }
        __syncthreads();
        if (A.prim && *(volatile uint32_t*)&A.st->need_grow) {  // re-run this level once the hash table grew
            status = kBfsGrow;
            break;
        }
        uint32_t run = 0;
        for (uint64_t base = 0; base < items; base += blockDim.x) {
            const uint64_t t = base + threadIdx.x;
            const bool win = t < items && item_wins(A, wb, t, A.k);
            uint32_t tot;
            const uint32_t e = block_exclusive_scan<kThreads>(win ? 1u : 0u, &tot, ws);
            if (win) {
                const uint32_t posn = run + e;
                const uint64_t r = we + posn;
                const unsigned long long key = A.item_key[t];
                A.rec.key[r] = key;
                A.rec.parent[r] = (uint32_t)(wb + t / A.k);
                A.rec.letter[r] = (uint32_t)(t % A.k);
                const bool fa = A.acc_a[key >> 32], fb = A.acc_b[(uint32_t)key];
                const bool fails = A.mode == DFAKIT_MODE_INCLUSION ? (fa && !fb) : (fa != fb);
                if (fails) atomicMin(&s_fail, posn);
            }
            run += tot;
        }
        __syncthreads();
        const uint32_t ff = s_fail, total = run;
        __syncthreads();  // s_fail is reset by the next level
        if (ff != kNone && A.mode != DFAKIT_MODE_FULL) {
            if (we + ff >= A.max_visited) {
                status = kBfsBudget;
            } else {
                status = kBfsFail;
                if (threadIdx.x == 0) st->fail_rec = (uint32_t)(we + ff);
            }
            we = we + ff + 1;
            break;
        }
        if (we + total > A.max_visited) {
            status = kBfsBudget;
            break;
        }
        if (ff != kNone && o.first_fail_all == ~0ull) o.first_fail_all = we + ff;
        ++levels;
        wb = we;
        we += total;
    }
    if (status == kBfsRunning && wb >= we) status = kBfsDone;
    o.wb = wb;
    o.we = we;
    o.levels = levels;
    o.status = status;
}

// the initial pair (record 0) fails the check: a counterexample at once
// (the empty word, one explored pair), or -- FULL mode -- the first failure
__global__ void bfs_init_kernel(const uint8_t* __restrict__ acc_a, const uint8_t* __restrict__ acc_b, uint32_t ia,
                                uint32_t ib, int mode, BfsState* st) {
    const bool fa = acc_a[ia] != 0, fb = acc_b[ib] != 0;
    if (!(mode == DFAKIT_MODE_INCLUSION ? (fa && !fb) : (fa != fb))) return;
    if (mode == DFAKIT_MODE_FULL) {
        st->first_fail_all = 0;
    } else {
        st->status = kBfsFail;
        st->fail_rec = 0;
    }
}

__global__ void __launch_bounds__(kThreads) bfs_persistent_kernel(BfsArgs A) {
    if (*(volatile uint32_t*)&A.st->status == kBfsFail) return;  // decided by bfs_init_kernel (uniform)
    cg::grid_group grid = cg::this_grid();
    auto tile = cg::tiled_partition<kTile>(cg::this_thread_block());
    __shared__ uint32_t ws[kThreads / 32];
    __shared__ uint32_t red[kThreads / 32];
    BfsState* st = A.st;
    uint64_t wb = st->wb, we = st->we;
    uint32_t levels = st->levels;
    unsigned long long first_fail_all = st->first_fail_all;
    uint32_t status = kBfsDone;
    const uint64_t mask = A.cap - 1;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    __shared__ SoloOut s_solo;
    while (wb < we) {
        const uint64_t items = (we - wb) * A.k;
        if (items <= kSoloItems) {
            // a run of small levels on CTA 0; everyone else waits at one barrier
            if (blockIdx.x == 0) {
                if (threadIdx.x == 0) s_solo = SoloOut{wb, we, first_fail_all, levels, kBfsRunning};
                __syncthreads();
                SoloOut o = s_solo;
                solo_levels(A, o);
                if (threadIdx.x == 0) {
                    st->wb = o.wb;
                    st->we = o.we;
                    st->levels = o.levels;
                    st->status = o.status;
                    st->first_fail_all = o.first_fail_all;
                }
            }
            grid.sync();
            if (threadIdx.x == 0) {
                volatile BfsState* vs = st;
                s_solo = SoloOut{vs->wb, vs->we, vs->first_fail_all, vs->levels, vs->status};
            }
            __syncthreads();
            const SoloOut o = s_solo;
            __syncthreads();
            wb = o.wb;
            we = o.we;
            levels = o.levels;
            first_fail_all = o.first_fail_all;
            if (o.status != kBfsRunning) {
                status = o.status;
                break;
            }
            continue;
        }
        if (items > A.item_cap || we + items > A.rec_cap || (!A.prim && 2 * (we + items) + 64 > A.cap)) {
            status = kBfsGrow;
            break;
        }
        // three slots: threads may still read level L-1's slot while level L
        // starts; level L-2's slot (= level L+1's) is free
        const uint32_t par = levels % 3;
        if (gtid == 0) {
            st->fail[par] = kNone;  // (a preceding run of solo levels did not reset it)
            st->fail[(levels + 1) % 3] = kNone;
        }
        // expand
        const uint64_t trips = (items + stride - 1) / stride;
        for (uint64_t it = 0; it < trips; ++it) {
            const uint64_t t = gtid + it * stride;
            const bool valid = t < items;
            unsigned long long key = 0, disc = 0;
            if (valid) {
                const uint64_t i = wb + t / A.k;
                const uint32_t la = (uint32_t)(t % A.k);
                const unsigned long long pk = __ldcg(A.rec.key + i);
                const uint32_t pa = A.da[(uint64_t)la * A.na + (uint32_t)(pk >> 32)];
                const uint32_t pb = A.db[(uint64_t)A.to_b[la] * A.nb + (uint32_t)pk];
                key = ((unsigned long long)pa << 32) | pb;
                disc = ((unsigned long long)(i + 1) << 32) | la;
            }
            const uint32_t sl = pair_find_or_insert(tile, valid, key, A, mask);
            if (valid && sl != kNone) {
                const unsigned long long old = atomicMin(disc_at(A, sl), disc);
                // a candidate winner only if the slot is new this level AND no
                // smaller discoverer got there first (a loser needs no re-check;
                // old == disc only on a re-run of the level, see solo_levels)
                A.item_slot[t] = (old >= ((unsigned long long)(wb + 1) << 32) && old >= disc) ? sl : kNone;
                A.item_key[t] = key;
            }
        }
        grid.sync();
        if (A.prim) {  // some insertion found no room: grow the hash table and re-run the level
            if (threadIdx.x == 0) red[0] = *(volatile uint32_t*)&A.st->need_grow;
            __syncthreads();
            const uint32_t ng = red[0];
            __syncthreads();
            if (ng) {
                status = kBfsGrow;
                break;
            }
        }
        // winner counts per contiguous chunk
        const uint64_t chunk = (items + gridDim.x - 1) / gridDim.x;
        const uint64_t c0 = min(items, blockIdx.x * chunk), c1 = min(items, c0 + chunk);
        uint32_t c = 0;
        for (uint64_t t = c0 + threadIdx.x; t < c1; t += blockDim.x) {
            const bool w = item_wins(A, wb, t, A.k);
            A.item_win[t] = w;
            c += w;
        }
        c = __reduce_add_sync(0xffffffffu, c);
        if ((threadIdx.x & 31u) == 0) red[threadIdx.x >> 5] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t tot = 0;
            for (int w = 0; w < kThreads / 32; ++w) tot += red[w];
            A.cta_cnt[blockIdx.x] = tot;
        }
        grid.sync();
        // prefix of this CTA, total of the level
        uint32_t pre = 0, total = 0;
        // four counts per 16-byte load (the count array is padded with zeros):
        // every CTA reads all of them, so this is gridDim^2 / 4 requests
        for (uint32_t j4 = threadIdx.x; j4 < (gridDim.x + 3) / 4; j4 += blockDim.x) {
            const uint4 v = __ldcg(reinterpret_cast<const uint4*>(A.cta_cnt) + j4);
            const uint32_t j = 4 * j4;
            total += v.x + v.y + v.z + v.w;
            pre += (j < blockIdx.x ? v.x : 0u) + (j + 1 < blockIdx.x ? v.y : 0u) + (j + 2 < blockIdx.x ? v.z : 0u) +
                   (j + 3 < blockIdx.x ? v.w : 0u);
        }
        pre = __reduce_add_sync(0xffffffffu, pre);
        total = __reduce_add_sync(0xffffffffu, total);
        __syncthreads();
        if ((threadIdx.x & 31u) == 0) {
            red[threadIdx.x >> 5] = pre;
            ws[threadIdx.x >> 5] = total;
        }
        __syncthreads();
        pre = 0;
        total = 0;
        for (int w = 0; w < kThreads / 32; ++w) {
            pre += red[w];
            total += ws[w];
        }
        __syncthreads();
        // emit in item order
        uint32_t run = pre;
        for (uint64_t base = c0; base < c1; base += blockDim.x) {
            const uint64_t t = base + threadIdx.x;
            const bool win = t < c1 && A.item_win[t];
            uint32_t tot;
            const uint32_t e = block_exclusive_scan<kThreads>(win ? 1u : 0u, &tot, ws);
            if (win) {
                const uint32_t posn = run + e;
                const uint64_t r = we + posn;
                const unsigned long long key = A.item_key[t];
                A.rec.key[r] = key;
                A.rec.parent[r] = (uint32_t)(wb + t / A.k);
                A.rec.letter[r] = (uint32_t)(t % A.k);
                const bool fa = A.acc_a[key >> 32], fb = A.acc_b[(uint32_t)key];
                const bool fails = A.mode == DFAKIT_MODE_INCLUSION ? (fa && !fb) : (fa != fb);
                if (fails) atomicMin(&st->fail[par], posn);
            }
            run += tot;
        }
        grid.sync();
        if (threadIdx.x == 0) red[0] = *(volatile uint32_t*)&st->fail[par];  // one read per CTA
        __syncthreads();
        const uint32_t ff = red[0];
        if (ff != kNone && A.mode != DFAKIT_MODE_FULL) {
            if (we + ff >= A.max_visited) {
                status = kBfsBudget;
            } else {
                status = kBfsFail;
                if (gtid == 0) st->fail_rec = (uint32_t)(we + ff);
            }
            we = we + ff + 1;  // explored count reported on failure
            break;
        }
        if (we + total > A.max_visited) {
            status = kBfsBudget;
            break;
        }
        if (ff != kNone && first_fail_all == ~0ull) first_fail_all = we + ff;
        ++levels;
        wb = we;
        we += total;
    }
    if (gtid == 0) {
        st->wb = wb;
        st->we = we;
        st->levels = levels;
        st->status = status;
        st->first_fail_all = first_fail_all;
    }
}

// union-find Hopcroft-Karp: one barrier per level
struct UfArgs {
    Rec rec;
    uint64_t cap;
    const uint32_t *da, *db;
    uint32_t na, nb, k;
    const uint8_t *acc_a, *acc_b;
    uint32_t* P;
    uint32_t* count;
    uint32_t* fail_rec;
    uint32_t* out;  // {levels, explored}
};

__global__ void __launch_bounds__(kThreads) uf_persistent_kernel(UfArgs A) {
    __shared__ uint32_t s_bc[2];
    cg::grid_group grid = cg::this_grid();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t wb = 0, we = 1;
    uint32_t levels = 0;
    while (wb < we) {
        const uint64_t items = (we - wb) * A.k;
        for (uint64_t t = gtid; t < items; t += stride) {
            const uint64_t i = wb + t / A.k;
            const uint32_t la = (uint32_t)(t % A.k);
            const unsigned long long pk = __ldcg(A.rec.key + i);
            const uint32_t pa = A.da[(uint64_t)la * A.na + (uint32_t)(pk >> 32)];
            const uint32_t pb = A.db[(uint64_t)la * A.nb + (uint32_t)pk];
            if (!uf_union(A.P, pa, A.na + pb)) continue;
            const uint32_t r = atomicAdd(A.count, 1u);
            if (r >= A.cap) continue;  // cannot happen: at most na+nb-1 unions
            A.rec.key[r] = ((unsigned long long)pa << 32) | pb;
            A.rec.parent[r] = (uint32_t)i;
            A.rec.letter[r] = la;
            if (A.acc_a[pa] != A.acc_b[pb]) atomicMin(A.fail_rec, r);
        }
        grid.sync();
        ++levels;
        if (threadIdx.x == 0) {  // one read per CTA
            s_bc[0] = *(volatile uint32_t*)A.fail_rec;
            s_bc[1] = *(volatile uint32_t*)A.count;
        }
        __syncthreads();
        if (s_bc[0] != kNone) break;
        wb = we;
        we = s_bc[1];
        grid.sync();  // every CTA has read count before the next level appends
    }
    if (gtid == 0) {
        A.out[0] = levels;
        A.out[1] = *(volatile uint32_t*)A.count;
    }
}

struct RecStore {
    DBuf<unsigned long long> key;
    DBuf<uint32_t> parent, letter;
    uint64_t cap = 0;
    void ensure(uint64_t need, uint64_t used, cudaStream_t s) {
        if (need <= cap) return;
        uint64_t nc = cap ? cap : 1024;
        while (nc < need) nc *= 2;
        DBuf<unsigned long long> k2(nc, s);
        DBuf<uint32_t> p2(nc, s), l2(nc, s);
        if (used) {
            DK_CUDA(cudaMemcpyAsync(k2.get(), key.get(), used * 8, cudaMemcpyDeviceToDevice, s));
            DK_CUDA(cudaMemcpyAsync(p2.get(), parent.get(), used * 4, cudaMemcpyDeviceToDevice, s));
            DK_CUDA(cudaMemcpyAsync(l2.get(), letter.get(), used * 4, cudaMemcpyDeviceToDevice, s));
        }
        key = std::move(k2);
        parent = std::move(p2);
        letter = std::move(l2);
        cap = nc;
    }
    Rec view() { return Rec{key.get(), parent.get(), letter.get()}; }
};

std::basic_string<uint32_t> walk_word(Ctx* ctx, RecStore& rs, uint32_t idx, cudaStream_t s) {
    DBuf<uint32_t> len(1, s);
    // words are at most (#levels + 1) long; size the buffer generously
    uint32_t cap = 1u << 16;
    for (;;) {
        DBuf<uint32_t> word(cap, s);
        DK_LAUNCH(ctx, walk_word_kernel, 1, 1, 0, s, rs.view(), idx, word.get(), cap, len.get());
        uint32_t l = 0;
        read_words(ctx, len.get(), 4, &l, s);
        if (l <= cap) {
            std::basic_string<uint32_t> w(l, 0u);
            if (l) {
                DK_CUDA(cudaMemcpyAsync(&w[0], word.get(), (size_t)l * 4, cudaMemcpyDeviceToHost, s));
                DK_CUDA(cudaStreamSynchronize(s));
            }
            return w;
        }
        cap = l;
    }
}

uint64_t next_pow2(uint64_t x) {
    uint64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

}  // namespace

ProductOut explore_product_device(Ctx* ctx, const DevDfa& a, const DevDfa& b, int mode, const uint32_t* letter_map,
                                  uint64_t max_visited, cudaStream_t s) {
    if (a.initial < 0 || b.initial < 0)
        throw Error(DFAKIT_E_INVALID, "product exploration requires initial states on both inputs");
    const uint32_t k = a.k;
    if (max_visited > 0xfffffffeull) max_visited = 0xfffffffeull;  // record indices are 32-bit
    ProductOut out;
    if (max_visited == 0) throw Error(DFAKIT_E_RESOURCE, "product exploration exceeded the visited-set budget of 0 pairs");
    // the initial pair's check runs on the device (bfs_init_kernel) ahead of
    // the exploration: no host round trip before the first launch
    uint64_t first_fail_all = ~0ull;

    DBuf<uint32_t> to_b(k ? k : 1, s);
    {
        std::vector<uint32_t> m(k);
        for (uint32_t i = 0; i < k; ++i) m[i] = letter_map ? letter_map[i] : i;
        // (pageable source: the copy is staged before the call returns)
        if (k) DK_CUDA(cudaMemcpyAsync(to_b.get(), m.data(), k * 4ull, cudaMemcpyHostToDevice, s));
    }
    RecStore rs;
    rs.ensure(1024, 0, s);
    const unsigned long long k0 = ((unsigned long long)(uint32_t)a.initial << 32) | (uint32_t)b.initial;
    const uint32_t zero = 0;
    DK_CUDA(cudaMemcpyAsync(rs.key.get(), &k0, 8, cudaMemcpyHostToDevice, s));
    DK_CUDA(cudaMemcpyAsync(rs.parent.get(), &zero, 4, cudaMemcpyHostToDevice, s));
    DK_CUDA(cudaMemcpyAsync(rs.letter.get(), &zero, 4, cudaMemcpyHostToDevice, s));

    DBuf<Slot> table;
    uint64_t cap = 0;
    DBuf<uint32_t> item_slot;
    DBuf<BfsState> dst(1, s);
    int per_sm = 0;
    DK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bfs_persistent_kernel, kThreads, 0));
    if (per_sm < 1) throw Error(DFAKIT_E_RESOURCE, "bfs kernel does not fit an SM");
    const unsigned grid_n = (unsigned)(per_sm * ctx->num_sms);
    DBuf<uint32_t> cta_cnt((grid_n + 3) / 4 * 4, s);  // padded for 16-byte reads
    DK_CUDA(cudaMemsetAsync(cta_cnt.get(), 0, cta_cnt.n * sizeof(uint32_t), s));
    BfsState hs{};
    hs.wb = 0;
    hs.we = 1;
    hs.first_fail_all = first_fail_all;
    hs.status = kBfsRunning;
    hs.fail[0] = hs.fail[1] = hs.fail[2] = kNone;
    DK_CUDA(cudaMemcpyAsync(dst.get(), &hs, sizeof(hs), cudaMemcpyHostToDevice, s));
    DK_LAUNCH(ctx, bfs_init_kernel, 1, 1, 0, s, a.acc, b.acc, (uint32_t)a.initial, (uint32_t)b.initial, mode,
              dst.get());
    uint64_t wb = 0, we = 1;
    DBuf<uint8_t> item_win;
    DBuf<unsigned long long> item_key;
    // first table: 2^20 slots at least.  DFAKIT_TEST_TABLE_LOG2=<b> (tests
    // only) starts at 2^b slots sized for nothing, so small explorations run
    // at load up to 1/2 -- home-slot collisions, the tile-cooperative
    // windows, growth and re-insertion all happen
    uint64_t min_slots = 1ull << 20;
    bool tiny = false;
    if (const char* t = getenv("DFAKIT_TEST_TABLE_LOG2")) {
        min_slots = 1ull << std::min(30, std::max(4, atoi(t)));
        tiny = true;
    }
    // primary mode (first automaton below 2^31 states; DFAKIT_BFS_NO_PRIMARY=1
    // turns it off): pair (pa, pb) is kept in slot pa of a direct-mapped
    // table -- pb and the discoverer, 16 B per state of A, nearer the L2's size
    // rather than 16-byte slots for max(nA, nB) pairs at load 1/2 -- unless
    // another pb already holds slot pa; only those pairs go to the hash
    // table, which then starts small and grows (x4) when its reservations
    // run out, re-running the level that ran out
    const bool prim = a.n < 0x80000000u && !getenv("DFAKIT_BFS_NO_PRIMARY");
    DBuf<PrimSlot> prim_tab;
    if (prim) {
        prim_tab.alloc(std::max<uint64_t>(1, a.n), s);
        DK_CUDA(cudaMemsetAsync(prim_tab.get(), 0xff, (size_t)a.n * sizeof(PrimSlot), s));
    }
    const uint64_t pairs_guess = tiny ? 0 : std::min<uint64_t>(max_visited, std::max(a.n, b.n)) + 64;
    for (;;) {
        // room for the next level: table at load <= 1/2; the record store and
        // the item buffers are sized with the table (cap / 2 each), so the
        // kernel comes back only when the table must grow (4x from 2^20)
        const uint64_t items = (we - wb) * k;
        const uint64_t need = prim ? (hs.need_grow ? cap * 4 : (cap ? cap : min_slots))
                                   : next_pow2(2 * (we + items) + 64);
        if (need > cap) {
            // first allocation sized for max(nA, nB) pairs at load 1/2 (the
            // usual size of an equivalence product; bounded by the visited
            // budget), so most explorations run in one launch without
            // re-insertion, and the table initialisation stays small
            const uint64_t guess = tiny || prim ? 0 : next_pow2(2 * pairs_guess);
            const uint64_t nc = cap ? std::max<uint64_t>(need, cap * 4)
                                    : std::max<uint64_t>(need, std::max<uint64_t>(min_slots, guess));
            table.alloc(nc, s);
            cap = nc;
            DK_CUDA(cudaMemsetAsync(table.get(), 0xff, cap * sizeof(Slot), s));
            if (prim) {  // reservations restart from the records actually in the hash table
                DK_CUDA(cudaMemsetAsync(&dst.get()->hkeys, 0, sizeof(unsigned long long), s));
                DK_CUDA(cudaMemsetAsync(&dst.get()->need_grow, 0, sizeof(uint32_t), s));
                hs.need_grow = 0;
            }
            DK_LAUNCH(ctx, reinsert_kernel, grid_for(we), kThreads, 0, s, rs.key.get(), we, table.get(), cap - 1,
                      prim ? prim_tab.get() : nullptr, prim ? &dst.get()->hkeys : nullptr);
        }
        const uint64_t base_cap = prim ? pairs_guess : cap / 2;
        rs.ensure(std::max<uint64_t>(base_cap, we + items), we, s);
        const uint64_t icap = std::max<uint64_t>(base_cap, items);
        if (icap > item_slot.n) {
            item_slot.alloc(icap, s);
            item_win.alloc(icap, s);
            item_key.alloc(icap, s);
        }
        BfsArgs A{rs.view(), rs.cap, table.get(), cap, item_slot.get(), item_win.get(), item_key.get(), item_slot.n,
                  cta_cnt.get(), a.delta, b.delta,
                  to_b.get(), a.n, b.n, k, a.acc, b.acc, mode, max_visited, dst.get(),
                  prim ? prim_tab.get() : nullptr};
        void* args[] = {(void*)&A};
        prof_begin_launch(ctx, s);
        DK_CUDA(cudaLaunchCooperativeKernel((const void*)bfs_persistent_kernel, grid_n, kThreads, args, 0, s));
        note_launch(ctx);
        prof_end_launch(ctx, s, "bfs_persistent_kernel", 0, 0);
        read_words(ctx, dst.get(), sizeof(hs), &hs, s);
        wb = hs.wb;
        we = hs.we;
        out.levels = hs.levels;
        first_fail_all = hs.first_fail_all;
        if (hs.status == kBfsFail) {
            out.verdict = DFAKIT_COUNTEREXAMPLE;
            out.explored = we;
            out.word = walk_word(ctx, rs, hs.fail_rec, s);
            return out;
        }
        if (hs.status == kBfsBudget)
            throw Error(DFAKIT_E_RESOURCE, "product exploration exceeded the visited-set budget of " +
                                               std::to_string(max_visited) + " pairs");
        if (hs.status == kBfsDone) break;
        // kBfsGrow: loop to grow and relaunch
        hs.status = kBfsRunning;
    }
    out.explored = we;
    if (mode == DFAKIT_MODE_FULL && first_fail_all != ~0ull) {
        out.verdict = DFAKIT_COUNTEREXAMPLE;
        out.word = walk_word(ctx, rs, (uint32_t)first_fail_all, s);
    } else {
        out.verdict = mode == DFAKIT_MODE_INCLUSION ? DFAKIT_INCLUDED : DFAKIT_EQUIVALENT;
    }
    return out;
}

ProductOut check_equiv_uf_device(Ctx* ctx, const DevDfa& a, const DevDfa& b, cudaStream_t s) {
    if (a.initial < 0 || b.initial < 0)
        throw Error(DFAKIT_E_INVALID, "equivalence checking requires initial states on both inputs");
    if (a.k != b.k) throw Error(DFAKIT_E_INVALID, "alphabet size mismatch");
    const uint32_t k = a.k;
    ProductOut out;
    uint8_t acc0[2];
    DK_CUDA(cudaMemcpyAsync(&acc0[0], a.acc + a.initial, 1, cudaMemcpyDeviceToHost, s));
    DK_CUDA(cudaMemcpyAsync(&acc0[1], b.acc + b.initial, 1, cudaMemcpyDeviceToHost, s));
    DK_CUDA(cudaStreamSynchronize(s));
    if (acc0[0] != acc0[1]) {
        out.verdict = DFAKIT_COUNTEREXAMPLE;
        out.explored = 1;
        return out;
    }
    const uint64_t total = (uint64_t)a.n + b.n;
    if (total >= 0xffffffffull) throw Error(DFAKIT_E_RESOURCE, "union-find: too many states");
    DBuf<uint32_t> P(total, s), cnt(1, s), fail(1, s);
    DK_LAUNCH(ctx, uf_init_kernel, grid_for(total), kThreads, 0, s, P.get(), total);
    DK_LAUNCH(ctx, uf_seed_kernel, 1, 1, 0, s, P.get(), (uint32_t)a.initial, a.n + (uint32_t)b.initial);
    RecStore rs;
    rs.ensure(total + 1, 0, s);  // at most total-1 unions + the seed record
    const unsigned long long k0 = ((unsigned long long)(uint32_t)a.initial << 32) | (uint32_t)b.initial;
    const uint32_t zero = 0, one = 1;
    DK_CUDA(cudaMemcpyAsync(rs.key.get(), &k0, 8, cudaMemcpyHostToDevice, s));
    DK_CUDA(cudaMemcpyAsync(rs.parent.get(), &zero, 4, cudaMemcpyHostToDevice, s));
    DK_CUDA(cudaMemcpyAsync(rs.letter.get(), &zero, 4, cudaMemcpyHostToDevice, s));
    DK_CUDA(cudaMemcpyAsync(cnt.get(), &one, 4, cudaMemcpyHostToDevice, s));
    DK_CUDA(cudaMemsetAsync(fail.get(), 0xff, 4, s));
    DBuf<uint32_t> res(2, s);
    int per_sm = 0;
    DK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, uf_persistent_kernel, kThreads, 0));
    if (per_sm < 1) throw Error(DFAKIT_E_RESOURCE, "union-find kernel does not fit an SM");
    UfArgs A{rs.view(), rs.cap, a.delta, b.delta, a.n, b.n, k, a.acc, b.acc, P.get(), cnt.get(), fail.get(),
             res.get()};
    void* args[] = {(void*)&A};
    prof_begin_launch(ctx, s);
    DK_CUDA(cudaLaunchCooperativeKernel((const void*)uf_persistent_kernel, (unsigned)(per_sm * ctx->num_sms), kThreads,
                                        args, 0, s));
    note_launch(ctx);
    prof_end_launch(ctx, s, "uf_persistent_kernel", 0, 0);
    uint32_t words[3] = {0, 0, 0};
    read_words(ctx, res.get(), 8, words, s);
    read_words(ctx, fail.get(), 4, &words[2], s);
    out.levels = words[0];
    const uint64_t we = words[1];
    if (words[2] != kNone) {
        out.verdict = DFAKIT_COUNTEREXAMPLE;
        out.explored = we;
        out.word = walk_word(ctx, rs, words[2], s);
        return out;
    }
    out.verdict = DFAKIT_EQUIVALENT;
    out.explored = we;
    return out;
}

}  // namespace dk
