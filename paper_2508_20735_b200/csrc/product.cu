// product.cu -- Hopcroft-Karp equivalence / inclusion checking (paper Alg. 6,
// reference src/equivalence.cpp:138-215) on B200.
//
// explore_product: level-synchronous BFS over the synchronous product with
// a lock-free open-addressing hash set of packed (qA, qB) pairs.  Each
// 16-byte slot holds the key and a "discoverer" word (parent record << 32 |
// letter); probing is tile-cooperative: 4 lanes inspect a 4-slot (64 B)
// window per step with ballots for match / empty, and the leader claims an
// empty slot with a 64-bit CAS.  Within a wave every (frontier record,
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

struct Rec {
    unsigned long long* key;
    uint32_t* parent;
    uint32_t* letter;
};

__device__ __forceinline__ uint64_t slot_hash(uint64_t key) { return mix64(key ^ 0x243F6A8885A308D3ull); }

// Tile-cooperative find-or-insert of every lane's key.  Returns the slot of
// this lane's key (kNone when !valid).
__device__ uint32_t tile_find_or_insert(cg::thread_block_tile<kTile> tile, bool valid, unsigned long long key,
                                        Slot* __restrict__ table, uint64_t mask) {
    uint32_t mine = kNone;
    const unsigned lane = tile.thread_rank();
    for (int j = 0; j < kTile; ++j) {
        const unsigned long long kj = tile.shfl(key, j);
        const bool vj = tile.shfl(valid, j);
        if (!vj) continue;
        uint64_t base = slot_hash(kj) & mask & ~(uint64_t)(kTile - 1);
        uint32_t found = kNone;
        for (;;) {
            const unsigned long long e = __ldcg(&table[base + lane].key);
            const unsigned match = tile.ballot(e == kj);
            if (match) {
                found = (uint32_t)(base + __ffs(match) - 1);
                break;
            }
            const unsigned empty = tile.ballot(e == kEmpty);
            if (empty) {
                const unsigned leader = __ffs(empty) - 1;
                unsigned long long old = 0;
                if (lane == leader) old = atomicCAS(&table[base + leader].key, kEmpty, kj);
                old = tile.shfl(old, leader);
                if (old == kEmpty || old == kj) {
                    found = (uint32_t)(base + leader);
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

// one item per (frontier record, letter)
__global__ void __launch_bounds__(kThreads) expand_kernel(Rec rec, uint64_t wb, uint64_t items, uint32_t k,
                                                          const uint32_t* __restrict__ da, uint32_t na,
                                                          const uint32_t* __restrict__ db, uint32_t nb,
                                                          const uint32_t* __restrict__ to_b, Slot* __restrict__ table,
                                                          uint64_t mask, uint32_t* __restrict__ item_slot) {
    auto tile = cg::tiled_partition<kTile>(cg::this_thread_block());
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t first = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    // uniform trip count so tiles stay converged
    const uint64_t trips = (items + stride - 1) / stride;
    for (uint64_t it = 0; it < trips; ++it) {
        const uint64_t t = first + it * stride;
        const bool valid = t < items;
        unsigned long long key = 0, disc = 0;
        if (valid) {
            const uint64_t i = wb + t / k;
            const uint32_t la = (uint32_t)(t % k);
            const unsigned long long pk = rec.key[i];
            const uint32_t qa = (uint32_t)(pk >> 32), qb = (uint32_t)pk;
            const uint32_t pa = da[(uint64_t)la * na + qa];
            const uint32_t pb = db[(uint64_t)to_b[la] * nb + qb];
            key = ((unsigned long long)pa << 32) | pb;
            disc = ((unsigned long long)(i + 1) << 32) | la;  // +1: reinserted slots hold 0
        }
        const uint32_t s = tile_find_or_insert(tile, valid, key, table, mask);
        if (valid) {
            const unsigned long long old = atomicMin(&table[s].disc, disc);
            // slots discovered in earlier waves carry a parent below wb (stored +1)
            item_slot[t] = (old >= ((unsigned long long)(wb + 1) << 32)) ? s : kNone;
        }
    }
}

__global__ void winner_flags_kernel(uint64_t wb, uint64_t items, uint32_t k, const Slot* __restrict__ table,
                                    const uint32_t* __restrict__ item_slot, uint32_t* __restrict__ flag) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < items;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = item_slot[t];
        uint32_t f = 0;
        if (s != kNone) {
            const unsigned long long disc = ((unsigned long long)(wb + t / k + 1) << 32) | (uint32_t)(t % k);
            f = __ldcg(&table[s].disc) == disc;
        }
        flag[t] = f;
    }
}

__global__ void emit_kernel(Rec rec, uint64_t wb, uint64_t we, uint64_t items, uint32_t k,
                            const Slot* __restrict__ table, const uint32_t* __restrict__ item_slot,
                            const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                            const uint8_t* __restrict__ acc_a, const uint8_t* __restrict__ acc_b, int mode,
                            uint32_t* __restrict__ first_fail) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < items;
         t += (uint64_t)gridDim.x * blockDim.x) {
        if (!flag[t]) continue;
        const unsigned long long key = table[item_slot[t]].key;
        const uint64_t r = we + pos[t];
        rec.key[r] = key;
        rec.parent[r] = (uint32_t)(wb + t / k);
        rec.letter[r] = (uint32_t)(t % k);
        const bool fa = acc_a[key >> 32], fb = acc_b[(uint32_t)key];
        const bool fails = mode == DFAKIT_MODE_INCLUSION ? (fa && !fb) : (fa != fb);
        if (fails) atomicMin(first_fail, pos[t]);
    }
}

__global__ void reinsert_kernel(const unsigned long long* __restrict__ keys, uint64_t count, Slot* __restrict__ table,
                                uint64_t mask) {
    auto tile = cg::tiled_partition<kTile>(cg::this_thread_block());
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t first = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t trips = (count + stride - 1) / stride;
    for (uint64_t it = 0; it < trips; ++it) {
        const uint64_t t = first + it * stride;
        const bool valid = t < count;
        const unsigned long long key = valid ? keys[t] : 0ull;
        const uint32_t s = tile_find_or_insert(tile, valid, key, table, mask);
        if (valid) table[s].disc = 0ull;  // discovered before any current wave
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

__global__ void __launch_bounds__(kThreads) uf_expand_kernel(Rec rec, uint64_t wb, uint64_t items, uint32_t k,
                                                             const uint32_t* __restrict__ da, uint32_t na,
                                                             const uint32_t* __restrict__ db, uint32_t nb,
                                                             const uint8_t* __restrict__ acc_a,
                                                             const uint8_t* __restrict__ acc_b, uint32_t* __restrict__ P,
                                                             uint32_t* __restrict__ count, uint64_t cap,
                                                             uint32_t* __restrict__ fail_rec) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < items;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = wb + t / k;
        const uint32_t la = (uint32_t)(t % k);
        const unsigned long long pk = rec.key[i];
        const uint32_t pa = da[(uint64_t)la * na + (uint32_t)(pk >> 32)];
        const uint32_t pb = db[(uint64_t)la * nb + (uint32_t)pk];
        if (!uf_union(P, pa, na + pb)) continue;
        const uint32_t r = atomicAdd(count, 1u);
        if (r >= cap) continue;  // cannot happen: at most na+nb-1 unions
        rec.key[r] = ((unsigned long long)pa << 32) | pb;
        rec.parent[r] = (uint32_t)i;
        rec.letter[r] = la;
        if (acc_a[pa] != acc_b[pb]) atomicMin(fail_rec, r);
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
    std::vector<uint8_t> acc0(2);
    DK_CUDA(cudaMemcpyAsync(&acc0[0], a.acc + a.initial, 1, cudaMemcpyDeviceToHost, s));
    DK_CUDA(cudaMemcpyAsync(&acc0[1], b.acc + b.initial, 1, cudaMemcpyDeviceToHost, s));
    DK_CUDA(cudaStreamSynchronize(s));
    if (max_visited == 0) throw Error(DFAKIT_E_RESOURCE, "product exploration exceeded the visited-set budget of 0 pairs");
    const bool fa = acc0[0], fb = acc0[1];
    const bool init_fails = mode == DFAKIT_MODE_INCLUSION ? (fa && !fb) : (fa != fb);
    if (init_fails && mode != DFAKIT_MODE_FULL) {
        out.verdict = DFAKIT_COUNTEREXAMPLE;
        out.explored = 1;
        return out;
    }
    uint64_t first_fail_all = init_fails ? 0 : ~0ull;

    DBuf<uint32_t> to_b(k ? k : 1, s);
    {
        std::vector<uint32_t> m(k);
        for (uint32_t i = 0; i < k; ++i) m[i] = letter_map ? letter_map[i] : i;
        if (k) DK_CUDA(cudaMemcpyAsync(to_b.get(), m.data(), k * 4ull, cudaMemcpyHostToDevice, s));
        DK_CUDA(cudaStreamSynchronize(s));
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
    DBuf<uint32_t> item_slot, flag, pos, ff(1, s), total(1, s);
    uint64_t wb = 0, we = 1;
    while (wb < we) {
        const uint64_t wave = we - wb;
        const uint64_t items = wave * k;
        // capacity for everything seen so far plus every possible new pair, at load <= 1/2
        const uint64_t need = next_pow2(2 * (we + items) + 64);
        if (need > cap) {
            table.alloc(need, s);
            cap = need;
            DK_CUDA(cudaMemsetAsync(table.get(), 0xff, need * sizeof(Slot), s));
            DK_LAUNCH(ctx, reinsert_kernel, grid_for(we), kThreads, 0, s, rs.key.get(), we, table.get(), cap - 1);
        }
        rs.ensure(we + items, we, s);
        if (items > item_slot.n) {
            item_slot.alloc(items, s);
            flag.alloc(items, s);
            pos.alloc(items, s);
        }
        if (items) {
            DK_LAUNCH_B(ctx, 44.0 * items, expand_kernel, grid_for(items), kThreads, 0, s, rs.view(), wb, items, k, a.delta, a.n,
                      b.delta, b.n, to_b.get(), table.get(), cap - 1, item_slot.get());
            DK_LAUNCH(ctx, winner_flags_kernel, grid_for(items), kThreads, 0, s, wb, items, k, table.get(),
                      item_slot.get(), flag.get());
            exclusive_scan_u32(ctx, flag.get(), pos.get(), items, total.get(), s);
            DK_CUDA(cudaMemsetAsync(ff.get(), 0xff, 4, s));
            DK_LAUNCH(ctx, emit_kernel, grid_for(items), kThreads, 0, s, rs.view(), wb, we, items, k, table.get(),
                      item_slot.get(), flag.get(), pos.get(), a.acc, b.acc, mode, ff.get());
        }
        uint32_t fresh = 0, first = kNone;
        if (items) {
            read_words(ctx, total.get(), 4, &fresh, s);
            read_words(ctx, ff.get(), 4, &first, s);
        }
        if (first != kNone && mode != DFAKIT_MODE_FULL) {
            if (we + first >= max_visited)
                throw Error(DFAKIT_E_RESOURCE, "product exploration exceeded the visited-set budget of " +
                                                   std::to_string(max_visited) + " pairs");
            out.verdict = DFAKIT_COUNTEREXAMPLE;
            out.explored = we + first + 1;
            out.word = walk_word(ctx, rs, (uint32_t)(we + first), s);
            return out;
        }
        if (we + fresh > max_visited)
            throw Error(DFAKIT_E_RESOURCE, "product exploration exceeded the visited-set budget of " +
                                               std::to_string(max_visited) + " pairs");
        if (first != kNone && first_fail_all == ~0ull) first_fail_all = we + first;
        ++out.levels;
        wb = we;
        we += fresh;
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
    uint64_t wb = 0, we = 1;
    while (wb < we) {
        const uint64_t items = (we - wb) * k;
        if (items)
            DK_LAUNCH(ctx, uf_expand_kernel, grid_for(items), kThreads, 0, s, rs.view(), wb, items, k, a.delta, a.n,
                      b.delta, b.n, a.acc, b.acc, P.get(), cnt.get(), rs.cap, fail.get());
        uint32_t words[2] = {0, 0};
        read_words(ctx, cnt.get(), 4, &words[0], s);
        read_words(ctx, fail.get(), 4, &words[1], s);
        ++out.levels;
        if (words[1] != kNone) {
            out.verdict = DFAKIT_COUNTEREXAMPLE;
            out.explored = words[0];
            out.word = walk_word(ctx, rs, words[1], s);
            return out;
        }
        wb = we;
        we = words[0];
    }
    out.verdict = DFAKIT_EQUIVALENT;
    out.explored = we;
    return out;
}

}  // namespace dk
