// refine_sort.cu -- sortPR (reference src/minimize.cpp:354-419, paper Alg. 4)
// re-designed for B200.
//
// Block labels are min-state ids (every block is named by its smallest
// member), so the canonical first-occurrence numbering of the reference's
// Partition::from_labels is one flag+scan away at any time, and a block's
// label never changes unless the block splits.
//
// Per pass, only states in non-singleton blocks ("active" states) take part:
//   1. signature kernel: gathers block[delta(q,a)] for every letter and
//      packs (block[q], sig[q][0..k-1]) into a 64-bit key -- exactly when the
//      fields fit, otherwise as a 64-bit fingerprint whose equal-key runs are
//      verified tuple-by-tuple afterwards (exactness never rests on the hash);
//   2. the keys are grouped either by direct addressing (keys of <= 20 bits:
//      a counting table, no sort) or by the LSD radix sort in prims.cu;
//   3. boundary flags (the reference's ARE_NEQ adjacent difference) and an
//      exclusive scan number the runs; every run's first element is its
//      minimum state (the sort is stable and the input order is increasing
//      within each block), which becomes the new block label;
//   4. counters give the new block count: the fixed-point test of l.19.
// Singleton runs leave the active list for good.
#include <vector>

#include "prims.cuh"
#include "refine.cuh"

namespace dk {

namespace {

constexpr uint32_t kTableBits = 20;

struct IterCounters {
    uint32_t runs;
    uint32_t active_blocks;
    uint32_t active_states;
    uint32_t collision;
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

// One thread per active state; delta rows are read with streaming loads
// (coalesced when the active list is the identity), block labels are
// gathered (the label array stays L2-resident for n <= ~25M).
__global__ void __launch_bounds__(kThreads) signature_kernel(const uint32_t* __restrict__ list, uint64_t m,
                                                             const uint32_t* __restrict__ delta, uint32_t n,
                                                             const uint32_t* __restrict__ lab,
                                                             const uint32_t* __restrict__ head, SigParams p,
                                                             uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t q = list ? list[i] : (uint32_t)i;
        uint64_t key;
        if (p.kind == kKeyPacked) {
            key = head ? head[i] : lab[q];
            for (uint32_t a = p.a0; a < p.a1; ++a) {
                uint32_t t = ld_stream(delta + (uint64_t)a * n + q);
                key = (key << p.field_bits) | lab[t];
            }
        } else {
            uint64_t h = fp_step(p.salt, lab[q]);
            for (uint32_t a = p.a0; a < p.a1; ++a) {
                uint32_t t = ld_stream(delta + (uint64_t)a * n + q);
                h = fp_step(h + a, lab[t]);
            }
            key = h & p.fp_mask;
        }
        keys[i] = key;
        vals[i] = q;
    }
}

// direct-address grouping for small packed keys
__global__ void table_insert_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, uint64_t m,
                                    uint32_t* __restrict__ tmin, uint32_t* __restrict__ tcnt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t key = (uint32_t)keys[i];
        atomicMin(&tmin[key], vals[i]);
        atomicAdd(&tcnt[key], 1u);
    }
}

__global__ void table_apply_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, uint64_t m,
                                   const uint32_t* __restrict__ tmin, const uint32_t* __restrict__ tcnt,
                                   uint32_t* __restrict__ lab, uint8_t* __restrict__ keep,
                                   IterCounters* __restrict__ ctr) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t key = (uint32_t)keys[i];
        const uint32_t q = vals[i];
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

__global__ void run_heads_kernel(const uint64_t* __restrict__ keys, uint64_t m, uint32_t* __restrict__ heads) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        heads[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}

// Exactness check of fingerprint runs: neighbours with equal keys must have
// identical (block, signature) tuples.
__global__ void verify_runs_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, uint64_t m,
                                   const uint32_t* __restrict__ delta, uint32_t n, uint32_t a0, uint32_t a1,
                                   const uint32_t* __restrict__ lab, IterCounters* __restrict__ ctr) {
    for (uint64_t i = 1 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (keys[i] != keys[i - 1]) continue;
        const uint32_t q = vals[i], r = vals[i - 1];
        bool same = lab[q] == lab[r];
        for (uint32_t a = a0; a < a1 && same; ++a) {
            const uint32_t* row = delta + (uint64_t)a * n;
            same = lab[row[q]] == lab[row[r]];
        }
        if (!same) atomicOr(&ctr->collision, 1u);
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
    DBuf<uint32_t> lab, list0, list1, vals0, vals1, heads, pos, run_start, scratch, dense, cur, tmin, tcnt;
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
        iota_u32(ctx, list_alt, n, s);
        m = compact_u32(ctx, list_alt, f.get(), n, list_buf, w.scratch.get(), s);
        list = list_buf;
    }

    const uint32_t label_bits = bits_for(n - 1);
    uint64_t salt = 0x5eed5eed5eedull;
    const uint64_t fp_mask = o.fingerprint_bits >= 64 ? ~0ull : ((1ull << o.fingerprint_bits) - 1ull);

    while (m > 0) {
        ++res.passes;
        const uint32_t dense_bits = bits_for(B ? B - 1 : 0);
        bool need_dense = false;
        bool fingerprint = false;
        bool chunked = false;
        uint32_t field_bits = 0;
        if ((uint64_t)(k + 1) * label_bits <= 64) {
            field_bits = label_bits;
        } else if ((uint64_t)(k + 1) * dense_bits <= 64) {
            field_bits = dense_bits;
            need_dense = true;
        } else if (!o.force_exact) {
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
        bool done_table = false;

        if (!chunked) {
            SigParams p{};
            p.kind = fingerprint ? kKeyFingerprint : kKeyPacked;
            p.a0 = 0;
            p.a1 = k;
            p.field_bits = field_bits;
            p.salt = salt;
            p.fp_mask = fp_mask;
            DK_LAUNCH_B(ctx, (double)m * (16.0 + 8.0 * k + (list ? 4.0 : 0.0)), signature_kernel, g, kThreads, 0, s, list, m, d.delta, n, keylab, nullptr, p, w.keys0.get(),
                      w.vals0.get());
            const uint32_t nbits = fingerprint ? 64u : (k + 1) * field_bits;
            if (!fingerprint && nbits <= kTableBits) {
                const uint64_t tsize = 1ull << nbits;
                if (w.tmin.n < tsize) {
                    w.tmin.alloc(tsize, s);
                    w.tcnt.alloc(tsize, s);
                }
                DK_CUDA(cudaMemsetAsync(w.tmin.get(), 0xff, tsize * sizeof(uint32_t), s));
                DK_CUDA(cudaMemsetAsync(w.tcnt.get(), 0, tsize * sizeof(uint32_t), s));
                DK_LAUNCH_B(ctx, 20.0 * m, table_insert_kernel, g, kThreads, 0, s, w.keys0.get(), w.vals0.get(), m, w.tmin.get(),
                          w.tcnt.get());
                DK_LAUNCH_B(ctx, 25.0 * m, table_apply_kernel, g, kThreads, 0, s, w.keys0.get(), w.vals0.get(), m, w.tmin.get(),
                          w.tcnt.get(), w.lab.get(), w.keep.get(), w.ctr.get());
                read_words(ctx, w.ctr.get(), sizeof(c), &c, s);
                done_table = true;
            } else {
                bool flip = radix_sort_pairs(ctx, rb, m, nbits, s);
                res.sorted += m;
                if (flip) {
                    skeys = w.keys1.get();
                    svals = w.vals1.get();
                }
                if (fingerprint) {
                    DK_LAUNCH(ctx, verify_runs_kernel, g, kThreads, 0, s, skeys, svals, m, d.delta, n, 0u, k,
                              w.lab.get(), w.ctr.get());
                    read_words(ctx, w.ctr.get(), sizeof(c), &c, s);
                    if (c.collision) {
                        // a genuine fingerprint collision: re-run this pass with
                        // a fresh salt, then exactly once retries run out
                        ++res.collisions;
                        --res.passes;
                        salt = mix64(salt + 0x1234567ull);
                        if (res.collisions % 3 == 0) {
                            // fall through to the chunked exact path for this pass
                            chunked = true;
                            need_dense = true;
                            field_bits = dense_bits;
                            if (!w.dense.get()) w.dense.alloc(n, s);
                            canonical_from_min_labels(ctx, w.lab.get(), n, w.dense.get(), w.scratch.get(), s);
                            keylab = w.dense.get();
                            ++res.passes;
                            DK_CUDA(cudaMemsetAsync(w.ctr.get(), 0, sizeof(IterCounters), s));
                        } else {
                            continue;
                        }
                    }
                }
            }
        }

        if (chunked) {
            // exact refinement letter-chunk by letter-chunk; the run index of
            // the previous chunk leads the next key
            if (!w.cur.get()) w.cur.alloc(n, s);
            DK_LAUNCH(ctx, gather_dense_kernel, g, kThreads, 0, s, list, m, keylab, w.cur.get());
            uint32_t cur_bits = field_bits;
            const uint32_t* elist = list;
            uint32_t a = 0;
            bool first = true;
            for (;;) {
                uint32_t c_letters = field_bits ? (64u - cur_bits) / field_bits : k;
                if (c_letters < 1) c_letters = 1;
                if (c_letters > k - a) c_letters = k - a;
                SigParams p{};
                p.kind = kKeyPacked;
                p.a0 = a;
                p.a1 = a + c_letters;
                p.field_bits = field_bits;
                DK_LAUNCH_B(ctx, (double)m * (24.0 + 8.0 * (p.a1 - p.a0)), signature_kernel, g, kThreads, 0, s, elist, m, d.delta, n, keylab, w.cur.get(), p,
                          w.keys0.get(), w.vals0.get());
                const uint32_t nbits = cur_bits + c_letters * field_bits;
                bool flip = radix_sort_pairs(ctx, rb, m, nbits, s);
                res.sorted += m;
                skeys = flip ? w.keys1.get() : w.keys0.get();
                svals = flip ? w.vals1.get() : w.vals0.get();
                a += c_letters;
                first = false;
                if (a >= k) break;
                // run indices for the next chunk, in sorted order
                DK_LAUNCH(ctx, run_heads_kernel, g, kThreads, 0, s, skeys, m, w.heads.get());
                exclusive_scan_u32(ctx, w.heads.get(), w.pos.get(), m, nullptr, s);
                DK_LAUNCH(ctx, run_index_kernel, g, kThreads, 0, s, w.heads.get(), w.pos.get(), m, w.cur.get());
                // the sorted state order becomes the element order
                DK_CUDA(cudaMemcpyAsync(list_alt, svals, m * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
                elist = list_alt;
                cur_bits = bits_for(m - 1);
            }
            (void)first;
        }

        if (!done_table) {
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

        const uint32_t newB = B - A + c.runs;
        if (newB == B) break;  // fixed point: no block split (reference l.411)
        ++res.iters;
        B = newB;
        A = c.active_blocks;
        // surviving active states, order preserved (sorted order groups runs,
        // increasing state order inside each run)
        const uint32_t* src = done_table ? w.vals0.get() : svals;
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
