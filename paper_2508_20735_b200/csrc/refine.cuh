// refine.cuh -- device entry points of the refinement and product engines.
#pragma once

#include "common.cuh"

namespace dk {

struct DevDfa {
    uint32_t n = 0;
    uint32_t k = 0;
    const uint32_t* delta = nullptr;  // device, letter-major
    const uint8_t* acc = nullptr;     // device
    int64_t initial = -1;
};

struct RefineResult {
    uint32_t num_blocks = 0;
    uint32_t iters = 0;
    uint32_t closure = 0;
    uint64_t passes = 0;
    uint64_t sorted = 0;
    uint32_t collisions = 0;
};

struct SortOptions {
    bool force_exact = false;
    uint32_t fingerprint_bits = 64;
    uint32_t grouping = 0;  // 0 = auto, 1 = LSD radix sort (literal Alg. 4), 2 = host-staged passes only
};

// Key plan of one sortPR pass (see plan_pass in refine_sort.cu).
enum : uint32_t { kPlanTable = 0, kPlanPacked = 1, kPlanFingerprint = 2, kPlanChunked = 3 };
struct PassPlan {
    uint32_t strategy = kPlanTable;
    uint32_t field_bits = 0;    // packed keys: bits per field
    uint32_t key_bits = 0;      // packed key width (64 for fingerprints)
    uint32_t keylab_bytes = 0;  // 0: gather min-state labels; 1/2/4: dense block ids of that width
};
PassPlan plan_pass(uint32_t n, uint32_t k, uint32_t B, uint64_t m, uint32_t collisions, bool force_exact);
// PassPlan::keylab_bytes tag for one-bit key labels (two-block partitions);
// used from kBitLabelsMinStates states on, where a byte per state would
// crowd the L2 (below it the byte array is resident and cheaper to gather)
constexpr uint32_t kKeylabBits = 255;
constexpr uint32_t kBitLabelsMinStates = 1u << 25;

// Sharded sortPR primitives (refine_sort.cu; driven by sharded.py).
// counters: device uint32[4] = {runs, active blocks, active states, collision}.
struct ShardInit {
    uint32_t num_blocks, active_blocks;
    uint64_t active_states;
};
ShardInit shard_init(Ctx* ctx, const DevDfa& d, uint32_t lo, uint32_t hi, uint32_t* lab, uint8_t* act,
                     cudaStream_t s, bool lazy = false);
void shard_keylab(Ctx* ctx, const uint32_t* lab, uint32_t n, uint32_t num_blocks, const PassPlan& plan, void* out,
                  uint32_t* scratch, cudaStream_t s,
                  const uint8_t* initial_acc = nullptr);
// list == nullptr: the active states are list_base .. list_base + m - 1
void shard_table_signature(Ctx* ctx, const DevDfa& d, const void* keylab, const PassPlan& plan, const uint32_t* list,
                           uint32_t list_base, uint64_t m, uint32_t* keys32, uint32_t* tmin, uint32_t* tcnt,
                           cudaStream_t s);
void shard_table_apply(Ctx* ctx, const PassPlan& plan, const uint32_t* list, uint32_t list_base,
                       const uint32_t* keys32, uint64_t m, const uint32_t* tmin, const uint32_t* tcnt, uint32_t* lab,
                       uint8_t* act, void* next_keylab, uint32_t* counters, cudaStream_t s);
void shard_sig_partition(Ctx* ctx, const DevDfa& d, const void* keylab, const PassPlan& plan, uint64_t salt,
                         const uint32_t* list, uint32_t list_base, uint64_t m, uint32_t world, uint4* send,
                         uint32_t* send_counts, cudaStream_t s);
// verify_lab: any injective labelling of the current blocks (verify_bytes
// 4 / 2 / 1 / kKeylabBits) -- the min-state labels, or the pass's key labels
void shard_group(Ctx* ctx, const DevDfa& d, const void* verify_lab, uint32_t verify_bytes, const PassPlan& plan,
                 const uint4* recv, uint64_t count, uint32_t* results, uint32_t* counters, cudaStream_t s);
// The same in two steps (the native driver): grouping into a workspace that
// keeps slot-ordered records, and the per-entry results from them -- needed
// only when the pass is not the last.
struct ShardGroupWs {
    DBuf<uint32_t> bcnt;
    DBuf<uint4> bent;
    DBuf<uint2> rec;
    uint32_t nb = 0, ovf = 0;
    uint64_t count = 0;
};
void shard_group_deferred(Ctx* ctx, const DevDfa& d, const void* verify_lab, uint32_t verify_bytes,
                          const PassPlan& plan, const uint4* recv, uint64_t count, ShardGroupWs& ws,
                          uint32_t* counters, cudaStream_t s);
void shard_group_results(Ctx* ctx, const ShardGroupWs& ws, uint32_t* results, cudaStream_t s);
// Owner-bucket layout of the native driver's wide passes: the sender's
// signature kernel appends straight into (owner, bucket) sub-buckets of cs
// slots (nb buckets per owner), which travel as they are; the owner groups
// the W senders' parts of each bucket together (no staging / partition /
// re-bucketing passes).  Sub-bucket overflow goes through a compact list and
// the global-table fallback.
struct OwnerPlan {
    uint32_t world = 1, nb = 1, cs = 0;
};
OwnerPlan owner_plan(uint64_t m_total, uint32_t world);
struct OwnerSend {
    DBuf<uint4> send;        // world * nb * cs slots: region o = nb sub-buckets of owner o
    DBuf<uint32_t> scur;     // sub-bucket cursors (kCntStride apart)
    DBuf<uint4> ovf, ovf_sorted;  // overflow entries, then sorted by owner
    DBuf<uint32_t> ovf_cnt;  // per owner, then the total
    DBuf<uint32_t> ovf_cur;
    DBuf<uint32_t> msg;      // per owner: nb counts + overflow count
    DBuf<uint64_t> part;     // partial keys of a sliced signature pass
};
struct OwnerSources {
    const uint4* base[8];
    const uint32_t* cnt[8];
};
// Where the sender's signature kernel puts owner o's sub-bucket entries
// (nb * cs slots) and their counts (nb + 1 words): its own send regions,
// exchanged afterwards, or -- peer mode -- this rank's region of owner o's
// receive buffers, written over NVLink by the kernel itself.
struct OwnerDst {
    uint4* entries[8];
    uint32_t* counts[8];
    int peer;  // some destinations are other GPUs' memory: system-scope fence before the kernel ends
};
// Owners' label writes into the senders' label / survivor-flag arrays (peer mode)
struct PeerLabels {
    uint32_t* lab[8];
    uint8_t* act[8];
};
// 16-bit labels below 4096 packed 12 bits apiece, five per 64-bit word;
// returns the KeyLab::bytes tag of the packed array (signature passes only)
// (eleven: 11-bit labels packed back to back instead; values below 2048)
uint32_t pack12_labels(Ctx* ctx, const uint16_t* keys16, uint32_t n, unsigned long long* out, cudaStream_t s,
                       bool eleven = false);
uint64_t pack_words(uint32_t n);  // words of the packed array (either layout)
bool pack11_unsliced(uint32_t n);  // 11-bit packed labels of n states need no slicing
int pack_choice(uint32_t n, uint32_t bits);  // 0 (16-bit labels), 11 or 12 (packed) for a big pass
void shard_sig_owner(Ctx* ctx, const DevDfa& d, const void* keylab, const PassPlan& plan, uint64_t salt,
                     const uint32_t* list, uint32_t list_base, uint64_t m, const OwnerPlan& op, OwnerSend& ws,
                     cudaStream_t s, const OwnerDst* dst = nullptr);
// peer mode, owner side: every received region entry's result straight into
// its sender's label (and survivor flag) -- the results' trip back and the
// sender's apply in one kernel
void shard_owner_scatter(Ctx* ctx, const OwnerPlan& op, const uint4* recv, const uint32_t* recv_cnt,
                         const uint32_t* results, const uint8_t* bsingle, const PeerLabels& out, cudaStream_t s);
// sender: the results of its overflow entries (peer mode: the region entries
// were applied by their owners)
void shard_apply_overflow(Ctx* ctx, const OwnerSend& ws, const uint32_t* back_ovf, uint32_t ovf_total, uint32_t* lab,
                          uint8_t* act, cudaStream_t s);
void shard_sort_overflow(Ctx* ctx, const OwnerPlan& op, OwnerSend& ws, uint32_t ovf_total, cudaStream_t s);
void shard_owner_ovf_counts(Ctx* ctx, const OwnerPlan& op, const uint32_t* recv_msg, uint32_t* out, cudaStream_t s);
void shard_group_owner(Ctx* ctx, const DevDfa& d, const void* verify_lab, uint32_t verify_bytes, const PassPlan& plan,
                       const OwnerPlan& op, const OwnerSources& in, const uint4* ovf_in, uint32_t ovf_total,
                       uint32_t* results, uint32_t* counters, cudaStream_t s, uint8_t* bsingle = nullptr);
void shard_apply_owner(Ctx* ctx, const OwnerPlan& op, const OwnerSend& ws, uint32_t rank, const uint32_t* own_res,
                       const uint32_t* back, const uint32_t* back_ovf, uint32_t ovf_total, uint32_t* lab,
                       uint8_t* act, cudaStream_t s);
void shard_apply(Ctx* ctx, const uint4* send, const uint32_t* results, uint64_t count, uint32_t* lab, uint8_t* act,
                 cudaStream_t s);
void shard_compact(Ctx* ctx, const uint8_t* act, uint32_t lo, uint32_t hi, uint32_t* list, uint32_t* count_dev,
                   cudaStream_t s);

// Native sharded driver over NCCL (shard_driver.cu).
struct NcclComm;
void nccl_unique_id(uint8_t out[128]);
NcclComm* nccl_comm_init(Ctx* ctx, const uint8_t id[128], int world, int rank);
void nccl_comm_destroy(NcclComm* c);
// in-process hub: `world` ranks as threads sharing one device (testing the
// driver's multi-rank path on a single GPU)
struct LocalHub;
LocalHub* local_hub_create(int world);
void local_hub_destroy(LocalHub* h);
NcclComm* local_comm_init(LocalHub* hub, int rank);
RefineResult sort_pr_sharded_device(Ctx* ctx, NcclComm* comm, const DevDfa& d, uint32_t* block_out, cudaStream_t s,
                                    uint64_t* exchanged);

// All block_out arrays are device arrays of n entries, canonical numbering.
// Host-buffer calls stream delta to the device in state-range chunks on a
// copy stream; pass 1 of sort_pr then consumes chunk c once ready[c] fired
// (range check + counting-table signatures), hiding under the PCIe copy.
struct DeltaStream {
    uint32_t chunks = 0;
    const uint32_t* bounds = nullptr;  // host, chunks + 1 state indices
    const cudaEvent_t* ready = nullptr;
};
RefineResult sort_pr_device(Ctx* ctx, const DevDfa& d, const SortOptions& o, uint32_t* block_out, cudaStream_t s,
                            const DeltaStream* ds = nullptr);
RefineResult naive_pr_device(Ctx* ctx, const DevDfa& d, int policy, uint64_t seed, uint32_t* block_out,
                             cudaStream_t s);
// ElectionPolicy::arbitrary(seed) with the reference's exact winner stream
RefineResult naive_pr_arbitrary_device(Ctx* ctx, const DevDfa& d, uint64_t seed, uint32_t* block_out,
                                       cudaStream_t s);
RefineResult naive_pr_fused_device(Ctx* ctx, const DevDfa& d, uint32_t* block_out, cudaStream_t s);
uint32_t floor_log2_u32(uint32_t n);
// out: k * (floor_log2(n)+1) * n entries (device)
void transitive_alphabet_device(Ctx* ctx, const DevDfa& d, uint32_t* out, cudaStream_t s);
RefineResult trans_pr_device(Ctx* ctx, const DevDfa& d, int policy, uint64_t seed, uint64_t max_transitions,
                             uint32_t* block_out, cudaStream_t s);
RefineResult trans_minimize_device(Ctx* ctx, const DevDfa& d, uint64_t max_pair_nodes, uint32_t* block_out,
                                   uint8_t* apart_dev, cudaStream_t s);

// Leader initialisation shared by naive/fused: min-index accepting and
// rejecting leaders; returns false when F or Q\F is empty (one block).
struct LeaderInfo {
    uint32_t min_acc, min_rej, cnt_acc, cnt_rej;
};
LeaderInfo leader_info(Ctx* ctx, const DevDfa& d, cudaStream_t s);
// Same, read back later: the kernel and a copy into the pinned mailbox are
// queued now; leader_info_wait() waits for that copy only (kernels queued
// after it keep the device busy meanwhile).
void leader_info_async(Ctx* ctx, const DevDfa& d, cudaStream_t s, uint8_t* dense2 = nullptr);
LeaderInfo leader_info_wait(Ctx* ctx);
void init_leader_labels(Ctx* ctx, const DevDfa& d, const LeaderInfo& li, uint32_t* lab, cudaStream_t s);

// product exploration
struct ProductOut {
    int32_t verdict = 0;
    uint32_t levels = 0;
    uint64_t explored = 0;
    std::basic_string<uint32_t> word;
};
ProductOut explore_product_device(Ctx* ctx, const DevDfa& a, const DevDfa& b, int mode, const uint32_t* letter_map,
                                  uint64_t max_visited, cudaStream_t s);
ProductOut check_equiv_uf_device(Ctx* ctx, const DevDfa& a, const DevDfa& b, cudaStream_t s);

// measured random-gather rate (gathers/s) from a table of table_words entries
double calibrate_gather(Ctx* ctx, uint64_t table_words, uint32_t elem_bytes, uint64_t gathers, cudaStream_t s,
                        float* ms_out);

// generators
void gen_synth_device(Ctx* ctx, uint32_t n, uint32_t k, uint64_t seed, uint32_t* delta, uint8_t* acc,
                      cudaStream_t s);
void gen_chain_device(Ctx* ctx, uint32_t n, uint32_t* delta, uint8_t* acc, cudaStream_t s);
uint32_t permute_states_device(Ctx* ctx, uint32_t n, uint32_t k, uint64_t seed, const uint32_t* delta,
                               const uint8_t* acc, uint32_t* out_delta, uint8_t* out_acc, cudaStream_t s);

}  // namespace dk
