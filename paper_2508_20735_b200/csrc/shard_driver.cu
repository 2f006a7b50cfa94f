// shard_driver.cu -- the sharded sortPR pass loop in C++ over NCCL.
//
// Same protocol as paper_2508_20735_b200/sharded.py (whose gloo CPU tests pin
// it), driven natively: one process per GPU, the shard primitives of
// refine_sort.cu on the caller's stream, NCCL collectives on the same
// stream.  Per pass:
//   table plans:  local (min, count) table -> ncclAllReduce MIN / SUM ->
//                 relabel own states (+ ranks as next key labels when the
//                 pass covered every state);
//   wide plans:   entries partitioned by owner -> grouped ncclSend/ncclRecv
//                 (16 B per active state) -> owner groups -> counters
//                 allreduced (collision => every rank retries with a new
//                 salt) -> results back (4 B per entry) -> apply;
//   then ncclAllGather of the label slices (the per-pass block-ID
//   allgather) and the next local active list.
// NCCL is resolved with dlopen at first use (the library has no link-time
// NCCL dependency; a process that already loaded NCCL, e.g. through torch,
// shares that copy).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <mutex>
#include <vector>

#include "prims.cuh"
#include "refine.cuh"

namespace dk {

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    const char* (*GetErrorString)(ncclResult_t);
};

const NcclApi& nccl() {
    static NcclApi api{};
    static std::string err;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = "libnccl.so.2 not found";
            return;
        }
        auto sym = [&](const char* n) {
            void* p = dlsym(h, n);
            if (!p) err = std::string("NCCL symbol missing: ") + n;
            return p;
        };
        api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
        api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
        api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
        api.Send = (decltype(api.Send))sym("ncclSend");
        api.Recv = (decltype(api.Recv))sym("ncclRecv");
        api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
        api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
        api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    });
    if (!err.empty()) throw Error(DFAKIT_E_RESOURCE, err);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Error(DFAKIT_E_CUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}

uint64_t mix64_host(uint64_t z) { return mix64(z); }

// one grouped send/recv round: element_bytes-sized elements, offsets and
// counts per peer
void grouped_all_to_all(const NcclApi& api, ncclComm_t comm, int world, const void* send,
                        const std::vector<uint64_t>& soff, const std::vector<uint64_t>& scount, void* recv,
                        const std::vector<uint64_t>& roff, const std::vector<uint64_t>& rcount, size_t element_bytes,
                        cudaStream_t s) {
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (int r = 0; r < world; ++r) {
        if (scount[r])
            nccl_check(api.Send(static_cast<const char*>(send) + soff[r] * element_bytes, scount[r] * element_bytes,
                                ncclUint8, r, comm, s),
                       "ncclSend");
        if (rcount[r])
            nccl_check(api.Recv(static_cast<char*>(recv) + roff[r] * element_bytes, rcount[r] * element_bytes,
                                ncclUint8, r, comm, s),
                       "ncclRecv");
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
}

}  // namespace

// Peer-memory workspace of a communicator (peer mode of the owner-bucket
// passes): every rank's receive regions, received counts, block labels and
// survivor flags, allocated with cudaMalloc (IPC-exportable) and mapped into
// every other rank (CUDA IPC over NVLink / NVSwitch between processes; plain
// pointers between the local hub's threads).  Kept across calls; grown
// collectively (every rank asks for the same sizes: they follow from n).
struct PeerSpace {
    int state = 0;  // 0 untried, 1 enabled, -1 disabled (setup or self-test failed)
    int device = 0;
    uint64_t recv_slots = 0, cnt_words = 0, lab_words = 0, act_bytes = 0;
    void* local[4] = {nullptr, nullptr, nullptr, nullptr};  // recv (uint4), cnt (u32), lab (u32), act (u8)
    std::vector<std::array<void*, 4>> peer;                  // per rank; own entry = local
    uint32_t* sync = nullptr;                                // barrier word
};

// Collectives of the pass loop on stream s.  NCCL in production; the local
// hub runs several ranks as threads of one process sharing a device (each
// with its own context), staging through host memory -- the way the
// driver's multi-rank path is tested on a single GPU.
struct NcclComm {
    virtual ~NcclComm() = default;
    int world = 1, rank = 0;
    PeerSpace peer;
    // every rank's local[4] pointers, mapped into this process (collective:
    // every rank calls it, valid or not; false when any mapping is missing)
    virtual bool exchange_peer_ptrs(cudaStream_t s, bool valid) = 0;
    virtual void release_peer_ptrs() = 0;
    // stream-ordered barrier: this rank's prior work on s is complete, and
    // work queued on s after it starts only once every rank's prior work is
    virtual void barrier(cudaStream_t s) = 0;
    virtual void allreduce_u32(uint32_t* buf, size_t count, bool use_min, cudaStream_t s) = 0;
    // full holds world slices of `bytes`; this rank's slice is at rank * bytes
    virtual void allgather(void* full, size_t bytes, cudaStream_t s) = 0;
    // element offsets per peer given explicitly (segments need not be packed)
    virtual void all_to_all_off(const void* send, const std::vector<uint64_t>& soff,
                                const std::vector<uint64_t>& scount, void* recv, const std::vector<uint64_t>& roff,
                                const std::vector<uint64_t>& rcount, size_t element_bytes, cudaStream_t s) = 0;
    void all_to_all_v(const void* send, const std::vector<uint64_t>& scount, void* recv,
                      const std::vector<uint64_t>& rcount, size_t element_bytes, cudaStream_t s) {
        std::vector<uint64_t> so(world), ro(world);
        for (int r = 1; r < world; ++r) {
            so[r] = so[r - 1] + scount[r - 1];
            ro[r] = ro[r - 1] + rcount[r - 1];
        }
        all_to_all_off(send, so, scount, recv, ro, rcount, element_bytes, s);
    }
};

namespace {

struct NcclImpl : NcclComm {
    ncclComm_t comm = nullptr;
    ~NcclImpl() override {
        release_peer_ptrs();
        if (comm) nccl().CommDestroy(comm);
    }
    void barrier(cudaStream_t s) override {
        nccl_check(nccl().AllReduce(peer.sync, peer.sync, 1, ncclUint32, ncclSum, comm, s), "barrier");
    }
    // CUDA IPC: every rank exports its four buffers, the 64-byte handles
    // travel by one ncclAllGather, and the peers' buffers are opened with
    // lazy peer access (NVLink / NVSwitch stores from this rank's kernels)
    bool exchange_peer_ptrs(cudaStream_t s, bool valid) override {
        // one extra byte per buffer flags a handle that could not be made
        constexpr size_t H = sizeof(cudaIpcMemHandle_t), E = H + 1;
        std::vector<unsigned char> mine(4 * E, 0), all((size_t)world * 4 * E);
        for (int i = 0; i < 4 && valid && world > 1; ++i) {
            const cudaError_t e =
                cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(mine.data() + i * E), peer.local[i]);
            if (e != cudaSuccess) {
                cudaGetLastError();
                valid = false;
            }
        }
        for (int i = 0; i < 4; ++i) mine[i * E + H] = valid ? 1 : 0;
        DBuf<unsigned char> dev((size_t)world * 4 * E, s);
        DK_CUDA(cudaMemcpyAsync(dev.get() + (size_t)rank * 4 * E, mine.data(), 4 * E, cudaMemcpyHostToDevice, s));
        nccl_check(nccl().AllGather(dev.get() + (size_t)rank * 4 * E, dev.get(), 4 * E, ncclUint8, comm, s),
                   "allgather (ipc handles)");
        DK_CUDA(cudaMemcpyAsync(all.data(), dev.get(), all.size(), cudaMemcpyDeviceToHost, s));
        DK_CUDA(cudaStreamSynchronize(s));
        peer.peer.assign(world, {nullptr, nullptr, nullptr, nullptr});
        bool ok = valid;
        for (int r = 0; r < world; ++r)
            for (int i = 0; i < 4; ++i) {
                if (r == rank) {
                    peer.peer[r][i] = valid ? peer.local[i] : nullptr;
                    continue;
                }
                const unsigned char* rec = all.data() + ((size_t)r * 4 + i) * E;
                if (!rec[H] || !valid) {
                    ok = false;
                    continue;
                }
                cudaIpcMemHandle_t h;
                std::memcpy(&h, rec, H);
                if (cudaIpcOpenMemHandle(&peer.peer[r][i], h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                    cudaGetLastError();
                    peer.peer[r][i] = nullptr;
                    ok = false;
                }
            }
        return ok;
    }
    void release_peer_ptrs() override {
        for (int r = 0; r < (int)peer.peer.size(); ++r)
            if (r != rank)
                for (void* p : peer.peer[r])
                    if (p) cudaIpcCloseMemHandle(p);
        peer.peer.clear();
    }
    void allreduce_u32(uint32_t* buf, size_t count, bool use_min, cudaStream_t s) override {
        nccl_check(nccl().AllReduce(buf, buf, count, ncclUint32, use_min ? ncclMin : ncclSum, comm, s), "allreduce");
    }
    void allgather(void* full, size_t bytes, cudaStream_t s) override {
        nccl_check(nccl().AllGather(static_cast<char*>(full) + (uint64_t)rank * bytes, full, bytes, ncclUint8, comm, s),
                   "allgather");
    }
    void all_to_all_off(const void* send, const std::vector<uint64_t>& soff, const std::vector<uint64_t>& scount,
                        void* recv, const std::vector<uint64_t>& roff, const std::vector<uint64_t>& rcount,
                        size_t element_bytes, cudaStream_t s) override {
        grouped_all_to_all(nccl(), comm, world, send, soff, scount, recv, roff, rcount, element_bytes, s);
    }
};

}  // namespace

struct LocalHub {
    explicit LocalHub(int w) : world(w), host(w), counts(w), ptrs(w) {}
    int world;
    std::vector<std::array<void*, 4>> ptrs;  // peer mode: the ranks' buffers (one device, plain pointers)
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    std::vector<std::vector<uint8_t>> host;
    std::vector<std::vector<uint64_t>> counts;
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const uint64_t gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

namespace {

struct LocalImpl : NcclComm {
    LocalHub* hub = nullptr;
    ~LocalImpl() override { release_peer_ptrs(); }
    void barrier(cudaStream_t s) override {
        DK_CUDA(cudaStreamSynchronize(s));
        hub->barrier();
    }
    bool exchange_peer_ptrs(cudaStream_t s, bool valid) override {
        DK_CUDA(cudaStreamSynchronize(s));
        for (int i = 0; i < 4; ++i) hub->ptrs[rank][i] = valid ? peer.local[i] : nullptr;
        hub->barrier();
        peer.peer = hub->ptrs;
        hub->barrier();
        bool ok = true;
        for (const auto& a : peer.peer)
            for (void* p : a) ok &= p != nullptr;
        return ok;
    }
    void release_peer_ptrs() override { peer.peer.clear(); }
    void publish(const void* dev, size_t bytes, cudaStream_t s) {
        auto& h = hub->host[rank];
        h.resize(bytes);
        if (bytes) DK_CUDA(cudaMemcpyAsync(h.data(), dev, bytes, cudaMemcpyDeviceToHost, s));
        DK_CUDA(cudaStreamSynchronize(s));
    }
    void allreduce_u32(uint32_t* buf, size_t count, bool use_min, cudaStream_t s) override {
        publish(buf, count * 4, s);
        hub->barrier();
        std::vector<uint32_t> acc(count);
        for (int r = 0; r < world; ++r) {
            const uint32_t* v = reinterpret_cast<const uint32_t*>(hub->host[r].data());
            for (size_t i = 0; i < count; ++i)
                acc[i] = r == 0 ? v[i] : (use_min ? std::min(acc[i], v[i]) : acc[i] + v[i]);
        }
        if (count) DK_CUDA(cudaMemcpyAsync(buf, acc.data(), count * 4, cudaMemcpyHostToDevice, s));
        DK_CUDA(cudaStreamSynchronize(s));
        hub->barrier();
    }
    void allgather(void* full, size_t bytes, cudaStream_t s) override {
        publish(static_cast<char*>(full) + (uint64_t)rank * bytes, bytes, s);
        hub->barrier();
        for (int r = 0; r < world; ++r)
            if (bytes)
                DK_CUDA(cudaMemcpyAsync(static_cast<char*>(full) + (uint64_t)r * bytes, hub->host[r].data(), bytes,
                                        cudaMemcpyHostToDevice, s));
        DK_CUDA(cudaStreamSynchronize(s));
        hub->barrier();
    }
    void all_to_all_off(const void* send, const std::vector<uint64_t>& soff, const std::vector<uint64_t>& scount,
                        void* recv, const std::vector<uint64_t>& roff, const std::vector<uint64_t>& rcount,
                        size_t element_bytes, cudaStream_t s) override {
        // stage every outgoing segment back to back; counts tell the peers where theirs is
        uint64_t total = 0;
        for (uint64_t c : scount) total += c;
        auto& h = hub->host[rank];
        h.resize(total * element_bytes);
        uint64_t at = 0;
        for (int r = 0; r < world; ++r) {
            if (scount[r])
                DK_CUDA(cudaMemcpyAsync(h.data() + at * element_bytes,
                                        static_cast<const char*>(send) + soff[r] * element_bytes,
                                        scount[r] * element_bytes, cudaMemcpyDeviceToHost, s));
            at += scount[r];
        }
        DK_CUDA(cudaStreamSynchronize(s));
        hub->counts[rank] = scount;
        hub->barrier();
        for (int r = 0; r < world; ++r) {
            uint64_t off = 0;
            for (int j = 0; j < rank; ++j) off += hub->counts[r][j];
            const uint64_t c = hub->counts[r][rank];
            if (c != rcount[r]) throw Error(DFAKIT_E_INVALID, "local hub: receive count mismatch");
            if (c)
                DK_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + roff[r] * element_bytes,
                                        hub->host[r].data() + off * element_bytes, c * element_bytes,
                                        cudaMemcpyHostToDevice, s));
        }
        DK_CUDA(cudaStreamSynchronize(s));
        hub->barrier();
    }
};

}  // namespace

void nccl_unique_id(uint8_t out[128]) {
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "NCCL unique id size");
    std::memcpy(out, &id, sizeof(id));
}

NcclComm* nccl_comm_init(Ctx* ctx, const uint8_t id[128], int world, int rank) {
    if (world < 1 || rank < 0 || rank >= world) throw Error(DFAKIT_E_INVALID, "comm_init: bad rank / world");
    DK_CUDA(cudaSetDevice(ctx->device));
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    NcclImpl* c = new NcclImpl();
    c->world = world;
    c->rank = rank;
    const ncclResult_t r = nccl().CommInitRank(&c->comm, world, uid, rank);
    if (r != ncclSuccess) {
        c->comm = nullptr;
        delete c;
        nccl_check(r, "ncclCommInitRank");
    }
    return c;
}

LocalHub* local_hub_create(int world) {
    if (world < 1 || world > 64) throw Error(DFAKIT_E_INVALID, "local hub: world size out of range");
    return new LocalHub(world);
}

void local_hub_destroy(LocalHub* h) { delete h; }

NcclComm* local_comm_init(LocalHub* hub, int rank) {
    if (!hub || rank < 0 || rank >= hub->world) throw Error(DFAKIT_E_INVALID, "local comm: bad rank");
    LocalImpl* c = new LocalImpl();
    c->hub = hub;
    c->world = hub->world;
    c->rank = rank;
    return c;
}

void peer_space_release(NcclComm* cm);

void nccl_comm_destroy(NcclComm* c) {
    if (!c) return;
    int cur = 0;
    cudaGetDevice(&cur);
    if (c->peer.state > 0) cudaSetDevice(c->peer.device);
    peer_space_release(c);
    cudaSetDevice(cur);
    delete c;
}

namespace {

__global__ void peer_probe_kernel(PeerLabels pl, int world, int rank) {
    // every rank stamps its id into word `rank` of every rank's label buffer
    const int r = threadIdx.x;
    if (r < world) pl.lab[r][rank] = 0xC0DE0000u | (uint32_t)rank;
}

void peer_free_local(PeerSpace& p) {
    for (void*& q : p.local)
        if (q) {
            cudaFree(q);
            q = nullptr;
        }
    if (p.sync) cudaFree(p.sync);
    p.sync = nullptr;
}

// Makes the peer workspace at least this large on every rank (collective:
// every rank passes the same sizes) and, the first time, proves the mapping
// with a stamp exchange; any failure turns peer mode off for the comm (the
// NCCL region exchange takes over).  Returns whether peer mode is on.
bool peer_ensure(Ctx* ctx, NcclComm* cm, uint64_t recv_slots, uint64_t cnt_words, uint64_t lab_words,
                 uint64_t act_bytes, cudaStream_t s) {
    PeerSpace& p = cm->peer;
    if (p.state < 0) return false;
    if (p.state > 0 && p.recv_slots >= recv_slots && p.cnt_words >= cnt_words && p.lab_words >= lab_words &&
        p.act_bytes >= act_bytes)
        return true;
    // every step below is taken by every rank, whatever failed locally, so
    // the collectives inside line up; the verdict is allreduced at the end
    const int world = cm->world, rank = cm->rank;
    const bool first = p.state == 0;
    DK_CUDA(cudaStreamSynchronize(s));
    if (!first) cm->barrier(s);  // nobody still writes into the old buffers
    DK_CUDA(cudaStreamSynchronize(s));
    cm->release_peer_ptrs();
    peer_free_local(p);
    p.device = ctx->device;
    p.recv_slots = std::max(p.recv_slots, recv_slots);
    p.cnt_words = std::max(p.cnt_words, cnt_words);
    p.lab_words = std::max(p.lab_words, std::max<uint64_t>(lab_words, (uint64_t)world));
    p.act_bytes = std::max(p.act_bytes, act_bytes);
    bool ok = true;
    const size_t bytes[4] = {std::max<uint64_t>(1, p.recv_slots) * sizeof(uint4),
                             std::max<uint64_t>(1, p.cnt_words) * sizeof(uint32_t), p.lab_words * sizeof(uint32_t),
                             std::max<uint64_t>(1, p.act_bytes)};
    for (int i = 0; i < 4 && ok; ++i)
        if (cudaMalloc(&p.local[i], bytes[i]) != cudaSuccess) {
            cudaGetLastError();
            p.local[i] = nullptr;
            ok = false;
        }
    DK_CUDA(cudaMalloc(reinterpret_cast<void**>(&p.sync), sizeof(uint32_t)));
    DK_CUDA(cudaMemsetAsync(p.sync, 0, sizeof(uint32_t), s));
    if (ok) DK_CUDA(cudaMemsetAsync(p.local[2], 0, (size_t)world * sizeof(uint32_t), s));
    ok = cm->exchange_peer_ptrs(s, ok);
    if (first) {
        // stamp exchange: every rank writes its id into word `rank` of every
        // rank's label buffer through the mapping, then checks its own
        cm->barrier(s);
        if (ok) {
            PeerLabels pl{};
            for (int r = 0; r < world; ++r) pl.lab[r] = static_cast<uint32_t*>(p.peer[r][2]);
            peer_probe_kernel<<<1, 32, 0, s>>>(pl, world, rank);
            if (cudaGetLastError() != cudaSuccess) ok = false;
        }
        cm->barrier(s);
        if (ok) {
            std::vector<uint32_t> got(world);
            DK_CUDA(cudaMemcpyAsync(got.data(), p.local[2], world * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
            DK_CUDA(cudaStreamSynchronize(s));
            for (int r = 0; r < world; ++r) ok &= got[r] == (0xC0DE0000u | (uint32_t)r);
        }
    }
    DBuf<uint32_t> v(1, s);
    const uint32_t mine = ok ? 1u : 0u;
    DK_CUDA(cudaMemcpyAsync(v.get(), &mine, 4, cudaMemcpyHostToDevice, s));
    cm->allreduce_u32(v.get(), 1, true, s);
    uint32_t all = 0;
    DK_CUDA(cudaMemcpyAsync(&all, v.get(), 4, cudaMemcpyDeviceToHost, s));
    DK_CUDA(cudaStreamSynchronize(s));
    if (all) {
        p.state = 1;
        return true;
    }
    cm->release_peer_ptrs();
    peer_free_local(p);
    if (!first) throw Error(DFAKIT_E_RESOURCE, "sharded sort_pr: growing the peer workspace failed");
    p.state = -1;
    return false;
}

}  // namespace

void peer_space_release(NcclComm* cm) {
    cm->release_peer_ptrs();
    peer_free_local(cm->peer);
}

RefineResult sort_pr_sharded_device(Ctx* ctx, NcclComm* cm, const DevDfa& d, uint32_t* block_out, cudaStream_t s,
                                    uint64_t* exchanged) {
    RefineResult res;
    const uint32_t n = d.n, k = d.k;
    const int world = cm->world, rank = cm->rank;
    if (n == 0) return res;
    if (n > 0x7fffffffu) throw Error(DFAKIT_E_INVALID, "sharded sort_pr: at most 2^31 - 1 states");
    // ranges start at multiples of four (the vectorised table apply)
    const uint32_t shard = (uint32_t)((((uint64_t)n + world - 1) / world + 3) / 4 * 4);
    const uint32_t lo = std::min<uint64_t>(n, (uint64_t)rank * shard);
    const uint32_t hi = std::min<uint64_t>(n, (uint64_t)(rank + 1) * shard);
    // owner-bucket layout (up to 8 ranks; DFAKIT_SHARD_STAGED=1 forces the
    // staged entries + partition + owner re-bucketing protocol of sharded.py)
    const bool owner_layout = world <= 8 && !getenv("DFAKIT_SHARD_STAGED");
    // peer mode (owner layout; DFAKIT_SHARD_PEER=0 turns it off): the
    // signature kernel stores each entry straight into its owner's receive
    // region and the owners write the results straight into the senders'
    // labels -- over NVLink between GPUs -- instead of two NCCL exchanges
    const char* peer_env = getenv("DFAKIT_SHARD_PEER");
    const OwnerPlan op_max = owner_plan(n, (uint32_t)world);
    const bool peer_mode = owner_layout && !(peer_env && peer_env[0] == '0') &&
                           peer_ensure(ctx, cm, (uint64_t)world * op_max.nb * op_max.cs,
                                       (uint64_t)world * (op_max.nb + 1), (uint64_t)world * shard, n, s);
    // DFAKIT_SHARD_PEER=2 (tests): peer mode required, its absence an error
    if (owner_layout && peer_env && peer_env[0] == '2' && !peer_mode)
        throw Error(DFAKIT_E_RESOURCE, "sharded sort_pr: peer mode required but unavailable");
    DBuf<uint32_t> lab_own, list(std::max(1u, hi - lo), s), scratch((uint64_t)n + 1, s);
    DBuf<uint8_t> act_own;
    if (!peer_mode) {
        lab_own.alloc((uint64_t)world * shard, s);
        act_own.alloc(n, s);
    }
    uint32_t* const LAB = peer_mode ? static_cast<uint32_t*>(cm->peer.local[2]) : lab_own.get();
    uint8_t* const ACT = peer_mode ? static_cast<uint8_t*>(cm->peer.local[3]) : act_own.get();
    DBuf<uint32_t> dctr(8, s), counts(2 * (uint64_t)world, s), keys32;  // [send counts | receive counts]
    DBuf<uint8_t> kl8;
    DBuf<uint16_t> kl16, next16;
    DBuf<uint32_t> kl32, next32, tmin, tcnt, results, back, bits;
    DBuf<uint4> send, recv;
    ShardGroupWs gws;  // owner-side grouping workspace (slot-ordered records)
    OwnerSend ows;
    DBuf<uint32_t> rmsg, small(2 * (uint64_t)world + 2, s);
    DBuf<uint4> rreg, rovf_buf;
    DBuf<uint32_t> back_ovf;
    DBuf<uint8_t> bsingle;  // peer mode: per owner bucket, 1 = every key distinct (no results written)
    DBuf<unsigned long long> pack12;  // packed 12-bit copy of the carried key labels
    auto read_u32 = [&](const uint32_t* p, size_t count, uint32_t* out) {
        for (size_t i = 0; i < count; i += 112)  // read_words moves at most 112 words
            read_words(ctx, p + i, std::min<size_t>(112, count - i) * sizeof(uint32_t), out + i, s);
    };

    const ShardInit si = shard_init(ctx, d, lo, hi, LAB, ACT, s, /*lazy=*/true);
    uint32_t B = si.num_blocks, A = si.active_blocks;
    uint64_t m_total = si.active_states;
    uint32_t m = 0;
    auto compact = [&] {
        shard_compact(ctx, ACT, lo, hi, list.get(), dctr.get() + 4, s);
        read_u32(dctr.get() + 4, 1, &m);
    };
    if (m_total == n) m = hi - lo;  // every state active: the identity range
    else compact();
    uint64_t salt = 0x5EED5EED5EEDull;
    uint32_t strikes = 0;
    const void* carried = nullptr;  // key labels of the current partition (ranks of a full table pass)
    bool lab_stale = false;         // other ranks' slices of `lab` not yet exchanged
    uint32_t carried_bytes = 0;
    uint64_t sent = 0;
    while (m_total > 0) {
        ++res.passes;
        PassPlan plan = plan_pass(n, k, B, m_total, std::min(strikes, 2u), false);
        if (plan.strategy == kPlanChunked) {  // sharded: fingerprints with fresh salts instead
            plan.strategy = kPlanFingerprint;
            plan.field_bits = 0;
            plan.key_bits = 64;
            plan.keylab_bytes = 0;
        }
        const uint32_t* lst = m == hi - lo ? nullptr : list.get();
        // the other ranks' min-state labels are needed unless the pass
        // gathers carried key labels
        if (lab_stale && !(plan.keylab_bytes && carried)) {
            cm->allgather(LAB, (size_t)shard * sizeof(uint32_t), s);
            lab_stale = false;
        }
        const void* keylab = LAB;
        if (plan.keylab_bytes) {
            if (carried) {
                keylab = carried;
                plan.keylab_bytes = carried_bytes;
            } else {
                void* out;
                if (plan.keylab_bytes == 1 && B <= 2 && n >= kBitLabelsMinStates) {  // two blocks, large n: a bitmap
                    if (!bits.get()) bits.alloc(((uint64_t)n + 31) / 32, s);
                    plan.keylab_bytes = kKeylabBits;
                    out = bits.get();
                } else if (plan.keylab_bytes == 1) {
                    if (!kl8.get()) kl8.alloc(n, s);
                    out = kl8.get();
                } else if (plan.keylab_bytes == 2) {
                    if (!kl16.get()) kl16.alloc(n, s);
                    out = kl16.get();
                } else {
                    if (!kl32.get()) kl32.alloc(n, s);
                    out = kl32.get();
                }
                shard_keylab(ctx, LAB, n, B, plan, out, scratch.get(), s, res.iters == 0 ? d.acc : nullptr);
                keylab = out;
            }
        }
        carried = nullptr;
        void* next_kl = nullptr;
        uint32_t ctr[4];
        if (plan.strategy == kPlanTable) {
            const uint64_t tsize = 1ull << plan.key_bits;
            if (tmin.n < tsize) {
                tmin.alloc(tsize, s);
                tcnt.alloc(tsize, s);
            }
            if (keys32.n < std::max(1u, m)) keys32.alloc(std::max(1u, hi - lo), s);
            shard_table_signature(ctx, d, keylab, plan, lst, lo, m, keys32.get(), tmin.get(), tcnt.get(), s);
            cm->allreduce_u32(tmin.get(), tsize, true, s);
            cm->allreduce_u32(tcnt.get(), tsize, false, s);
            if (hi > lo) DK_CUDA(cudaMemsetAsync(ACT + lo, 0, hi - lo, s));
            if (m_total == n) {
                // every block of the next partition is one table key
                if (plan.key_bits <= 16) {
                    if (!next16.get()) next16.alloc((uint64_t)world * shard, s);
                    next_kl = next16.get();
                } else {
                    if (!next32.get()) next32.alloc((uint64_t)world * shard, s);
                    next_kl = next32.get();
                }
            }
            shard_table_apply(ctx, plan, lst, lo, keys32.get(), m, tmin.get(), tcnt.get(), LAB, ACT,
                              next_kl, dctr.get(), s);
            // only this rank's slice of `lab` was written (after a lazy
            // shard_init the other slices were never initialised): a fixed
            // point reached here must still exchange them before numbering
            lab_stale = true;
            cm->allreduce_u32(dctr.get(), 4, false, s);
            read_u32(dctr.get(), 4, ctr);
        } else if (owner_layout) {
            // wide pass, owner-bucket layout: the signature kernel fills
            // (owner, bucket) sub-buckets that travel as they are
            const OwnerPlan op = owner_plan(m_total, (uint32_t)world);
            const uint64_t msgw = op.nb + 1, region = (uint64_t)op.nb * op.cs;
            // carried 16-bit ranks below 4096 over a large automaton: the
            // signature gathers them packed 12 bits apiece (fewer label bytes
            // in the L2; the verification keeps the 16-bit array)
            const void* sig_keylab = keylab;
            PassPlan sig_plan = plan;
            // (identity ranges only: the packed layouts' sliced sweeps take no state list)
            const int pack = plan.keylab_bytes == 2 && keylab != LAB && k <= 16 && lst == nullptr
                                 ? pack_choice(n, B <= 2048 ? 11u : B <= 4096 ? 12u : 16u)
                                 : 0;
            if (pack) {
                if (pack12.n < pack_words(n)) pack12.alloc(pack_words(n), s);
                sig_plan.keylab_bytes =
                    pack12_labels(ctx, static_cast<const uint16_t*>(keylab), n, pack12.get(), s, pack == 11);
                sig_keylab = pack12.get();
            }
            uint4* const precv = peer_mode ? static_cast<uint4*>(cm->peer.local[0]) : nullptr;
            uint32_t* const pcnt = peer_mode ? static_cast<uint32_t*>(cm->peer.local[1]) : nullptr;
            if (peer_mode) {
                // this rank's region of every owner's receive buffer
                OwnerDst dst{};
                dst.peer = world > 1;
                for (int o = 0; o < world; ++o) {
                    dst.entries[o] = static_cast<uint4*>(cm->peer.peer[o][0]) + (uint64_t)rank * region;
                    dst.counts[o] = static_cast<uint32_t*>(cm->peer.peer[o][1]) + (uint64_t)rank * msgw;
                }
                shard_sig_owner(ctx, d, sig_keylab, sig_plan, salt, lst, lo, m, op, ows, s, &dst);
                cm->barrier(s);  // every sender's entries and counts have landed
            } else {
                shard_sig_owner(ctx, d, sig_keylab, sig_plan, salt, lst, lo, m, op, ows, s);
                if (rmsg.n < world * msgw) rmsg.alloc(world * msgw, s);
                const std::vector<uint64_t> mcount(world, msgw);
                cm->all_to_all_v(ows.msg.get(), mcount, rmsg.get(), mcount, sizeof(uint32_t), s);
            }
            const uint32_t* const rcnt_all = peer_mode ? pcnt : rmsg.get();
            // overflow counts: received per sender, own per owner, own total
            shard_owner_ovf_counts(ctx, op, rcnt_all, small.get(), s);
            DK_CUDA(cudaMemcpyAsync(small.get() + world, ows.ovf_cnt.get(), (world + 1) * sizeof(uint32_t),
                                    cudaMemcpyDeviceToDevice, s));
            std::vector<uint32_t> w32(2 * (size_t)world + 1);
            read_u32(small.get(), w32.size(), w32.data());
            std::vector<uint64_t> rovf(world), sovf(world);
            uint64_t rovf_total = 0;
            for (int r = 0; r < world; ++r) {
                rovf_total += (rovf[r] = w32[r]);
                sovf[r] = w32[world + r];
            }
            const uint32_t own_ovf = w32[2 * world];
            shard_sort_overflow(ctx, op, ows, own_ovf, s);
            // regions: every peer's region of this rank's send buffer; its own stays put
            std::vector<uint64_t> soff(world), scnt(world), roff(world), rcnt(world);
            for (int r = 0; r < world; ++r) {
                soff[r] = (uint64_t)r * region;
                scnt[r] = rcnt[r] = r == rank ? 0 : region;
                roff[r] = r == rank ? 0 : (uint64_t)(r - (r > rank)) * region;
            }
            const uint64_t peers_slots = peer_mode ? 0 : (uint64_t)(world - 1) * region;
            if (peers_slots && rreg.n < peers_slots) rreg.alloc(peers_slots, s);
            if (peers_slots) cm->all_to_all_off(ows.send.get(), soff, scnt, rreg.get(), roff, rcnt, sizeof(uint4), s);
            if (rovf_buf.n < std::max<uint64_t>(1, rovf_total)) rovf_buf.alloc(std::max<uint64_t>(1, rovf_total), s);
            cm->all_to_all_v(ows.ovf_sorted.get(), sovf, rovf_buf.get(), rovf, sizeof(uint4), s);
            sent += m;
            OwnerSources in{};
            for (int r = 0; r < world; ++r) {
                in.base[r] = peer_mode ? precv + (uint64_t)r * region
                                       : (r == rank ? ows.send.get() + (uint64_t)rank * region : rreg.get() + roff[r]);
                in.cnt[r] = rcnt_all + (uint64_t)r * msgw;
            }
            const uint64_t rslots = (uint64_t)world * region + rovf_total;
            if (results.n < rslots) results.alloc(rslots, s);
            // peer mode: buckets of distinct keys write no results (the owner's
            // scatter takes their states from the entries)
            if (peer_mode && bsingle.n < op.nb) bsingle.alloc(op.nb, s);
            uint8_t* const bs = peer_mode ? bsingle.get() : nullptr;
            if (lab_stale)
                shard_group_owner(ctx, d, keylab, plan.keylab_bytes ? plan.keylab_bytes : 4, plan, op, in,
                                  rovf_buf.get(), (uint32_t)rovf_total, results.get(), dctr.get(), s, bs);
            else
                shard_group_owner(ctx, d, LAB, 4, plan, op, in, rovf_buf.get(), (uint32_t)rovf_total,
                                  results.get(), dctr.get(), s, bs);
            // peer mode: the owners will write this rank's flags; zeroed before
            // the counter exchange, which every owner passes before writing
            if (peer_mode && hi > lo) DK_CUDA(cudaMemsetAsync(ACT + lo, 0, hi - lo, s));
            cm->allreduce_u32(dctr.get(), 4, false, s);
            read_u32(dctr.get(), 4, ctr);
            if (ctr[3]) {
                ++res.collisions;
                --res.passes;
                if (++strikes > 16) throw Error(DFAKIT_E_RESOURCE, "sharded sort_pr: repeated fingerprint collisions");
                salt = mix64_host(salt + 0x1234567ull);
                continue;
            }
            if (B - A + ctr[0] == B) break;  // fixed point (reference l.411)
            if (B - A + ctr[0] == n) {       // all singletons: nothing travels back
                ++res.iters;
                B = n;
                break;
            }
            if (peer_mode) {
                // owners: region results straight into the senders' labels and
                // flags; the overflow results travel back as before
                PeerLabels pl{};
                for (int r = 0; r < world; ++r) {
                    pl.lab[r] = static_cast<uint32_t*>(cm->peer.peer[r][2]);
                    pl.act[r] = static_cast<uint8_t*>(cm->peer.peer[r][3]);
                }
                shard_owner_scatter(ctx, op, precv, pcnt, results.get(), bs, pl, s);
                if (back_ovf.n < std::max<uint32_t>(1, own_ovf)) back_ovf.alloc(std::max<uint32_t>(1, own_ovf), s);
                cm->all_to_all_v(results.get() + (uint64_t)world * region, rovf, back_ovf.get(), sovf,
                                 sizeof(uint32_t), s);
                shard_apply_overflow(ctx, ows, back_ovf.get(), own_ovf, LAB, ACT, s);
                cm->barrier(s);  // every owner's label writes into this rank have landed
                goto pass_done;
            }
            // results back: each sender's padded part of every region, then the overflow results
            if (peers_slots && back.n < peers_slots) back.alloc(peers_slots, s);
            if (peers_slots)
                cm->all_to_all_off(results.get(), soff, scnt, back.get(), roff, rcnt, sizeof(uint32_t), s);
            if (back_ovf.n < std::max<uint32_t>(1, own_ovf)) back_ovf.alloc(std::max<uint32_t>(1, own_ovf), s);
            cm->all_to_all_v(results.get() + (uint64_t)world * region, rovf, back_ovf.get(), sovf, sizeof(uint32_t),
                             s);
            if (hi > lo) DK_CUDA(cudaMemsetAsync(ACT + lo, 0, hi - lo, s));
            shard_apply_owner(ctx, op, ows, (uint32_t)rank, results.get() + (uint64_t)rank * region, back.get(),
                              back_ovf.get(), own_ovf, LAB, ACT, s);
        } else {
            if (send.n < std::max(1u, m)) send.alloc(std::max(1u, hi - lo), s);
            shard_sig_partition(ctx, d, keylab, plan, salt, lst, lo, m, (uint32_t)world, send.get(), counts.get(), s);
            // counts: one word to every peer, then both vectors in one readback
            std::vector<uint32_t> c32(2 * (size_t)world);
            std::vector<uint64_t> scount(world), rcount(world), ones(world, 1);
            cm->all_to_all_v(counts.get(), ones, counts.get() + world, ones, sizeof(uint32_t), s);
            read_u32(counts.get(), 2 * (size_t)world, c32.data());
            const uint32_t* sc32 = c32.data();
            const uint32_t* rc32 = c32.data() + world;
            for (int r = 0; r < world; ++r) scount[r] = sc32[r];
            uint64_t rtotal = 0;
            for (int r = 0; r < world; ++r) rtotal += (rcount[r] = rc32[r]);
            if (recv.n < std::max<uint64_t>(1, rtotal)) recv.alloc(std::max<uint64_t>(1, rtotal) * 5 / 4, s);
            cm->all_to_all_v(send.get(), scount, recv.get(), rcount, sizeof(uint4), s);
            sent += m;
            if (results.n < std::max<uint64_t>(1, rtotal)) results.alloc(std::max<uint64_t>(1, rtotal) * 5 / 4, s);
            // verification compares any injective labelling: the key labels when
            // the min-state labels of other ranks are stale
            if (lab_stale)
                shard_group_deferred(ctx, d, keylab, plan.keylab_bytes ? plan.keylab_bytes : 4, plan, recv.get(),
                                     rtotal, gws, dctr.get(), s);
            else
                shard_group_deferred(ctx, d, LAB, 4, plan, recv.get(), rtotal, gws, dctr.get(), s);
            cm->allreduce_u32(dctr.get(), 4, false, s);
            read_u32(dctr.get(), 4, ctr);
            if (ctr[3]) {
                // verified fingerprint collision on some owner: nothing applied
                ++res.collisions;
                --res.passes;
                if (++strikes > 16) throw Error(DFAKIT_E_RESOURCE, "sharded sort_pr: repeated fingerprint collisions");
                salt = mix64_host(salt + 0x1234567ull);
                continue;
            }
            if (B - A + ctr[0] == B) break;  // fixed point (reference l.411)
            if (B - A + ctr[0] == n) {
                // every block a singleton (the usual last pass): the numbering
                // is the identity, so the results need not travel back nor
                // become labels (a random 4-byte store per state)
                ++res.iters;
                B = n;
                break;
            }
            shard_group_results(ctx, gws, results.get(), s);
            if (back.n < std::max(1u, m)) back.alloc(std::max(1u, hi - lo), s);
            cm->all_to_all_v(results.get(), rcount, back.get(), scount, sizeof(uint32_t), s);
            if (hi > lo) DK_CUDA(cudaMemsetAsync(ACT + lo, 0, hi - lo, s));
            shard_apply(ctx, send.get(), back.get(), m, LAB, ACT, s);
        }
    pass_done:
        strikes = 0;
        const uint32_t newB = B - A + ctr[0];
        if (newB == B) break;  // fixed point
        ++res.iters;
        B = newB;
        A = ctr[1];
        m_total = ctr[2];
        // label exchange: the carried key labels when the next pass gathers
        // them (the min-state labels follow only when a pass or the final
        // numbering needs them), else the min-state labels
        if (next_kl) {
            const size_t es = plan.key_bits <= 16 ? 2 : 4;
            cm->allgather(next_kl, (size_t)shard * es, s);
            carried = next_kl;
            carried_bytes = (uint32_t)es;
            lab_stale = true;
        } else if (B < n) {
            cm->allgather(LAB, (size_t)shard * sizeof(uint32_t), s);
            lab_stale = false;
        } else {
            lab_stale = true;  // all singletons: the numbering needs no labels
        }
        if (m_total == n) m = hi - lo;  // every state survives: the identity range, no compaction
        else if (m_total) compact();     // (none left: the loop ends, nothing to compact)
    }
    // an all-singleton partition is numbered by identity (no label exchange)
    if (lab_stale && B < n) cm->allgather(LAB, (size_t)shard * sizeof(uint32_t), s);
    res.num_blocks = canonical_from_min_labels(ctx, LAB, n, block_out, scratch.get(), s, B);
    if (exchanged) *exchanged = sent;
    return res;
}

}  // namespace dk
