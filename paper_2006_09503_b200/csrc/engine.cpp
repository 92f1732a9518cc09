// Stage executor: interprets the per-stage op programs on CUDA streams.
//
// Mirrors reference pipelined_execute (core/src/semantics.cpp:238-375):
//   - the same round-robin "run each stage until blocked" issue order (:270-361),
//     except that "blocked" means "the producing op has not been *issued* yet":
//     ordering on the GPU is carried by CUDA events, so the host never waits;
//   - the same version bookkeeping (versions map, prune rules :213-234, the
//     "needs discarded weight version" check :282-287, max_versions_held);
//   - the same deadlock detection and error text (:360).
// Buffers: every stage owns a receive ring for its input activations (which is
// also the stash of its first-layer input) and one for its output gradient.
// The producing stage's last kernel writes straight into those slots, so a
// stage hand-off is a peer store over NVLink when stages sit on different GPUs
// of this process.  Stages in another process (one process per GPU) are reached
// through CUDA IPC: the producer writes a local staging slot, a copy stream moves
// it into the consumer's ring and bumps a sequence flag in the consumer's block;
// slot reuse is gated by the consumer's backward progress, pushed back the same
// way (transport.cu).
#include "engine.h"

#include <algorithm>
#include <cstring>
#include <nlohmann/json.hpp>

#include "nccl_dl.h"
#include "pipesim/schedule.hpp"
#include "profiler.h"
#include "transport.h"

namespace p2bw {

namespace {

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        check_cuda(cudaGetDevice(&prev), "cudaGetDevice");
        if (prev != dev) check_cuda(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

int weight_slots_for(int policy, int depth) {
    switch (policy) {
        case P2BW_POLICY_2BW: return 2;          // exactly two versions (paper §3.1)
        case P2BW_POLICY_1F1B: return depth + 1; // weight stashing worst case + the new one
        default: return 1;                       // flush policies update in place
    }
}

}  // namespace

Engine::Engine(const EngineConfig& cfg) : cfg_(cfg) {
    if (cfg_.depth < 1) throw Error("depth must be >= 1");
    if (cfg_.layers < 1) throw Error("layer count must be >= 1");
    if (cfg_.stage_layers.empty()) {
        if (cfg_.layers % cfg_.depth != 0)
            throw Error("block count " + std::to_string(cfg_.layers) + " not divisible by depth " +
                        std::to_string(cfg_.depth));
    } else {
        int sum = 0;
        for (int n : cfg_.stage_layers) {
            if (n < 1) throw Error("every stage needs at least one layer");
            sum += n;
        }
        if (static_cast<int>(cfg_.stage_layers.size()) != cfg_.depth || sum != cfg_.layers)
            throw Error("stage_layers must hold depth entries summing to the layer count");
    }
    if (cfg_.microbatches < 1) throw Error("m must be >= 1");
    if (cfg_.policy == P2BW_POLICY_2BW && cfg_.microbatches < cfg_.depth)
        throw Error("2bw requires m >= d (m=" + std::to_string(cfg_.microbatches) +
                    ", d=" + std::to_string(cfg_.depth) + ")");
    if (cfg_.devices.empty()) {
        int dev = 0;
        check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
        cfg_.devices.assign(static_cast<size_t>(cfg_.depth), dev);
    }
    if (static_cast<int>(cfg_.devices.size()) != cfg_.depth)
        throw Error("device list must have one entry per stage");
    if (cfg_.local_count < 0 || cfg_.first_local < 0 || cfg_.first_local + cfg_.local_count > cfg_.depth)
        throw Error("local stage range [" + std::to_string(cfg_.first_local) + ", " +
                    std::to_string(cfg_.first_local + cfg_.local_count) + ") outside the pipeline");
    const int lo_local = cfg_.local_count == 0 ? 0 : cfg_.first_local;
    const int hi_local = cfg_.local_count == 0 ? cfg_.depth : cfg_.first_local + cfg_.local_count;

    // Peer access between devices of adjacent local stages (NVLink / NVSwitch).
    for (int s = lo_local; s + 1 < hi_local; ++s) {
        const int a = cfg_.devices[s], b = cfg_.devices[s + 1];
        if (a == b) continue;
        for (auto [x, y] : {std::pair{a, b}, std::pair{b, a}}) {
            DeviceGuard g(x);
            int can = 0;
            check_cuda(cudaDeviceCanAccessPeer(&can, x, y), "cudaDeviceCanAccessPeer");
            if (!can) throw Error("no peer access between GPU " + std::to_string(x) + " and " +
                                  std::to_string(y));
            const cudaError_t e = cudaDeviceEnablePeerAccess(y, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                check_cuda(e, "cudaDeviceEnablePeerAccess");
            cudaGetLastError();
        }
    }

    // Ring sizes come from the policy's programs: the peak in-flight count of a
    // stage bounds its stash; one extra input slot lets the upstream stage run
    // its next forward without waiting for this stage's oldest backward.
    const int per = cfg_.layers / cfg_.depth;
    stages_.resize(static_cast<size_t>(cfg_.depth));
    // Forward of microbatch k+1 overlaps the Backward of k on its own stream
    // (transformer stages; recomputation re-runs forwards inside the Backward into a
    // single shared slot, so it keeps one stream).  P2BW_SERIAL_STAGE=1 turns it off.
    // A function of the configuration only: every process derives the same ring sizes.
    const char* serial = std::getenv("P2BW_SERIAL_STAGE");
    const bool overlap =
        cfg_.model_kind != P2BW_MODEL_LINEAR_F64 && !cfg_.recompute && !(serial && serial[0] == '1');
    try {
        for (int s = 0; s < cfg_.depth; ++s) {
            Stage& st = stages_[s];
            st.index = s;
            st.device = cfg_.devices[s];
            if (cfg_.stage_layers.empty()) {
                st.lo = s * per;
                st.hi = st.lo + per;
            } else {
                st.lo = s == 0 ? 0 : stages_[static_cast<size_t>(s) - 1].hi;
                st.hi = st.lo + cfg_.stage_layers[static_cast<size_t>(s)];
            }
            const int warm = std::min(cfg_.depth - s, cfg_.microbatches);
            int inflight;
            switch (cfg_.policy) {
                case P2BW_POLICY_GPIPE: inflight = cfg_.microbatches; break;
                case P2BW_POLICY_NONE: inflight = 1; break;
                default: inflight = std::max(warm, 1); break;
            }
            st.stash_slots = inflight + (s > 0 ? 1 : 0);
            // one more slot lets Forward k+1 (own stream) run while Backward k holds its slot
            if (overlap) st.stash_slots = std::max(st.stash_slots, 2 + (s > 0 ? 1 : 0));
            st.grad_slots = st.stash_slots;
            st.weight_slots = weight_slots_for(cfg_.policy, cfg_.depth);
            st.local = s >= lo_local && s < hi_local;
            if (!st.local) continue;  // another process runs it; connect_stage maps its block
            DeviceGuard g(st.device);
            st.stream = make_stage_stream("main");
            if (overlap) {
                st.fstream = make_stage_stream("fwd");
                st.dstream = make_stage_stream("data");
                // 2BW: AllReduce + WeightUpdate of batch t on their own stream, overlapping the
                // Backwards of batch t+1 (which accumulate into the other gradient buffer)
                if (cfg_.policy == P2BW_POLICY_2BW)
                    st.ustream = make_stage_stream("update");
            }
            check_cuda(cudaEventCreate(&st.t0), "cudaEventCreate");
            check_cuda(cudaEventCreate(&st.t1), "cudaEventCreate");
            if (cfg_.model_kind == P2BW_MODEL_LINEAR_F64) {
                st.model = make_linear_f64_stage(cfg_, s, st.lo, st.hi, st.stash_slots,
                                                 st.weight_slots);
            } else if (cfg_.model_kind == P2BW_MODEL_LINEAR_BF16) {
                st.model = make_linear_bf16_stage(cfg_, s, st.lo, st.hi, st.stash_slots,
                                                  st.weight_slots);
            } else if (cfg_.model_kind == P2BW_MODEL_TRANSFORMER) {
                st.model = make_transformer_stage(cfg_, s, st.lo, st.hi, st.stash_slots,
                                                  st.weight_slots);
            } else {
                throw Error("unknown model kind " + std::to_string(cfg_.model_kind));
            }
            st.model->bind_stream(st.stream);
            if (st.dstream) st.model->bind_data_stream(st.dstream);
            if (st.ustream && !st.model->enable_grad_double_buffer()) {
                cudaStreamDestroy(st.ustream);
                st.ustream = nullptr;
            }
            // Receive block: [act ring][grad ring][flags], one allocation so that a
            // single IPC handle exports it.
            const size_t nb = st.model->boundary_bytes();
            auto al = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
            const size_t act_b = s > 0 ? al(nb * st.stash_slots) : 0;
            const size_t grad_b = s + 1 < cfg_.depth ? al(nb * st.grad_slots) : 0;
            check_cuda(cudaMalloc(&st.block, act_b + grad_b + 256), "cudaMalloc(receive block)");
            uint8_t* base = static_cast<uint8_t*>(st.block);
            if (s > 0)
                for (int i = 0; i < st.stash_slots; ++i) st.act_ring.push_back(base + i * nb);
            if (s + 1 < cfg_.depth)
                for (int i = 0; i < st.grad_slots; ++i) st.grad_ring.push_back(base + act_b + i * nb);
            st.flags = reinterpret_cast<uint32_t*>(base + act_b + grad_b);
            check_cuda(cudaMemset(st.flags, 0, 256), "cudaMemset(flags)");
            st.version_slot[0] = 0;
        }
        // Staging slots and copy streams towards neighbours in other processes.
        for (int s = lo_local; s < hi_local; ++s) {
            Stage& st = stages_[s];
            DeviceGuard g(st.device);
            const size_t nb = st.model->boundary_bytes();
            if (s + 1 < cfg_.depth && !stages_[s + 1].local) {
                for (auto& p : st.send_act) check_cuda(cudaMalloc(&p, nb), "cudaMalloc(send slot)");
                check_cuda(cudaStreamCreateWithFlags(&st.copy_fwd, cudaStreamNonBlocking), "cudaStreamCreate");
            }
            if (s > 0 && !stages_[s - 1].local) {
                for (auto& p : st.send_grad) check_cuda(cudaMalloc(&p, nb), "cudaMalloc(send slot)");
                check_cuda(cudaStreamCreateWithFlags(&st.copy_bwd, cudaStreamNonBlocking), "cudaStreamCreate");
            }
        }
        check_cuda(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    } catch (...) {
        free_buffers();
        throw;
    }
}

Engine::~Engine() { free_buffers(); }

void Engine::join_replicas(const void* ids, int nranks, int rank) {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw Error("bad data-parallel rank / size");
    for (Stage& st : stages_) {
        if (!st.local) continue;
        if (st.comm) throw Error("stage already joined a replica group");
        // a single replica needs no communicator (AllReduce is then a no-op);
        // P2BW_NCCL_SINGLE_RANK=1 builds one anyway so one-GPU tests run the NCCL path
        if (nranks == 1 && std::getenv("P2BW_NCCL_SINGLE_RANK") == nullptr) continue;
        ncclUniqueId id;
        std::memcpy(&id, static_cast<const uint8_t*>(ids) + sizeof(ncclUniqueId) * st.index, sizeof(id));
        DeviceGuard g(st.device);
        st.comm = nccl_comm_init(id, nranks, rank);
        st.replicas = nranks;
    }
}

Engine::Stage& Engine::local_stage(int s) {
    if (s < 0 || s >= cfg_.depth) throw Error("stage " + std::to_string(s) + " out of range");
    Stage& st = stages_[static_cast<size_t>(s)];
    if (!st.local) throw Error("stage " + std::to_string(s) + " runs in another process");
    return st;
}

StageBlob Engine::export_stage(int s) {
    Stage& st = local_stage(s);
    StageBlob b{};
    cudaIpcMemHandle_t h;
    DeviceGuard g(st.device);
    check_cuda(cudaIpcGetMemHandle(&h, st.block), "cudaIpcGetMemHandle");
    static_assert(sizeof(h) == sizeof(b.ipc), "IPC handle size");
    std::memcpy(b.ipc, &h, sizeof(h));
    b.stage = s;
    b.stash_slots = st.stash_slots;
    b.grad_slots = st.grad_slots;
    b.slot_bytes = st.model->boundary_bytes();
    const uint8_t* base = static_cast<const uint8_t*>(st.block);
    b.act_off = st.act_ring.empty() ? 0 : static_cast<const uint8_t*>(st.act_ring[0]) - base;
    b.grad_off = st.grad_ring.empty() ? 0 : static_cast<const uint8_t*>(st.grad_ring[0]) - base;
    b.flag_off = reinterpret_cast<const uint8_t*>(st.flags) - base;
    return b;
}

void Engine::connect_stage(const StageBlob& b) {
    const int s = b.stage;
    if (s < 0 || s >= cfg_.depth) throw Error("connect: stage " + std::to_string(s) + " out of range");
    Stage& st = stages_[static_cast<size_t>(s)];
    if (st.local) throw Error("connect: stage " + std::to_string(s) + " runs in this process");
    if (st.connected) throw Error("connect: stage " + std::to_string(s) + " is already connected");
    const bool left = s + 1 < cfg_.depth && stages_[s + 1].local, right = s > 0 && stages_[s - 1].local;
    if (!left && !right) throw Error("connect: stage " + std::to_string(s) + " is not adjacent to a local stage");
    if (b.stash_slots != st.stash_slots || b.grad_slots != st.grad_slots)
        throw Error("connect: stage " + std::to_string(s) + " ring sizes differ between processes");
    Stage& nb = stages_[static_cast<size_t>(left ? s + 1 : s - 1)];
    if (b.slot_bytes != nb.model->boundary_bytes())
        throw Error("connect: boundary tensor size differs between processes");
    DeviceGuard g(nb.device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, b.ipc, sizeof(h));
    check_cuda(cudaIpcOpenMemHandle(&st.block, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    st.block_mapped = true;
    uint8_t* base = static_cast<uint8_t*>(st.block);
    st.act_ring.clear();
    st.grad_ring.clear();
    if (s > 0)
        for (int i = 0; i < st.stash_slots; ++i) st.act_ring.push_back(base + b.act_off + i * b.slot_bytes);
    if (s + 1 < cfg_.depth)
        for (int i = 0; i < st.grad_slots; ++i) st.grad_ring.push_back(base + b.grad_off + i * b.slot_bytes);
    st.flags = reinterpret_cast<uint32_t*>(base + b.flag_off);
    st.connected = true;
}

ReplicaBlob Engine::export_replica(int s) {
    Stage& st = local_stage(s);
    DeviceGuard g(st.device);
    ReplicaBlob b{};
    static_assert(sizeof(cudaIpcMemHandle_t) == sizeof(b.block_ipc), "IPC handle size");
    b.magic = kReplicaBlobMagic;
    b.stage = s;
    b.weight_slots = st.weight_slots;
    b.weight_bytes = st.model->weight_bytes_public();
    cudaIpcMemHandle_t h;
    check_cuda(cudaIpcGetMemHandle(&h, st.block), "cudaIpcGetMemHandle(block)");
    std::memcpy(b.block_ipc, &h, sizeof(h));
    b.flag_off = static_cast<uint64_t>(reinterpret_cast<const uint8_t*>(st.flags) -
                                       static_cast<const uint8_t*>(st.block));
    const std::vector<void*> bufs = st.model->replica_buffers();
    if (bufs.empty()) throw Error("this stage model cannot join a peer-memory replica group");
    if (bufs.size() > static_cast<size_t>(kMaxReplicaBufs)) throw Error("too many replica buffers");
    b.nbuf = static_cast<int>(bufs.size());
    for (size_t i = 0; i < bufs.size(); ++i) {
        if (!bufs[i]) continue;
        size_t off = 0;
        void* base = allocation_base(bufs[i], &off);
        check_cuda(cudaIpcGetMemHandle(&h, base), "cudaIpcGetMemHandle(replica buffer)");
        std::memcpy(b.buf_ipc[i], &h, sizeof(h));
        b.buf_off[i] = off;
        b.buf_present[i] = 1;
    }
    return b;
}

void Engine::join_replicas_ipc(int s, const std::vector<ReplicaBlob>& blobs, int rank) {
    Stage& st = local_stage(s);
    const int w = static_cast<int>(blobs.size());
    if (w < 1 || w > kMaxReplicas || rank < 0 || rank >= w) throw Error("bad data-parallel rank / size");
    if (st.comm || st.ipc_group) throw Error("stage already joined a replica group");
    if (w == 1) return;  // AllReduce is a no-op (semantics.cpp:351-354)
    DeviceGuard g(st.device);
    const std::vector<void*> mine = st.model->replica_buffers();
    std::map<std::string, void*> opened;  // one mapping per exported allocation
    auto open = [&](const char* ipc) -> void* {
        const std::string key(ipc, 64);
        auto it = opened.find(key);
        if (it != opened.end()) return it->second;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, ipc, sizeof(h));
        void* p = nullptr;
        check_cuda(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle(replica)");
        st.ipc_opened.push_back(p);
        opened[key] = p;
        return p;
    };
    st.peer_bufs.assign(static_cast<size_t>(w), {});
    st.peer_flags.assign(static_cast<size_t>(w), nullptr);
    for (int q = 0; q < w; ++q) {
        const ReplicaBlob& b = blobs[static_cast<size_t>(q)];
        if (b.magic != kReplicaBlobMagic || b.stage != s)
            throw Error("replica blob " + std::to_string(q) + " is not stage " + std::to_string(s) + "'s");
        if (b.weight_bytes != st.model->weight_bytes_public() || b.weight_slots != st.weight_slots ||
            b.nbuf != static_cast<int>(mine.size()))
            throw Error("replica " + std::to_string(q) + " of stage " + std::to_string(s) + " has a different shape");
        if (q == rank) {
            st.peer_bufs[static_cast<size_t>(q)] = mine;
            continue;
        }
        std::vector<void*> v(static_cast<size_t>(b.nbuf), nullptr);
        for (int i = 0; i < b.nbuf; ++i)
            if (b.buf_present[i]) v[static_cast<size_t>(i)] = static_cast<uint8_t*>(open(b.buf_ipc[i])) + b.buf_off[i];
        st.peer_bufs[static_cast<size_t>(q)] = std::move(v);
        st.peer_flags[static_cast<size_t>(q)] =
            reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(open(b.block_ipc)) + b.flag_off);
    }
    st.ipc_group = true;
    st.replica_rank = rank;
    st.replicas = w;
}

// WeightUpdate of a peer-memory replica group, on the update stream `us`:
//   1. tell every peer this replica's gradient is complete (and its in-flight Forwards no
//      longer read the destination slot the peers are about to write);
//   2. wait until every peer said the same;
//   3. the fused reduce-scatter + optimizer + all-gather kernel (this replica's shard);
//   4. tell every peer, wait for every peer: all shards of the new version have landed
//      here and nobody reads this replica's gradient buffer any more.
// Flags are sequence numbers in each replica's own block (peers write them, the owner
// waits with a stream memory op: no SM spins).
void Engine::issue_update_replicas(Stage& st, int src_slot, int dst_slot, cudaStream_t us) {
    const int w = st.replicas, r = st.replica_rank;
    const uint32_t n = ++st.ar_seq;
    std::vector<uint32_t*> ready, done;
    for (int q = 0; q < w; ++q)
        if (q != r) {
            ready.push_back(st.peer_flags[static_cast<size_t>(q)] + kReplicaReady + r);
            done.push_back(st.peer_flags[static_cast<size_t>(q)] + kReplicaDone + r);
        }
    stream_signal_many(ready.data(), static_cast<int>(ready.size()), n, us);
    for (int q = 0; q < w; ++q)
        if (q != r) stream_wait_geq(st.flags + kReplicaReady + q, n, us);
    st.model->update_replicas(src_slot, dst_slot, st.grad_count * w, st.peer_bufs, r, us);
    stream_signal_many(done.data(), static_cast<int>(done.size()), n, us);
    for (int q = 0; q < w; ++q)
        if (q != r) stream_wait_geq(st.flags + kReplicaDone + q, n, us);
}

void Engine::signal_remote(uint32_t* flag, uint32_t value, cudaStream_t s) { stream_signal(flag, value, s); }

void Engine::wait_flag(const uint32_t* flag, uint32_t value, cudaStream_t s) {
    if (value != 0) stream_wait_geq(flag, value, s);
}

void Engine::free_buffers() {
    for (TraceRec& r : trace_) cudaEventDestroy(r.e0), cudaEventDestroy(r.e1);
    trace_.clear();
    for (Stage& st : stages_) {
        if (!st.local) {
            if (st.block_mapped) cudaIpcCloseMemHandle(st.block);
            st.block = nullptr;
            st.block_mapped = false;
            continue;
        }
        DeviceGuard g(st.device);
        if (st.stream) cudaStreamSynchronize(st.stream);
        if (st.copy_fwd) cudaStreamSynchronize(st.copy_fwd);
        if (st.copy_bwd) cudaStreamSynchronize(st.copy_bwd);
        if (st.block) cudaFree(st.block);
        st.block = nullptr;
        for (void*& p : st.send_act) cudaFree(p), p = nullptr;
        for (void*& p : st.send_grad) cudaFree(p), p = nullptr;
        if (st.copy_fwd) cudaStreamDestroy(st.copy_fwd);
        if (st.copy_bwd) cudaStreamDestroy(st.copy_bwd);
        st.copy_fwd = st.copy_bwd = nullptr;
        st.act_ring.clear();
        st.grad_ring.clear();
        st.model.reset();
        if (st.comm) nccl_comm_destroy(static_cast<ncclComm_t>(st.comm));
        st.comm = nullptr;
        if (st.ustream) cudaStreamSynchronize(st.ustream);
        for (void* p : st.ipc_opened) cudaIpcCloseMemHandle(p);
        st.ipc_opened.clear();
        st.peer_bufs.clear();
        st.peer_flags.clear();
        st.ipc_group = false;
        if (st.fstream) cudaStreamSynchronize(st.fstream), cudaStreamDestroy(st.fstream);
        st.fstream = nullptr;
        if (st.dstream) cudaStreamSynchronize(st.dstream), cudaStreamDestroy(st.dstream);
        st.dstream = nullptr;
        if (st.ustream) cudaStreamSynchronize(st.ustream), cudaStreamDestroy(st.ustream);
        st.ustream = nullptr;
        if (st.t0) cudaEventDestroy(st.t0);
        if (st.t1) cudaEventDestroy(st.t1);
        if (st.stream) cudaStreamDestroy(st.stream);
        st.stream = nullptr;
        st.t0 = st.t1 = nullptr;
    }
}

// Per-run event tables: one event per (stage, microbatch, pass), created lazily
// when the op is issued, plus a timing event after every WeightUpdate.
// Destroying an event with pending waits is legal.
struct EventTable {
    std::vector<std::map<int, cudaEvent_t>> fwd, bwd;
    std::vector<std::map<int, cudaEvent_t>> cpf, cpb;  // sends to remote neighbours done
    std::vector<std::vector<cudaEvent_t>> upd;
    std::vector<std::map<int, cudaEvent_t>> data;  // data-ring copy of microbatch k done
    explicit EventTable(size_t d) : fwd(d), bwd(d), cpf(d), cpb(d), upd(d), data(d) {}
    ~EventTable() {
        for (auto* t : {&fwd, &bwd, &cpf, &cpb, &data})
            for (auto& m : *t)
                for (auto& kv : m) cudaEventDestroy(kv.second);
        for (auto& v : upd)
            for (cudaEvent_t e : v) cudaEventDestroy(e);
    }
};

void Engine::EventTableDeleter::operator()(EventTable* t) const { delete t; }

namespace {

cudaEvent_t record(std::map<int, cudaEvent_t>& tab, int k, cudaStream_t s) {
    cudaEvent_t e;
    check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    check_cuda(cudaEventRecord(e, s), "cudaEventRecord");
    tab[k] = e;
    return e;
}

void wait_on(const std::map<int, cudaEvent_t>& tab, int k, cudaStream_t s) {
    const auto it = tab.find(k);
    if (it == tab.end()) throw Error("internal: missing event for microbatch " + std::to_string(k));
    check_cuda(cudaStreamWaitEvent(s, it->second, 0), "cudaStreamWaitEvent");
}

}  // namespace

int Engine::resolve_version(const Stage& st, const OpRec& op) const {
    // Program versions count from the engine's version at begin() (0 on a fresh engine).
    return op.weight_version == P2BW_LATEST_VERSION ? st.updates_done : st.version_base + op.weight_version;
}

bool Engine::ready(const Stage& st, const OpRec& op) const {
    const int s = st.index, d = cfg_.depth, k = op.microbatch;
    auto issued = [](const std::map<int, bool>& m, int key) { return key < 1 || m.count(key); };
    // Neighbours in another process are ordered on the GPU by sequence flags.
    const bool prev_l = s > 0 && stages_[s - 1].local, next_l = s + 1 < d && stages_[s + 1].local;
    if (op.kind == P2BW_OP_FORWARD) {
        if (prev_l && !issued(stages_[s - 1].fwd_issued, k)) return false;  // semantics.cpp:279
        if (!issued(st.bwd_issued, k - st.stash_slots)) return false;       // own stash slot
        if (next_l && !issued(stages_[s + 1].bwd_issued, k - stages_[s + 1].stash_slots))
            return false;  // next stage's receive slot
        return true;
    }
    if (op.kind == P2BW_OP_BACKWARD) {
        if (next_l && !issued(stages_[s + 1].bwd_issued, k)) return false;  // :301
        if (prev_l && !issued(stages_[s - 1].bwd_issued, k - stages_[s - 1].grad_slots))
            return false;  // previous stage's gradient slot
        return true;
    }
    return true;
}

void Engine::issue_forward(Stage& st, const OpRec& op) {
    const int s = st.index, d = cfg_.depth, k = op.microbatch;
    const int v = resolve_version(st, op);
    const auto vit = st.version_slot.find(v);
    if (vit == st.version_slot.end())
        throw Error("stage " + std::to_string(s) + " forward of microbatch " + std::to_string(k) +
                    " needs discarded weight version " + std::to_string(v));
    if (k < 1) throw Error("forward of microbatch " + std::to_string(k));
    const int sslot = (k - 1) % st.stash_slots;
    const bool prev_remote = s > 0 && !stages_[s - 1].local;
    const bool next_remote = s + 1 < d && !stages_[s + 1].local;
    const cudaStream_t fs = op_stream(st, P2BW_OP_FORWARD);
    if (st.fstream && ev_->data[static_cast<size_t>(s)].count(k))  // this microbatch's data copy
        wait_on(ev_->data[static_cast<size_t>(s)], k, fs);
    if (st.fstream) {
        // what the single stream ordered implicitly: the update that produced version
        // v, the backward that last held this stash slot, and this stage's data
        const int u = v - st.version_base;  // 1-based update of this run (<= 0: earlier run)
        if (u >= 1) {
            const auto& ue = ev_->upd[static_cast<size_t>(s)];
            if (u > static_cast<int>(ue.size())) throw Error("internal: forward before its version's update");
            check_cuda(cudaStreamWaitEvent(fs, ue[static_cast<size_t>(u - 1)], 0), "cudaStreamWaitEvent(version)");
        }
        if (k > st.stash_slots) wait_on(ev_->bwd[s], k - st.stash_slots, fs);
    }
    if (prev_remote) wait_flag(&st.flags[kActReady], seq(k), fs);
    else if (s > 0) wait_on(ev_->fwd[s - 1], k, fs);
    void* x_out = nullptr;
    if (next_remote) {  // staging slot, freed by the copy of microbatch k - 2
        if (k > 2) wait_on(ev_->cpf[s], k - 2, fs);
        x_out = st.send_act[(k - 1) % 2];
    } else if (s + 1 < d) {
        const Stage& nx = stages_[s + 1];
        if (k > nx.stash_slots) wait_on(ev_->bwd[s + 1], k - nx.stash_slots, fs);
        x_out = nx.act_ring[(k - 1) % nx.stash_slots];
    }
    const void* x_in = s > 0 ? st.act_ring[sslot] : nullptr;
    if (trace_on_ && trace_open_) check_cuda(cudaEventRecord(trace_open_, fs), "cudaEventRecord(trace)");  // after the waits
    st.model->forward(k, vit->second, sslot, x_in, x_out, fs);
    record(ev_->fwd[s], k, fs);
    st.last_fwd = std::max(st.last_fwd, k);
    if (next_remote) {  // copy into the next process's ring once its slot is free
        const Stage& nx = stages_[s + 1];
        const cudaStream_t c = st.copy_fwd;
        wait_on(ev_->fwd[s], k, c);
        wait_flag(&st.flags[kNextBwd], k > nx.stash_slots ? seq(k - nx.stash_slots) : seq(0), c);
        check_cuda(cudaMemcpyAsync(nx.act_ring[(k - 1) % nx.stash_slots], x_out, st.model->boundary_bytes(),
                                   cudaMemcpyDeviceToDevice, c),
                   "cudaMemcpyAsync(stage send)");
        signal_remote(&nx.flags[kActReady], seq(k), c);
        record(ev_->cpf[s], k, c);
    }
    st.stash_version[k] = v;
    st.fwd_issued[k] = true;
}

void Engine::issue_backward(Stage& st, const OpRec& op) {
    const int s = st.index, d = cfg_.depth, k = op.microbatch;
    const auto sit = st.stash_version.find(k);
    if (sit == st.stash_version.end())
        throw Error("backward before forward for microbatch " + std::to_string(k));  // :304
    const int v = sit->second;
    if (op.weight_version != P2BW_LATEST_VERSION && st.version_base + op.weight_version != v)
        stats_.version_consistent = false;
    const int wslot = st.version_slot.at(v);
    const int sslot = (k - 1) % st.stash_slots;
    const bool prev_remote = s > 0 && !stages_[s - 1].local;
    const bool next_remote = s + 1 < d && !stages_[s + 1].local;
    if (st.fstream) wait_on(ev_->fwd[s], k, st.stream);  // its own Forward (other stream)
    const void* g_in = nullptr;
    if (s + 1 < d) {
        if (next_remote) wait_flag(&st.flags[kGradReady], seq(k), st.stream);
        else wait_on(ev_->bwd[s + 1], k, st.stream);
        g_in = st.grad_ring[(k - 1) % st.grad_slots];
    }
    void* g_out = nullptr;
    if (prev_remote) {
        if (k > 2) wait_on(ev_->cpb[s], k - 2, st.stream);
        g_out = st.send_grad[(k - 1) % 2];
    } else if (s > 0) {
        const Stage& pv = stages_[s - 1];
        if (k > pv.grad_slots) wait_on(ev_->bwd[s - 1], k - pv.grad_slots, st.stream);
        g_out = pv.grad_ring[(k - 1) % pv.grad_slots];
    }
    if (st.ustream && st.grad_count == 0) {
        // first Backward of a batch: its gradient buffer was last read by the AllReduce /
        // WeightUpdate two batches back (update stream)
        const auto& ue = ev_->upd[static_cast<size_t>(s)];
        if (ue.size() >= 2) check_cuda(cudaStreamWaitEvent(st.stream, ue[ue.size() - 2], 0), "cudaStreamWaitEvent(grad)");
    }
    if (trace_on_ && trace_open_) check_cuda(cudaEventRecord(trace_open_, st.stream), "cudaEventRecord(trace)");
    if (cfg_.recompute) {  // Recompute op (simulator.cpp:242-247): the stage input is in its ring slot
        st.model->recompute(k, wslot, sslot, s > 0 ? st.act_ring[sslot] : nullptr, st.stream);
        if (trace_on_) trace_split(st, OpRec{P2BW_OP_RECOMPUTE, k, op.weight_version});
    }
    st.model->backward(k, wslot, sslot, g_in, g_out, st.grad_count == 0, st.stream);
    record(ev_->bwd[s], k, st.stream);
    st.last_bwd = std::max(st.last_bwd, k);
    // Backward k released this stage's act slot and grad slot of microbatch k:
    // tell the remote producers (their flags live in their own blocks).
    if (prev_remote) signal_remote(&stages_[s - 1].flags[kNextBwd], seq(k), st.stream);
    if (next_remote) signal_remote(&stages_[s + 1].flags[kPrevBwd], seq(k), st.stream);
    if (prev_remote) {
        const Stage& pv = stages_[s - 1];
        const cudaStream_t c = st.copy_bwd;
        wait_on(ev_->bwd[s], k, c);
        wait_flag(&st.flags[kPrevBwd], k > pv.grad_slots ? seq(k - pv.grad_slots) : seq(0), c);
        check_cuda(cudaMemcpyAsync(pv.grad_ring[(k - 1) % pv.grad_slots], g_out, st.model->boundary_bytes(),
                                   cudaMemcpyDeviceToDevice, c),
                   "cudaMemcpyAsync(stage send)");
        signal_remote(&pv.flags[kGradReady], seq(k), c);
        record(ev_->cpb[s], k, c);
    }
    st.grad_count += 1;
    st.stash_version.erase(sit);
    st.bwd_issued[k] = true;
}

// semantics.cpp:213-234, applied to a version set.
void Engine::prune_versions(Stage& st) {
    const int latest = st.updates_done;
    auto& vs = st.version_slot;
    if (cfg_.policy == P2BW_POLICY_2BW) {
        vs.erase(latest - 2);
        return;
    }
    if (cfg_.policy == P2BW_POLICY_1F1B) {
        for (auto it = vs.begin(); it != vs.end();) {
            bool referenced = it->first == latest;
            for (const auto& kv : st.stash_version) referenced = referenced || kv.second == it->first;
            it = referenced ? std::next(it) : vs.erase(it);
        }
        return;
    }
    for (auto it = vs.begin(); it != vs.end();) it = it->first == latest ? std::next(it) : vs.erase(it);
}

// WeightUpdate (semantics.cpp:335-350): new version u+1 from the latest u.
void Engine::issue_update(Stage& st) {
    if (st.grad_count == 0) throw Error("weight update with no gradients");
    const int src_version = st.updates_done;
    const int src_slot = st.version_slot.at(src_version);
    // Which versions survive once u+1 exists?  Its buffer may be any slot not
    // holding one of them (the source slot itself when the source is dropped).
    Stage probe_state;  // only the bookkeeping fields are used
    probe_state.updates_done = src_version + 1;
    probe_state.version_slot = st.version_slot;
    probe_state.version_slot[src_version + 1] = -1;
    probe_state.stash_version = st.stash_version;
    prune_versions(probe_state);
    std::vector<bool> used(static_cast<size_t>(st.weight_slots), false);
    for (const auto& kv : probe_state.version_slot)
        if (kv.first != src_version + 1) used[static_cast<size_t>(kv.second)] = true;
    int dst_slot = -1;
    if (!used[static_cast<size_t>(src_slot)] && !probe_state.version_slot.count(src_version))
        dst_slot = src_slot;
    for (int i = 0; i < st.weight_slots && dst_slot < 0; ++i)
        if (!used[static_cast<size_t>(i)]) dst_slot = i;
    if (dst_slot < 0)
        throw Error("stage " + std::to_string(st.index) + ": no free weight buffer for version " +
                    std::to_string(src_version + 1));
    const cudaStream_t us = update_stream(st);  // after this batch's Backwards (update stream)
    // the new version's buffer may be one an in-flight Forward (own stream) still reads
    if (st.fstream && st.last_fwd > 0 && ev_->fwd[static_cast<size_t>(st.index)].count(st.last_fwd))
        wait_on(ev_->fwd[static_cast<size_t>(st.index)], st.last_fwd, us);
    // gradients are summed over grad_count microbatches (and over the replicas by
    // the AllReduce): divide by both (semantics.cpp:338-340; PAPER §3 "w replicas")
    if (st.ipc_group) issue_update_replicas(st, src_slot, dst_slot, us);
    else st.model->update(src_slot, dst_slot, st.grad_count * st.replicas, us);
    st.updates_done += 1;
    st.version_slot[st.updates_done] = dst_slot;
    prune_versions(st);
    st.grad_count = 0;
    st.updates_issued += 1;
    {
        cudaEvent_t e;
        check_cuda(cudaEventCreate(&e), "cudaEventCreate");
        check_cuda(cudaEventRecord(e, us), "cudaEventRecord");
        ev_->upd[static_cast<size_t>(st.index)].push_back(e);
    }
    stats_.max_versions_held =
        std::max(stats_.max_versions_held, static_cast<int>(st.version_slot.size()));
    if (snapshots_on_) {
        std::vector<uint8_t> buf(st.model->weight_bytes_public());
        st.model->snapshot_weights(dst_slot, buf.data(), buf.size(), us);
        st.snaps.push_back(std::move(buf));
    }
}

void Engine::begin(const std::vector<Program>& programs) {
    if (static_cast<int>(programs.size()) != cfg_.depth)
        throw Error("expected one program per stage");
    for (int s = 0; s < cfg_.depth; ++s) {
        const Stage& st = stages_[static_cast<size_t>(s)];
        if (st.local) continue;
        const bool adjacent = (s > 0 && stages_[s - 1].local) || (s + 1 < cfg_.depth && stages_[s + 1].local);
        if (adjacent && !st.connected)
            throw Error("stage " + std::to_string(s) + " runs in another process and is not connected");
    }
    sync();
    ev_.reset(new EventTable(stages_.size()));
    for (TraceRec& r : trace_) cudaEventDestroy(r.e0), cudaEventDestroy(r.e1);
    trace_.clear();
    progs_ = programs;
    total_ops_ = 0;
    done_ops_ = 0;
    // Flag sequence numbers continue across runs (every process sees the same programs).
    mb_base_ += run_max_mb_;
    run_max_mb_ = 0;
    for (const Program& p : progs_)
        for (const OpRec& op : p) run_max_mb_ = std::max(run_max_mb_, op.microbatch);
    for (int s = 0; s < cfg_.depth; ++s)
        if (stages_[static_cast<size_t>(s)].local) total_ops_ += progs_[static_cast<size_t>(s)].size();
    for (Stage& st : stages_) {
        if (!st.local) continue;
        st.ptr = 0;
        st.fwd_issued.clear();
        st.bwd_issued.clear();
        st.snaps.clear();
        st.updates_issued = 0;
        st.last_fwd = 0;
        st.last_bwd = 0;
        st.version_base = st.updates_done;
        DeviceGuard g(st.device);
        check_cuda(cudaEventRecord(st.t0, st.stream), "cudaEventRecord");
    }
}

// Round-robin issue (semantics.cpp:270-361) until every stage has issued the
// updates of batches 1..upto_batch of this run (or its whole program).
void Engine::issue(int upto_batch) {
    if (!ev_) throw Error("issue() before begin()");
    const int per_batch = cfg_.policy == P2BW_POLICY_1F1B ? cfg_.microbatches : 1;
    const long long target = static_cast<long long>(upto_batch) * per_batch;
    while (true) {
        bool progress = false, pending = false;
        for (Stage& st : stages_) {
            if (!st.local) continue;
            const Program& prog = progs_[static_cast<size_t>(st.index)];
            DeviceGuard g(st.device);
            while (st.ptr < prog.size() && st.updates_issued < target) {
                const OpRec& op = prog[st.ptr];
                if (!ready(st, op)) break;
                if (trace_on_) trace_begin(st, op);
                switch (op.kind) {
                    case P2BW_OP_FORWARD: issue_forward(st, op); break;
                    case P2BW_OP_BACKWARD: issue_backward(st, op); break;
                    case P2BW_OP_UPDATE: issue_update(st); break;
                    case P2BW_OP_ALLREDUCE:  // sum the coalesced gradient over the w replicas
                        if (st.comm) {       // (w == 1: no-op, semantics.cpp:351-354; peer-memory
                                             // groups reduce inside WeightUpdate)
                            void* buf = nullptr;
                            size_t n = 0;
                            int dt = 0;
                            st.model->grad_buffer(&buf, &n, &dt);
                            const cudaStream_t us = update_stream(st);
                            nccl_allreduce_sum(buf, n, dt == 1 ? ncclFloat64 : ncclFloat32,
                                               static_cast<ncclComm_t>(st.comm), us);
                        }
                        break;
                    case P2BW_OP_FLUSH:  // ordering is already implied by stream order
                        break;
                    default:
                        throw Error("op kind " + std::to_string(op.kind) +
                                    " is not executable by the stage executor");
                }
                if (trace_on_) trace_end(st, op);
                st.ptr += 1;
                done_ops_ += 1;
                stats_.ops_executed += 1;
                progress = true;
            }
            if (st.ptr < prog.size() && st.updates_issued < target) pending = true;
        }
        if (!pending) break;
        if (!progress) throw Error("dependency deadlock in toy-model replay");
    }
}

void Engine::finish() {
    if (done_ops_ != total_ops_) issue(1 << 30);
    if (capturing_) return;  // run_graph times the launches instead
    for (Stage& st : stages_) {
        if (!st.local) continue;
        DeviceGuard g(st.device);
        check_cuda(cudaEventRecord(st.t1, st.stream), "cudaEventRecord");
    }
}

double Engine::run_graph(const std::vector<Program>& programs, int launches) {
    if (launches < 1) throw Error("graph mode: launches must be >= 1");
    if (trace_on_ || snapshots_on_) throw Error("graph mode: tracing and snapshots must be off");
    Stage* origin_st = nullptr;
    for (Stage& st : stages_) {
        if (!st.local || st.comm || st.ipc_group)
            throw Error("graph mode runs single-process engines without replica groups");
        if (!origin_st) origin_st = &st;
        else if (st.device != origin_st->device) throw Error("graph mode: all stages on one device");
    }
    // The graph bakes in the slots each update writes and each op reads, chosen from the
    // pre-run state: a replay is another run only if the latest version sits in the same
    // slot again afterwards (2BW: an even number of updates; flush policies: one slot).
    std::vector<int> latest_before;
    for (const Stage& st : stages_) latest_before.push_back(st.version_slot.at(st.updates_done));
    begin(programs);
    DeviceGuard g(origin_st->device);
    const cudaStream_t origin = origin_st->stream;
    std::vector<cudaStream_t> others;
    for (Stage& st : stages_)
        for (cudaStream_t x : {st.stream, st.fstream, st.dstream, st.ustream})
            if (x && x != origin) others.push_back(x);
    cudaEvent_t fork = nullptr;
    std::vector<cudaEvent_t> joins(others.size(), nullptr);
    check_cuda(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming), "cudaEventCreate");
    for (auto& e : joins) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    check_cuda(cudaStreamBeginCapture(origin, cudaStreamCaptureModeRelaxed), "cudaStreamBeginCapture");
    capturing_ = true;
    try {
        // every stream of the run joins the capture through the origin
        check_cuda(cudaEventRecord(fork, origin), "cudaEventRecord(fork)");
        for (cudaStream_t x : others) check_cuda(cudaStreamWaitEvent(x, fork, 0), "cudaStreamWaitEvent(fork)");
        issue(1 << 30);
        finish();
        for (size_t i = 0; i < others.size(); ++i) {
            check_cuda(cudaEventRecord(joins[i], others[i]), "cudaEventRecord(join)");
            check_cuda(cudaStreamWaitEvent(origin, joins[i], 0), "cudaStreamWaitEvent(join)");
        }
        capturing_ = false;
        check_cuda(cudaStreamEndCapture(origin, &graph), "cudaStreamEndCapture");
        check_cuda(cudaGraphInstantiate(&exec, graph, 0), "cudaGraphInstantiate");
    } catch (...) {
        capturing_ = false;
        cudaGraph_t partial = nullptr;
        cudaStreamEndCapture(origin, &partial);
        if (partial) cudaGraphDestroy(partial);
        if (graph) cudaGraphDestroy(graph);
        cudaEventDestroy(fork);
        for (auto e : joins) cudaEventDestroy(e);
        throw;
    }
    // more than one launch replays the run: the slots must have returned to their places
    bool periodic = cfg_.policy != P2BW_POLICY_1F1B;  // 1F1B's stash-pinned versions: launch once
    for (size_t i = 0; i < stages_.size(); ++i)
        periodic = periodic && stages_[i].version_slot.at(stages_[i].updates_done) == latest_before[i];
    if (launches > 1 && !periodic) {
        cudaGraphExecDestroy(exec);
        cudaGraphDestroy(graph);
        cudaEventDestroy(fork);
        for (auto e : joins) cudaEventDestroy(e);
        throw Error("graph mode: this run does not return the weight-version slots to their places; launch it once");
    }
    cudaEvent_t e0, e1;
    check_cuda(cudaEventCreate(&e0), "cudaEventCreate");
    check_cuda(cudaEventCreate(&e1), "cudaEventCreate");
    check_cuda(cudaEventRecord(e0, origin), "cudaEventRecord");
    for (int i = 0; i < launches; ++i) check_cuda(cudaGraphLaunch(exec, origin), "cudaGraphLaunch");
    check_cuda(cudaEventRecord(e1, origin), "cudaEventRecord");
    check_cuda(cudaEventSynchronize(e1), "cudaEventSynchronize");
    float ms = 0.0f;
    check_cuda(cudaEventElapsedTime(&ms, e0, e1), "cudaEventElapsedTime");
    // host bookkeeping: the extra launches are further runs of the same programs
    for (Stage& st : stages_) {
        const int upd = st.updates_done - st.version_base;
        const int extra = upd * (launches - 1);
        if (extra == 0) continue;
        std::map<int, int> shifted;
        for (const auto& kv : st.version_slot) shifted[kv.first + extra] = kv.second;
        st.version_slot = std::move(shifted);
        st.updates_done += extra;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    cudaEventDestroy(fork);
    for (auto e : joins) cudaEventDestroy(e);
    return static_cast<double>(ms) / launches;
}

void Engine::run(const std::vector<Program>& programs) {
    begin(programs);
    issue(1 << 30);
    finish();
}

double Engine::update_elapsed_ms(int s, int u0, int u1) {
    Stage& st = local_stage(s);
    const auto& ev = ev_->upd.at(static_cast<size_t>(s));
    if (u0 < 1 || u1 > static_cast<int>(ev.size()) || u0 > u1)
        throw Error("no update events for that range");
    DeviceGuard g(st.device);
    check_cuda(cudaEventSynchronize(ev[static_cast<size_t>(u1 - 1)]), "cudaEventSynchronize");
    float ms = 0.0f;
    check_cuda(cudaEventElapsedTime(&ms, ev[static_cast<size_t>(u0 - 1)], ev[static_cast<size_t>(u1 - 1)]),
               "cudaEventElapsedTime");
    return ms;
}

void Engine::sync() {
    for (Stage& st : stages_) {
        if (!st.local) continue;
        DeviceGuard g(st.device);
        check_cuda(cudaStreamSynchronize(st.stream), "cudaStreamSynchronize");
        if (st.fstream) check_cuda(cudaStreamSynchronize(st.fstream), "cudaStreamSynchronize");
        if (st.dstream) check_cuda(cudaStreamSynchronize(st.dstream), "cudaStreamSynchronize");
        if (st.ustream) check_cuda(cudaStreamSynchronize(st.ustream), "cudaStreamSynchronize");
        if (st.copy_fwd) check_cuda(cudaStreamSynchronize(st.copy_fwd), "cudaStreamSynchronize");
        if (st.copy_bwd) check_cuda(cudaStreamSynchronize(st.copy_bwd), "cudaStreamSynchronize");
    }
}

double Engine::elapsed_ms_last_run() {
    sync();
    double worst = 0.0;
    for (Stage& st : stages_) {
        if (!st.local) continue;
        float ms = 0.0f;
        check_cuda(cudaEventElapsedTime(&ms, st.t0, st.t1), "cudaEventElapsedTime");
        worst = std::max(worst, static_cast<double>(ms));
    }
    return worst;
}

std::vector<double> Engine::losses(int first_mb, int count) {
    Stage& st = local_stage(cfg_.depth - 1);
    if (st.fstream) check_cuda(cudaStreamSynchronize(st.fstream), "cudaStreamSynchronize");
    std::vector<double> out(static_cast<size_t>(count));
    DeviceGuard g(st.device);
    st.model->read_losses(out.data(), first_mb, count, st.stream);
    check_cuda(cudaStreamSynchronize(st.stream), "cudaStreamSynchronize");
    return out;
}

void Engine::load_stage_weights(int s, const void* host, size_t bytes) {
    Stage& st = local_stage(s);
    sync();
    DeviceGuard g(st.device);
    const int slot = st.version_slot.at(st.updates_done);
    st.model->load_weights(slot, host, bytes);
    st.version_slot.clear();
    st.version_slot[st.updates_done] = slot;
}

void Engine::read_version(int s, int version, void* host, size_t bytes) {
    Stage& st = local_stage(s);
    sync();  // updates may run on the update stream
    const auto it = st.version_slot.find(version);
    if (it == st.version_slot.end())
        throw Error("stage " + std::to_string(s) + " no longer holds weight version " +
                    std::to_string(version));
    DeviceGuard g(st.device);
    st.model->read_weights(it->second, host, bytes, st.stream);
    check_cuda(cudaStreamSynchronize(st.stream), "cudaStreamSynchronize");
}

void Engine::trace_begin(Stage& st, const OpRec& op) {
    check_cuda(cudaEventCreate(&trace_open_), "cudaEventCreate(trace)");
    check_cuda(cudaEventRecord(trace_open_, op_stream(st, op.kind)), "cudaEventRecord(trace)");
}

void Engine::trace_end(Stage& st, const OpRec& op) {
    TraceRec r{};
    r.stage = st.index;
    r.kind = op.kind;
    r.microbatch = op.microbatch;
    r.version = op.weight_version;
    r.versions_held = static_cast<int>(st.version_slot.size());
    r.stashes = static_cast<int>(st.stash_version.size());
    r.e0 = trace_open_;
    trace_open_ = nullptr;
    check_cuda(cudaEventCreate(&r.e1), "cudaEventCreate(trace)");
    check_cuda(cudaEventRecord(r.e1, op_stream(st, op.kind)), "cudaEventRecord(trace)");
    trace_.push_back(r);
}

void Engine::copy_losses_async(float* host, int first_mb, int count) {
    Stage& st = local_stage(cfg_.depth - 1);
    DeviceGuard g(st.device);
    if (st.fstream && ev_) {  // the losses are written by the Forwards (forward stream)
        const auto& fe = ev_->fwd[static_cast<size_t>(st.index)];
        const int last = first_mb + count - 1;
        if (fe.count(last)) wait_on(fe, last, st.stream);
        else if (st.last_fwd > 0 && fe.count(st.last_fwd)) wait_on(fe, st.last_fwd, st.stream);
    }
    st.model->copy_losses_async(host, first_mb, count, st.stream);
}

cudaStream_t Engine::update_stream(Stage& st) {
    if (!st.ustream) return st.stream;
    // the batch's gradient is complete once its last Backward (stage stream) is
    if (st.last_bwd > 0 && ev_->bwd[static_cast<size_t>(st.index)].count(st.last_bwd))
        wait_on(ev_->bwd[static_cast<size_t>(st.index)], st.last_bwd, st.ustream);
    return st.ustream;
}

cudaStream_t Engine::op_stream(const Stage& st, int kind) const {
    return kind == P2BW_OP_FORWARD && st.fstream && !prof::enabled() ? st.fstream : st.stream;
}

void Engine::before_data_set(int s) {
    Stage& st = local_stage(s);
    if (!st.dstream || !ev_ || st.last_bwd < 1) return;
    const auto& be = ev_->bwd[static_cast<size_t>(st.index)];
    if (!be.count(st.last_bwd)) return;
    DeviceGuard g(st.device);
    wait_on(be, st.last_bwd, st.dstream);
}

void Engine::after_data_set(int s, int first_mb, int count) {
    Stage& st = local_stage(s);
    if (!st.dstream) return;
    DeviceGuard g(st.device);
    if (!ev_) {  // before the first run: nothing waits on events, finish the copies now
        check_cuda(cudaStreamSynchronize(st.dstream), "cudaStreamSynchronize(data)");
        return;
    }
    auto& de = ev_->data[static_cast<size_t>(st.index)];
    for (int k = first_mb; k < first_mb + count; ++k) {
        auto it = de.find(k);
        if (it != de.end()) cudaEventDestroy(it->second), de.erase(it);
        record(de, k, st.dstream);
    }
}

void Engine::trace_split(Stage& st, const OpRec& first_part) {
    trace_end(st, first_part);
    trace_begin(st, OpRec{P2BW_OP_BACKWARD, first_part.microbatch, first_part.weight_version});
}

namespace {

std::string op_name(int kind) { return pipesim::to_string(static_cast<pipesim::OpKind>(kind)); }

std::string policy_name(int p) { return pipesim::to_string(static_cast<pipesim::PipelinePolicy>(p)); }

}  // namespace

std::string Engine::trace_report() {
    if (trace_.empty()) throw Error("no traced run: enable tracing before begin()");
    sync();
    using json = nlohmann::json;
    const int d = cfg_.depth;
    // time base: the begin() event of the first local stage on each device
    std::map<int, cudaEvent_t> base;
    for (const Stage& st : stages_)
        if (st.local && !base.count(st.device)) base[st.device] = st.t0;
    struct Entry {
        int worker, kind, mb, ver, versions, stashes;
        double start, end;
    };
    std::vector<Entry> tl;
    tl.reserve(trace_.size());
    for (const TraceRec& r : trace_) {
        const Stage& st = stages_[static_cast<size_t>(r.stage)];
        DeviceGuard g(st.device);
        float a = 0.0f, b = 0.0f;
        check_cuda(cudaEventElapsedTime(&a, base[st.device], r.e0), "cudaEventElapsedTime(trace)");
        check_cuda(cudaEventElapsedTime(&b, base[st.device], r.e1), "cudaEventElapsedTime(trace)");
        tl.push_back({r.stage, r.kind, r.microbatch, r.version, r.versions_held, r.stashes, a * 1e-3, b * 1e-3});
    }
    // steady state from the batch-boundary updates of the last stage, excluding the
    // first and last batch (simulator.cpp:298-309)
    const int per_batch = cfg_.policy == P2BW_POLICY_1F1B ? cfg_.microbatches : 1;
    std::vector<std::vector<double>> upd(static_cast<size_t>(d));
    for (const Entry& e : tl)
        if (e.kind == P2BW_OP_UPDATE) upd[static_cast<size_t>(e.worker)].push_back(e.end);
    auto batch_update_time = [&](int s, int t) {
        const auto& u = upd[static_cast<size_t>(s)];
        const size_t idx = static_cast<size_t>(t) * per_batch - 1;
        if (idx >= u.size()) throw Error("missing batch updates in program");
        return u[idx];
    };
    int last = d - 1;
    while (last >= 0 && !stages_[static_cast<size_t>(last)].local) --last;
    const int num_batches = static_cast<int>(upd[static_cast<size_t>(last)].size()) / per_batch;
    int replicas = 1;
    for (const Stage& st : stages_)
        if (st.local) replicas = std::max(replicas, st.replicas);
    const double global_batch = static_cast<double>(cfg_.microbatch_size) * cfg_.microbatches * replicas;
    double steady = 0.0, throughput = 0.0, bubble = 0.0;
    if (num_batches >= 3) {
        steady = (batch_update_time(last, num_batches - 1) - batch_update_time(last, 1)) / (num_batches - 2);
        throughput = steady > 0 ? global_batch / steady : 0.0;
        double window = 0.0, busy = 0.0;  // simulator.cpp:311-329
        for (int s = 0; s < d; ++s) {
            if (!stages_[static_cast<size_t>(s)].local) continue;
            const double w0 = batch_update_time(s, 1), w1 = batch_update_time(s, num_batches - 1);
            window += w1 - w0;
            for (const Entry& e : tl) {
                if (e.worker != s) continue;
                if (e.kind != P2BW_OP_FORWARD && e.kind != P2BW_OP_BACKWARD && e.kind != P2BW_OP_RECOMPUTE) continue;
                const double lo = std::max(e.start, w0), hi = std::min(e.end, w1);
                if (hi > lo) busy += hi - lo;
            }
        }
        bubble = window > 0.0 ? 1.0 - busy / window : 0.0;
    }
    std::stable_sort(tl.begin(), tl.end(), [](const Entry& a, const Entry& b) {
        if (a.worker != b.worker) return a.worker < b.worker;
        return a.start < b.start;
    });
    json doc;
    doc["policy"] = policy_name(cfg_.policy);
    // ParallelConfig (profile.hpp:49-62) has m = depth * grad_accum; when m is not a
    // multiple of d, grad_accum is rounded down and the exact m rides beside it
    doc["config"] = {{"width", replicas},
                     {"depth", d},
                     {"microbatch_size", cfg_.microbatch_size},
                     {"recompute", cfg_.recompute},
                     {"grad_accum", std::max(cfg_.microbatches / d, 1)},
                     {"microbatches_per_batch", cfg_.microbatches}};
    doc["num_batches"] = num_batches;
    doc["throughput"] = throughput;
    doc["bubble_fraction"] = bubble;
    doc["steady_batch_time"] = steady;
    doc["measured"] = true;
    doc["timeline"] = json::array();
    for (const Entry& e : tl) {
        const bool comm = e.kind == P2BW_OP_ALLREDUCE || (e.kind >= P2BW_OP_ACT_SEND && e.kind <= P2BW_OP_GRAD_RECV);
        doc["timeline"].push_back({{"worker", e.worker},
                                   {"lane", comm ? "comm" : "compute"},
                                   {"op", op_name(e.kind)},
                                   {"mb", e.mb},
                                   {"ver", e.ver},
                                   {"start", e.start},
                                   {"end", e.end}});
    }
    doc["memory"] = json::array();
    for (int s = 0; s < d; ++s) {
        json jt = json::array();
        const Stage& st = stages_[static_cast<size_t>(s)];
        if (st.local) {
            const double vb = st.model->version_bytes(), sb = st.model->stash_bytes();
            for (const Entry& e : tl) {
                if (e.worker != s) continue;
                jt.push_back({{"time", e.end},
                              {"versions", e.versions},
                              {"stashes", e.stashes},
                              {"bytes", e.versions * vb + e.stashes * sb}});
            }
        }
        doc["memory"].push_back(std::move(jt));
    }
    return doc.dump(2);
}

}  // namespace p2bw
