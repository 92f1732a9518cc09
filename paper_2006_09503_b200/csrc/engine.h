// The B200 stage executor: the third interpreter of pipesim's op stream
// (reference interpreters: semantics.cpp:270-361 numerically, simulator.cpp:195-290
// for timing).  One CUDA stream per pipeline stage; cross-stage hand-offs are
// producer kernels writing straight into the consumer stage's receive ring
// (same device or an NVLink peer), ordered by CUDA events.  The host issues
// every op asynchronously in the reference's round-robin order; nothing blocks
// on the GPU inside run().
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "p2bw.h"
#include "util.h"

namespace p2bw {

struct EventTable;  // engine.cpp

struct OpRec {
    int kind = 0;
    int microbatch = 0;
    int weight_version = 0;
};
using Program = std::vector<OpRec>;

struct EngineConfig {
    int model_kind = P2BW_MODEL_LINEAR_F64;
    int policy = P2BW_POLICY_2BW;
    int depth = 1;
    int microbatches = 1;     // m
    int microbatch_size = 1;  // b (columns / sequences)
    // linear chain
    int dim = 0;
    // shared
    int layers = 0;
    // transformer
    int hidden = 0, heads = 0, seq_len = 0, vocab = 0, causal = 0, head_rows = 0;
    double lr = 0.0, momentum = 0.0;
    uint64_t seed = 0;
    std::vector<int> devices;  // per stage
    // Cross-process pipeline: this process runs stages [first_local, first_local +
    // local_count); 0 = all stages.  Remote neighbours are reached through CUDA IPC
    // (export_stage / connect_stage).
    int first_local = 0, local_count = 0;
    // Activation recomputation: forwards keep only the stage input; each backward
    // first re-runs the stage forward (Recompute op, simulator.cpp:242-247).
    bool recompute = false;
    // WeightUpdate optimizer: P2BW_OPT_MOMENTUM_SGD (reference) or P2BW_OPT_ADAM
    int optimizer = 0;
    double beta2 = 0.999, eps = 1e-8;
    // fp64 linear chain: reference_loop's per-microbatch 1/m gradient scaling
    // (semantics.cpp:145) instead of pipelined_execute's sum / count (:338-340).
    bool loop_scaling = false;
    // Layers per stage (B200 extension, e.g. from pipesim::partition_balanced); empty:
    // the reference's equal split, which needs layers % depth == 0.
    std::vector<int> stage_layers;
};

// Receive-side block of one stage, exported over CUDA IPC to its neighbours'
// processes: the activation ring, the output-gradient ring and four u32 flags.
struct StageBlob {
    char ipc[64];       // cudaIpcMemHandle_t of the block
    int stage;
    int stash_slots, grad_slots;
    uint64_t slot_bytes;
    uint64_t act_off, grad_off, flag_off;  // byte offsets inside the block
};

// One stage of one data-parallel replica, for the peer-memory replica group
// (Engine::join_replicas_ipc): CUDA IPC handles of the stage's flag block and of the
// buffers StageModel::replica_buffers() lists.
constexpr int kMaxReplicaBufs = 12;
struct ReplicaBlob {
    uint32_t magic;
    int32_t stage, nbuf, weight_slots;
    uint64_t weight_bytes;  // public weight bytes of the stage (shape check)
    char block_ipc[64];
    uint64_t flag_off;
    char buf_ipc[kMaxReplicaBufs][64];
    uint64_t buf_off[kMaxReplicaBufs];
    uint8_t buf_present[kMaxReplicaBufs];
};
constexpr uint32_t kReplicaBlobMagic = 0x42523250u;  // "P2RB"

// One pipeline stage's model slice: parameters, version buffers, stash and the
// kernels of the Forward / Backward / WeightUpdate ops.
class StageModel {
public:
    virtual ~StageModel() = default;
    virtual size_t num_params() const = 0;
    // Elements of the boundary tensor handed to the next stage (and of its gradient).
    virtual size_t boundary_bytes() const = 0;
    // Forward of microbatch k on weight slot `wslot`, stash slot `sslot`.
    //   x_in : this stage's input (receive-ring slot), nullptr on stage 0 (data)
    //   x_out: next stage's receive-ring slot, nullptr on the last stage
    virtual void forward(int k, int wslot, int sslot, const void* x_in, void* x_out,
                         cudaStream_t s) = 0;
    //   g_in : gradient of this stage's output, nullptr on the last stage (loss)
    //   g_out: previous stage's gradient ring slot, nullptr on stage 0
    //   first: first backward since the last update (gradient buffer is overwritten)
    virtual void backward(int k, int wslot, int sslot, const void* g_in, void* g_out,
                          bool first, cudaStream_t s) = 0;
    // Recompute op: re-run the forward of microbatch k (weights wslot, input x_in, the
    // stage's ring slot; nullptr on stage 0) so that backward() finds its activations.
    virtual void recompute(int k, int wslot, int sslot, const void* x_in, cudaStream_t s) {
        (void)k, (void)wslot, (void)sslot, (void)x_in, (void)s;
        throw Error("this stage model does not support activation recomputation");
    }
    // Fused optimizer: new version into dst_slot from src_slot (may alias).
    virtual void update(int src_slot, int dst_slot, int grad_count, cudaStream_t s) = 0;
    // Host <-> device weights of one version slot, in the model's public layout.
    virtual void load_weights(int wslot, const void* host, size_t bytes) = 0;
    virtual void read_weights(int wslot, void* host, size_t bytes, cudaStream_t s) = 0;
    // Trajectory snapshot of the version just written into wslot (semantics.cpp:363-373);
    // mixed-precision models return their fp32 master (the bf16 version is its rounding).
    virtual void snapshot_weights(int wslot, void* host, size_t bytes, cudaStream_t s) {
        read_weights(wslot, host, bytes, s);
    }
    virtual size_t weight_bytes_public() const = 0;
    // Per-microbatch training loss (last stage only), indexed like the data ring.
    virtual void read_losses(double* host, int first_mb, int count, cudaStream_t s) {
        (void)host, (void)first_mb, (void)count, (void)s;
        throw Error("this stage computes no loss");
    }
    virtual void bind_stream(cudaStream_t s) { (void)s; }
    // Stream for set_data's host-to-device copies (default: the bound stream).
    virtual void bind_data_stream(cudaStream_t s) { (void)s; }
    // Two coalesced-gradient buffers used alternately per batch, so the AllReduce and
    // WeightUpdate of batch t (update stream) overlap the Backwards of batch t+1.
    // Returns false if the model keeps a single buffer.
    virtual bool enable_grad_double_buffer() { return false; }
    // The coalesced gradient buffer (all-reduced across data-parallel replicas).
    // dtype: 0 = fp32, 1 = fp64.
    virtual void grad_buffer(void** ptr, size_t* count, int* dtype) = 0;
    // Data-parallel replicas on one node (Engine::join_replicas_ipc, CUDA IPC): the
    // buffers the fused AllReduce + WeightUpdate touches in every replica, in a fixed
    // order: [0], [1] coalesced gradient buffers (null when single), [2] fp32 master
    // (null when the versions are the master), [3 + i] weight slot i.
    virtual std::vector<void*> replica_buffers() { return {}; }
    // WeightUpdate with the AllReduce fused in (replica `rank` owns parameter shard
    // `rank`): sum the shard of every replica's current gradient, update its optimizer
    // state, store the new version of the shard into every replica.  peers[q] is
    // replica q's replica_buffers() as mapped in this process (peers[rank]: local).
    virtual void update_replicas(int src_slot, int dst_slot, int count, const std::vector<std::vector<void*>>& peers,
                                 int rank, cudaStream_t s) {
        (void)src_slot, (void)dst_slot, (void)count, (void)peers, (void)rank, (void)s;
        throw Error("this stage model has no fused replica update");
    }
    // Asynchronous D2H of fp32 losses into (pinned) host memory, stream-ordered.
    virtual void copy_losses_async(float* host, int first_mb, int count, cudaStream_t s) {
        (void)host, (void)first_mb, (void)count, (void)s;
        throw Error("this stage computes no fp32 loss");
    }
    // Bytes one weight version / one stash slot occupies (memory trace of a measured run).
    virtual double version_bytes() const { return static_cast<double>(weight_bytes_public()); }
    virtual double stash_bytes() const { return 0.0; }
    // fp32 master weights (models that keep one), public layout.
    virtual void read_master(void* host, size_t bytes) {
        (void)host, (void)bytes;
        throw Error("this model keeps no separate master weights");
    }
    // Deterministic synthetic initial weights (version 0) from a seed.
    virtual void init_weights(uint64_t seed) {
        (void)seed;
        throw Error("this model takes its initial weights from the caller");
    }
    virtual void set_data(const void* inputs, const void* targets, int first_mb, int count) = 0;
    // Dataset microbatches generated on the device from a seed (linear chain: ToyModel::make).
    virtual void make_toy_data(uint64_t seed, int first_mb, int count) {
        (void)seed, (void)first_mb, (void)count;
        throw Error("this stage model has no device-side toy dataset");
    }
    virtual int data_capacity() const = 0;
};

std::unique_ptr<StageModel> make_linear_f64_stage(const EngineConfig& cfg, int stage, int lo,
                                                   int hi, int stash_slots, int weight_slots);
std::unique_ptr<StageModel> make_linear_bf16_stage(const EngineConfig& cfg, int stage, int lo,
                                                    int hi, int stash_slots, int weight_slots);
std::unique_ptr<StageModel> make_transformer_stage(const EngineConfig& cfg, int stage, int lo,
                                                    int hi, int stash_slots, int weight_slots);

struct RunStats {
    bool version_consistent = true;
    int max_versions_held = 1;
    long long ops_executed = 0;
};

class Engine {
public:
    explicit Engine(const EngineConfig& cfg);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    const EngineConfig& config() const { return cfg_; }
    int depth() const { return cfg_.depth; }
    StageModel& model(int s) { return *local_stage(s).model; }
    // Initial weights of stage s: written into the buffer of its latest version, which
    // then becomes the stage's only live version.
    void load_stage_weights(int s, const void* host, size_t bytes);

    // Interpret one program per stage (asynchronous; call sync() to wait).
    void run(const std::vector<Program>& programs);
    // Incremental form of run(): begin() installs the programs, issue(t) issues
    // ops until every stage has issued the weight updates of batches 1..t,
    // finish() issues the rest.  Lets a caller stream data in batch by batch.
    void begin(const std::vector<Program>& programs);
    void issue(int upto_batch);
    void finish();
    // CUDA-graph mode (one process, no replica group, tracing and snapshots off): the
    // whole run is captured into one graph across the stages' streams and launched
    // `launches` times.  Every launch after the first runs the same programs again on
    // the current weights, exactly as another run() would, which needs each stage's
    // version slots to be back where they started (an even number of 2BW updates per
    // run; checked).  Returns the device ms per launch (events around the launches);
    // the per-update events of a captured run are not timed.
    double run_graph(const std::vector<Program>& programs, int launches);
    // Device time between a stage's u0-th and u1-th update of the current run.
    double update_elapsed_ms(int stage, int u0, int u1);
    // Data parallelism: stage s of this pipeline joins the communicator of its
    // `nranks` replicas (one NCCL unique id per stage, 128 bytes each).  The
    // AllReduce op then sums the coalesced gradient across replicas and the
    // update divides by count * nranks (the replicas' average).
    void join_replicas(const void* ids, int nranks, int rank);
    void sync();
    // Weights of stage s for the version created by its u-th update (0 = initial).
    void read_version(int s, int version, void* host, size_t bytes);
    void set_snapshot_every_update(bool on) { snapshots_on_ = on; }
    const std::vector<std::vector<uint8_t>>& snapshots(int s) const { return stages_.at(s).snaps; }
    const RunStats& stats() const { return stats_; }
    double elapsed_ms_last_run();
    // Losses of microbatches [first_mb, first_mb + count) (last stage), after sync.
    std::vector<double> losses(int first_mb, int count);
    void copy_losses_async(float* host, int first_mb, int count);
    // Around the host's refill of stage s's data ring: with a forward stream the copies
    // run on a data stream, after every Backward issued so far (stage 0's embedding
    // gradient reads the token ids of the slots being overwritten), and each Forward
    // waits only for the copy of its own microbatch (after_data_set records them).
    void before_data_set(int s);
    void after_data_set(int s, int first_mb, int count);
    bool is_local(int s) const { return s >= 0 && s < cfg_.depth && stages_[static_cast<size_t>(s)].local; }
    // Measured timeline: with tracing on, every issued op of a
    // local stage is bracketed by CUDA events; trace_report() renders the last run
    // as the reference's SimReport document (simulator.cpp:356-390) with
    // throughput, steady batch time and bubble fraction computed exactly as
    // simulate() does (simulator.cpp:298-329), from measured times.
    void set_trace(bool on) { trace_on_ = on; }
    std::string trace_report();
    // CUDA IPC hand-off between processes (one process per stage group).
    StageBlob export_stage(int s);
    void connect_stage(const StageBlob& blob);
    // Data-parallel replicas of stage s on one node, one process each, without NCCL:
    // blobs[q] = replica q's export_replica(s).  The AllReduce op then happens inside
    // WeightUpdate: one fused kernel reduce-scatters the coalesced gradients over peer
    // memory, applies the optimizer to this replica's shard and all-gathers the new
    // version (StageModel::update_replicas), between two stream-ordered flag barriers.
    ReplicaBlob export_replica(int s);
    void join_replicas_ipc(int s, const std::vector<ReplicaBlob>& blobs, int rank);

private:
    // Flags in a stage's receive block (seq numbers, monotonically increasing).
    enum Flag { kActReady = 0, kGradReady = 1, kNextBwd = 2, kPrevBwd = 3, kNumFlags = 4 };
    // replica-group barriers: kReplicaReady + q / kReplicaDone + q written by replica q
    static constexpr int kReplicaReady = 16, kReplicaDone = 32;

    struct Stage {
        int index = 0;
        int device = 0;
        bool local = true;
        bool connected = false;  // remote stage: its block is mapped into this process
        int lo = 0, hi = 0;
        cudaStream_t stream = nullptr;   // Backward / WeightUpdate / AllReduce (and Forward unless fstream)
        cudaStream_t fstream = nullptr;  // Forward, overlapping the previous microbatch's Backward
        int last_fwd = 0;                // latest microbatch whose Forward was issued
        int last_bwd = 0;                // latest microbatch whose Backward was issued
        cudaStream_t dstream = nullptr;  // set_data host-to-device copies (with fstream)
        cudaStream_t ustream = nullptr;  // AllReduce + WeightUpdate (2BW with double-buffered gradients)
        std::unique_ptr<StageModel> model;
        int stash_slots = 1;
        int grad_slots = 1;
        int weight_slots = 1;
        // receive rings owned by this stage (written by the neighbours)
        std::vector<void*> act_ring;   // [stash_slots] boundary tensors (stage input)
        std::vector<void*> grad_ring;  // [grad_slots] gradient of this stage's output
        void* block = nullptr;         // one allocation: rings + flags (IPC-exportable)
        uint32_t* flags = nullptr;     // [kNumFlags] inside `block`
        bool block_mapped = false;     // opened with cudaIpcOpenMemHandle (remote stage)
        // sends to a remote neighbour: local staging slots + a copy stream each way
        void* send_act[2] = {nullptr, nullptr};
        void* send_grad[2] = {nullptr, nullptr};
        cudaStream_t copy_fwd = nullptr, copy_bwd = nullptr;
        // host-side interpreter state (mirrors semantics.cpp:198-211)
        size_t ptr = 0;
        int updates_done = 0;
        int updates_issued = 0;  // in the current run
        void* comm = nullptr;    // ncclComm_t over this stage's data-parallel replicas
        int replicas = 1;
        // peer-memory replica group (join_replicas_ipc)
        bool ipc_group = false;
        int replica_rank = 0;
        std::vector<std::vector<void*>> peer_bufs;  // [replica] -> replica_buffers() mapped here
        std::vector<uint32_t*> peer_flags;          // [replica] -> its flag block (null for this one)
        std::vector<void*> ipc_opened;              // bases to cudaIpcCloseMemHandle
        uint32_t ar_seq = 0;                        // fused all-reduce updates so far (flag values)
        int version_base = 0;    // updates_done at begin()
        std::map<int, int> version_slot;  // live version -> weight slot
        std::map<int, int> stash_version; // in-flight microbatch -> version
        int grad_count = 0;
        std::map<int, bool> fwd_issued, bwd_issued;
        std::vector<std::vector<uint8_t>> snaps;  // snapshot per update (optional)
        cudaEvent_t t0 = nullptr, t1 = nullptr;
    };

    struct TraceRec {
        int stage, kind, microbatch, version;
        int versions_held, stashes;  // after the op (host bookkeeping)
        cudaEvent_t e0, e1;
    };
    void trace_begin(Stage& st, const OpRec& op);
    void trace_end(Stage& st, const OpRec& op);
    // Forwards run on the forward stream, except while per-launch profiling is on
    // (the roofline wants every launch timed alone).
    cudaStream_t op_stream(const Stage& st, int kind) const;
    // Stream of AllReduce / WeightUpdate, ordered after the stage's last issued Backward.
    cudaStream_t update_stream(Stage& st);
    void trace_split(Stage& st, const OpRec& first_part);  // close first_part, open the rest

    void issue_forward(Stage& st, const OpRec& op);
    void issue_backward(Stage& st, const OpRec& op);
    void issue_update(Stage& st);
    void issue_update_replicas(Stage& st, int src_slot, int dst_slot, cudaStream_t us);
    bool ready(const Stage& st, const OpRec& op) const;
    int resolve_version(const Stage& st, const OpRec& op) const;
    void prune_versions(Stage& st);
    void free_buffers();
    Stage& local_stage(int s);
    uint32_t seq(int k) const { return static_cast<uint32_t>(mb_base_ + k); }
    void signal_remote(uint32_t* flag, uint32_t value, cudaStream_t s);
    void wait_flag(const uint32_t* flag, uint32_t value, cudaStream_t s);

    struct EventTableDeleter {
        void operator()(struct EventTable* t) const;
    };

    EngineConfig cfg_;
    std::vector<Stage> stages_;
    std::vector<Program> progs_;
    size_t total_ops_ = 0, done_ops_ = 0;
    std::unique_ptr<struct EventTable, EventTableDeleter> ev_;
    RunStats stats_;
    bool snapshots_on_ = false;
    bool trace_on_ = false;
    std::vector<TraceRec> trace_;
    cudaEvent_t trace_open_ = nullptr;  // e0 of the op being issued
    long long mb_base_ = 0;  // microbatches of earlier runs (flag sequence numbers)
    bool capturing_ = false;  // inside run_graph's stream capture
    int run_max_mb_ = 0;
};

}  // namespace p2bw
