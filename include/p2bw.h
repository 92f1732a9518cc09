/*
 * p2bw.h — C-ABI of libp2bw.so, the B200-native PipeDream-2BW engine.
 *
 * This is the drop-in boundary for the reference's pipelined training path
 * (pipesim, /root/reference/proj/core/include/pipesim/ headers).  The reference
 * has no FFI of its own; every entry point below names the C++ interface it
 * replaces (file:line, relative to /root/reference/proj).  Plain pointers and
 * sizes only: no torch / C++ types cross this boundary.
 *
 * Conventions
 *   - Every function returns P2BW_OK (0) or a nonzero status; the message of
 *     the last failure on the calling thread is p2bw_last_error().  The message
 *     text keeps the reference's pipesim::Error wording (core/include/pipesim/
 *     error.hpp:9-12) so callers can rethrow it unchanged.
 *   - Host buffers are borrowed for the duration of the call only.
 *   - An engine is not reentrant (the reference is single-threaded,
 *     SPEC.md:83); internally it drives one CUDA stream per pipeline stage.
 */
#ifndef P2BW_H
#define P2BW_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define P2BW_OK 0
#define P2BW_ERR 1     /* pipesim::Error equivalent (invariant / infeasible / CUDA failure) */
#define P2BW_ERR_ARG 2 /* malformed argument */

/* ---- library ------------------------------------------------------------ */

const char* p2bw_last_error(void);
const char* p2bw_version(void);

/* ---- policies and ops: schedule.hpp:10-51 ---------------------------------- */

/* == pipesim::PipelinePolicy (schedule.hpp:10-16), same order. */
enum {
    P2BW_POLICY_NONE = 0,
    P2BW_POLICY_GPIPE = 1,
    P2BW_POLICY_1F1B = 2,
    P2BW_POLICY_FLUSH = 3,
    P2BW_POLICY_2BW = 4
};

/* == pipesim::OpKind (schedule.hpp:21-32), same order. */
enum {
    P2BW_OP_FORWARD = 0,
    P2BW_OP_BACKWARD = 1,
    P2BW_OP_RECOMPUTE = 2,
    P2BW_OP_UPDATE = 3,
    P2BW_OP_FLUSH = 4,
    P2BW_OP_ACT_SEND = 5,
    P2BW_OP_ACT_RECV = 6,
    P2BW_OP_GRAD_SEND = 7,
    P2BW_OP_GRAD_RECV = 8,
    P2BW_OP_ALLREDUCE = 9
};

#define P2BW_LATEST_VERSION (-1) /* == pipesim::kLatestVersion (schedule.hpp:36) */

/* Stage model families the executor can run. */
enum {
    P2BW_MODEL_LINEAR_F64 = 0,  /* the reference ToyModel (semantics.hpp:31-43), fp64, bit-exact */
    P2BW_MODEL_TRANSFORMER = 1, /* pre-LN transformer blocks, bf16 tcgen05 kernels, fp32 master */
    P2BW_MODEL_LINEAR_BF16 = 2  /* the ToyModel on the production path: bf16 tcgen05 GEMMs, fp32
                                   master / momentum / gradient, fused optimizer, the transformer's
                                   streams; same public fp64 layout as P2BW_MODEL_LINEAR_F64 */
};

/* == pipesim::ScheduledOp (schedule.hpp:40-46). */
typedef struct {
    int kind;
    int microbatch;
    int weight_version;
} p2bw_op;

/* ---- schedule: schedule.hpp:53-65 ------------------------------------------ */

typedef struct p2bw_schedule p2bw_schedule; /* == std::vector<StageProgram> */

/* weight_version_2bw (schedule.hpp:53-55 / schedule.cpp:58-62). */
int p2bw_weight_version_2bw(int k, int m, int* out);
/* required_versions (schedule.hpp:57-58). */
int p2bw_required_versions(int policy, int d, int m, int* out);
/* generate_schedule (schedule.hpp:60-61 / schedule.cpp:148-175). */
int p2bw_schedule_generate(int policy, int d, int m, int num_batches, p2bw_schedule** out);
/* parse_programs (schedule.hpp:64 / schedule.cpp:197-242). */
int p2bw_schedule_parse(const char* text, p2bw_schedule** out);
int p2bw_schedule_num_stages(const p2bw_schedule* sched, int* out);
/* Borrowed view of one StageProgram's ops, valid until p2bw_schedule_destroy. */
int p2bw_schedule_ops(const p2bw_schedule* sched, int stage, const p2bw_op** ops, size_t* n);
/* serialize_programs (schedule.hpp:63 / schedule.cpp:177-195); free with p2bw_free. */
int p2bw_schedule_serialize(const p2bw_schedule* sched, char** text);
void p2bw_schedule_destroy(p2bw_schedule* sched);
/* Policy names: to_string / parse_policy (schedule.hpp:18-19). */
int p2bw_policy_name(int policy, const char** name);
int p2bw_policy_parse(const char* name, int* policy);

void p2bw_free(void* p);

/* ---- planner and partition: planner.hpp:40-41, profile.hpp:76 ------------- */

/* plan(load_model_profile(model_json), load_cluster_spec(cluster_json), B, policy)
 * rendered by plan_to_json (planner.cpp:160-186) or plan_to_text (:139-158).
 * JSON inputs use the reference's profile / cluster documents (profile.cpp:162-241). */
int p2bw_plan(const char* model_json, const char* cluster_json, long long max_batch, int policy,
              int as_text, char** out);
/* partition_equal (profile.cpp:104-131) rendered as a JSON array of stages
 * {fwd_time, bwd_time, weight_bytes, act_total_bytes, act_input_bytes,
 *  act_output_bytes} in SI units (seconds, bytes), keys = microbatch sizes. */
int p2bw_partition_equal(const char* model_json, int d, char** out_json);
/* B200 extension: pipesim::partition_balanced (include/pipesim/profile.hpp) -- the d + 1
 * block boundaries of the contiguous split minimising the slowest stage's fwd + bwd
 * time at microbatch size b, as a JSON array. */
int p2bw_partition_balanced(const char* model_json, int d, int b, char** out_json);

/* ---- the stage executor: pipelined_execute (semantics.hpp:73-74) ---------- */

typedef struct p2bw_engine p2bw_engine;

typedef struct {
    int model_kind;      /* P2BW_MODEL_* */
    int policy;          /* P2BW_POLICY_* */
    int depth;           /* pipeline stages d (layers split by partition_equal) */
    int width;           /* data-parallel replicas w (1 in this process) */
    int microbatches;    /* m: microbatches per batch (TrainerConfig, semantics.hpp:45-52) */
    int microbatch_size; /* b: columns (linear) or sequences (transformer) */
    int layers;          /* blocks */
    int dim;             /* linear chain width (ToyModel::dim) */
    int hidden, heads, seq_len, vocab;
    int causal;          /* 1: GPT decoder mask, 0: BERT encoder */
    int head_rows;       /* LM-head rows per sequence (0: every position) */
    double learning_rate;
    double momentum;
    unsigned long long seed;
    const int* devices;  /* one CUDA device per stage, or NULL: all on the current device */
    /* Cross-process pipeline (one process per GPU): this process runs stages
     * [first_local_stage, first_local_stage + local_stages); local_stages == 0 runs
     * every stage here.  Neighbours in other processes are connected with
     * p2bw_engine_export_stage / p2bw_engine_connect_stage before the first run. */
    int first_local_stage;
    int local_stages;
    /* Activation recomputation (the planner's r flag, planner.cpp:21-22; timed by
     * simulate() as a Recompute op before each Backward, simulator.cpp:242-247):
     * a Forward keeps only the stage input, the Backward re-runs the stage forward
     * into one shared workspace first.  Numerics are unchanged. */
    int recompute;
    /* Optimizer of the WeightUpdate op: P2BW_OPT_MOMENTUM_SGD is the reference's
     * momentum SGD with (1 - beta) dampening (semantics.cpp:153-165); P2BW_OPT_ADAM is
     * Adam with bias correction (the paper's optimizer, absent from
     * the reference): beta1 = momentum, beta2, eps; transformer stages only. */
    int optimizer;
    double beta2;
    double eps;
    /* Gradient normalisation of the fp64 linear chain.  0: pipelined_execute's -- sum the
     * batch's microbatch gradients, divide by grad_count at the update (semantics.cpp:329,
     * 338-340).  1: reference_loop's -- scale each microbatch's gradient by 1/m as it is
     * accumulated and apply the sum (semantics.cpp:145); the two agree bit for bit only
     * when m is a power of two. */
    int loop_scaling;
    /* Layers per stage (depth entries), or NULL for the reference's equal split
     * (partition_equal, profile.cpp:104-131; requires layers % depth == 0).  A B200
     * extension: p2bw_partition_balanced picks the split whose slowest stage is fastest,
     * so the first / last stages, which also carry the embedding / LM head, get fewer
     * layers.  Weights depend only on the global layer index, so a run is comparable
     * across splits. */
    const int* stage_layers;
} p2bw_desc;

enum { P2BW_OPT_MOMENTUM_SGD = 0, P2BW_OPT_ADAM = 1 };

typedef struct {
    int version_consistent; /* PipelinedResult::version_consistent */
    int max_versions_held;  /* PipelinedResult::max_versions_held */
    long long ops_executed;
    double last_run_ms;     /* device time of the last run, max over stages (CUDA events) */
} p2bw_counters;

int p2bw_engine_create(const p2bw_desc* desc, p2bw_engine** out);
void p2bw_engine_destroy(p2bw_engine* eng);
/* Bytes of one stage's weights in the public layout (linear: fp64 column-major
 * matrices of the stage's layers; transformer: fp32 flat parameter vector). */
int p2bw_engine_stage_weight_bytes(p2bw_engine* eng, int stage, size_t* bytes);
/* Initial weights (version 0) of one stage (host buffer, borrowed). */
int p2bw_engine_load_stage_weights(p2bw_engine* eng, int stage, const void* host, size_t bytes);
/* Deterministic initial weights from desc->seed (transformer: scaled-uniform init;
 * bf16 linear chain: ToyModel::make's W_l = I + 0.2 U, semantics.cpp:89-95). */
int p2bw_engine_init_weights(p2bw_engine* eng);
/* Microbatches [first_mb, first_mb+count), 1-based like ScheduledOp::microbatch.
 * Linear: inputs/targets fp64 [count][dim*b] column-major (ToyModel::dataset).
 * Transformer: int32 token ids / targets [count][b*seq_len]. */
int p2bw_engine_set_data(p2bw_engine* eng, const void* inputs, const void* targets, int first_mb,
                         int count);
/* P2BW_MODEL_LINEAR_BF16: microbatches [first_mb, first_mb+count) of ToyModel::make's
 * dataset (semantics.cpp:85-109) for desc->seed, generated on the device draw for draw
 * from the same splitmix64 stream (x exact up to the bf16 rounding; y = A x by the bf16
 * GEMM) -- the bench's same-config workload without a host-side dataset.  The matching
 * initial weights come from p2bw_engine_init_weights. */
int p2bw_engine_make_toy_data(p2bw_engine* eng, int first_mb, int count);
/* Interpret one program per stage (n_ops[s] ops at programs[s]).  Asynchronous. */
int p2bw_engine_run(p2bw_engine* eng, const p2bw_op* const* programs, const size_t* n_ops,
                    int snapshot_updates);
/* generate_schedule(desc->policy, d, m, num_batches) followed by p2bw_engine_run. */
int p2bw_engine_run_schedule(p2bw_engine* eng, int num_batches, int snapshot_updates);
/* CUDA-graph form of run_schedule (one process, no replica group; tracing and snapshots
 * off): the run is captured across the stages' streams into one graph and launched
 * `launches` times -- each launch after the first is another run of the same programs
 * on the current weights (allowed when the run returns every stage's weight-version
 * slots to their places, e.g. an even number of 2BW batches).  ms_per_launch: device
 * time per launch. */
int p2bw_engine_run_schedule_graph(p2bw_engine* eng, int num_batches, int launches, double* ms_per_launch);
/* Streaming form of run_schedule: begin() installs generate_schedule(policy, d, m,
 * num_batches); issue(t) issues every stage's ops up to and including its weight
 * update of batch t (so batch t+1's data must already be set: 2BW forwards of the
 * next batch are admitted before the update); finish() issues the remainder. */
int p2bw_engine_begin(p2bw_engine* eng, int num_batches);
int p2bw_engine_issue(p2bw_engine* eng, int upto_batch);
int p2bw_engine_finish(p2bw_engine* eng);
/* Device time between stage `stage`'s u0-th and u1-th WeightUpdate of the current
 * run (CUDA events on the stage's stream; waits for u1). */
int p2bw_engine_update_elapsed_ms(p2bw_engine* eng, int stage, int u0, int u1, double* ms);
/* Data-parallel width w > 1 (planner's "width", profile.hpp:50-62): one process
 * per pipeline replica.  Rank 0 makes one 128-byte NCCL unique id per stage and
 * shares them; every replica calls join_replicas with the same ids.  The
 * AllReduce op (schedule.cpp:80-84) then sums each stage's coalesced gradient
 * across its w replicas (NCCL, on the stage's stream) and WeightUpdate divides
 * by count * w -- the replicas' average, as costmodel.cpp:23-27 prices it. */
int p2bw_nccl_unique_id(void* out, size_t bytes);
int p2bw_engine_join_replicas(p2bw_engine* eng, const void* ids, int nranks, int rank);
/* Data-parallel replicas on one node without NCCL: every replica exports each local
 * stage (p2bw_engine_export_replica), the blobs are exchanged (any transport), and each
 * stage joins with the blobs of its w replicas in replica order.  The AllReduce op
 * (schedule.cpp:80-84) is then fused into WeightUpdate: one kernel per replica sums its
 * shard of every replica's coalesced gradient over CUDA-IPC peer memory (NVLink),
 * applies the optimizer to that shard and stores the new version of the shard into
 * every replica -- the update the reference prices as allreduce + apply
 * (costmodel.cpp:23-27, semantics.cpp:335-350), divided by count * w.  Replicas may
 * share a GPU (one process each).  nranks <= 8. */
#define P2BW_REPLICA_BLOB_BYTES 1024
int p2bw_engine_export_replica(p2bw_engine* eng, int stage, void* blob, size_t bytes);
int p2bw_engine_join_replicas_ipc(p2bw_engine* eng, int stage, const void* blobs, int nranks, int rank);
/* Cross-process pipelines: the reference interprets all stages in one loop
 * (semantics.cpp:270-361); here each process interprets its own stages and the
 * hand-offs of out_act (:299) / grad_to_prev (:333) to a stage in another process
 * go through that stage's receive block, exported with CUDA IPC.  Each process
 * exports its local stages' blobs, exchanges them (any transport), and connects
 * every remote stage adjacent to one of its own.  Ordering between processes is
 * GPU-side (sequence flags), so the host still never waits. */
#define P2BW_STAGE_BLOB_BYTES 128
int p2bw_engine_is_local(p2bw_engine* eng, int stage, int* out);
int p2bw_engine_export_stage(p2bw_engine* eng, int stage, void* blob, size_t bytes);
int p2bw_engine_connect_stage(p2bw_engine* eng, const void* blob, size_t bytes);
int p2bw_engine_sync(p2bw_engine* eng);
/* Measured timeline.  With tracing on, every op the engine
 * issues is bracketed by CUDA events on its stage stream (set before begin / run).
 * trace_report renders the last run as the reference's SimReport document
 * (report_to_json, simulator.cpp:356-390): timeline entries per worker in seconds,
 * throughput / steady_batch_time / bubble_fraction computed as simulate() does
 * (simulator.cpp:298-329) but from measured times, and per-op memory samples
 * (live versions, stashes, bytes).  Free with p2bw_free. */
int p2bw_engine_set_trace(p2bw_engine* eng, int on);
int p2bw_engine_trace_report(p2bw_engine* eng, char** out_json);
int p2bw_engine_counters(p2bw_engine* eng, p2bw_counters* out);
/* Weights created by a stage's update_index-th update of the last run (snapshots on). */
int p2bw_engine_read_snapshot(p2bw_engine* eng, int stage, int update_index, void* host,
                              size_t bytes);
/* A live weight version of a stage (at most 2 under 2BW). */
int p2bw_engine_read_version(p2bw_engine* eng, int stage, int version, void* host, size_t bytes);
/* fp32 master weights of a stage (transformer: the latest version, unrounded). */
int p2bw_engine_read_master(p2bw_engine* eng, int stage, void* host, size_t bytes);
/* Stream-ordered async copy of fp32 losses into (pinned) host memory; no sync. */
int p2bw_engine_losses_async(p2bw_engine* eng, int first_mb, int count, float* host);
/* Training losses of microbatches [first_mb, first_mb+count) (last stage). */
int p2bw_engine_losses(p2bw_engine* eng, int first_mb, int count, double* out);

/* ---- B200 block profiler -> planner ------------------- */

/* Times every block of the transformer described by *desc (one layer per block;
 * the embedding folds into block 0, LNf + LM head + loss into the last block) on
 * the current device at each microbatch size, running the stage executor's own
 * Forward / Backward kernels, and returns the profile document the reference's
 * load_model_profile reads (profile.cpp:162-193; fwd_ms / bwd_ms / weight_bytes /
 * act_*_bytes keyed by microbatch size).  Feed it to p2bw_plan.  Free with p2bw_free. */
int p2bw_profile_blocks(const p2bw_desc* desc, const int* microbatch_sizes, int n_sizes, int warmup,
                        int iters, const char* name, char** out_json);

/* ---- measurement --------------------------------------------------------- */

/* Kernels launched by this library since load (all stage kernels count). */
long long p2bw_launch_count(void);
/* Per-launch CUDA-event timing of every stage kernel, grouped by class. */
void p2bw_profile_enable(int on);
typedef struct {
    char name[32];
    long long launches;
    double ms;     /* summed device time of the class's launches */
    double flops;  /* algorithmic FLOPs (GEMM / attention) */
    double bytes;  /* algorithmic HBM bytes (memory-bound kernels) */
} p2bw_kernel_class;
/* Waits for and folds the recorded launches into classes (clears them). */
int p2bw_profile_collect(p2bw_kernel_class* out, int cap, int* n);

/* ---- stage kernels (parity-test hooks; device pointers, CUDA stream) ------- */

/* Epilogue of p2bw_kernel_gemm_bf16. kind: 0 = bf16 store with optional
 * bias / GELU (pre-activation copy in preact) / residual; 1 = fp32
 * D = beta*D + alpha*acc (wgrad accumulation, semantics.cpp:329);
 * 2 = bf16 D = alpha*acc*gelu'(aux). */
typedef struct {
    int kind;
    void* d;
    long long ldd;
    const void* bias;
    const void* residual;
    long long ldr;
    void* preact;
    int gelu;
    const void* aux;
    float alpha;
    float beta;
    /* Optional fp32 workspace of >= m*n floats (NULL: none).  Lets a plain bf16 store
     * (kind 0 without bias / GELU / residual) with few output tiles and a long K run
     * split-K into it and be cast to bf16 afterwards. */
    void* workspace;
    long long workspace_floats;
    /* Optional: the bias gradient of the layer whose output gradient A is, summed
     * from the A tiles the GEMM already stages in SMEM.  MN-major A (the wgrad, kind 1):
     * bias_grad[r] (=|+=) sum over K of A[r, :], bias_scratch >= (K / 512 + 1) * m
     * floats.  K-major A (the dgrad, any kind): bias_grad[c] (=|+=) sum over M of
     * A[:, c], bias_scratch >= 2 * ceil(m / 128) * k floats. */
    void* bias_grad;
    int bias_grad_accumulate;
    void* bias_scratch;
    long long bias_scratch_floats;
} p2bw_gemm_epilogue;

/* D[m x n] = A[m x k] . B[n x k]^T on tcgen05 tensor cores (bf16 in, fp32 acc).
 * major 0: element (r,k) at ptr[r*ld+k]; major 1: at ptr[k*ld+r].
 * Replaces matmul / matmul_tn / matmul_nt (semantics.hpp:23-25). */
int p2bw_kernel_gemm_bf16(const void* a, long long lda, int a_major, const void* b,
                          long long ldb, int b_major, int m, int n, int k,
                          const p2bw_gemm_epilogue* epi, void* stream);

/* Attention over qkv [b*seq x 3h] (heads of 64): o [b*seq x h], lse [b*heads*seq] fp32. */
int p2bw_kernel_attention_fwd(const void* qkv, void* o, void* lse, int batch, int seq, int heads,
                              int causal, void* stream);
/* dqkv [b*seq x 3h] from dO; delta scratch [b*heads*seq] fp32. */
int p2bw_kernel_attention_bwd(const void* qkv, const void* o, const void* dout, const void* lse,
                              void* dqkv, void* delta, int batch, int seq, int heads, int causal,
                              void* stream);
/* The same for heads of head_dim = 64 or 128 columns (h = heads * head_dim). */
int p2bw_kernel_attention_fwd_hd(const void* qkv, void* o, void* lse, int batch, int seq, int heads,
                                 int head_dim, int causal, void* stream);
int p2bw_kernel_attention_bwd_hd(const void* qkv, const void* o, const void* dout, const void* lse,
                                 void* dqkv, void* delta, int batch, int seq, int heads, int head_dim,
                                 int causal, void* stream);
/* LayerNorm forward / backward (bf16 rows, fp32 stats and parameter gradients). */
int p2bw_kernel_layernorm_fwd(const void* x, const void* g, const void* b, void* y, void* mean,
                              void* rstd, int rows, int h, void* stream);
/* dsum (optional, fp32 [h]): (=|+=) column sums of bf16(dx), the fused bias gradient
 * of the layer whose output gradient dx is.  dx may alias dy. */
int p2bw_kernel_layernorm_bwd(const void* dy, const void* x, const void* mean, const void* rstd,
                              const void* g, const void* dres, void* dx, void* dg, void* db, void* dsum,
                              int overwrite, int rows, int h, void* stream);
/* Debug: per-CTA phase clocks of the tcgen05 attention forward (16 uint64 per CTA)
 * and backward (64 uint64 per CTA) into a device buffer (NULL switches it off). */
int p2bw_debug_attention_timing(void* dev_buf);
/* Debug: per-CTA phase timestamps (%globaltimer ns) of the tcgen05 GEMM, 8 uint64 per
 * CTA: entry, setup done, last load issued, first stage consumed, last MMA commit,
 * first accumulator seen by the epilogue, epilogue done, teardown done (NULL = off). */
int p2bw_debug_gemm_timing(void* dev_buf);
/* Debug: the launch plan p2bw_kernel_gemm_bf16 makes for a shape (epilogue kind as in
 * p2bw_gemm_epilogue, bias_grad != 0 for a fused bias gradient): out[4] = {BN, CTAs per
 * cluster, split-K slices, tail-split K parts (1 = none)}.  The tail split runs the
 * ragged last wave's tiles as K parts on idle SMs with an in-kernel fp32 fixup;
 * P2BW_GEMM_TAIL=0 disables it. */
int p2bw_debug_gemm_plan(int m, int n, int k, int a_major, int b_major, int kind, int bias_grad, int* out);
/* Column sums of a bf16 matrix (bias gradients): out (=|+=) sum_r x[r, :]. */
int p2bw_kernel_colsum(const void* x, int rows, int n, int ld, void* out, int overwrite, void* stream);
/* Fused softmax cross-entropy: logits [rows x vp] -> dlogits in place, row_loss [rows]. */
int p2bw_kernel_softmax_xent(void* logits, const void* targets, int rows, int vocab, int vp,
                             float grad_scale, void* row_loss, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* P2BW_H */
