// Linear-chain stage (the reference ToyModel, semantics.hpp:31-43) on the
// PRODUCTION path: bf16 weights / activations on the tcgen05 GEMM (gemm.cu),
// fp32 master / momentum / coalesced gradient, the fused optimizer k_sgd writing
// the next bf16 version into the alternate buffer, and the transformer stage's
// streams (Forward stream, weight-gradient side stream, update stream).  It is
// the one model the reference itself pins numerically, so it ties the benched
// kernels to pipesim::pipelined_execute (semantics.cpp:238-375) within a bf16
// tolerance (tests/test_linear_bf16_gpu.py).
//
//   Forward   semantics.cpp:278-299   cur = W_l cur per layer (stash each input)
//   loss      semantics.cpp:312-319   g = (out - y) / b, loss = sum (out - y)^2 / (2b)
//   Backward  semantics.cpp:320-334   grad_sum[l] += g in_l^T (wgrad GEMM epilogue:
//                                     beta 0 on the batch's first microbatch, TMA
//                                     reduce-add afterwards); g = W_l^T g except at
//                                     stage 0 / layer 0 (:330)
//   Update    semantics.cpp:153-165, 335-350   v = beta v + (1-beta) grad/count;
//                                     w -= lr v; next bf16 version = bf16(w)
//
// Layout: the reference Mat is column-major dim x cols (semantics.hpp:12-21), which
// is a row-major [cols x dim] matrix with one sample per row -- the GEMM's
// activation layout as is.  Weights stay column-major on the device too (fp32
// master, bf16 versions): the forward reads W as an MN-major B operand, the dgrad
// as a K-major one, and the wgrad's [dim x dim] row-major output is exactly the
// column-major dW.  No transposes are materialised.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "engine.h"
#include "profiler.h"
#include "ptx.cuh"
#include "tkernels.h"

namespace p2bw {
namespace {

constexpr int kLossBlocks = 296;  // 2 x 148 SMs: fixed, so the loss sum order is fixed

int grid_1d(size_t n) { return static_cast<int>(std::min<size_t>((n + 255) / 256, 148u * 32u)); }

__global__ void k_f64_to_bf16(const double* __restrict__ in, bf16* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        out[i] = __float2bfloat16_rn(static_cast<float>(in[i]));
}

__global__ void k_f64_to_f32(const double* __restrict__ in, float* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<float>(in[i]);
}

__global__ void k_f32_to_f64(const float* __restrict__ in, double* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<double>(in[i]);
}

__global__ void k_bf16_to_f64(const bf16* __restrict__ in, double* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<double>(__bfloat162float(in[i]));
}

// ToyModel::make on the device (semantics.cpp:64-109): draw `skip + i + 1` of
// splitmix64(seed), as a double in [-0.5, 0.5), times `scale`, plus 1 where i is on
// the diagonal of a column-major square matrix (i % diag_stride == 0; 0 = none), then
// rounded once to the stored type.  The integer stream and the fp64 arithmetic are the
// reference's, so the values are its own rounded to fp32 / bf16.
template <class T>
__global__ void k_toy_uniform(T* __restrict__ out, size_t n, unsigned long long seed, unsigned long long skip,
                              double scale, unsigned long long diag_stride) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        unsigned long long z = seed + (skip + i + 1) * 0x9e3779b97f4a7c15ULL;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        z ^= z >> 31;
        double v = (static_cast<double>(z >> 11) * (1.0 / 9007199254740992.0) - 0.5) * scale;
        if (diag_stride != 0 && i % diag_stride == 0) v += 1.0;
        if constexpr (sizeof(T) == 4) out[i] = static_cast<float>(v);
        else out[i] = __float2bfloat16_rn(static_cast<float>(v));
    }
}

// Quadratic loss and its gradient (semantics.cpp:312-319) from the fp32 network
// output: g = bf16((out - y) / b); part[block] = this block's share of
// sum (out - y)^2 / (2b).  Four elements per thread (n % 4 == 0), fixed grid.
__global__ void __launch_bounds__(256) k_lin_loss(const float4* __restrict__ out, const float4* __restrict__ y,
                                                  uint2* __restrict__ g, float* __restrict__ part, size_t n4,
                                                  float inv_b) {
    float acc = 0.0f;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const float4 o = out[i], t = y[i];
        const float d0 = o.x - t.x, d1 = o.y - t.y, d2 = o.z - t.z, d3 = o.w - t.w;
        acc += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
        g[i] = make_uint2(ptx::pack_bf16x2(d0 * inv_b, d1 * inv_b), ptx::pack_bf16x2(d2 * inv_b, d3 * inv_b));
    }
    __shared__ float red[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        float s = 0.0f;
        for (int w = 0; w < 8; ++w) s += red[w];
        part[blockIdx.x] = s * (0.5f * inv_b);
    }
}

class LinearBF16Stage final : public StageModel {
public:
    LinearBF16Stage(const EngineConfig& cfg, int stage, int lo, int hi, int sslots, int wslots)
        : cfg_(cfg), n_(cfg.dim), cols_(cfg.microbatch_size), lo_(lo), layers_(hi - lo), stage0_(stage == 0),
          stageL_(stage == cfg.depth - 1), sslots_(sslots), wslots_(wslots) {
        if (n_ < 32 || n_ % 32 != 0) throw Error("bf16 linear chain: dim must be a multiple of 32");
        if (cols_ < 8 || cols_ % 8 != 0) throw Error("bf16 linear chain: microbatch columns must be a multiple of 8");
        mat_ = static_cast<size_t>(n_) * n_;
        act_ = static_cast<size_t>(n_) * cols_;
        nparam_ = static_cast<size_t>(layers_) * mat_;
        master_ = dalloc<float>(nparam_);
        vel_ = dalloc<float>(nparam_);
        grad_ = grad_bufs_[0] = dalloc<float>(nparam_);
        for (int i = 0; i < wslots_; ++i) wbf_.push_back(dalloc<bf16>(nparam_));
        staging_ = dalloc<double>(nparam_);
        check_cuda(cudaMemset(vel_, 0, nparam_ * sizeof(float)), "memset");
        check_cuda(cudaMemset(grad_, 0, nparam_ * sizeof(float)), "memset");
        stash_ = dalloc<bf16>(static_cast<size_t>(sslots_) * layers_ * act_);
        gtmp_[0] = dalloc<bf16>(act_);
        gtmp_[1] = dalloc<bf16>(act_);
        rc_out_ = dalloc<bf16>(act_);
        if (stageL_) {
            out32_ = dalloc<float>(act_);
            gloss_ = dalloc<bf16>(static_cast<size_t>(sslots_) * act_);
            lpart_ = dalloc<float>(kLossBlocks);
        }
        xin_.assign(static_cast<size_t>(sslots_), nullptr);
        side_stream_ = make_stage_stream("side");
        for (cudaEvent_t& e : ev_) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    }

    ~LinearBF16Stage() override {
        if (side_stream_) cudaStreamSynchronize(side_stream_);
        for (cudaEvent_t e : ev_)
            if (e) cudaEventDestroy(e);
        if (side_stream_) cudaStreamDestroy(side_stream_);
        for (void* p : allocs_) cudaFree(p);
        for (void* p : {static_cast<void*>(x_), static_cast<void*>(y_), static_cast<void*>(loss_),
                        static_cast<void*>(dstage_)})
            cudaFree(p);
    }

    size_t num_params() const override { return nparam_; }
    size_t boundary_bytes() const override { return act_ * sizeof(bf16); }
    size_t weight_bytes_public() const override { return nparam_ * sizeof(double); }
    double version_bytes() const override { return static_cast<double>(nparam_) * sizeof(bf16); }
    double stash_bytes() const override { return static_cast<double>(layers_) * act_ * sizeof(bf16); }
    int data_capacity() const override { return capacity_; }
    void bind_stream(cudaStream_t s) override { stream_ = s; }
    void bind_data_stream(cudaStream_t s) override { data_stream_ = s; }
    bool enable_grad_double_buffer() override {
        if (!grad_bufs_[1]) {
            grad_bufs_[1] = dalloc<float>(nparam_);
            check_cuda(cudaMemset(grad_bufs_[1], 0, nparam_ * sizeof(float)), "memset");
        }
        return true;
    }
    void grad_buffer(void** ptr, size_t* count, int* dtype) override {
        *ptr = grad_;
        *count = nparam_;
        *dtype = 0;
    }

    std::vector<void*> replica_buffers() override {
        std::vector<void*> v{grad_bufs_[0], grad_bufs_[1], master_};
        for (bf16* w : wbf_) v.push_back(w);
        return v;
    }
    void update_replicas(int src_slot, int dst_slot, int grad_count, const std::vector<std::vector<void*>>& peers,
                         int rank, cudaStream_t s) override {
        (void)src_slot;
        ReplicaShard r;
        r.w = static_cast<int>(peers.size());
        r.rank = rank;
        for (int q = 0; q < r.w && q < kMaxReplicas; ++q) {
            r.grad[q] = static_cast<const float*>(peers[q].at(static_cast<size_t>(grad_cur_)));
            r.master[q] = static_cast<float*>(peers[q].at(2));
            r.version[q] = static_cast<bf16*>(peers[q].at(3 + static_cast<size_t>(dst_slot)));
        }
        sgd_momentum_update_replicas(r, vel_, nparam_, 1.0f / static_cast<float>(grad_count),
                                     static_cast<float>(cfg_.lr), static_cast<float>(cfg_.momentum), s);
        if (grad_bufs_[1]) {
            grad_cur_ ^= 1;
            grad_ = grad_bufs_[grad_cur_];
        }
    }

    // Public layout: fp64 column-major matrices of the stage's layers (like LinearF64Stage).
    void load_weights(int wslot, const void* host, size_t bytes) override {
        if (bytes != weight_bytes_public()) throw Error("load_weights: size mismatch");
        check_cuda(cudaStreamSynchronize(stream_), "sync");
        // stream-ordered: a pageable cudaMemcpy may return before its DMA lands, and the
        // conversion below runs on a non-blocking stream that would not wait for it
        check_cuda(cudaMemcpyAsync(staging_, host, bytes, cudaMemcpyHostToDevice, stream_), "H2D W");
        k_f64_to_f32<<<grid_1d(nparam_), 256, 0, stream_>>>(staging_, master_, nparam_);
        cast_f32_bf16(master_, wbf_[static_cast<size_t>(wslot)], nparam_, stream_);
        check_cuda(cudaMemsetAsync(vel_, 0, nparam_ * sizeof(float), stream_), "memset vel");
        check_cuda(cudaStreamSynchronize(stream_), "load sync");
    }
    // A bf16 weight version, widened to fp64.
    void read_weights(int wslot, void* host, size_t bytes, cudaStream_t s) override {
        if (bytes != weight_bytes_public()) throw Error("read_weights: size mismatch");
        k_bf16_to_f64<<<grid_1d(nparam_), 256, 0, s>>>(wbf_[static_cast<size_t>(wslot)], staging_, nparam_);
        check_cuda(cudaMemcpyAsync(host, staging_, bytes, cudaMemcpyDeviceToHost, s), "D2H W");
        check_cuda(cudaStreamSynchronize(s), "read sync");
    }
    // Trajectory snapshots are the fp32 master (the weights the update produced; the
    // bf16 version is its rounding), widened to fp64.
    void snapshot_weights(int wslot, void* host, size_t bytes, cudaStream_t s) override {
        (void)wslot;
        if (bytes != weight_bytes_public()) throw Error("snapshot: size mismatch");
        k_f32_to_f64<<<grid_1d(nparam_), 256, 0, s>>>(master_, staging_, nparam_);
        check_cuda(cudaMemcpyAsync(host, staging_, bytes, cudaMemcpyDeviceToHost, s), "D2H master");
        check_cuda(cudaStreamSynchronize(s), "snapshot sync");
    }
    void read_master(void* host, size_t bytes) override { snapshot_weights(0, host, bytes, stream_); }

    void read_losses(double* host, int first_mb, int count, cudaStream_t s) override {
        if (!stageL_) throw Error("this stage computes no loss");
        if (capacity_ == 0) throw Error("no data has been set");
        std::vector<float> tmp(static_cast<size_t>(capacity_));
        check_cuda(cudaMemcpyAsync(tmp.data(), loss_, sizeof(float) * capacity_, cudaMemcpyDeviceToHost, s), "D2H loss");
        check_cuda(cudaStreamSynchronize(s), "loss sync");
        for (int i = 0; i < count; ++i) host[i] = tmp[static_cast<size_t>((first_mb - 1 + i) % capacity_)];
    }
    void copy_losses_async(float* host, int first_mb, int count, cudaStream_t s) override {
        if (!stageL_ || capacity_ == 0) throw Error("this stage computes no loss");
        for (int i = 0; i < count;) {
            const int slot = (first_mb - 1 + i) % capacity_;
            const int run = std::min(count - i, capacity_ - slot);
            check_cuda(cudaMemcpyAsync(host + i, loss_ + slot, sizeof(float) * run, cudaMemcpyDeviceToHost, s),
                       "D2H loss");
            i += run;
        }
    }

    // Initial weights W_l = I + 0.2 U of the stage's layers [lo, hi), drawn at the
    // offsets ToyModel::make gives them (layer l's matrix is draws l*dim^2 + 1 ...).
    void init_weights(uint64_t seed) override {
        for (int l = 0; l < layers_; ++l)
            k_toy_uniform<float><<<grid_1d(mat_), 256, 0, stream_>>>(master_ + static_cast<size_t>(l) * mat_, mat_, seed,
                                                                  static_cast<unsigned long long>(lo_ + l) * mat_, 0.2,
                                                                  static_cast<unsigned long long>(n_) + 1);
        check_cuda(cudaGetLastError(), "toy init");
        cast_f32_bf16(master_, wbf_[0], nparam_, stream_);
        check_cuda(cudaMemsetAsync(vel_, 0, nparam_ * sizeof(float), stream_), "memset vel");
        check_cuda(cudaStreamSynchronize(stream_), "init sync");
    }

    // Microbatches [first_mb, first_mb + count) of ToyModel::make's dataset generated in
    // place: x = U (dim x b) at draws (L+1) dim^2 + (k-1) dim b + 1 ...; y = A x with the
    // hidden map A = I + 0.3 U (draws L dim^2 + 1 ...) formed by the bf16 GEMM (fp32 out).
    // The x values are the reference's (rounded to bf16); y carries the GEMM's rounding.
    void make_toy_data(uint64_t seed, int first_mb, int count) override {
        if (count < 1) throw Error("toy data: empty microbatch range");
        const cudaStream_t ds = data_stream_ ? data_stream_ : stream_;
        ensure_ring(count, ds);
        const unsigned long long L = static_cast<unsigned long long>(cfg_.layers);
        bf16 *xs = nullptr, *a = nullptr;
        if (stageL_) {
            check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&a), mat_ * sizeof(bf16), ds), "cudaMallocAsync");
            check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&xs), act_ * sizeof(bf16), ds), "cudaMallocAsync");
            k_toy_uniform<bf16><<<grid_1d(mat_), 256, 0, ds>>>(a, mat_, seed, L * mat_, 0.3,
                                                                static_cast<unsigned long long>(n_) + 1);
        }
        for (int i = 0; i < count; ++i) {
            const int k = first_mb + i, slot = (k - 1) % capacity_;
            const unsigned long long skip = (L + 1) * mat_ + static_cast<unsigned long long>(k - 1) * act_;
            bf16* x = stage0_ ? x_ + static_cast<size_t>(slot) * act_ : xs;
            if (stage0_ || stageL_) k_toy_uniform<bf16><<<grid_1d(act_), 256, 0, ds>>>(x, act_, seed, skip, 1.0, 0);
            if (stageL_) {
                GemmEpilogue e;
                e.kind = EpiKind::StoreF32;
                e.d = y_ + static_cast<size_t>(slot) * act_;
                e.ldd = n_;
                gemm_bf16({x, n_, Major::K}, {a, n_, Major::MN}, cols_, n_, n_, e, ds);
            }
        }
        check_cuda(cudaGetLastError(), "toy data");
        if (a) check_cuda(cudaFreeAsync(a, ds), "cudaFreeAsync");
        if (xs) check_cuda(cudaFreeAsync(xs, ds), "cudaFreeAsync");
    }

    // inputs / targets: fp64 [count][dim * b] column-major (ToyModel::dataset), like the
    // fp64 stage.  They land in a ring of max(count, 2m) microbatches (x as bf16, y as
    // fp32), so a caller may stream batch after batch like the transformer's token ring.
    void set_data(const void* inputs, const void* targets, int first_mb, int count) override {
        if (count < 1) throw Error("set_data: empty microbatch range");
        const cudaStream_t ds = data_stream_ ? data_stream_ : stream_;
        ensure_ring(count, ds);
        if (static_cast<size_t>(count) > dstage_mb_) {  // fp64 staging for the conversion
            check_cuda(cudaStreamSynchronize(ds), "sync");
            cudaFree(dstage_);
            check_cuda(cudaMalloc(&dstage_, static_cast<size_t>(count) * act_ * sizeof(double)), "cudaMalloc(stage)");
            dstage_mb_ = static_cast<size_t>(count);
        }
        for (int pass = 0; pass < 2; ++pass) {
            const void* src = pass == 0 ? inputs : targets;
            if (src == nullptr) continue;
            check_cuda(cudaMemcpyAsync(dstage_, src, static_cast<size_t>(count) * act_ * sizeof(double),
                                       cudaMemcpyHostToDevice, ds), "H2D data");
            for (int i = 0; i < count;) {  // contiguous ring runs
                const int slot = (first_mb - 1 + i) % capacity_;
                const int run = std::min(count - i, capacity_ - slot);
                const size_t n = static_cast<size_t>(run) * act_;
                const double* from = dstage_ + static_cast<size_t>(i) * act_;
                if (pass == 0) k_f64_to_bf16<<<grid_1d(n), 256, 0, ds>>>(from, x_ + static_cast<size_t>(slot) * act_, n);
                else k_f64_to_f32<<<grid_1d(n), 256, 0, ds>>>(from, y_ + static_cast<size_t>(slot) * act_, n);
                i += run;
            }
            check_cuda(cudaGetLastError(), "set_data convert");
        }
    }

    void forward(int k, int wslot, int sslot, const void* x_in, void* x_out, cudaStream_t s) override {
        const bf16* W = wbf_[static_cast<size_t>(wslot)];
        const bf16* cur = stage0_ ? data_x(k) : static_cast<const bf16*>(x_in);
        xin_[static_cast<size_t>(sslot)] = cur;
        for (int l = 0; l < layers_; ++l) {
            const bf16* wl = W + static_cast<size_t>(l) * mat_;
            GemmEpilogue e;
            e.ldd = n_;
            if (l + 1 == layers_ && stageL_) {  // network output in fp32 for the loss
                e.kind = EpiKind::StoreF32;
                e.d = out32_;
                e.beta = 0.0f;
            } else {
                e.kind = EpiKind::StoreBF16;
                e.d = l + 1 < layers_ ? stash_ptr(sslot, l + 1) : static_cast<bf16*>(x_out);
            }
            // Y[c][i] = sum_k X[c][k] W(i, k): A = X (K-major), B(i, k) = W at k*dim + i (MN-major)
            gemm_bf16({cur, n_, Major::K}, {wl, n_, Major::MN}, cols_, n_, n_, e, s);
            cur = static_cast<const bf16*>(e.d);
        }
        if (stageL_) {
            prof::Scope scope("linear_loss", 0.0, 10.0 * static_cast<double>(act_), 2, s);
            k_lin_loss<<<kLossBlocks, 256, 0, s>>>(reinterpret_cast<const float4*>(out32_),
                                                   reinterpret_cast<const float4*>(data_y(k)),
                                                   reinterpret_cast<uint2*>(gloss_ + static_cast<size_t>(sslot) * act_),
                                                   lpart_, act_ / 4, 1.0f / static_cast<float>(cols_));
            check_cuda(cudaGetLastError(), "linear loss");
            sum_scaled(lpart_, kLossBlocks, 1.0f, loss_ + (k - 1) % capacity_, s);
        }
    }

    void recompute(int k, int wslot, int sslot, const void* x_in, cudaStream_t s) override {
        forward(k, wslot, sslot, x_in, stageL_ ? nullptr : rc_out_, s);
    }

    void backward(int k, int wslot, int sslot, const void* g_in, void* g_out, bool first,
                  cudaStream_t s) override {
        (void)k;
        const bf16* W = wbf_[static_cast<size_t>(wslot)];
        const float beta = first ? 0.0f : 1.0f;
        const bf16* g = stageL_ ? gloss_ + static_cast<size_t>(sslot) * act_ : static_cast<const bf16*>(g_in);
        // weight gradients on the side stream (off the dgrad chain's critical path), as
        // in the transformer stage; per-launch profiling keeps them on the stage stream
        side_ = prof::enabled() ? s : side_stream_;
        // ev_[0 / 1] were last recorded by the previous backward (joined at its end): re-record
        // them after a fork so the first wait below refers to this backward (CUDA-graph capture)
        fork(s);
        for (int e = 0; e < 2; ++e) check_cuda(cudaEventRecord(ev_[e], side_), "cudaEventRecord(side)");
        int flip = 0;
        for (int l = layers_ - 1; l >= 0; --l) {
            const bf16* in = l == 0 ? xin_[static_cast<size_t>(sslot)] : stash_ptr(sslot, l);
            fork(s);  // g is ready
            GemmEpilogue w;
            w.kind = EpiKind::StoreF32;
            w.d = grad_ + static_cast<size_t>(l) * mat_;
            w.ldd = n_;
            w.beta = beta;
            // dW[j][i] (= column-major dW(i, j)) = sum_c in[c][j] g[c][i]: A = in, B = g, both MN-major
            gemm_bf16({in, n_, Major::MN}, {g, n_, Major::MN}, n_, n_, cols_, w, side_);
            check_cuda(cudaEventRecord(ev_[flip], side_), "cudaEventRecord(side)");
            if (l > 0 || !stage0_) {
                bf16* dst = l == 0 ? static_cast<bf16*>(g_out) : gtmp_[flip];
                // gtmp_[flip] was last read by the wgrad two layers up
                if (l != 0) check_cuda(cudaStreamWaitEvent(s, ev_[flip ^ 1], 0), "cudaStreamWaitEvent(side)");
                GemmEpilogue e;
                e.kind = EpiKind::StoreBF16;
                e.d = dst;
                e.ldd = n_;
                // G'[c][i] = sum_k G[c][k] W(k, i): B(i, k) = W at i*dim + k (K-major)
                gemm_bf16({g, n_, Major::K}, {W + static_cast<size_t>(l) * mat_, n_, Major::K}, cols_, n_, n_, e, s);
                g = dst;
                flip ^= 1;
            }
        }
        check_cuda(cudaEventRecord(ev_[2], side_), "cudaEventRecord(side)");
        check_cuda(cudaStreamWaitEvent(s, ev_[2], 0), "cudaStreamWaitEvent(side)");
    }

    void update(int src_slot, int dst_slot, int grad_count, cudaStream_t s) override {
        (void)src_slot;  // the fp32 master holds the latest version (semantics.cpp:341)
        sgd_momentum_update(master_, vel_, grad_, wbf_[static_cast<size_t>(dst_slot)], nparam_,
                            1.0f / static_cast<float>(grad_count), static_cast<float>(cfg_.lr),
                            static_cast<float>(cfg_.momentum), s);
        if (grad_bufs_[1]) {
            grad_cur_ ^= 1;
            grad_ = grad_bufs_[grad_cur_];
        }
    }

private:
    // The data ring: max(count of the first call, 2m) microbatches, like the transformer's.
    void ensure_ring(int count, cudaStream_t ds) {
        if (capacity_ == 0) {
            capacity_ = std::max(count, 2 * cfg_.microbatches);
            check_cuda(cudaMalloc(&x_, static_cast<size_t>(capacity_) * act_ * sizeof(bf16)), "cudaMalloc(x)");
            check_cuda(cudaMalloc(&y_, static_cast<size_t>(capacity_) * act_ * sizeof(float)), "cudaMalloc(y)");
            check_cuda(cudaMalloc(&loss_, static_cast<size_t>(capacity_) * sizeof(float)), "cudaMalloc(loss)");
            check_cuda(cudaMemsetAsync(loss_, 0, sizeof(float) * capacity_, ds), "memset loss");
        }
        if (count > capacity_) throw Error("set_data: more microbatches than the data ring holds");
    }

    template <class T>
    T* dalloc(size_t n) {
        void* p = nullptr;
        check_cuda(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc(linear bf16)");
        allocs_.push_back(p);
        return static_cast<T*>(p);
    }
    void fork(cudaStream_t s) {
        check_cuda(cudaEventRecord(ev_[3], s), "cudaEventRecord(fork)");
        check_cuda(cudaStreamWaitEvent(side_, ev_[3], 0), "cudaStreamWaitEvent(fork)");
    }
    bf16* stash_ptr(int slot, int l) const { return stash_ + (static_cast<size_t>(slot) * layers_ + l) * act_; }
    const bf16* data_x(int k) const {
        if (capacity_ == 0) throw Error("no input data has been set");
        return x_ + static_cast<size_t>((k - 1) % capacity_) * act_;
    }
    const float* data_y(int k) const {
        if (capacity_ == 0) throw Error("no target data has been set");
        return y_ + static_cast<size_t>((k - 1) % capacity_) * act_;
    }

    EngineConfig cfg_;
    int n_, cols_, lo_, layers_;
    bool stage0_, stageL_;
    int sslots_, wslots_;
    size_t mat_ = 0, act_ = 0, nparam_ = 0;
    cudaStream_t stream_ = nullptr, data_stream_ = nullptr;
    cudaStream_t side_stream_ = nullptr, side_ = nullptr;
    cudaEvent_t ev_[4] = {};
    std::vector<void*> allocs_;
    float *master_ = nullptr, *vel_ = nullptr, *grad_ = nullptr;
    float* grad_bufs_[2] = {nullptr, nullptr};
    int grad_cur_ = 0;
    std::vector<bf16*> wbf_;
    double* staging_ = nullptr;
    bf16* stash_ = nullptr;
    bf16* gtmp_[2] = {nullptr, nullptr};
    bf16* rc_out_ = nullptr;
    float* out32_ = nullptr;
    bf16* gloss_ = nullptr;
    float* lpart_ = nullptr;
    std::vector<const bf16*> xin_;
    int capacity_ = 0;
    bf16* x_ = nullptr;
    float* y_ = nullptr;
    float* loss_ = nullptr;
    double* dstage_ = nullptr;
    size_t dstage_mb_ = 0;
};

}  // namespace

std::unique_ptr<StageModel> make_linear_bf16_stage(const EngineConfig& cfg, int stage, int lo, int hi,
                                                    int stash_slots, int weight_slots) {
    return std::make_unique<LinearBF16Stage>(cfg, stage, lo, hi, stash_slots, weight_slots);
}

}  // namespace p2bw
