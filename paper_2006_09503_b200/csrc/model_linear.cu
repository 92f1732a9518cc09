// Linear-chain stage (the reference ToyModel, semantics.hpp:31-43) in fp64 on
// the GPU.  This is the engine's reference-pinned numeric mode: each output
// element is produced by one thread that accumulates in the reference's loop
// order with explicitly rounded (__dmul_rn / __dadd_rn, no FMA contraction)
// operations, so trajectories are bit-identical to pipesim::pipelined_execute.
//   matmul     semantics.cpp:9-19   Y(i,j)  = sum_k W(i,k) X(k,j)     (k ascending)
//   matmul_tn  semantics.cpp:21-32  G'(i,j) = sum_k W(k,i) G(k,j)
//   matmul_nt  semantics.cpp:34-44  T(i,j)  = sum_c G(i,c) X(j,c); grad += T (axpy :329)
//   loss grad  semantics.cpp:314-319  g = (out - y) / b
//   update     semantics.cpp:153-165, 335-350
// Layout: column-major dim x cols, exactly the reference Mat (semantics.hpp:12-21).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "engine.h"

namespace p2bw {
namespace {

constexpr int kThreads = 256;

int blocks_for(long n) { return static_cast<int>(std::min<long>((n + kThreads - 1) / kThreads, 65535L * 8)); }

// Y = W X  (W: n x n, X: n x c)
__global__ void k_matmul_nn(const double* __restrict__ w, const double* __restrict__ x,
                            double* __restrict__ y, int n, int c) {
    const long total = static_cast<long>(n) * c;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(idx % n), j = static_cast<int>(idx / n);
        double acc = 0.0;
        for (int k = 0; k < n; ++k) acc = __dadd_rn(acc, __dmul_rn(w[static_cast<long>(k) * n + i], x[static_cast<long>(j) * n + k]));
        y[idx] = acc;
    }
}

// Y = W^T G  (W: n x n, G: n x c)
__global__ void k_matmul_tn(const double* __restrict__ w, const double* __restrict__ g,
                            double* __restrict__ y, int n, int c) {
    const long total = static_cast<long>(n) * c;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(idx % n), j = static_cast<int>(idx / n);
        double acc = 0.0;
        for (int k = 0; k < n; ++k) acc = __dadd_rn(acc, __dmul_rn(w[static_cast<long>(i) * n + k], g[static_cast<long>(j) * n + k]));
        y[idx] = acc;
    }
}

// grad (=|+=) scale * G X^T  (G, X: n x c; grad: n x n).  The product is formed first
// and then added, like axpy(1.0, matmul_nt(g, in), grad_sum) (semantics.cpp:329), or
// axpy(1.0 / m, ...) in reference_loop (semantics.cpp:145) when scale != 1.
__global__ void k_wgrad_nt(const double* __restrict__ g, const double* __restrict__ x,
                           double* __restrict__ grad, int n, int c, int overwrite, double scale) {
    const long total = static_cast<long>(n) * n;
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(idx % n), j = static_cast<int>(idx / n);
        double acc = 0.0;
        for (int k = 0; k < c; ++k) acc = __dadd_rn(acc, __dmul_rn(g[static_cast<long>(k) * n + i], x[static_cast<long>(k) * n + j]));
        if (scale != 1.0) acc = __dmul_rn(scale, acc);
        grad[idx] = overwrite ? __dadd_rn(0.0, acc) : __dadd_rn(grad[idx], acc);
    }
}

// g = (out - y) / b   (semantics.cpp:314-319)
__global__ void k_loss_grad(const double* __restrict__ out, const double* __restrict__ y,
                            double* __restrict__ g, long total, double b) {
    for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long>(gridDim.x) * blockDim.x)
        g[idx] = __ddiv_rn(__dsub_rn(out[idx], y[idx]), b);
}

// loss = sum (out - y)^2 / (2b), one block, fixed summation order (deterministic).
__global__ void k_loss(const double* __restrict__ out, const double* __restrict__ y, long total,
                       double b, double* __restrict__ loss) {
    __shared__ double part[kThreads];
    double acc = 0.0;
    for (long i = threadIdx.x; i < total; i += kThreads) {
        const double diff = out[i] - y[i];
        acc += diff * diff / (2.0 * b);
    }
    part[threadIdx.x] = acc;
    __syncthreads();
    for (int w = kThreads / 2; w > 0; w >>= 1) {
        if (static_cast<int>(threadIdx.x) < w) part[threadIdx.x] += part[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *loss = part[0];
}

// v = beta v + (1-beta) (gsum / count);  W_dst = W_src + (-lr) v
__global__ void k_update(const double* __restrict__ wsrc, double* __restrict__ wdst,
                         double* __restrict__ vel, const double* __restrict__ gsum, long total,
                         double count, double lr, double beta) {
    for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long>(gridDim.x) * blockDim.x) {
        const double g = __ddiv_rn(gsum[i], count);
        const double v = __dadd_rn(__dmul_rn(beta, vel[i]), __dmul_rn(__dsub_rn(1.0, beta), g));
        vel[i] = v;
        wdst[i] = __dadd_rn(wsrc[i], __dmul_rn(-lr, v));
    }
}

// Data-parallel replicas (Engine::join_replicas_ipc): the AllReduce fused into the
// update.  This replica owns elements [lo, hi); gsum is the replicas' sum in replica
// order, then k_update's arithmetic; the new weights go to every replica's dst slot.
constexpr int kMaxRep = 8;
struct F64Peers {
    const double* g[kMaxRep];
    double* wdst[kMaxRep];
};
__global__ void k_update_replicas(F64Peers p, int nrep, const double* __restrict__ wsrc, double* __restrict__ vel,
                                  long lo, long hi, double count, double lr, double beta) {
    for (long i = lo + blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < hi;
         i += static_cast<long>(gridDim.x) * blockDim.x) {
        double gs = p.g[0][i];
        for (int q = 1; q < nrep; ++q) gs = __dadd_rn(gs, p.g[q][i]);
        const double g = __ddiv_rn(gs, count);
        const double v = __dadd_rn(__dmul_rn(beta, vel[i]), __dmul_rn(__dsub_rn(1.0, beta), g));
        vel[i] = v;
        const double w = __dadd_rn(wsrc[i], __dmul_rn(-lr, v));
        for (int q = 0; q < nrep; ++q) p.wdst[q][i] = w;
    }
}

class LinearF64Stage final : public StageModel {
public:
    LinearF64Stage(const EngineConfig& cfg, int stage, int lo, int hi, int sslots, int wslots)
        : n_(cfg.dim), cols_(cfg.microbatch_size), layers_(hi - lo), stage0_(stage == 0),
          stageL_(stage == cfg.depth - 1), sslots_(sslots), wslots_(wslots), lr_(cfg.lr),
          beta_(cfg.momentum), loop_scale_(cfg.loop_scaling ? 1.0 / cfg.microbatches : 1.0),
          loop_scaling_(cfg.loop_scaling) {
        if (n_ < 1 || cols_ < 1) throw Error("toy model dimensions must be >= 1");
        mat_ = static_cast<size_t>(n_) * n_;
        act_ = static_cast<size_t>(n_) * cols_;
        alloc(&w_, static_cast<size_t>(wslots_) * layers_ * mat_);
        alloc(&vel_, layers_ * mat_);
        alloc(&gsum_, layers_ * mat_);
        alloc(&stash_, static_cast<size_t>(sslots_) * layers_ * act_);
        alloc(&gtmp_, 2 * act_);
        if (stageL_) alloc(&out_, static_cast<size_t>(sslots_) * act_);
        check_cuda(cudaMemset(vel_, 0, layers_ * mat_ * sizeof(double)), "cudaMemset");
        xin_.assign(static_cast<size_t>(sslots_), nullptr);
    }
    ~LinearF64Stage() override {
        for (double* p : {w_, vel_, gsum_, stash_, gtmp_, out_, x_, y_, loss_}) cudaFree(p);
    }

    size_t num_params() const override { return layers_ * mat_; }
    void grad_buffer(void** ptr, size_t* count, int* dtype) override {
        *ptr = gsum_;
        *count = layers_ * mat_;
        *dtype = 1;
    }
    size_t boundary_bytes() const override { return act_ * sizeof(double); }
    double stash_bytes() const override { return static_cast<double>(layers_) * act_ * sizeof(double); }
    size_t weight_bytes_public() const override { return layers_ * mat_ * sizeof(double); }
    int data_capacity() const override { return capacity_; }

    void bind_stream(cudaStream_t s) override { stream_ = s; }

    // Dataset microbatches [first_mb, first_mb + count).  Growing the buffers keeps the
    // microbatches already uploaded; the copies are ordered on the stage stream, so a
    // call between runs never races the kernels still reading the old contents.
    void set_data(const void* inputs, const void* targets, int first_mb, int count) override {
        if (count < 1) throw Error("set_data: empty microbatch range");
        if (first_mb + count - 1 > capacity_) {
            check_cuda(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
            const int cap = first_mb + count - 1;
            double *x = nullptr, *y = nullptr, *loss = nullptr;
            alloc(&x, static_cast<size_t>(cap) * act_);
            alloc(&y, static_cast<size_t>(cap) * act_);
            alloc(&loss, static_cast<size_t>(cap));
            check_cuda(cudaMemsetAsync(loss, 0, sizeof(double) * cap, stream_), "cudaMemset");
            if (capacity_ > 0) {
                const size_t keep = static_cast<size_t>(capacity_) * act_ * sizeof(double);
                check_cuda(cudaMemcpyAsync(x, x_, keep, cudaMemcpyDeviceToDevice, stream_), "D2D x");
                check_cuda(cudaMemcpyAsync(y, y_, keep, cudaMemcpyDeviceToDevice, stream_), "D2D y");
                check_cuda(cudaMemcpyAsync(loss, loss_, sizeof(double) * capacity_, cudaMemcpyDeviceToDevice, stream_), "D2D loss");
            }
            // stage 0's stash points into the dataset for in-flight microbatches: rebase it
            for (auto& p : xin_)
                if (p != nullptr && x_ != nullptr && p >= x_ && p < x_ + static_cast<size_t>(capacity_) * act_)
                    p = x + (p - x_);
            check_cuda(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
            for (double* p : {x_, y_, loss_}) cudaFree(p);
            x_ = x, y_ = y, loss_ = loss;
            capacity_ = cap;
        }
        const size_t off = static_cast<size_t>(first_mb - 1) * act_;
        const size_t bytes = static_cast<size_t>(count) * act_ * sizeof(double);
        if (inputs) check_cuda(cudaMemcpyAsync(x_ + off, inputs, bytes, cudaMemcpyHostToDevice, stream_), "H2D x");
        if (targets) check_cuda(cudaMemcpyAsync(y_ + off, targets, bytes, cudaMemcpyHostToDevice, stream_), "H2D y");
        check_cuda(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");  // host buffers are borrowed
    }

    void load_weights(int wslot, const void* host, size_t bytes) override {
        if (bytes != weight_bytes_public()) throw Error("load_weights: size mismatch");
        // stream-ordered: a pageable cudaMemcpy may return before its DMA lands, and the
        // stage's kernels run on a non-blocking stream
        check_cuda(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
        check_cuda(cudaMemcpyAsync(wslot_ptr(wslot, 0), host, bytes, cudaMemcpyHostToDevice, stream_), "H2D W");
        check_cuda(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
    }
    void read_weights(int wslot, void* host, size_t bytes, cudaStream_t s) override {
        if (bytes != weight_bytes_public()) throw Error("read_weights: size mismatch");
        check_cuda(cudaMemcpyAsync(host, wslot_ptr(wslot, 0), bytes, cudaMemcpyDeviceToHost, s), "D2H W");
        check_cuda(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    }
    void read_losses(double* host, int first_mb, int count, cudaStream_t s) override {
        if (!stageL_) throw Error("this stage computes no loss");
        if (first_mb < 1 || first_mb + count - 1 > capacity_) throw Error("loss index out of range");
        check_cuda(cudaMemcpyAsync(host, loss_ + first_mb - 1, sizeof(double) * count,
                                   cudaMemcpyDeviceToHost, s), "D2H loss");
    }

    // Recompute op: the forward again into the same stash slot (the output goes to a
    // scratch row block; the loss path reads out_).  Bit-identical by construction.
    void recompute(int k, int wslot, int sslot, const void* x_in, cudaStream_t s) override {
        forward(k, wslot, sslot, x_in, gtmp_, s);
    }

    void forward(int k, int wslot, int sslot, const void* x_in, void* x_out, cudaStream_t s) override {
        const double* cur = stage0_ ? data_x(k) : static_cast<const double*>(x_in);
        xin_[static_cast<size_t>(sslot)] = cur;
        for (int l = 0; l < layers_; ++l) {
            double* y;
            if (l + 1 < layers_) y = stash_ptr(sslot, l + 1);
            else y = stageL_ ? out_ + static_cast<size_t>(sslot) * act_ : static_cast<double*>(x_out);
            k_matmul_nn<<<blocks_for(static_cast<long>(act_)), kThreads, 0, s>>>(wslot_ptr(wslot, l), cur, y, n_, cols_);
            cur = y;
        }
        check_cuda(cudaGetLastError(), "linear forward");
    }

    void backward(int k, int wslot, int sslot, const void* g_in, void* g_out, bool first,
                  cudaStream_t s) override {
        const double* g = static_cast<const double*>(g_in);
        int flip = 0;
        if (stageL_) {
            double* lg = gtmp_ + static_cast<size_t>(flip) * act_;
            flip ^= 1;
            const double* out = out_ + static_cast<size_t>(sslot) * act_;
            k_loss<<<1, kThreads, 0, s>>>(out, data_y(k), static_cast<long>(act_),
                                          static_cast<double>(cols_), loss_ + (k - 1));
            k_loss_grad<<<blocks_for(static_cast<long>(act_)), kThreads, 0, s>>>(
                out, data_y(k), lg, static_cast<long>(act_), static_cast<double>(cols_));
            g = lg;
        }
        for (int l = layers_ - 1; l >= 0; --l) {
            const double* in = l == 0 ? xin_[static_cast<size_t>(sslot)] : stash_ptr(sslot, l);
            k_wgrad_nt<<<blocks_for(static_cast<long>(mat_)), kThreads, 0, s>>>(
                g, in, gsum_ + static_cast<size_t>(l) * mat_, n_, cols_, first ? 1 : 0, loop_scale_);
            if (l > 0 || !stage0_) {
                double* dst = l == 0 ? static_cast<double*>(g_out) : gtmp_ + static_cast<size_t>(flip) * act_;
                flip ^= 1;
                k_matmul_tn<<<blocks_for(static_cast<long>(act_)), kThreads, 0, s>>>(wslot_ptr(wslot, l), g, dst, n_, cols_);
                g = dst;
            }
        }
        check_cuda(cudaGetLastError(), "linear backward");
    }

    void update(int src_slot, int dst_slot, int count, cudaStream_t s) override {
        if (loop_scaling_) count = 1;  // reference_loop applies the pre-scaled sum (semantics.cpp:145, :163)
        const long total = static_cast<long>(layers_ * mat_);
        k_update<<<blocks_for(total), kThreads, 0, s>>>(wslot_ptr(src_slot, 0), wslot_ptr(dst_slot, 0), vel_,
                                                        gsum_, total, static_cast<double>(count), lr_, beta_);
        check_cuda(cudaGetLastError(), "linear update");
    }

    std::vector<void*> replica_buffers() override {
        std::vector<void*> v{gsum_, nullptr, nullptr};
        for (int i = 0; i < wslots_; ++i) v.push_back(wslot_ptr(i, 0));
        return v;
    }
    void update_replicas(int src_slot, int dst_slot, int count, const std::vector<std::vector<void*>>& peers,
                         int rank, cudaStream_t s) override {
        if (loop_scaling_) count = 1;
        const int w = static_cast<int>(peers.size());
        if (w < 1 || w > kMaxRep) throw Error("replica update: bad width");
        F64Peers p{};
        for (int q = 0; q < w; ++q) {
            p.g[q] = static_cast<const double*>(peers[q].at(0));
            p.wdst[q] = static_cast<double*>(peers[q].at(3 + static_cast<size_t>(dst_slot)));
        }
        const long total = static_cast<long>(layers_ * mat_);
        const long lo = total * rank / w, hi = total * (rank + 1) / w;
        k_update_replicas<<<blocks_for(std::max(hi - lo, 1L)), kThreads, 0, s>>>(
            p, w, wslot_ptr(src_slot, 0), vel_, lo, hi, static_cast<double>(count), lr_, beta_);
        check_cuda(cudaGetLastError(), "linear update (replicas)");
    }

private:
    static void alloc(double** p, size_t n) {
        check_cuda(cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(double)), "cudaMalloc");
    }
    double* wslot_ptr(int slot, int l) const { return w_ + (static_cast<size_t>(slot) * layers_ + l) * mat_; }
    double* stash_ptr(int slot, int l) const { return stash_ + (static_cast<size_t>(slot) * layers_ + l) * act_; }
    const double* data_x(int k) const { check_k(k); return x_ + static_cast<size_t>(k - 1) * act_; }
    const double* data_y(int k) const { check_k(k); return y_ + static_cast<size_t>(k - 1) * act_; }
    void check_k(int k) const {
        if (k < 1 || k > capacity_) throw Error("toy dataset has too few microbatches for the requested run");
    }

    int n_, cols_, layers_;
    bool stage0_, stageL_;
    int sslots_, wslots_;
    double lr_, beta_;
    double loop_scale_;
    bool loop_scaling_;
    cudaStream_t stream_ = nullptr;
    size_t mat_ = 0, act_ = 0;
    int capacity_ = 0;
    double *w_ = nullptr, *vel_ = nullptr, *gsum_ = nullptr, *stash_ = nullptr, *gtmp_ = nullptr,
           *out_ = nullptr, *x_ = nullptr, *y_ = nullptr, *loss_ = nullptr;
    std::vector<const double*> xin_;
};

}  // namespace

std::unique_ptr<StageModel> make_linear_f64_stage(const EngineConfig& cfg, int stage, int lo,
                                                   int hi, int stash_slots, int weight_slots) {
    return std::make_unique<LinearF64Stage>(cfg, stage, lo, hi, stash_slots, weight_slots);
}

}  // namespace p2bw
