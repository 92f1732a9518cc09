// Transformer pipeline stage: pre-LN blocks (GPT-2 / BERT family) in bf16 with
// fp32 statistics, gradients, momentum and master weights.
//
//   block(x):  xn1 = LN1(x); qkv = xn1 Wqkv^T + bqkv; o = attn(qkv)
//              x1 = o Wo^T + bo + x; xn2 = LN2(x1); u = xn2 W1^T + b1; a = gelu(u)
//              x2 = a W2^T + b2 + x1
//   stage 0 :  x0 = tok_emb[ids] + pos_emb[pos]
//   last    :  xf = LNf(x_L[head rows]); logits = xf Whead^T; CE (mean over head rows)
//
// The reference has no layer arithmetic; this stage follows its
// trainer-step *semantics* (semantics.cpp:238-375): Forward stashes per-
// microbatch activations under the version it used, Backward accumulates the
// coalesced weight gradient (summed over the batch's microbatches, divided by
// the count at the update, :329/:338-340), WeightUpdate applies momentum SGD
// with dampening (:153-165) and writes the next version into the other bf16
// buffer.  Every dense contraction is the tcgen05 GEMM (gemm.cu); wgrad lands
// in the fp32 gradient buffer through the GEMM epilogue (beta = 0 on the first
// microbatch after an update, 1 afterwards).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "engine.h"
#include "profiler.h"
#include "tkernels.h"

namespace p2bw {

namespace {
// Timing diagnostic only (P2BW_DEBUG_DUP bit mask): issue a kernel class twice to read
// its marginal cost inside the overlapped step.  1 LN fwd, 2 LN bwd, 4 bias colsum,
// 8 attention fwd, 16 attention bwd, 32 the QKV GEMM.  Duplicates are idempotent except for the
// accumulated gradients they double -- never set outside timing runs.
int debug_dup(int bit) {
    static const int mask = [] {
        const char* e = std::getenv("P2BW_DEBUG_DUP");
        return e ? std::atoi(e) : 0;
    }();
    return (mask & bit) ? 2 : 1;
}

// Two alternating attention dQ accumulators per stage (zero-fill inside the previous
// layer's backward kernel instead of the delta kernel); P2BW_ATTN_DQ_DBUF=0 turns it off.
bool dq_double_buffer() {
    static const bool on = [] {
        const char* e = std::getenv("P2BW_ATTN_DQ_DBUF");
        return e == nullptr || std::atoi(e) != 0;
    }();
    return on;
}
}  // namespace

namespace {


size_t align64(size_t n) { return (n + 63) & ~static_cast<size_t>(63); }

struct LayerOff {
    size_t ln1g, ln1b, wqkv, bqkv, wo, bo, ln2g, ln2b, w1, b1, w2, b2;
};

// One stash slot: everything the backward of one microbatch reads.
struct Slot {
    std::vector<bf16*> x;       // layer inputs (x[0] used on stage 0 only)
    std::vector<bf16*> xn1, qkv, o, x1, xn2, u, a;
    std::vector<float*> mean1, rstd1, mean2, rstd2, lse;
    const bf16* xin0 = nullptr;  // layer-0 input (ring slot on stages > 0)
    bf16* xl = nullptr;          // last-layer output (last stage)
    bf16* hg = nullptr;          // gathered head rows (last stage, head_rows > 0)
    bf16* xf = nullptr;          // LNf output
    float *meanf = nullptr, *rstdf = nullptr;
    bf16* logits = nullptr;      // logits -> dlogits (in place)
};

class TransformerStage final : public StageModel {
public:
    TransformerStage(const EngineConfig& c, int stage, int lo, int hi, int sslots, int wslots)
        : cfg_(c), stage_(stage), lo_(lo), layers_(hi - lo), first_(stage == 0), last_(stage == c.depth - 1),
          sslots_(c.recompute ? 1 : sslots), wslots_(wslots), recompute_(c.recompute) {
        h_ = c.hidden;
        heads_ = c.heads;
        seq_ = c.seq_len;
        b_ = c.microbatch_size;
        vocab_ = c.vocab;
        vp_ = static_cast<int>((static_cast<size_t>(vocab_) + 127) / 128 * 128);
        T_ = b_ * seq_;
        if (h_ <= 0 || heads_ <= 0 || (h_ != heads_ * 64 && h_ != heads_ * 128))
            throw Error("transformer: hidden must equal heads * 64 or heads * 128 (head dim 64 / 128)");
        hd_ = h_ / heads_;
        if (!attention_tc_supported(seq_))
            throw Error("transformer: seq_len must be a positive multiple of 128 (tcgen05 attention tiles)");
        if (b_ < 1 || vocab_ < 2) throw Error("transformer: bad microbatch size or vocab");
        rows_per_seq_ = c.head_rows > 0 ? c.head_rows : seq_;
        if (rows_per_seq_ > seq_) throw Error("transformer: head_rows exceeds seq_len");
        R_ = b_ * rows_per_seq_;
        layout_params();
        alloc_all();
    }

    ~TransformerStage() override {
        if (side_stream_) cudaStreamSynchronize(side_stream_);
        for (cudaEvent_t e : ev_)
            if (e) cudaEventDestroy(e);
        if (side_stream_) cudaStreamDestroy(side_stream_);
        for (void* p : allocs_) cudaFree(p);
    }

    size_t num_params() const override { return nparam_; }
    size_t boundary_bytes() const override { return static_cast<size_t>(T_) * h_ * sizeof(bf16); }
    size_t weight_bytes_public() const override { return nparam_ * sizeof(float); }
    double version_bytes() const override { return static_cast<double>(nparam_) * sizeof(bf16); }
    // with recomputation a microbatch's stash is its input (the ring slot)
    double stash_bytes() const override { return recompute_ ? static_cast<double>(boundary_bytes()) : stash_bytes_; }
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

    void init_weights(uint64_t seed) override {
        const float hw = static_cast<float>(0.02 * std::sqrt(3.0));  // U(-a, a), std of N(0, 0.02)
        cudaStream_t s = stream_;
        fill_f32(master_, nparam_, 0.0f, s);
        for (int l = 0; l < layers_; ++l) {
            const LayerOff& o = lay_[l];
            const uint64_t uid = static_cast<uint64_t>(lo_ + l) * 16;
            fill_f32(master_ + o.ln1g, h_, 1.0f, s);
            fill_f32(master_ + o.ln2g, h_, 1.0f, s);
            init_uniform(master_ + o.wqkv, 3ull * h_ * h_, seed, uid + 1, hw, s);
            init_uniform(master_ + o.wo, 1ull * h_ * h_, seed, uid + 2, hw, s);
            init_uniform(master_ + o.w1, 4ull * h_ * h_, seed, uid + 3, hw, s);
            init_uniform(master_ + o.w2, 4ull * h_ * h_, seed, uid + 4, hw, s);
        }
        if (first_) {
            init_uniform(master_ + off_tok_, static_cast<size_t>(vocab_) * h_, seed, 1ull << 40, hw, s);
            init_uniform(master_ + off_pos_, static_cast<size_t>(seq_) * h_, seed, (1ull << 40) + 1, hw, s);
        }
        if (last_) {
            fill_f32(master_ + off_lnfg_, h_, 1.0f, s);
            init_uniform(master_ + off_head_, static_cast<size_t>(vocab_) * h_, seed, 1ull << 41, hw, s);
        }
        cast_f32_bf16(master_, wbf_[0], nparam_, s);
        check_cuda(cudaMemsetAsync(vel_, 0, nparam_ * sizeof(float), s), "memset vel");
        if (vel2_) check_cuda(cudaMemsetAsync(vel2_, 0, nparam_ * sizeof(float), s), "memset vel2");
        adam_step_ = 0;
        check_cuda(cudaStreamSynchronize(s), "init sync");
    }

    void load_weights(int wslot, const void* host, size_t bytes) override {
        if (bytes != weight_bytes_public()) throw Error("load_weights: expected the flat fp32 parameter vector");
        check_cuda(cudaStreamSynchronize(stream_), "sync");
        // stream-ordered (a pageable cudaMemcpy may return before its DMA lands)
        check_cuda(cudaMemcpyAsync(master_, host, bytes, cudaMemcpyHostToDevice, stream_), "H2D master");
        cast_f32_bf16(master_, wbf_[wslot], nparam_, stream_);
        check_cuda(cudaMemsetAsync(vel_, 0, nparam_ * sizeof(float), stream_), "memset vel");
        if (vel2_) check_cuda(cudaMemsetAsync(vel2_, 0, nparam_ * sizeof(float), stream_), "memset vel2");
        adam_step_ = 0;
        check_cuda(cudaStreamSynchronize(stream_), "load sync");
    }

    void read_weights(int wslot, void* host, size_t bytes, cudaStream_t s) override {
        if (bytes != weight_bytes_public()) throw Error("read_weights: size mismatch");
        // bf16 -> host, widened there (no parameter-sized device scratch)
        std::vector<uint16_t> raw(nparam_);
        check_cuda(cudaMemcpyAsync(raw.data(), wbf_[wslot], nparam_ * sizeof(bf16), cudaMemcpyDeviceToHost, s),
                   "D2H weights");
        check_cuda(cudaStreamSynchronize(s), "read sync");
        float* out = static_cast<float*>(host);
        for (size_t i = 0; i < nparam_; ++i) {
            const uint32_t bits = static_cast<uint32_t>(raw[i]) << 16;
            std::memcpy(out + i, &bits, sizeof(float));
        }
    }

    void read_master(void* host, size_t bytes) override {
        if (bytes != weight_bytes_public()) throw Error("read_master: size mismatch");
        check_cuda(cudaMemcpyAsync(host, master_, bytes, cudaMemcpyDeviceToHost, stream_), "D2H master");
        check_cuda(cudaStreamSynchronize(stream_), "read sync");
    }

    void read_losses(double* host, int first_mb, int count, cudaStream_t s) override {
        if (!last_) throw Error("this stage computes no loss");
        if (capacity_ == 0) throw Error("no data has been set");
        std::vector<float> tmp(static_cast<size_t>(capacity_));
        check_cuda(cudaMemcpyAsync(tmp.data(), loss_, sizeof(float) * capacity_, cudaMemcpyDeviceToHost, s),
                   "D2H loss");
        check_cuda(cudaStreamSynchronize(s), "loss sync");
        for (int i = 0; i < count; ++i) host[i] = tmp[static_cast<size_t>((first_mb - 1 + i) % capacity_)];
    }

    void copy_losses_async(float* host, int first_mb, int count, cudaStream_t s) override {
        if (!last_ || capacity_ == 0) throw Error("this stage computes no loss");
        for (int i = 0; i < count;) {
            const int slot = (first_mb - 1 + i) % capacity_;
            const int run = std::min(count - i, capacity_ - slot);
            check_cuda(cudaMemcpyAsync(host + i, loss_ + slot, sizeof(float) * run, cudaMemcpyDeviceToHost, s),
                       "D2H loss");
            i += run;
        }
    }

    // inputs: int32 [count][T] token ids (stage 0); targets: int32 [count][R] (last stage).
    void set_data(const void* inputs, const void* targets, int first_mb, int count) override {
        if (count < 1) throw Error("set_data: empty microbatch range");
        const cudaStream_t ds = data_stream_ ? data_stream_ : stream_;
        if (capacity_ == 0) {
            capacity_ = std::max(count, 2 * cfg_.microbatches);
            ids_ = dalloc<int>(static_cast<size_t>(capacity_) * T_);
            tgt_ = dalloc<int>(static_cast<size_t>(capacity_) * R_);
            loss_ = dalloc<float>(static_cast<size_t>(capacity_));
            check_cuda(cudaMemsetAsync(loss_, 0, sizeof(float) * capacity_, ds), "memset loss");
        }
        if (count > capacity_) throw Error("set_data: more microbatches than the data ring holds");
        for (int i = 0; i < count; ++i) {
            const int slot = (first_mb - 1 + i) % capacity_;
            if (inputs)
                check_cuda(cudaMemcpyAsync(ids_ + static_cast<size_t>(slot) * T_,
                                           static_cast<const int*>(inputs) + static_cast<size_t>(i) * T_,
                                           sizeof(int) * T_, cudaMemcpyHostToDevice, ds), "H2D ids");
            if (targets)
                check_cuda(cudaMemcpyAsync(tgt_ + static_cast<size_t>(slot) * R_,
                                           static_cast<const int*>(targets) + static_cast<size_t>(i) * R_,
                                           sizeof(int) * R_, cudaMemcpyHostToDevice, ds), "H2D targets");
        }
    }

    // With recomputation every microbatch shares stash slot 0: a Forward only produces
    // its output (and loss); the Backward's Recompute refills the slot first.
    void recompute(int k, int wslot, int sslot, const void* x_in, cudaStream_t s) override {
        if (!recompute_) throw Error("recompute op on a stage built without activation recomputation");
        forward(k, wslot, sslot, x_in, last_ ? nullptr : rc_out_, s);
    }

    void forward(int k, int wslot, int sslot, const void* x_in, void* x_out, cudaStream_t s) override {
        const bf16* W = wbf_[wslot];
        Slot& st = slots_[recompute_ ? 0 : sslot];
        const bf16* cur;
        if (first_) {
            embed_fwd(data_ids(k), W + off_tok_, W + off_pos_, st.x[0], T_, seq_, h_, s);
            cur = st.x[0];
        } else {
            cur = static_cast<const bf16*>(x_in);
        }
        st.xin0 = cur;
        for (int l = 0; l < layers_; ++l) {
            const LayerOff& o = lay_[l];
            for (int dup_ = 0; dup_ < debug_dup(1); ++dup_) layernorm_fwd(cur, W + o.ln1g, W + o.ln1b, st.xn1[l], st.mean1[l], st.rstd1[l], T_, h_, s);
            for (int dup_ = 0; dup_ < debug_dup(32); ++dup_) gemm_store(st.xn1[l], h_, T_, W + o.wqkv, 3 * h_, h_, st.qkv[l], W + o.bqkv, nullptr, false, nullptr, s);
            for (int dup_ = 0; dup_ < debug_dup(8); ++dup_) attention_fwd(st.qkv[l], st.o[l], st.lse[l], b_, seq_, heads_, cfg_.causal != 0, s, hd_);
            gemm_store(st.o[l], h_, T_, W + o.wo, h_, h_, st.x1[l], W + o.bo, cur, false, nullptr, s);
            for (int dup_ = 0; dup_ < debug_dup(1); ++dup_) layernorm_fwd(st.x1[l], W + o.ln2g, W + o.ln2b, st.xn2[l], st.mean2[l], st.rstd2[l], T_, h_, s);
            gemm_store(st.xn2[l], h_, T_, W + o.w1, 4 * h_, h_, st.a[l], W + o.b1, nullptr, true, st.u[l], s);
            bf16* dst = l + 1 < layers_ ? st.x[l + 1] : (last_ ? st.xl : static_cast<bf16*>(x_out));
            gemm_store(st.a[l], 4 * h_, T_, W + o.w2, h_, 4 * h_, dst, W + o.b2, st.x1[l], false, nullptr, s);
            cur = dst;
        }
        if (last_) {
            const bf16* hsrc = cur;
            if (R_ < T_) {
                gather_rows(cur, head_idx_, st.hg, R_, h_, s);
                hsrc = st.hg;
            }
            layernorm_fwd(hsrc, W + off_lnfg_, W + off_lnfb_, st.xf, st.meanf, st.rstdf, R_, h_, s);
            gemm_store(st.xf, h_, R_, W + off_head_, vp_, h_, st.logits, nullptr, nullptr, false, nullptr, s);
            softmax_xent(st.logits, data_tgt(k), R_, vocab_, vp_, 1.0f / R_, row_loss_, s);
            sum_scaled(row_loss_, R_, 1.0f / R_, loss_ + (k - 1) % capacity_, s);
        }
    }

    void backward(int k, int wslot, int sslot, const void* g_in, void* g_out, bool first,
                  cudaStream_t s) override {
        const bf16* W = wbf_[wslot];
        Slot& st = slots_[recompute_ ? 0 : sslot];
        const float beta = first ? 0.0f : 1.0f;
        const bf16* g = static_cast<const bf16*>(g_in);
        // With per-launch profiling on, the weight gradients stay on the main stream so
        // that every kernel's event-timed duration is its own (the roofline report).
        side_ = prof::enabled() ? s : side_stream_;
        fork(kEvStart, s);  // the side stream follows the previous update (grad_ overwrite with beta 0)
        // The "side task done" events the main stream waits on before a side task of THIS
        // backward re-records them were last recorded by the previous backward, whose end
        // already joined the side stream: re-record them here (trivially complete) so no wait
        // refers to work outside the current CUDA-graph capture (Engine::run_graph).
        for (int e : {kEvDoneA, kEvDoneB, kEvDoneC, kEvDoneD}) done(e);
        if (last_) {
            // logits now hold dloss/dlogits (softmax_xent ran in the forward)
            bf16* dxf = R_ < T_ ? gH_ : gA_;
            gemm_store_mn_b(st.logits, vp_, W + off_head_, h_, R_, h_, vp_, dxf, s, head_ws_,
                            static_cast<int64_t>(R_) * h_);
            gemm_wgrad(st.logits, vp_, st.xf, h_, vp_, h_, R_, grad_ + off_head_, beta, side_);
            bf16* dsrc = dxf;
            bf16* dhead = R_ < T_ ? gB_ : gA_;
            // the LNf gradient is the top layer's FC2 output gradient: its column sum is
            // that layer's b2 gradient (rows outside the head are zero)
            layernorm_bwd(dsrc, R_ < T_ ? st.hg : st.xl, st.meanf, st.rstdf, W + off_lnfg_, nullptr, dhead,
                          grad_ + off_lnfg_, grad_ + off_lnfb_, first, R_, h_, red_scratch_, s,
                          grad_ + lay_[layers_ - 1].b2);
            if (R_ < T_) {
                check_cuda(cudaMemsetAsync(gA_, 0, static_cast<size_t>(T_) * h_ * sizeof(bf16), s), "memset");
                scatter_rows(dhead, head_idx_, gA_, R_, h_, s);
            }
            g = gA_;
        }
        // Weight gradients run on a side stream, concurrently with the dgrad / attention /
        // LayerNorm chain of the main stream (they are off the critical path and fill
        // the ragged last waves of the main chain's kernels).  fork(e): the side stream
        // waits for main's progress; done(e) marks a side task; wait_side(e) holds main
        // before it overwrites a buffer that side task reads.
        for (int l = layers_ - 1; l >= 0; --l) {
            const LayerOff& o = lay_[l];
            const bf16* x = l == 0 ? st.xin0 : st.x[l];
            fork(kEvG, s);  // g (this layer's output gradient) is ready
            // FC2 (+ GELU'): du = (g W2) * gelu'(u)
            wait_side(kEvDoneB, s);  // g4_ free (previous layer's W1 / b1 gradients)
            gemm_dgelu(g, h_, W + o.w2, 4 * h_, T_, 4 * h_, h_, st.u[l], g4_, s);
            gemm_wgrad(g, h_, st.a[l], 4 * h_, h_, 4 * h_, T_, grad_ + o.w2, beta, side_);
            // b2: fused into the LayerNorm backward that produced g (LNf or the layer
            // above's LN1); only the gradient received from the next stage needs a pass
            if (l == layers_ - 1 && !last_) colsum_bf16(g, T_, h_, h_, grad_ + o.b2, first, side_red_, side_);
            done(kEvDoneA);
            fork(kEvG4, s);
            // FC1: dxn2 = du W1
            gemm_store_mn_b(g4_, 4 * h_, W + o.w1, h_, T_, h_, 4 * h_, gX_, s);
            gemm_wgrad(g4_, 4 * h_, st.xn2[l], h_, 4 * h_, h_, T_, grad_ + o.w1, beta, side_);
            // b1 = colsum(du) as its own side-stream pass: summing the A tiles inside the
            // wgrad GEMM (GemmEpilogue::bias_grad) measured no faster, as it rules out
            // CTA-pair tiles, and inside the FC1 dgrad 1.3% slower (critical path)
            for (int dup_ = 0; dup_ < debug_dup(4); ++dup_) colsum_bf16(g4_, T_, 4 * h_, 4 * h_, grad_ + o.b1, first, side_red_, side_);
            done(kEvDoneB);
            // LN2 (+ residual): dx1 = LN2'(dxn2) + g
            // (+ bo = colsum(dx1), fused)
            wait_side(kEvDoneC, s);  // gB_ free (previous layer's Wo gradient)
            for (int dup_ = 0; dup_ < debug_dup(2); ++dup_) layernorm_bwd(gX_, st.x1[l], st.mean2[l], st.rstd2[l], W + o.ln2g, g, gB_, grad_ + o.ln2g,
                          grad_ + o.ln2b, first, T_, h_, red_scratch_, s, grad_ + o.bo);
            fork(kEvGB, s);
            // proj: do = dx1 Wo
            gemm_store_mn_b(gB_, h_, W + o.wo, h_, T_, h_, h_, gX_, s);
            gemm_wgrad(gB_, h_, st.o[l], h_, h_, h_, T_, grad_ + o.wo, beta, side_);
            done(kEvDoneC);
            // attention
            wait_side(kEvDoneD, s);  // g3_ free (previous layer's Wqkv / bqkv gradients)
            // the layers' calls alternate two dQ accumulators (each call's kernel zeroes the
            // next one's, attention_bwd_tc); debug duplicates keep the single-buffer path
            for (int dup_ = 0; dup_ < debug_dup(16); ++dup_)
                attention_bwd(st.qkv[l], st.o[l], gX_, st.lse[l], g3_, delta_, attn_scratch_, b_, seq_, heads_,
                              cfg_.causal != 0, s, hd_, debug_dup(16) > 1 ? nullptr : attn_dq_alt_,
                              layers_ - 1 - l, l == 0);
            fork(kEvG3, s);
            // QKV: dxn1 = dqkv Wqkv
            gemm_store_mn_b(g3_, 3 * h_, W + o.wqkv, h_, T_, h_, 3 * h_, gX_, s);
            gemm_wgrad(g3_, 3 * h_, st.xn1[l], h_, 3 * h_, h_, T_, grad_ + o.wqkv, beta, side_);
            for (int dup_ = 0; dup_ < debug_dup(4); ++dup_) colsum_bf16(g3_, T_, 3 * h_, 3 * h_, grad_ + o.bqkv, first, side_red_, side_);
            done(kEvDoneD);
            // LN1 (+ residual): dx = LN1'(dxn1) + dx1
            bf16* dst = (l > 0 || first_) ? gA_ : static_cast<bf16*>(g_out);
            wait_side(kEvDoneA, s);  // g (gA_) read by this layer's W2 gradient
            // (+ b2 of the layer below = colsum(dx), fused)
            for (int dup_ = 0; dup_ < debug_dup(2); ++dup_) layernorm_bwd(gX_, x, st.mean1[l], st.rstd1[l], W + o.ln1g, gB_, dst, grad_ + o.ln1g, grad_ + o.ln1b,
                          first, T_, h_, red_scratch_, s, l > 0 ? grad_ + lay_[l - 1].b2 : nullptr);
            g = dst;
        }
        if (first_) {
            if (first)
                check_cuda(cudaMemsetAsync(grad_ + off_tok_, 0, static_cast<size_t>(vocab_) * h_ * sizeof(float), s),
                           "memset dtok");
            embed_bwd(data_ids(k), g, grad_ + off_tok_, grad_ + off_pos_, T_, seq_, h_, first, s);
        }
        done(kEvEnd);
        wait_side(kEvEnd, s);  // every weight gradient of this microbatch is in grad_
    }

    // side-stream plumbing of backward()
    enum { kEvStart, kEvG, kEvG4, kEvGB, kEvG3, kEvDoneA, kEvDoneB, kEvDoneC, kEvDoneD, kEvEnd, kNumEv };
    void fork(int e, cudaStream_t s) {
        check_cuda(cudaEventRecord(ev_[e], s), "cudaEventRecord(fork)");
        check_cuda(cudaStreamWaitEvent(side_, ev_[e], 0), "cudaStreamWaitEvent(fork)");
    }
    void done(int e) { check_cuda(cudaEventRecord(ev_[e], side_), "cudaEventRecord(side)"); }
    void wait_side(int e, cudaStream_t s) { check_cuda(cudaStreamWaitEvent(s, ev_[e], 0), "cudaStreamWaitEvent(side)"); }

    void update(int src_slot, int dst_slot, int grad_count, cudaStream_t s) override {
        (void)src_slot;  // the fp32 master always holds the latest version
        if (cfg_.optimizer == P2BW_OPT_ADAM) {
            adam_update(master_, vel_, vel2_, grad_, wbf_[dst_slot], nparam_, 1.0f / grad_count,
                        static_cast<float>(cfg_.lr), static_cast<float>(cfg_.momentum), static_cast<float>(cfg_.beta2),
                        static_cast<float>(cfg_.eps), ++adam_step_, s);
            flip_grad();
            return;
        }
        sgd_momentum_update(master_, vel_, grad_, wbf_[dst_slot], nparam_, 1.0f / grad_count,
                            static_cast<float>(cfg_.lr), static_cast<float>(cfg_.momentum), s);
        flip_grad();
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
        if (cfg_.optimizer == P2BW_OPT_ADAM)
            adam_update_replicas(r, vel_, vel2_, nparam_, 1.0f / grad_count, static_cast<float>(cfg_.lr),
                                 static_cast<float>(cfg_.momentum), static_cast<float>(cfg_.beta2),
                                 static_cast<float>(cfg_.eps), ++adam_step_, s);
        else
            sgd_momentum_update_replicas(r, vel_, nparam_, 1.0f / grad_count, static_cast<float>(cfg_.lr),
                                         static_cast<float>(cfg_.momentum), s);
        flip_grad();
    }

    // Next batch accumulates into the other buffer (when double-buffered).
    void flip_grad() {
        if (grad_bufs_[1]) {
            grad_cur_ ^= 1;
            grad_ = grad_bufs_[grad_cur_];
        }
    }

private:
    template <class T>
    T* dalloc(size_t n) {
        void* p = nullptr;
        check_cuda(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc(transformer)");
        allocs_.push_back(p);
        return static_cast<T*>(p);
    }

    void layout_params() {
        size_t off = 0;
        auto take = [&](size_t n) {
            const size_t at = off;
            off += align64(n);
            return at;
        };
        const size_t h = static_cast<size_t>(h_);
        if (first_) {
            off_tok_ = take(static_cast<size_t>(vp_) * h);
            off_pos_ = take(static_cast<size_t>(seq_) * h);
        }
        lay_.resize(static_cast<size_t>(layers_));
        for (auto& o : lay_) {
            o.ln1g = take(h);
            o.ln1b = take(h);
            o.wqkv = take(3 * h * h);
            o.bqkv = take(3 * h);
            o.wo = take(h * h);
            o.bo = take(h);
            o.ln2g = take(h);
            o.ln2b = take(h);
            o.w1 = take(4 * h * h);
            o.b1 = take(4 * h);
            o.w2 = take(4 * h * h);
            o.b2 = take(h);
        }
        if (last_) {
            off_lnfg_ = take(h);
            off_lnfb_ = take(h);
            off_head_ = take(static_cast<size_t>(vp_) * h);
        }
        nparam_ = off;
    }

    void alloc_all() {
        const size_t T = static_cast<size_t>(T_), h = static_cast<size_t>(h_);
        master_ = dalloc<float>(nparam_);
        vel_ = dalloc<float>(nparam_);
        if (cfg_.optimizer == P2BW_OPT_ADAM) {
            vel2_ = dalloc<float>(nparam_);
            check_cuda(cudaMemset(vel2_, 0, nparam_ * sizeof(float)), "memset");
        }
        grad_ = grad_bufs_[0] = dalloc<float>(nparam_);
        for (int i = 0; i < wslots_; ++i) wbf_.push_back(dalloc<bf16>(nparam_));
        check_cuda(cudaMemset(master_, 0, nparam_ * sizeof(float)), "memset");
        check_cuda(cudaMemset(vel_, 0, nparam_ * sizeof(float)), "memset");
        check_cuda(cudaMemset(grad_, 0, nparam_ * sizeof(float)), "memset");
        for (bf16* w : wbf_) check_cuda(cudaMemset(w, 0, nparam_ * sizeof(bf16)), "memset");
        slots_.resize(static_cast<size_t>(sslots_));
        const size_t stat = static_cast<size_t>(b_) * heads_ * seq_;
        const double tbytes = static_cast<double>(T) * h * sizeof(bf16);
        stash_bytes_ = layers_ * (16.0 * tbytes + 16.0 * T + 4.0 * stat) + (last_ ? 2.0 * tbytes : 0.0);
        for (Slot& st : slots_) {
            for (int l = 0; l < layers_; ++l) {
                st.x.push_back(l == 0 && !first_ ? nullptr : dalloc<bf16>(T * h));
                st.xn1.push_back(dalloc<bf16>(T * h));
                st.qkv.push_back(dalloc<bf16>(T * 3 * h));
                st.o.push_back(dalloc<bf16>(T * h));
                st.x1.push_back(dalloc<bf16>(T * h));
                st.xn2.push_back(dalloc<bf16>(T * h));
                st.u.push_back(dalloc<bf16>(T * 4 * h));
                st.a.push_back(dalloc<bf16>(T * 4 * h));
                st.mean1.push_back(dalloc<float>(T));
                st.rstd1.push_back(dalloc<float>(T));
                st.mean2.push_back(dalloc<float>(T));
                st.rstd2.push_back(dalloc<float>(T));
                st.lse.push_back(dalloc<float>(stat));
            }
            if (last_) {
                const size_t R = static_cast<size_t>(R_);
                st.xl = dalloc<bf16>(T * h);
                if (R_ < T_) st.hg = dalloc<bf16>(R * h);
                st.xf = dalloc<bf16>(R * h);
                st.meanf = dalloc<float>(R);
                st.rstdf = dalloc<float>(R);
                st.logits = dalloc<bf16>(R * static_cast<size_t>(vp_));
            }
        }
        if (recompute_ && !last_) rc_out_ = dalloc<bf16>(T * h);  // the Recompute's discarded output
        gA_ = dalloc<bf16>(T * h);
        gB_ = dalloc<bf16>(T * h);
        gX_ = dalloc<bf16>(T * h);
        g3_ = dalloc<bf16>(T * 3 * h);
        g4_ = dalloc<bf16>(T * 4 * h);
        delta_ = dalloc<float>(stat);
        attn_scratch_ = dalloc<float>(attention_bwd_scratch_floats(b_, seq_, heads_, hd_));
        if (dq_double_buffer()) attn_dq_alt_ = dalloc<float>(static_cast<size_t>(T_) * h_);
        if (last_) {
            row_loss_ = dalloc<float>(static_cast<size_t>(R_));
            head_ws_ = dalloc<float>(static_cast<size_t>(R_) * h);
            if (R_ < T_) gH_ = dalloc<bf16>(static_cast<size_t>(R_) * h);
            // evenly spaced head positions, identical for every sequence of every microbatch
            std::vector<int> idx(static_cast<size_t>(R_));
            for (int bb = 0; bb < b_; ++bb)
                for (int j = 0; j < rows_per_seq_; ++j)
                    idx[static_cast<size_t>(bb) * rows_per_seq_ + j] =
                        bb * seq_ + static_cast<int>((static_cast<long>(j) * seq_) / rows_per_seq_);
            head_idx_ = dalloc<int>(idx.size());
            check_cuda(cudaMemcpyAsync(head_idx_, idx.data(), idx.size() * sizeof(int), cudaMemcpyHostToDevice,
                                       cudaStreamPerThread), "H2D idx");
            check_cuda(cudaStreamSynchronize(cudaStreamPerThread), "sync idx");
        }
        const size_t red = std::max({layernorm_bwd_scratch_floats(T_, h_), colsum_scratch_floats(T_, 4 * h_),
                                     layernorm_bwd_scratch_floats(R_, h_)});
        red_scratch_ = dalloc<float>(red);
        // colsum partials of the side stream, and the wgrad bias partials (splits x rows,
        // splits <= T / 512)
        side_red_floats_ = static_cast<int64_t>(std::max({colsum_scratch_floats(T_, 4 * h_), colsum_scratch_floats(T_, h_),
                                                          static_cast<size_t>(T_ / 512 + 1) * 4 * h}));
        side_red_ = dalloc<float>(static_cast<size_t>(side_red_floats_));
        side_stream_ = make_stage_stream("side");
        side_ = side_stream_;
        for (cudaEvent_t& e : ev_) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    }

    const int* data_ids(int k) const {
        if (capacity_ == 0) throw Error("no token data has been set");
        return ids_ + static_cast<size_t>((k - 1) % capacity_) * T_;
    }
    const int* data_tgt(int k) const {
        if (capacity_ == 0) throw Error("no target data has been set");
        return tgt_ + static_cast<size_t>((k - 1) % capacity_) * R_;
    }

    // D[m x n] = A[m x k] B[n x k]^T, A and B K-major (forward layout), bf16 epilogue.
    void gemm_store(const bf16* a, int lda, int m, const bf16* b, int n, int k, bf16* d, const bf16* bias,
                    const bf16* residual, bool gelu, bf16* preact, cudaStream_t s) const {
        GemmEpilogue e;
        e.kind = EpiKind::StoreBF16;
        e.d = d;
        e.ldd = n;
        e.bias = bias;
        e.residual = residual;
        e.ldr = n;
        e.gelu = gelu;
        e.preact = preact;
        gemm_bf16({a, lda, Major::K}, {b, k, Major::K}, m, n, k, e, s);
    }

    // dgrad: D[m x n] = A[m x k] . B where B is stored [k x n] (weights [out x in]).
    void gemm_store_mn_b(const bf16* a, int lda, const bf16* w, int ldw, int m, int n, int k, bf16* d,
                         cudaStream_t s, float* ws = nullptr, int64_t ws_floats = 0) const {
        GemmEpilogue e;
        e.kind = EpiKind::StoreBF16;
        e.d = d;
        e.ldd = n;
        e.workspace = ws;  // split-K over the vocabulary for the LM-head dgrad
        e.workspace_floats = ws_floats;
        gemm_bf16({a, lda, Major::K}, {w, ldw, Major::MN}, m, n, k, e, s);
    }

    void gemm_dgelu(const bf16* a, int lda, const bf16* w, int ldw, int m, int n, int k, const bf16* u, bf16* d,
                    cudaStream_t s) const {
        GemmEpilogue e;
        e.kind = EpiKind::DGeluBF16;
        e.d = d;
        e.ldd = n;
        e.aux = u;
        gemm_bf16({a, lda, Major::K}, {w, ldw, Major::MN}, m, n, k, e, s);
    }

    // wgrad: G[m x n] (=|+=) dY^T X with dY [tokens x m] and X [tokens x n], fp32 out.
    // bias (optional): bias (=|+=) column sums of dY, computed inside the GEMM.
    void gemm_wgrad(const bf16* dy, int lddy, const bf16* x, int ldx, int m, int n, int tokens, float* g,
                    float beta, cudaStream_t s, float* bias = nullptr, bool bias_overwrite = false) const {
        GemmEpilogue e;
        e.kind = EpiKind::StoreF32;
        e.d = g;
        e.ldd = n;
        e.alpha = 1.0f;
        e.beta = beta;
        if (bias != nullptr) {
            e.bias_grad = bias;
            e.bias_grad_accumulate = !bias_overwrite;
            e.bias_scratch = side_red_;
            e.bias_scratch_floats = side_red_floats_;
        }
        gemm_bf16({dy, lddy, Major::MN}, {x, ldx, Major::MN}, m, n, tokens, e, s);
    }

    EngineConfig cfg_;
    int stage_, lo_, layers_;
    bool first_, last_;
    int sslots_, wslots_;
    bool recompute_ = false;
    bf16* rc_out_ = nullptr;
    int h_ = 0, heads_ = 0, hd_ = 64, seq_ = 0, b_ = 0, vocab_ = 0, vp_ = 0, T_ = 0, R_ = 0, rows_per_seq_ = 0;
    cudaStream_t stream_ = nullptr;
    cudaStream_t data_stream_ = nullptr;  // set_data copies (the forward stream), else stream_
    std::vector<void*> allocs_;
    std::vector<LayerOff> lay_;
    size_t off_tok_ = 0, off_pos_ = 0, off_lnfg_ = 0, off_lnfb_ = 0, off_head_ = 0, nparam_ = 0;
    float *master_ = nullptr, *vel_ = nullptr, *grad_ = nullptr;
    float* vel2_ = nullptr;  // Adam second moment
    float* grad_bufs_[2] = {nullptr, nullptr};  // coalesced gradient, double-buffered per batch (2BW)
    int grad_cur_ = 0;
    int adam_step_ = 0;
    std::vector<bf16*> wbf_;
    std::vector<Slot> slots_;
    bf16 *gA_ = nullptr, *gB_ = nullptr, *gX_ = nullptr, *g3_ = nullptr, *g4_ = nullptr, *gH_ = nullptr;
    float* delta_ = nullptr;
    float* attn_scratch_ = nullptr;
    float* attn_dq_alt_ = nullptr;    // second dQ accumulator [T x h] (dq_double_buffer)
    float* red_scratch_ = nullptr;
    float* side_red_ = nullptr;       // colsum / wgrad-bias partials of the side stream
    int64_t side_red_floats_ = 0;
    cudaStream_t side_stream_ = nullptr;  // weight-gradient stream of backward()
    cudaStream_t side_ = nullptr;         // side_stream_, or the main stream while profiling
    cudaEvent_t ev_[kNumEv] = {};
    float* row_loss_ = nullptr;
    float* head_ws_ = nullptr;
    int* head_idx_ = nullptr;
    double stash_bytes_ = 0.0;
    int capacity_ = 0;
    int* ids_ = nullptr;
    int* tgt_ = nullptr;
    float* loss_ = nullptr;
};

}  // namespace

std::unique_ptr<StageModel> make_transformer_stage(const EngineConfig& cfg, int stage, int lo, int hi,
                                                    int stash_slots, int weight_slots) {
    return std::make_unique<TransformerStage>(cfg, stage, lo, hi, stash_slots, weight_slots);
}

}  // namespace p2bw
