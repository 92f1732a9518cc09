// Persistent, warp-specialised tcgen05 GEMM for the stage executor.
//
//   D[M x N] = A[M x K] . B[N x K]^T     (bf16 operands, fp32 accumulation in TMEM)
//
// One kernel serves the three dense contractions of every stage layer
// (reference: semantics.cpp:9-19 matmul -> forward, :21-32 matmul_tn -> dgrad,
// :34-44 matmul_nt -> wgrad accumulated like axpy at :329):
//   forward  Y  = X  . W^T    A = X  (K-major),  B = W (K-major)
//   dgrad    dX = dY . W      A = dY (K-major),  B = W (MN-major)
//   wgrad    dW += dY^T . X   A = dY (MN-major), B = X (MN-major), fp32 += epilogue
//
// Roles (256 threads, 1 CTA per SM, grid = min(tiles, #SMs), static round-robin tiles):
//   warp 0  : TMA producer  (one lane)   global -> SMEM ring of kStages stages
//   warp 1  : MMA issuer    (one lane)   tcgen05.mma 128 x BN x 16, commit -> mbarriers
//   warp 2  : TMEM allocator (2 x BN fp32 columns: double-buffered accumulator)
//   warps 4-7: epilogue     tcgen05.ld -> registers -> fused bias/GELU/residual -> global
// The epilogue of tile i overlaps the main loop of tile i+1 through the two TMEM buffers.
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <stdexcept>
#include <string>

#include "kernels.h"
#include "profiler.h"
#include "ptx.cuh"
#include "util.h"

namespace p2bw {
namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 bf16 = 128 bytes = one swizzle row
constexpr int kThreads = 256;

template <int BN>
struct GemmCfg {
    static constexpr int kStages = BN == 256 ? 4 : 6;
    static constexpr int kABytes = kBM * kBK * 2;
    static constexpr int kBBytes = BN * kBK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kTmemCols = 2 * BN;  // 256 or 512: a power of two
    static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

__device__ __forceinline__ float gelu_fwd(float x) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(k0 * (x + k1 * x * x * x)));
    return 0.5f * x * (1.0f + t);
}

__device__ __forceinline__ float gelu_bwd(float x) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    const float x2 = x * x;
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(k0 * (x + k1 * x * x2)));
    return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * k0 * (1.0f + 3.0f * k1 * x2);
}

struct KParams {
    int m, n, k;
    GemmEpilogue epi;
};

// One 32-column chunk of the epilogue for one output row (this thread's TMEM lane).
template <EpiKind kKind>
__device__ __forceinline__ void epilogue_chunk(const KParams& p, int64_t row, int col,
                                               const uint32_t (&v)[32]) {
    const GemmEpilogue& e = p.epi;
    if constexpr (kKind == EpiKind::StoreF32) {
        float* d = static_cast<float*>(e.d) + row * e.ldd + col;
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
            float4 acc = make_float4(__uint_as_float(v[j]) * e.alpha, __uint_as_float(v[j + 1]) * e.alpha,
                                     __uint_as_float(v[j + 2]) * e.alpha,
                                     __uint_as_float(v[j + 3]) * e.alpha);
            if (e.beta != 0.0f) {
                const float4 old = *reinterpret_cast<const float4*>(d + j);
                acc.x += e.beta * old.x;
                acc.y += e.beta * old.y;
                acc.z += e.beta * old.z;
                acc.w += e.beta * old.w;
            }
            *reinterpret_cast<float4*>(d + j) = acc;
        }
    } else if constexpr (kKind == EpiKind::DGeluBF16) {
        bf16* d = static_cast<bf16*>(e.d) + row * e.ldd + col;
        const bf16* u = e.aux + row * e.ldd + col;
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
            const uint4 uu = *reinterpret_cast<const uint4*>(u + j);
            const uint32_t uw[4] = {uu.x, uu.y, uu.z, uu.w};
            uint32_t out[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 uf = ptx::unpack_bf16x2(uw[q]);
                const float a0 = __uint_as_float(v[j + 2 * q]) * e.alpha * gelu_bwd(uf.x);
                const float a1 = __uint_as_float(v[j + 2 * q + 1]) * e.alpha * gelu_bwd(uf.y);
                out[q] = ptx::pack_bf16x2(a0, a1);
            }
            *reinterpret_cast<uint4*>(d + j) = make_uint4(out[0], out[1], out[2], out[3]);
        }
    } else {
        bf16* d = static_cast<bf16*>(e.d) + row * e.ldd + col;
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
            float x[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) x[q] = __uint_as_float(v[j + q]) * e.alpha;
            if (e.bias != nullptr) {
                const uint4 bb = *reinterpret_cast<const uint4*>(e.bias + col + j);
                const uint32_t bw[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float2 bf = ptx::unpack_bf16x2(bw[q]);
                    x[2 * q] += bf.x;
                    x[2 * q + 1] += bf.y;
                }
            }
            if (e.gelu) {
                if (e.preact != nullptr) {
                    uint32_t pre[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) pre[q] = ptx::pack_bf16x2(x[2 * q], x[2 * q + 1]);
                    *reinterpret_cast<uint4*>(e.preact + row * e.ldd + col + j) =
                        make_uint4(pre[0], pre[1], pre[2], pre[3]);
                    // GELU is applied to the bf16-rounded pre-activation so that the
                    // backward (which only sees the stored bf16 u) differentiates the
                    // exact function the forward evaluated.
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float2 r = ptx::unpack_bf16x2(pre[q]);
                        x[2 * q] = r.x;
                        x[2 * q + 1] = r.y;
                    }
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) x[q] = gelu_fwd(x[q]);
            }
            if (e.residual != nullptr) {
                const uint4 rr = *reinterpret_cast<const uint4*>(e.residual + row * e.ldr + col + j);
                const uint32_t rw[4] = {rr.x, rr.y, rr.z, rr.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float2 rf = ptx::unpack_bf16x2(rw[q]);
                    x[2 * q] += rf.x;
                    x[2 * q + 1] += rf.y;
                }
            }
            uint32_t out[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) out[q] = ptx::pack_bf16x2(x[2 * q], x[2 * q + 1]);
            *reinterpret_cast<uint4*>(d + j) = make_uint4(out[0], out[1], out[2], out[3]);
        }
    }
}

template <int BN, bool kAMN, bool kBMN, EpiKind kKind>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_a,
                   const __grid_constant__ CUtensorMap tmap_b, const KParams p) {
    using Cfg = GemmCfg<BN>;
    constexpr int S = Cfg::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* s_a = smem;
    uint8_t* s_b = smem + S * Cfg::kABytes;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
    uint64_t* empty_bar = full_bar + S;
    uint64_t* tfull_bar = empty_bar + S;   // [2]
    uint64_t* tempty_bar = tfull_bar + 2;  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int tiles_m = (p.m + kBM - 1) / kBM;
    const int tiles_n = p.n / BN + (p.n % BN != 0);
    const int num_tiles = tiles_m * tiles_n;
    const int kblocks = (p.k + kBK - 1) / kBK;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmap_a);
        ptx::tma_prefetch_desc(&tmap_b);
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full_bar[s], 1);
            ptx::mbar_init(&empty_bar[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull_bar[i], 1);
            ptx::mbar_init(&tempty_bar[i], 4);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 2) ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                const int m0 = (tile % tiles_m) * kBM;
                const int n0 = (tile / tiles_m) * BN;
                for (int kb = 0; kb < kblocks; ++kb) {
                    ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
                    ptx::mbar_arrive_expect_tx(&full_bar[stage], Cfg::kStageBytes);
                    uint8_t* da = s_a + stage * Cfg::kABytes;
                    uint8_t* db = s_b + stage * Cfg::kBBytes;
                    const int k0 = kb * kBK;
                    if constexpr (kAMN) {
#pragma unroll
                        for (int j = 0; j < kBM / 64; ++j)
                            ptx::tma_load_2d(da + j * 64 * kBK * 2, &tmap_a, &full_bar[stage],
                                             m0 + j * 64, k0);
                    } else {
                        ptx::tma_load_2d(da, &tmap_a, &full_bar[stage], k0, m0);
                    }
                    if constexpr (kBMN) {
#pragma unroll
                        for (int j = 0; j < BN / 64; ++j)
                            ptx::tma_load_2d(db + j * 64 * kBK * 2, &tmap_b, &full_bar[stage],
                                             n0 + j * 64, k0);
                    } else {
                        ptx::tma_load_2d(db, &tmap_b, &full_bar[stage], k0, n0);
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_bf16(kBM, BN, kAMN, kBMN);
            // K-major SW128: rows of 128 B, 8-row groups 1024 B apart; a K step of 16
            // elements is +32 B inside the swizzle atom.  MN-major SW128: 64-element MN
            // groups one TMA box (kBK rows x 128 B) apart, 8-row K groups 1024 B apart;
            // a K step of 16 rows is +2048 B.
            constexpr uint32_t a_lbo = kAMN ? kBK * 128 : 16, a_sbo = 1024;
            constexpr uint32_t b_lbo = kBMN ? kBK * 128 : 16, b_sbo = 1024;
            constexpr uint32_t a_kstep = kAMN ? 16 * 128 : 32;
            constexpr uint32_t b_kstep = kBMN ? 16 * 128 : 32;
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                ptx::mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
                for (int kb = 0; kb < kblocks; ++kb) {
                    ptx::mbar_wait(&full_bar[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t a_addr = ptx::smem_u32(s_a + stage * Cfg::kABytes);
                    const uint32_t b_addr = ptx::smem_u32(s_b + stage * Cfg::kBBytes);
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        const uint64_t ad = ptx::sdesc_sw128(a_addr + kk * a_kstep, a_lbo, a_sbo);
                        const uint64_t bd = ptx::sdesc_sw128(b_addr + kk * b_kstep, b_lbo, b_sbo);
                        ptx::umma_bf16(d_tmem, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
                    }
                    ptx::umma_commit(&empty_bar[stage]);
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ptx::umma_commit(&tfull_bar[acc]);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            const int m0 = (tile % tiles_m) * kBM;
            const int n0 = (tile / tiles_m) * BN;
            ptx::mbar_wait(&tfull_bar[acc], acc_phase);
            ptx::tc_fence_after();
            const int64_t row = m0 + q * 32 + lane;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t v[32];
                const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                                       static_cast<uint32_t>(acc * BN + c * 32);
                ptx::tmem_ld_32x32b_x32(taddr, v);
                ptx::tmem_ld_wait();
                const int col = n0 + c * 32;
                if (row < p.m && col < p.n) epilogue_chunk<kKind>(p, row, col, v);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tempty_bar[acc]);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<Cfg::kTmemCols>(tmem_base);
    }
}

// ---- host side -------------------------------------------------------------

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        check_cuda(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q),
                   "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
        if (p == nullptr || q != cudaDriverEntryPointSuccess)
            throw Error("cuTensorMapEncodeTiled is unavailable in this driver");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// 2-D bf16 tensor map with a 64-element (128 B) inner box and 128 B swizzle.
CUtensorMap make_map(const bf16* ptr, uint64_t inner, uint64_t outer, int64_t ld_elems,
                     uint32_t box_outer) {
    CUtensorMap map;
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_elems) * 2};
    const cuuint32_t box[2] = {64, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                   const_cast<bf16*>(ptr), dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error("cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return map;
}

template <int BN, bool kAMN, bool kBMN, EpiKind kKind>
void launch(const CUtensorMap& ta, const CUtensorMap& tb, const KParams& p, cudaStream_t s) {
    using Cfg = GemmCfg<BN>;
    auto kern = gemm_tc_kernel<BN, kAMN, kBMN, kKind>;
    static std::atomic<uint32_t> configured{0};  // one attribute call per device
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    const uint32_t bit = 1u << (dev & 31);
    if ((configured.load() & bit) == 0) {
        check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        Cfg::kSmemBytes),
                   "cudaFuncSetAttribute(gemm smem)");
        configured.fetch_or(bit);
    }
    const int tiles = ((p.m + kBM - 1) / kBM) * ((p.n + BN - 1) / BN);
    const int grid = tiles < num_sms() ? tiles : num_sms();
    kern<<<grid, kThreads, Cfg::kSmemBytes, s>>>(ta, tb, p);
    check_cuda(cudaGetLastError(), "gemm_tc_kernel launch");
}

template <int BN, bool kAMN, bool kBMN>
void dispatch_epi(const CUtensorMap& ta, const CUtensorMap& tb, const KParams& p, cudaStream_t s) {
    switch (p.epi.kind) {
        case EpiKind::StoreBF16: launch<BN, kAMN, kBMN, EpiKind::StoreBF16>(ta, tb, p, s); break;
        case EpiKind::StoreF32: launch<BN, kAMN, kBMN, EpiKind::StoreF32>(ta, tb, p, s); break;
        case EpiKind::DGeluBF16: launch<BN, kAMN, kBMN, EpiKind::DGeluBF16>(ta, tb, p, s); break;
    }
}

template <int BN>
void dispatch_major(bool amn, bool bmn, const CUtensorMap& ta, const CUtensorMap& tb,
                    const KParams& p, cudaStream_t s) {
    if (!amn && !bmn) dispatch_epi<BN, false, false>(ta, tb, p, s);
    else if (!amn && bmn) dispatch_epi<BN, false, true>(ta, tb, p, s);
    else if (amn && !bmn) dispatch_epi<BN, true, false>(ta, tb, p, s);
    else dispatch_epi<BN, true, true>(ta, tb, p, s);
}

// Pick the N tile that wastes the fewest MMA slots over whole waves of SMs.
int choose_bn(int m, int n) {
    if (n % 256 != 0) return 128;
    const long tm = (m + kBM - 1) / kBM;
    const long sms = num_sms();
    auto cost = [&](long bn) {
        const long tiles = tm * ((n + bn - 1) / bn);
        const long waves = (tiles + sms - 1) / sms;
        return waves * bn;  // proportional to the busiest SM's MMA time
    };
    return cost(256) <= cost(128) ? 256 : 128;
}

}  // namespace

void gemm_bf16(const GemmOperand& a, const GemmOperand& b, int m, int n, int k,
               const GemmEpilogue& epi, cudaStream_t stream) {
    if (m <= 0 || n <= 0 || k <= 0) throw Error("gemm: empty problem");
    if (n % 32 != 0) throw Error("gemm: N must be a multiple of 32");
    if ((a.ld % 8) != 0 || (b.ld % 8) != 0) throw Error("gemm: leading dims must be multiples of 8");
    const int bn = choose_bn(m, n);
    const bool amn = a.major == Major::MN, bmn = b.major == Major::MN;
    // A: rows = m (tile kBM), B: rows = n (tile bn).  K-major maps put k innermost.
    const CUtensorMap ta = amn ? make_map(a.ptr, m, k, a.ld, kBK) : make_map(a.ptr, k, m, a.ld, kBM);
    const CUtensorMap tb = bmn ? make_map(b.ptr, n, k, b.ld, kBK) : make_map(b.ptr, k, n, b.ld, bn);
    KParams p{m, n, k, epi};
    const double out_bytes = epi.kind == EpiKind::StoreF32 ? (epi.beta != 0.0f ? 8.0 : 4.0) : 2.0;
    prof::Scope scope("gemm", 2.0 * m * n * k,
                      2.0 * (static_cast<double>(m) * k + static_cast<double>(n) * k) +
                          out_bytes * m * n,
                      1, stream);
    if (bn == 256) dispatch_major<256>(amn, bmn, ta, tb, p, stream);
    else dispatch_major<128>(amn, bmn, ta, tb, p, stream);
}

int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
        check_cuda(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev),
                   "cudaDeviceGetAttribute(SM count)");
    }
    return n;
}

}  // namespace p2bw
