// tcgen05 implicit-GEMM core used by every contraction of the training step
// (Convolv fwd / bwd-data / bwd-filter and the FC MatMul forms).
//
//   D[m, n] (+)= sum_k A[m, k] * B[n, k]        bf16 operands, fp32 accumulate in TMEM
//
// Operand sources (per operand, chosen at launch):
//   OP_TMA_K    row-major [rows, K] matrix, TMA 2D box {64 K, rows}, SW128 K-major smem
//   OP_TMA_MN   row-major [K, rows] matrix, TMA 2D box {64 rows, 64 K}, SW128 MN-major smem
//   OP_GATHER_K implicit im2col rows of an NHWC activation (fprop: x, bwd-data: dy),
//               16-byte cp.async gathers with zero fill, written pre-swizzled (A only)
//   OP_GATHER_MN implicit im2col of x transposed for bwd-filter (B only)
//
// Warp roles (256 threads, one output tile per CTA):
//   warp 0   TMA producer (elected lane)
//   warp 1   MMA issuer (elected lane) -> tcgen05.mma into TMEM, tcgen05.commit frees smem stages
//   warp 2   TMEM allocator
//   warps 4-7  gather producers during the main loop, then the epilogue
//              (warp%4 selects the 32 TMEM lanes = tile rows it may read)
#pragma once

#include <cuda_bf16.h>

#include "ptx.cuh"

namespace tcb {

enum OperandMode : int { OP_TMA_K = 0, OP_TMA_MN = 1, OP_GATHER_K = 2, OP_GATHER_MN = 3 };
enum GatherKind : int { GATHER_FPROP = 0, GATHER_DGRAD = 1 };
enum EpiMode : int { EPI_BF16 = 0, EPI_F32 = 1, EPI_F32_PARTIAL = 2 };

// Implicit-GEMM geometry. Activations are NHWC with a channel stride that is a
// multiple of 8 (16-byte chunks never straddle two filter taps).
struct ConvGeom {
    int N, H, W, C;      // input image (fprop / wgrad source) or dx image (dgrad rows)
    int R, S, stride, pad;
    int Ho, Wo, Co;      // output image; Co = channel stride of dy (dgrad source)
};

struct GemmParams {
    CUtensorMap tmA;  // valid when a_mode is a TMA mode
    CUtensorMap tmB;  // valid when b_mode is a TMA mode
    int M, N, K;
    int a_mode, b_mode;
    int gather_kind;          // GatherKind for OP_GATHER_K
    const __nv_bfloat16* gsrc;  // gather source tensor
    ConvGeom g;
    int kb_per_split;         // k-blocks handled by one blockIdx.z
    int num_kb;               // total k-blocks
    // epilogue
    int epi;
    void* D;
    long long ldd;            // row stride of D in elements
    long long split_stride;   // elements between split partial slabs (EPI_F32_PARTIAL)
    const float* bias;        // per-column bias (EPI_BF16 / EPI_F32), may be null
    int n_bias;               // bias is read for n < n_bias (padded channels get 0)
    int relu;
    float alpha;              // D = alpha * acc (+ beta * D_old for EPI_F32 when beta != 0)
    float beta;
};

constexpr int BK = 64;          // bf16 elements per k-block = one 128-byte swizzle row
constexpr int BM = 128;
constexpr int kNumThreads = 256;

template <int BN>
struct TileCfg {
    static constexpr int kStages = BN >= 256 ? 4 : (BN >= 128 ? 6 : 8);
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = BN * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;
};

// Byte offset of 16B chunk `j` of row `r` inside a SW128 tile (1024B-aligned base).
__device__ __forceinline__ uint32_t sw128_off(int r, int j) {
    return static_cast<uint32_t>(r * 128 + ((j ^ (r & 7)) << 4));
}

// ---- im2col gathers -------------------------------------------------------
// A rows (K-major): thread owns one tile row, fills its 8 chunks for k-block kb.
__device__ __forceinline__ void gather_rows_kmajor(const GemmParams& p, uint32_t sA, int row, int m0, int kb,
                                                   bool row_valid, int rn, int ry, int rx) {
    const ConvGeom& g = p.g;
    const int k0 = kb * BK;
    const int C = (p.gather_kind == GATHER_FPROP) ? g.C : g.Co;
    int tap = k0 / C;
    int c = k0 - tap * C;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int k = k0 + j * 8;
        const void* src = p.gsrc;
        uint32_t bytes = 0;
        if (row_valid && k < p.K) {
            const int kh = tap / g.S;
            const int kw = tap - kh * g.S;
            if (p.gather_kind == GATHER_FPROP) {
                const int iy = ry * g.stride - g.pad + kh;
                const int ix = rx * g.stride - g.pad + kw;
                if (iy >= 0 && iy < g.H && ix >= 0 && ix < g.W) {
                    src = p.gsrc + ((static_cast<long long>(rn) * g.H + iy) * g.W + ix) * g.C + c;
                    bytes = 16;
                }
            } else {
                const int ny = ry + g.pad - kh;
                const int nx = rx + g.pad - kw;
                if (ny >= 0 && nx >= 0) {
                    const int oy = ny / g.stride, ox = nx / g.stride;
                    if (oy * g.stride == ny && ox * g.stride == nx && oy < g.Ho && ox < g.Wo) {
                        src = p.gsrc + ((static_cast<long long>(rn) * g.Ho + oy) * g.Wo + ox) * g.Co + c;
                        bytes = 16;
                    }
                }
            }
        }
        cp_async_16(sA + sw128_off(row, j), src, bytes);
        c += 8;
        if (c >= C) { c -= C; ++tap; }
    }
    (void)m0;
}

// B for bwd-filter (MN-major): rows of the smem atoms are k = output pixels,
// columns are n = (kh, kw, c). Thread handles pixel row `kr` and every other chunk.
template <int BN>
__device__ __forceinline__ void gather_wgrad_mn(const GemmParams& p, uint32_t sB, int kr, int half, int n0, int kb) {
    const ConvGeom& g = p.g;
    const int pix = kb * BK + kr;
    const int npix = g.N * g.Ho * g.Wo;
    const bool pv = pix < npix;
    int rn = 0, oy = 0, ox = 0;
    if (pv) {
        rn = pix / (g.Ho * g.Wo);
        const int rem = pix - rn * g.Ho * g.Wo;
        oy = rem / g.Wo;
        ox = rem - oy * g.Wo;
    }
    constexpr int kChunks = (BN / 64) * 8;
#pragma unroll
    for (int cc = half; cc < kChunks; cc += 2) {
        const int atom = cc >> 3, j = cc & 7;
        const int n = n0 + atom * 64 + j * 8;
        const void* src = p.gsrc;
        uint32_t bytes = 0;
        if (pv && n < p.N) {
            const int tap = n / g.C;
            const int c = n - tap * g.C;
            const int kh = tap / g.S, kw = tap - (tap / g.S) * g.S;
            const int iy = oy * g.stride - g.pad + kh;
            const int ix = ox * g.stride - g.pad + kw;
            if (iy >= 0 && iy < g.H && ix >= 0 && ix < g.W) {
                src = p.gsrc + ((static_cast<long long>(rn) * g.H + iy) * g.W + ix) * g.C + c;
                bytes = 16;
            }
        }
        cp_async_16(sB + atom * (BK * 128) + sw128_off(kr, j), src, bytes);
    }
}

template <int BN>
__global__ void __launch_bounds__(kNumThreads, 1) tc_gemm_kernel(const __grid_constant__ GemmParams p) {
    using Cfg = TileCfg<BN>;
    constexpr int S = Cfg::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + S * Cfg::kABytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
    uint64_t* empty = full + S;
    uint64_t* tmem_full = empty + S;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * BM;
    const int n0 = blockIdx.y * BN;
    const int kb_begin = blockIdx.z * p.kb_per_split;
    const int kb_end = min(p.num_kb, kb_begin + p.kb_per_split);
    const int nkb = max(0, kb_end - kb_begin);
    const bool a_gather = p.a_mode == OP_GATHER_K;
    const bool b_gather = p.b_mode == OP_GATHER_MN;
    const bool any_gather = a_gather || b_gather;

    if (warp == 0 && lane == 0) {
        if (!a_gather) tma_prefetch(&p.tmA);
        if (!b_gather) tma_prefetch(&p.tmB);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1 + (any_gather ? 128 : 0));
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, Cfg::kTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer
        if (lane == 0) {
            uint32_t tx = 0;
            if (!a_gather) tx += Cfg::kABytes;
            if (!b_gather) tx += Cfg::kBBytes;
            for (int i = 0; i < nkb; ++i) {
                const int s = i % S;
                const uint32_t use = i / S;
                mbar_wait(&empty[s], (use & 1) ^ 1);
                const int kb = kb_begin + i;
                uint8_t* a_dst = sA + s * Cfg::kABytes;
                uint8_t* b_dst = sB + s * Cfg::kBBytes;
                if (p.a_mode == OP_TMA_K) {
                    tma_load_2d(a_dst, &p.tmA, &full[s], kb * BK, m0);
                } else if (p.a_mode == OP_TMA_MN) {
#pragma unroll
                    for (int a = 0; a < BM / 64; ++a) tma_load_2d(a_dst + a * BK * 128, &p.tmA, &full[s], m0 + a * 64, kb * BK);
                }
                if (p.b_mode == OP_TMA_K) {
                    tma_load_2d(b_dst, &p.tmB, &full[s], kb * BK, n0);
                } else if (p.b_mode == OP_TMA_MN) {
#pragma unroll
                    for (int a = 0; a < BN / 64; ++a) tma_load_2d(b_dst + a * BK * 128, &p.tmB, &full[s], n0 + a * 64, kb * BK);
                }
                mbar_arrive_expect_tx(&full[s], tx);
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        const uint32_t idesc = umma_idesc_bf16(BM, BN, p.a_mode == OP_TMA_MN ? 1u : 0u,
                                               (p.b_mode == OP_TMA_MN || p.b_mode == OP_GATHER_MN) ? 1u : 0u);
        const bool a_mn = p.a_mode == OP_TMA_MN;
        const bool b_mn = p.b_mode == OP_TMA_MN || p.b_mode == OP_GATHER_MN;
        for (int i = 0; i < nkb; ++i) {
            const int s = i % S;
            const uint32_t use = i / S;
            mbar_wait(&full[s], use & 1);
            tc_fence_after();
            if (lane == 0) {
                const uint32_t a_base = smem_u32(sA + s * Cfg::kABytes);
                const uint32_t b_base = smem_u32(sB + s * Cfg::kBBytes);
#pragma unroll
                for (int k = 0; k < BK / 16; ++k) {
                    // K-major: advance 32 bytes along the swizzled row.
                    // MN-major: advance two 8-row k-groups (2 x 1024 bytes).
                    const uint64_t ad = a_mn ? umma_desc_sw128(a_base + k * 2048, BK * 128, 1024)
                                             : umma_desc_sw128(a_base + k * 32, 0, 1024);
                    const uint64_t bd = b_mn ? umma_desc_sw128(b_base + k * 2048, BK * 128, 1024)
                                             : umma_desc_sw128(b_base + k * 32, 0, 1024);
                    umma_bf16(tmem_base, ad, bd, idesc, (i > 0 || k > 0) ? 1u : 0u);
                }
                umma_commit(&empty[s]);
                if (i == nkb - 1) umma_commit(tmem_full);
            }
            __syncwarp();
        }
        if (nkb == 0 && lane == 0) mbar_arrive(tmem_full);
    } else if (warp >= 4) {
        const int et = threadIdx.x - 128;  // 0..127
        // ---------------- gather producers
        if (any_gather) {
            constexpr int LAG = 2;
            // Precompute this thread's output-row coordinates for A gathers.
            int rn = 0, ry = 0, rx = 0;
            bool row_valid = false;
            if (a_gather) {
                const int m = m0 + et;
                row_valid = m < p.M;
                if (row_valid) {
                    const int hw = (p.gather_kind == GATHER_FPROP) ? p.g.Ho * p.g.Wo : p.g.H * p.g.W;
                    const int wd = (p.gather_kind == GATHER_FPROP) ? p.g.Wo : p.g.W;
                    rn = m / hw;
                    const int rem = m - rn * hw;
                    ry = rem / wd;
                    rx = rem - ry * wd;
                }
            }
            for (int i = 0; i < nkb; ++i) {
                const int s = i % S;
                const uint32_t use = i / S;
                mbar_wait(&empty[s], (use & 1) ^ 1);
                const int kb = kb_begin + i;
                if (a_gather) {
                    gather_rows_kmajor(p, smem_u32(sA + s * Cfg::kABytes), et, m0, kb, row_valid, rn, ry, rx);
                } else {
                    gather_wgrad_mn<BN>(p, smem_u32(sB + s * Cfg::kBBytes), et & 63, et >> 6, n0, kb);
                }
                cp_async_commit();
                if (i >= LAG) {
                    cp_async_wait<LAG>();
                    fence_proxy_async_smem();
                    mbar_arrive(&full[(i - LAG) % S]);
                }
            }
            cp_async_wait<0>();
            fence_proxy_async_smem();
            for (int i = max(0, nkb - LAG); i < nkb; ++i) mbar_arrive(&full[i % S]);
        }

        // ---------------- epilogue
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        const int ew = warp - 4;  // TMEM lane quarter
        const int row = m0 + ew * 32 + lane;
        const bool rv = row < p.M;
        for (int c0 = 0; c0 < BN; c0 += 32) {
            uint32_t r[32];
            tmem_ld32(tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + c0, r);
            tmem_ld_wait();
            if (!rv) continue;
            const int nb = n0 + c0;
            if (nb >= p.N) continue;
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * p.alpha;
            if (p.epi == EPI_F32_PARTIAL) {
                float* out = reinterpret_cast<float*>(p.D) + blockIdx.z * p.split_stride + row * p.ldd + nb;
                if (nb + 32 <= p.N && (p.ldd & 3) == 0) {
#pragma unroll
                    for (int j = 0; j < 32; j += 4)
                        *reinterpret_cast<float4*>(out + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                } else {
                    for (int j = 0; j < 32 && nb + j < p.N; ++j) out[j] = v[j];
                }
                continue;
            }
            if (p.bias) {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (nb + j < p.n_bias) v[j] += __ldg(p.bias + nb + j);
            }
            if (p.relu) {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
            }
            if (p.epi == EPI_BF16) {
                __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.D) + row * p.ldd + nb;
                if (nb + 32 <= p.N && (p.ldd & 7) == 0) {
#pragma unroll
                    for (int j = 0; j < 32; j += 8) {
                        uint4 q;
                        q.x = pack_bf16x2(v[j], v[j + 1]);
                        q.y = pack_bf16x2(v[j + 2], v[j + 3]);
                        q.z = pack_bf16x2(v[j + 4], v[j + 5]);
                        q.w = pack_bf16x2(v[j + 6], v[j + 7]);
                        *reinterpret_cast<uint4*>(out + j) = q;
                    }
                } else {
                    for (int j = 0; j < 32 && nb + j < p.N; ++j) out[j] = __float2bfloat16_rn(v[j]);
                }
            } else {  // EPI_F32
                float* out = reinterpret_cast<float*>(p.D) + row * p.ldd + nb;
                for (int j = 0; j < 32 && nb + j < p.N; ++j) out[j] = p.beta != 0.f ? v[j] + p.beta * out[j] : v[j];
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, Cfg::kTmemCols);
    }
}

}  // namespace tcb
