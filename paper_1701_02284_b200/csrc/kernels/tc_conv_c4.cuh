// First-layer convolution forward over a channel-stride-4 image (3 colour channels + 1 zero pad,
// 8 bytes per pixel: VGG-16 conv1_1 3x3/1, GoogLeNet / ResNet-50 conv1 7x7/2).
//
// The generic path gathers the im2col rows of such a layer with one 8-byte cp.async per filter tap
// and pixel straight from global memory, and a 128-pixel tile holds a single short k-block, so
// the kernel was paced by per-tile overhead (VGG conv1_1: 36 TF/s, 1.8 us per tile).  Here each
// 128-pixel tile first stages the input rows it touches (one 1-D bulk copy per row, 8 bytes per
// pixel, zero margins and zero rows for the padding) and 128 builder threads assemble the
// SWIZZLE_128B K-major A tile from shared memory (k = tap * 4 + channel, 16 taps per 64-wide
// k-block); the filter (B, K-major [Cout][R*S*4]) stays resident for the whole launch.
//
// Warp roles (512 threads): 0 row loader, 1 MMA issuer, 2 TMEM allocator, 3 filter loader,
// 4-7 and 12-15 two A-builder groups taking alternate k-blocks (one tile row per thread),
// 8-11 epilogue (bias / ReLU, bf16, TMA store).
#pragma once

#include <cuda_bf16.h>

#include "ptx.cuh"
#include "tc_gemm.cuh"

namespace tcb {

struct ConvC4Params {
    CUtensorMap tmB;  // filter [Cout][Kw] K-major, box {64, BN}
    CUtensorMap tmD;  // output store {ks, M, 1}, box {64 bf16 columns, 32 rows, 1}
    const __nv_bfloat16* x;  // NHWC, channel stride 4
    int H, W, Ho, Wo, R, S, stride, pad;
    int taps;         // R * S
    int nkb;          // k-blocks (16 taps each)
    int margin;       // zero pixels left of each staged row (even: 16-byte aligned rows)
    int rows_in;      // staged input rows per tile (max)
    int pitch;        // bytes per staged row
    int tiles;        // 128-pixel tiles (N * Ho * Wo / 128)
    int a_stages;     // A ring slots (16 KB each)
    int h_slots;      // staged-row slots (the loader runs up to h_slots tiles ahead of the builders)
    const float* bias;
    int n_bias, relu;
};

template <int BN>
struct ConvC4Cfg {
    static constexpr int kBBytes = BN * BK * 2;  // per k-block
    static constexpr int kAcc = 4;
    static constexpr uint32_t kTmemCols = kAcc * BN < 32 ? 32 : kAcc * BN;
};

constexpr int kC4Threads = 512;

template <int BN>
__global__ void __launch_bounds__(kC4Threads, 1) tc_conv_c4_fwd_kernel(const __grid_constant__ ConvC4Params p) {
    using Cfg = ConvC4Cfg<BN>;
    constexpr int NACC = Cfg::kAcc;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sB = smem;                                                   // nkb x kBBytes
    uint8_t* sA = sB + p.nkb * Cfg::kBBytes;                              // a_stages x 16 KB
    uint8_t* sHalo = sA + p.a_stages * (BM * 128);                        // h_slots x rows_in x pitch
    uint8_t* sStage = sHalo + ((p.h_slots * p.rows_in * p.pitch + 1023) & ~1023);  // 4 warps x 4 x 4 KB
    uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + 16 * kStagingBytes);
    uint64_t* b_full = bars;
    uint64_t* h_full = bars + 1;   // [8]
    uint64_t* h_empty = bars + 9;  // [8]
    uint64_t* a_full = bars + 17;  // [8]
    uint64_t* a_empty = bars + 25; // [8]
    uint64_t* tfull = bars + 33;   // [NACC]
    uint64_t* tempty = tfull + NACC;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NACC);

    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    const int AS = p.a_stages;
    const int HW = p.Ho * p.Wo;
    const uint32_t row_bytes = static_cast<uint32_t>(p.W) * 8;

    // zero the staged-row slots once: the margins are never written again
    for (uint32_t i = threadIdx.x; i < static_cast<uint32_t>(p.h_slots * p.rows_in * p.pitch) / 16; i += blockDim.x)
        st_shared_v4(smem_u32(sHalo) + i * 16, 0u, 0u, 0u, 0u);
    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.tmB);
        tma_prefetch(&p.tmD);
        mbar_init(b_full, 1);
        for (int s = 0; s < p.h_slots; ++s) {
            mbar_init(&h_full[s], 1);
            mbar_init(&h_empty[s], 256);  // both builder groups read every tile's rows
        }
        for (int s = 0; s < AS; ++s) {
            mbar_init(&a_full[s], 128);
            mbar_init(&a_empty[s], 1);
        }
        for (int b = 0; b < NACC; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4);
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<1>(tmem_slot, Cfg::kTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_trigger();
    pdl_wait();

    if (warp == 0) {
        // ---------------- halo loader: the input rows of tile u, one bulk copy per image row
        int hs = 0;
        uint32_t hph = 0;
        for (int u = blockIdx.x; u < p.tiles; u += gridDim.x) {
            mbar_wait(&h_empty[hs], hph ^ 1);
            const int m0 = u * BM;
            const int n = m0 / HW;
            const int y0 = (m0 - n * HW) / p.Wo, y1 = (m0 + BM - 1 - n * HW) / p.Wo;
            const int iy0 = y0 * p.stride - p.pad;
            const int rows = (y1 - y0) * p.stride + p.R;
            uint8_t* slot = sHalo + hs * p.rows_in * p.pitch;
            int valid = 0;
            for (int r = 0; r < rows; ++r) {
                const int iy = iy0 + r;
                if (iy >= 0 && iy < p.H) {
                    ++valid;
                } else {  // padding row: zero the interior (the margins are already zero)
                    for (uint32_t o = lane * 16; o < row_bytes; o += 32 * 16)
                        st_shared_v4(smem_u32(slot + r * p.pitch + p.margin * 8) + o, 0u, 0u, 0u, 0u);
                }
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive_expect_tx(&h_full[hs], valid * row_bytes);
                for (int r = 0; r < rows; ++r) {
                    const int iy = iy0 + r;
                    if (iy < 0 || iy >= p.H) continue;
                    const __nv_bfloat16* src = p.x + (static_cast<long long>(n) * p.H + iy) * p.W * 4;
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            smem_u32(slot + r * p.pitch + p.margin * 8)),
                        "l"(src), "r"(row_bytes), "r"(smem_u32(&h_full[hs]))
                        : "memory");
                }
            }
            __syncwarp();
            if (++hs == p.h_slots) {
                hs = 0;
                hph ^= 1;
            }
        }
    } else if (warp == 3) {
        // ---------------- filter loader (resident for the launch)
        for (int kb = 0; kb < p.nkb; ++kb) tma_load_2d_e<1>(sB + kb * Cfg::kBBytes, &p.tmB, smem_u32(b_full), kb * BK, 0);
        mbar_arrive_expect_tx_e(b_full, p.nkb * Cfg::kBBytes);
    } else if ((warp >= 4 && warp < 8) || warp >= 12) {
        // ---------------- A builders: two groups of 128 threads (thread t = tile row t) take
        // alternate k-blocks of the global k-block sequence (alternate tiles when a tile has one)
        const int bg = warp >= 12 ? 1 : 0;
        const int t = threadIdx.x - (bg ? 384 : 128);
        int hs = 0, as = 0, q = 0;
        uint32_t hph = 0, aph = 0;
        for (int u = blockIdx.x; u < p.tiles; u += gridDim.x) {
            const int m0 = u * BM;
            const int n = m0 / HW;
            const int y0 = (m0 - n * HW) / p.Wo;
            const int pix = m0 + t - n * HW;
            const int oy = pix / p.Wo, ox = pix - (pix / p.Wo) * p.Wo;
            mbar_wait(&h_full[hs], hph);
            // tap (kh, kw) of this pixel: staged row (oy - y0) * stride + kh, column ox * stride - pad + kw
            const uint32_t base = smem_u32(sHalo + hs * p.rows_in * p.pitch) +
                                  static_cast<uint32_t>((oy - y0) * p.stride * p.pitch + (ox * p.stride - p.pad + p.margin) * 8);
            for (int kb = 0; kb < p.nkb; ++kb, ++q) {
                if ((q & 1) == bg) {
                    mbar_wait(&a_empty[as], aph ^ 1);
                    const uint32_t dst = smem_u32(sA + as * (BM * 128)) + t * 128;
                    int kh = (kb * 16) / p.S, kw = kb * 16 - kh * p.S;
#pragma unroll
                    for (int j = 0; j < 16; j += 2) {
                        uint32_t v[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            if (kb * 16 + j + h < p.taps) {
                                asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];"
                                             : "=r"(v[2 * h]), "=r"(v[2 * h + 1])
                                             : "r"(base + kh * p.pitch + kw * 8));
                                if (++kw == p.S) {
                                    kw = 0;
                                    ++kh;
                                }
                            }
                        }
                        st_shared_v4(dst + (((j >> 1) ^ (t & 7)) << 4), v[0], v[1], v[2], v[3]);
                    }
                    fence_proxy_async_smem();
                    mbar_arrive(&a_full[as]);
                }
                if (++as == AS) {
                    as = 0;
                    aph ^= 1;
                }
            }
            mbar_arrive(&h_empty[hs]);
            if (++hs == p.h_slots) {
                hs = 0;
                hph ^= 1;
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        const uint32_t idesc = umma_idesc_bf16(BM, BN, 0u, 0u);
        const uint64_t a0 = umma_desc_sw128(smem_u32(sA), 0, 1024);
        const uint64_t b0 = umma_desc_sw128(smem_u32(sB), 0, 1024);
        mbar_wait(b_full, 0);
        tc_fence_after();
        int as = 0, tc = 0;
        uint32_t aph = 0;
        for (int u = blockIdx.x; u < p.tiles; u += gridDim.x, ++tc) {
            const int buf = tc % NACC;
            mbar_wait(&tempty[buf], ((tc / NACC) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d = tmem_base + buf * BN;
            for (int kb = 0; kb < p.nkb; ++kb) {
                mbar_wait(&a_full[as], aph);
                tc_fence_after();
                const uint64_t a_s = a0 + static_cast<uint64_t>(as * (BM * 128 >> 4));
                const uint64_t b_s = b0 + static_cast<uint64_t>(kb * (Cfg::kBBytes >> 4));
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                    umma_bf16_elect<1>(d, a_s + static_cast<uint64_t>(k * 2), b_s + static_cast<uint64_t>(k * 2), idesc,
                                       (kb > 0 || k > 0) ? 1u : 0u);
                umma_commit_elect<1>(&a_empty[as]);
                if (++as == AS) {
                    as = 0;
                    aph ^= 1;
                }
            }
            umma_commit_elect<1>(&tfull[buf]);
        }
    } else if (warp >= 8) {
        // ---------------- epilogue: warp q = rows 32 q .. +32, BN columns in 64-column chunks
        const int quarter = warp - 8;
        uint8_t* stg = sStage + quarter * 4 * kStagingBytes;
        int nstore = 0, tc = 0;
        for (int u = blockIdx.x; u < p.tiles; u += gridDim.x, ++tc) {
            const int buf = tc % NACC;
            mbar_wait(&tfull[buf], (tc / NACC) & 1);
            tc_fence_after();
            const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + buf * BN;
            for (int c0 = 0; c0 < BN; c0 += 64) {
                uint32_t r0[32], r1[32];
                tmem_ld32(t_row + c0, r0);
                tmem_ld32(t_row + c0 + 32, r1);
                float b0 = 0.f, b1 = 0.f;
                if (p.bias) {
                    if (c0 + lane < p.n_bias) b0 = __ldg(p.bias + c0 + lane);
                    if (c0 + 32 + lane < p.n_bias) b1 = __ldg(p.bias + c0 + 32 + lane);
                }
                tmem_ld_wait();
                if (c0 + 64 >= BN) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[buf]);
                }
                uint32_t packed[32];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    float x0 = __uint_as_float(r0[2 * j]) + __shfl_sync(0xffffffffu, b0, 2 * j);
                    float x1 = __uint_as_float(r0[2 * j + 1]) + __shfl_sync(0xffffffffu, b0, 2 * j + 1);
                    float x2 = __uint_as_float(r1[2 * j]) + __shfl_sync(0xffffffffu, b1, 2 * j);
                    float x3 = __uint_as_float(r1[2 * j + 1]) + __shfl_sync(0xffffffffu, b1, 2 * j + 1);
                    if (p.relu) {
                        x0 = fmaxf(x0, 0.f);
                        x1 = fmaxf(x1, 0.f);
                        x2 = fmaxf(x2, 0.f);
                        x3 = fmaxf(x3, 0.f);
                    }
                    packed[j] = pack_bf16x2(x0, x1);
                    packed[16 + j] = pack_bf16x2(x2, x3);
                }
                uint8_t* buf_s = stg + (nstore & 3) * kStagingBytes;
                if (nstore >= 4) bulk_wait_read<3>();
                __syncwarp();
                const uint32_t row_addr = smem_u32(buf_s);
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    st_shared_v4(row_addr + sw128_off(lane, q), packed[4 * q], packed[4 * q + 1], packed[4 * q + 2],
                                 packed[4 * q + 3]);
                fence_proxy_async_smem();
                __syncwarp();
                tma_store_3d_e(&p.tmD, buf_s, c0, u * BM + quarter * 32, 0);
                bulk_commit();
                ++nstore;
            }
        }
        bulk_wait<0>();
        __syncwarp();
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<1>(tmem_base, Cfg::kTmemCols);
    }
}

// Filter gradient of the same layers:  dW^T[k][cout] = sum_p A[p][k] * dy[p][cout]  with the A
// tiles (k = tap * 4 + channel) assembled exactly as in the forward from staged input rows.  The
// built [128 pixel][64 k] k-blocks are MN-major operands for M = k (two k-blocks per 128-row MMA,
// LBO = one k-block), dy tiles ([128 pixel][64 cout], one TMA box) are the MN-major N = 64 side,
// and the accumulators (ceil(nkb / 2) x 64 TMEM columns) live for the CTA's whole pixel range;
// fp32 partials go out transposed to [split][cout][Kw] for the fixed-order reduce.
struct ConvC4WgradParams {
    CUtensorMap tmDy;  // dy [M pixels][ks] K... box {64 cout, 128 pixels}, SW128
    CUtensorMap tmWs;  // partials {Kw, K, splits} fp32, box {32, 32, 1}
    const __nv_bfloat16* x;
    int H, W, Ho, Wo, R, S, stride, pad, taps, nkb, nkb2;  // nkb2 = nkb rounded up to even
    int margin, rows_in, pitch, h_slots;
    int K, Kw;
    int tiles, tiles_per_split;
    float* bias_ws;  // folded bias gradient: per-split dy column sums [splits][K], or nullptr
};

__global__ void __launch_bounds__(kC4Threads, 1) tc_conv_c4_wgrad_kernel(const __grid_constant__ ConvC4WgradParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t tile_bytes = static_cast<uint32_t>(p.nkb2) * BM * 128 + BM * 128;  // A k-blocks + dy
    uint8_t* sT = smem;                                                    // 2 tile slots
    uint8_t* sHalo = sT + 2 * tile_bytes;                                  // h_slots x rows_in x pitch
    uint8_t* sStage = sHalo + ((p.h_slots * p.rows_in * p.pitch + 1023) & ~1023);  // 4 warps x 4 KB
    uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + 4 * kStagingBytes);
    uint64_t* h_full = bars;        // [8]
    uint64_t* h_empty = bars + 8;   // [8]
    uint64_t* t_full = bars + 16;   // [2]
    uint64_t* t_empty = bars + 18;  // [2]
    uint64_t* tdone = bars + 20;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 21);

    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    const int HW = p.Ho * p.Wo;
    const uint32_t row_bytes = static_cast<uint32_t>(p.W) * 8;
    const int sp = blockIdx.x;
    const int tile0 = sp * p.tiles_per_split, tile1 = min(p.tiles, tile0 + p.tiles_per_split);
    const int halves = p.nkb2 / 2;
    const uint32_t tmem_cols = halves * 64 <= 64 ? 64 : halves * 64 <= 128 ? 128 : 256;

    // zero the staged-row slots (margins) and both tile slots (an odd nkb leaves one k-block
    // per tile that the builders never write: it must read as zeros)
    for (uint32_t i = threadIdx.x; i < (2 * tile_bytes) / 16; i += blockDim.x) st_shared_v4(smem_u32(sT) + i * 16, 0u, 0u, 0u, 0u);
    for (uint32_t i = threadIdx.x; i < static_cast<uint32_t>(p.h_slots * p.rows_in * p.pitch) / 16; i += blockDim.x)
        st_shared_v4(smem_u32(sHalo) + i * 16, 0u, 0u, 0u, 0u);
    fence_proxy_async_smem();
    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.tmDy);
        tma_prefetch(&p.tmWs);
        for (int s = 0; s < p.h_slots; ++s) {
            mbar_init(&h_full[s], 1);
            mbar_init(&h_empty[s], 256);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&t_full[s], 256 + 1);  // both builder groups + the dy load's arrive
            mbar_init(&t_empty[s], p.bias_ws ? 5 : 1);  // + the 4 epilogue warps summing dy
        }
        mbar_init(tdone, 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<1>(tmem_slot, tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_trigger();
    pdl_wait();

    if (warp == 0) {
        // ---------------- loader: staged input rows of the tile + its dy box
        int hs = 0, ts = 0;
        uint32_t hph = 0, tph = 0;
        for (int u = tile0; u < tile1; ++u) {
            mbar_wait(&h_empty[hs], hph ^ 1);
            const int m0 = u * BM;
            const int n = m0 / HW;
            const int y0 = (m0 - n * HW) / p.Wo, y1 = (m0 + BM - 1 - n * HW) / p.Wo;
            const int iy0 = y0 * p.stride - p.pad;
            const int rows = (y1 - y0) * p.stride + p.R;
            uint8_t* slot = sHalo + hs * p.rows_in * p.pitch;
            int valid = 0;
            for (int r = 0; r < rows; ++r) {
                const int iy = iy0 + r;
                if (iy >= 0 && iy < p.H) {
                    ++valid;
                } else {
                    for (uint32_t o = lane * 16; o < row_bytes; o += 32 * 16)
                        st_shared_v4(smem_u32(slot + r * p.pitch + p.margin * 8) + o, 0u, 0u, 0u, 0u);
                }
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive_expect_tx(&h_full[hs], valid * row_bytes);
                for (int r = 0; r < rows; ++r) {
                    const int iy = iy0 + r;
                    if (iy < 0 || iy >= p.H) continue;
                    const __nv_bfloat16* src = p.x + (static_cast<long long>(n) * p.H + iy) * p.W * 4;
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            smem_u32(slot + r * p.pitch + p.margin * 8)),
                        "l"(src), "r"(row_bytes), "r"(smem_u32(&h_full[hs]))
                        : "memory");
                }
            }
            __syncwarp();
            // dy of the tile into the tile slot (after the MMA released it)
            mbar_wait(&t_empty[ts], tph ^ 1);
            tma_load_2d_e<1>(sT + ts * tile_bytes + p.nkb2 * BM * 128, &p.tmDy, smem_u32(&t_full[ts]), 0, m0);
            mbar_arrive_expect_tx_e(&t_full[ts], BM * 128);
            if (++hs == p.h_slots) {
                hs = 0;
                hph ^= 1;
            }
            if (++ts == 2) {
                ts = 0;
                tph ^= 1;
            }
        }
    } else if ((warp >= 4 && warp < 8) || warp >= 12) {
        // ---------------- A builders (as in the forward), k-blocks alternating between the groups
        const int bg = warp >= 12 ? 1 : 0;
        const int t = threadIdx.x - (bg ? 384 : 128);
        int hs = 0, ts = 0;
        uint32_t hph = 0, tph = 0;
        for (int u = tile0; u < tile1; ++u) {
            const int m0 = u * BM;
            const int n = m0 / HW;
            const int y0 = (m0 - n * HW) / p.Wo;
            const int pix = m0 + t - n * HW;
            const int oy = pix / p.Wo, ox = pix - (pix / p.Wo) * p.Wo;
            mbar_wait(&h_full[hs], hph);
            mbar_wait(&t_empty[ts], tph ^ 1);
            const uint32_t base = smem_u32(sHalo + hs * p.rows_in * p.pitch) +
                                  static_cast<uint32_t>((oy - y0) * p.stride * p.pitch + (ox * p.stride - p.pad + p.margin) * 8);
            for (int kb = bg; kb < p.nkb; kb += 2) {
                const uint32_t dst = smem_u32(sT + ts * tile_bytes + kb * (BM * 128)) + t * 128;
                int kh = (kb * 16) / p.S, kw = kb * 16 - kh * p.S;
#pragma unroll
                for (int j = 0; j < 16; j += 2) {
                    uint32_t v[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (kb * 16 + j + h < p.taps) {
                            asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];"
                                         : "=r"(v[2 * h]), "=r"(v[2 * h + 1])
                                         : "r"(base + kh * p.pitch + kw * 8));
                            if (++kw == p.S) {
                                kw = 0;
                                ++kh;
                            }
                        }
                    }
                    st_shared_v4(dst + (((j >> 1) ^ (t & 7)) << 4), v[0], v[1], v[2], v[3]);
                }
            }
            fence_proxy_async_smem();
            mbar_arrive(&t_full[ts]);
            mbar_arrive(&h_empty[hs]);
            if (++hs == p.h_slots) {
                hs = 0;
                hph ^= 1;
            }
            if (++ts == 2) {
                ts = 0;
                tph ^= 1;
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA: M = 128 k (two k-blocks), N = 64 cout, K = 128 pixels per tile
        const uint32_t idesc = umma_idesc_bf16(BM, 64, 1u, 1u);
        int ts = 0;
        uint32_t tph = 0;
        bool first = true;
        for (int u = tile0; u < tile1; ++u) {
            mbar_wait(&t_full[ts], tph);
            tc_fence_after();
            const uint32_t tb = smem_u32(sT + ts * tile_bytes);
            const uint64_t b0 = umma_desc_sw128(tb + p.nkb2 * BM * 128, 0, 1024);
            for (int h = 0; h < halves; ++h) {
                const uint64_t a0 = umma_desc_sw128(tb + 2 * h * BM * 128, BM * 128, 1024);
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    umma_bf16_elect<1>(tmem_base + h * 64, a0 + static_cast<uint64_t>(k * 128),
                                       b0 + static_cast<uint64_t>(k * 128), idesc, (!first || k > 0) ? 1u : 0u);
            }
            first = false;
            umma_commit_elect<1>(&t_empty[ts]);
            if (++ts == 2) {
                ts = 0;
                tph ^= 1;
            }
        }
        umma_commit_elect<1>(tdone);
    } else if (warp >= 8 && warp < 12) {
        // ---------------- epilogue: warp q holds k = 128 h + 32 q + lane; transposed 32 x 32 stores
        const int quarter = warp - 8;
        uint8_t* stg = sStage + quarter * kStagingBytes;
        if (p.bias_ws) {
            // folded bias gradient (as wgrad_bias_sums): thread e sums 16-byte chunk kc of the
            // tile's dy rows rg, rg + 16, ... (SW128 chunk kc ^ (rg & 7)) while the MMA runs
            const int e = threadIdx.x - 256, kc = e & 7, rg = e >> 3;
            float acc[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = 0.f;
            int ts = 0;
            uint32_t tph = 0;
            for (int u = tile0; u < tile1; ++u) {
                mbar_wait(&t_full[ts], tph);
                const uint32_t src = smem_u32(sT + ts * tile_bytes + p.nkb2 * BM * 128) + rg * 128 + ((kc ^ (rg & 7)) << 4);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    uint4 v;
                    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                                 : "r"(src + i * 16 * 128)
                                 : "memory");
                    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float2 f = __bfloat1622float2(h[q]);
                        acc[2 * q] += f.x;
                        acc[2 * q + 1] += f.y;
                    }
                }
                fence_proxy_async_smem();  // generic reads ordered before the slot's async-proxy refill
                __syncwarp();
                if (lane == 0) mbar_arrive(&t_empty[ts]);
                if (++ts == 2) {
                    ts = 0;
                    tph ^= 1;
                }
            }
            float* red = reinterpret_cast<float*>(sStage);  // [16 row groups][64 channels]
#pragma unroll
            for (int j = 0; j < 8; ++j) red[rg * 64 + kc * 8 + j] = acc[j];
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (e < 64) {
                float sum = 0.f;
                for (int g = 0; g < 16; ++g) sum += red[g * 64 + e];
                if (e < p.K) p.bias_ws[static_cast<long long>(sp) * p.K + e] = sum;
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");  // the staging is reused below
        }
        if (tile1 > tile0) {
            mbar_wait(tdone, 0);
            tc_fence_after();
        }
        int nstore = 0;
        for (int h = 0; h < halves; ++h) {
            for (int c0 = 0; c0 < 64; c0 += 32) {
                uint32_t r[32];
                if (tile1 > tile0) {
                    tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + h * 64 + c0, r);
                    tmem_ld_wait();
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) r[j] = 0u;
                }
                if (nstore > 0) bulk_wait_read<0>();
                __syncwarp();
                const uint32_t base = smem_u32(stg);
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    asm volatile("st.shared.b32 [%0], %1;" ::"r"(base + j * 128 + ((((lane >> 2) ^ (j & 7)) << 4) | ((lane & 3) << 2))),
                                 "r"(r[j])
                                 : "memory");
                fence_proxy_async_smem();
                __syncwarp();
                const int k0 = h * 128 + quarter * 32;
                if (k0 < p.Kw && c0 < p.K) tma_store_3d_e(&p.tmWs, stg, k0, c0, sp);
                bulk_commit();
                ++nstore;
            }
        }
        bulk_wait<0>();
        __syncwarp();
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<1>(tmem_base, tmem_cols);
    }
}

}  // namespace tcb
