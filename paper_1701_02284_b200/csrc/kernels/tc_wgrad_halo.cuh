// Halo-tile filter gradient for stride-1 convolutions:
//
//   dW[k][tap][c] = sum over output pixels p of dy[p][k] * x[p + off(tap)][c]
//
// The im2col form (tc_gemm_kernel with an OP_IM2COL_MN B operand) streams x from L2 once per filter
// tap.  Here a pixel tile is 128 positions laid out with row stride wr (th = 128 / wr output rows of
// wv = wr - (S - 1) pixels each); per tile ONE tiled TMA box per 64-channel block stages the
// (th + R - 1) x wr input halo, and every tap of the unit's tap group reads it as a row-shifted
// MN-major SW128 view (start shifted by kh * wr + kw rows; the swizzle is address-based).  dy is
// staged one output row at a time (box {64, wv, 1, 1}) into the same row-stride-wr layout, so the
// wr - wv gap positions of every row stay zero (written once at kernel start) and contribute nothing
// (they pair with wrapped halo rows).
//
//   unit  = (128-channel block of k (M), tap group (nt taps), channel group (CB x 64 c), pixel split)
//   TMEM  = nt accumulators of CB * 64 fp32 columns, live for the whole pixel range of the unit
//   MMA   = per tile, per tap, 8 k-steps of 16 pixels: M = 128 (k), N = CB * 64 (c), MN-major A / B
//   out   = fp32 partials [split][K][R*S][wcs] (TMA store), summed in fixed order by splitk_reduce
//
// Warp roles (256 threads): 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 4-7 epilogue.
#pragma once

#include <cuda_bf16.h>

#include "ptx.cuh"
#include "tc_gemm.cuh"

namespace tcb {

struct WgradHaloParams {
    CUtensorMap tmX;   // 4-D tiled {cs, W, H, N} over x, box {64, wr, hh, 1}, SW128
    CUtensorMap tmDy;  // 4-D tiled {ks, Wo, Ho, N} over dy, box {64, wv, 1, 1}, SW128
    CUtensorMap tmWs;  // 3-D store {R*S*wcs, K, splits} fp32, box {32, 32, 1}, SW128
    int K;             // output channels (GEMM M)
    int R, S, pad;
    int wr, th, hh, wv, xt, yt, nimg;
    int Ho, Wo;
    int ntap, ntg;     // taps per group (accumulators), tap groups
    int ncg;           // channel groups of CB x 64 channels
    int nc;            // MMA N / accumulator columns per tap: CB * 64, or (one group) cs rounded up to 32
    int cs;            // x channel stride
    int wcs;           // workspace columns per tap (cs rounded up to 32: D column of tap t, channel c: t * wcs + c)
    int mt;            // 128-row blocks of K
    int splits, tiles, tiles_per_split;
    uint32_t dy_bytes;    // dy tile: 2 k-atoms x 128 rows x 128 B
    uint32_t halo_bytes;  // per 64-channel halo (1024-aligned, includes the over-read slack)
    uint32_t stage_bytes; // dy tile + CB halos
    int stages;
    float* bias_ws;       // folded bias gradient: per-split partial sums [splits][K] of dy, or nullptr
};

// Folded bias gradient, run by the 4 epilogue warps (threads 128..255) of one unit per (k block,
// split) while the MMA consumes the same stages: per staged dy tile (natoms k-atoms of 128 rows x
// 64 k, SW128, zero gap rows) the column sums over the 128 rows; each stage is released by one
// arrival per warp (the stage's empty barrier counts the MMA commit + 4).  Thread e owns the
// 16-byte chunk kc of atom a over rows rg, rg + rgs, ...: with rgs a multiple of 8 the SW128
// chunk of all its rows is kc ^ (rg & 7).  The row groups are summed in fixed order at the end,
// through the (not yet used) epilogue staging; out: bias_ws[sp][k_base + k].
__device__ __forceinline__ void wgrad_bias_sums(const WgradHaloParams& p, const uint8_t* smem, uint8_t* sStage,
                                                uint64_t* full, uint64_t* empty, int tile0, int tile1, int natoms,
                                                int k_base, int sp, int lane) {
    const int e = threadIdx.x - 128;
    const int combos = natoms * 8, rgs = 128 / combos;
    const int combo = e % combos, rg = e / combos, a = combo >> 3, kc = combo & 7;
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    int s = 0;
    uint32_t ph = 0;
    for (int t = tile0; t < tile1; ++t) {
        mbar_wait(&full[s], ph);
        const uint32_t src = smem_u32(smem) + s * p.stage_bytes + a * (BM * 128) + rg * 128 + ((kc ^ (rg & 7)) << 4);
        for (int i = 0; i < 128 / rgs; ++i) {
            uint4 v;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                         : "r"(src + i * rgs * 128)
                         : "memory");
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 f = __bfloat1622float2(h[q]);
                acc[2 * q] += f.x;
                acc[2 * q + 1] += f.y;
            }
        }
        // generic-proxy reads of a TMA-written stage must be ordered before the async-proxy refill
        // the release enables (without this fence a refill could land under the last reads: rare
        // wrong tiles in the sums, seen only with a concurrent side-stream kernel)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == p.stages) {
            s = 0;
            ph ^= 1;
        }
    }
    float* red = reinterpret_cast<float*>(sStage);  // [rgs][natoms * 64]
    const int row = natoms * 64;
#pragma unroll
    for (int j = 0; j < 8; ++j) red[rg * row + combo * 8 + j] = acc[j];
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (e < row) {
        float sum = 0.f;
        for (int g = 0; g < rgs; ++g) sum += red[g * row + e];
        const int k = k_base + e;
        if (k < p.K) p.bias_ws[static_cast<long long>(sp) * p.K + k] = sum;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");  // the staging is reused by the stores that follow
}

template <int CB>
__global__ void __launch_bounds__(256, 1) tc_wgrad_halo_kernel(const __grid_constant__ WgradHaloParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages;
    uint8_t* sStage = smem + S * p.stage_bytes;  // epilogue staging: 4 warps x 4 KB
    uint64_t* full = reinterpret_cast<uint64_t*>(sStage + 4 * kStagingBytes);
    uint64_t* empty = full + 4;
    uint64_t* tdone = empty + 4;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tdone + 1);

    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;

    // unit decode: m block fastest (units sharing a tile of x / dy run side by side)
    int u = blockIdx.x;
    const int mb = u % p.mt;
    u /= p.mt;
    const int cg = u % p.ncg;
    u /= p.ncg;
    const int tg = u % p.ntg;
    const int sp = u / p.ntg;
    const int t0 = tg * p.ntap;
    const int taps_here = min(p.ntap, p.R * p.S - t0);
    const int tile0 = sp * p.tiles_per_split;
    const int tile1 = min(p.tiles, tile0 + p.tiles_per_split);
    const uint32_t ncols = static_cast<uint32_t>(p.ntap) * p.nc;
    // the (channel group 0, tap group 0) unit of each (m block, split) also sums its dy tiles over
    // the pixels (the bias gradient): its epilogue warps read every staged dy tile from shared
    // memory while the MMA runs, so each stage is released by the MMA commit + 4 warp arrivals
    const bool do_bias = p.bias_ws != nullptr && cg == 0 && tg == 0;
    const uint32_t tmem_cols = ncols <= 32 ? 32 : ncols <= 64 ? 64 : ncols <= 128 ? 128 : ncols <= 256 ? 256 : 512;

    // zero every stage and the staging once: the dy gap positions (wr - wv per row) and the halo
    // over-read slack are never written by TMA (gap rows must be 0, slack rows finite: they meet
    // in the products of the wrapped positions)
    for (uint32_t i = threadIdx.x; i < (S * p.stage_bytes + 4 * kStagingBytes) / 16; i += blockDim.x)
        st_shared_v4(smem_u32(smem) + i * 16, 0u, 0u, 0u, 0u);
    fence_proxy_async_smem();
    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.tmX);
        tma_prefetch(&p.tmDy);
        tma_prefetch(&p.tmWs);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], do_bias ? 5 : 1);
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

    const int per_img = p.yt * p.xt;
    if (warp == 0) {
        // ---------------- TMA producer: per tile, th dy row loads per k-atom + CB halo boxes
        int s = 0;
        uint32_t ph = 0;
        const uint32_t tx = static_cast<uint32_t>(2 * p.th * p.wv * 128) + CB * static_cast<uint32_t>(p.hh * p.wr * 128);
        for (int t = tile0; t < tile1; ++t) {
            mbar_wait(&empty[s], ph ^ 1);
            const int img = t / per_img;
            const int r = t - img * per_img;
            const int ty = r / p.xt;
            const int y0 = ty * p.th, x0 = (r - ty * p.xt) * p.wv;
            uint8_t* st = smem + s * p.stage_bytes;
            const uint32_t bar = smem_u32(&full[s]);
            for (int a = 0; a < 2; ++a)
                for (int j = 0; j < p.th; ++j)
                    tma_load_4d_e(st + a * (p.dy_bytes / 2) + j * p.wr * 128, &p.tmDy, bar, mb * 128 + a * 64, x0,
                                  y0 + j, img);
            for (int c = 0; c < CB; ++c)
                tma_load_4d_e(st + p.dy_bytes + c * p.halo_bytes, &p.tmX, bar, (cg * CB + c) * 64, x0 - p.pad,
                              y0 - p.pad, img);
            mbar_arrive_expect_tx_e(&full[s], tx);
            if (++s == S) {
                s = 0;
                ph ^= 1;
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        const uint32_t idesc = umma_idesc_bf16(BM, static_cast<uint32_t>(p.nc), 1u, 1u);
        // A = dy tile, MN-major: k-atoms 128 rows x 128 B apart (LBO), 8-row groups 1 KB (SBO);
        // a k-step of 16 pixels = 2 KB.  B = halo, MN-major: channel blocks halo_bytes apart.
        const uint64_t a0 = umma_desc_sw128(smem_u32(smem), p.dy_bytes / 2, 1024);
        const uint64_t b0 = umma_desc_sw128(smem_u32(smem) + p.dy_bytes, p.halo_bytes, 1024);
        const uint64_t step16 = p.stage_bytes >> 4;
        int s = 0;
        uint32_t ph = 0;
        bool first = true;
        for (int t = tile0; t < tile1; ++t) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint64_t so = static_cast<uint64_t>(s) * step16;
            int kh = t0 / p.S, kw = t0 - (t0 / p.S) * p.S;
            for (int j = 0; j < taps_here; ++j) {
                const uint64_t b_tap = b0 + so + static_cast<uint64_t>((kh * p.wr + kw) * 8);
                const uint32_t d = tmem_base + j * p.nc;
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    umma_bf16_elect<1>(d, a0 + so + static_cast<uint64_t>(k * 128), b_tap + static_cast<uint64_t>(k * 128),
                                       idesc, (!first || k > 0) ? 1u : 0u);
                if (++kw == p.S) {
                    kw = 0;
                    ++kh;
                }
            }
            first = false;
            umma_commit_elect<1>(&empty[s]);
            if (++s == S) {
                s = 0;
                ph ^= 1;
            }
        }
        umma_commit_elect<1>(tdone);
    } else if (warp >= 4) {
        // ---------------- epilogue: warp e reads TMEM lanes 32 (e - 4) .. +32 (rows k)
        const int quarter = warp - 4;
        uint8_t* stg = sStage + quarter * kStagingBytes;
        if (do_bias) wgrad_bias_sums(p, smem, sStage, full, empty, tile0, tile1, 2, mb * 128, sp, lane);
        mbar_wait(tdone, 0);
        tc_fence_after();
        const int m0 = mb * 128 + quarter * 32;
        int nstore = 0;
        if (tile1 > tile0) {
            for (int j = 0; j < taps_here; ++j) {
                for (int c0 = 0; c0 < p.nc; c0 += 32) {
                    uint32_t r[32];
                    tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + j * p.nc + c0, r);
                    tmem_ld_wait();
                    if (nstore > 0) bulk_wait_read<0>();
                    __syncwarp();
                    const uint32_t row_addr = smem_u32(stg);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        st_shared_v4(row_addr + sw128_off(lane, q), r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
                    fence_proxy_async_smem();
                    __syncwarp();
                    const int col = (t0 + j) * p.wcs + cg * CB * 64 + c0;
                    if (m0 < p.K && cg * CB * 64 + c0 < p.cs) tma_store_3d_e(&p.tmWs, stg, col, m0, sp);
                    bulk_commit();
                    ++nstore;
                }
            }
        } else {
            // empty pixel range: this split's partial is zero
            for (int i = lane; i < 32 * 32; i += 32) reinterpret_cast<uint32_t*>(stg)[i] = 0u;
            fence_proxy_async_smem();
            __syncwarp();
            for (int j = 0; j < taps_here; ++j)
                for (int c0 = 0; c0 < p.nc; c0 += 32) {
                    if (nstore > 0) bulk_wait_read<0>();
                    __syncwarp();
                    if (m0 < p.K && cg * CB * 64 + c0 < p.cs)
                        tma_store_3d_e(&p.tmWs, stg, (t0 + j) * p.wcs + cg * CB * 64 + c0, m0, sp);
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

// Narrow-k form (K <= 64 output channels, e.g. VGG conv1_2, or K < 128 not a multiple of 64,
// e.g. AlexNet conv1's 96): the transposed product
//   dW^T[(tap, c)][k] = sum_p x[p + off(tap)][c] * dy[p][k]
// with M = two taps x 64 channels of the halo (two MN-major atoms of one halo, LBO = the two taps'
// shift difference), N = K rounded to 16 (one or two 64-channel dy atoms), so the 128-row MMA is
// full where the direct form would fill K of its rows.  Up to 512 TMEM columns of tap pairs per
// unit (8 pairs at K <= 64, 4 at K <= 128); the epilogue transposes each 32 x 32 chunk through
// shared memory into the [k][tap][c] partials.
__global__ void __launch_bounds__(256, 1) tc_wgrad_halo_swap_kernel(const __grid_constant__ WgradHaloParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages;
    uint8_t* sStage = smem + S * p.stage_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(sStage + 4 * kStagingBytes);
    uint64_t* empty = full + 4;
    uint64_t* tdone = empty + 4;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tdone + 1);

    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    int u = blockIdx.x;
    const int cg = u % p.ncg;
    u /= p.ncg;
    const int tg = u % p.ntg;
    const int sp = u / p.ntg;
    const int t0 = tg * p.ntap;
    const int taps_here = min(p.ntap, p.R * p.S - t0);
    const int pairs = (taps_here + 1) / 2;
    const int tile0 = sp * p.tiles_per_split;
    const int tile1 = min(p.tiles, tile0 + p.tiles_per_split);
    const int NK = p.K <= 64 ? 64 : 128;  // accumulator columns per tap pair (k padded to 64 / 128)
    const uint32_t ncols = static_cast<uint32_t>((p.ntap + 1) / 2) * NK;
    const uint32_t tmem_cols = ncols <= 64 ? 64 : ncols <= 128 ? 128 : ncols <= 256 ? 256 : 512;
    const bool do_bias = p.bias_ws != nullptr && cg == 0 && tg == 0;  // see wgrad_bias_sums

    for (uint32_t i = threadIdx.x; i < (S * p.stage_bytes + 4 * kStagingBytes) / 16; i += blockDim.x)
        st_shared_v4(smem_u32(smem) + i * 16, 0u, 0u, 0u, 0u);
    fence_proxy_async_smem();
    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.tmX);
        tma_prefetch(&p.tmDy);
        tma_prefetch(&p.tmWs);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], do_bias ? 5 : 1);
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

    const int per_img = p.yt * p.xt;
    if (warp == 0) {
        int s = 0;
        uint32_t ph = 0;
        const int natoms = NK / 64;  // 64-channel dy atoms
        const uint32_t tx = static_cast<uint32_t>(natoms * p.th * p.wv * 128) + static_cast<uint32_t>(p.hh * p.wr * 128);
        for (int t = tile0; t < tile1; ++t) {
            mbar_wait(&empty[s], ph ^ 1);
            const int img = t / per_img;
            const int r = t - img * per_img;
            const int ty = r / p.xt;
            const int y0 = ty * p.th, x0 = (r - ty * p.xt) * p.wv;
            uint8_t* st = smem + s * p.stage_bytes;
            const uint32_t bar = smem_u32(&full[s]);
            for (int a = 0; a < natoms; ++a)
                for (int j = 0; j < p.th; ++j)
                    tma_load_4d_e(st + a * (BM * 128) + j * p.wr * 128, &p.tmDy, bar, a * 64, x0, y0 + j, img);
            tma_load_4d_e(st + p.dy_bytes, &p.tmX, bar, cg * 64, x0 - p.pad, y0 - p.pad, img);
            mbar_arrive_expect_tx_e(&full[s], tx);
            if (++s == S) {
                s = 0;
                ph ^= 1;
            }
        }
    } else if (warp == 1) {
        // N = the real output channels rounded to 16 (MN-major dy atoms of 64 channels, LBO = one atom)
        const uint32_t idesc = umma_idesc_bf16(BM, static_cast<uint32_t>((p.K + 15) / 16 * 16), 1u, 1u);
        const uint64_t step16 = p.stage_bytes >> 4;
        const uint64_t b0 = umma_desc_sw128(smem_u32(smem), BM * 128, 1024);
        int s = 0;
        uint32_t ph = 0;
        bool first = true;
        for (int t = tile0; t < tile1; ++t) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint32_t halo = smem_u32(smem) + s * p.stage_bytes + p.dy_bytes;
            const uint64_t so = static_cast<uint64_t>(s) * step16;
            for (int q = 0; q < pairs; ++q) {
                const int ta = t0 + 2 * q, tb = min(ta + 1, t0 + taps_here - 1);
                const int sa = (ta / p.S) * p.wr + ta % p.S, sb = (tb / p.S) * p.wr + tb % p.S;
                // atom 1 (rows 64-127 of M) = tap tb's view: LBO = the shift difference (>= 0;
                // a lone last tap repeats itself and its rows are not stored)
                const uint64_t a_pair = umma_desc_sw128(halo + sa * 128, (sb - sa) * 128, 1024);
                const uint32_t d = tmem_base + q * NK;
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    umma_bf16_elect<1>(d, a_pair + static_cast<uint64_t>(k * 128), b0 + so + static_cast<uint64_t>(k * 128),
                                       idesc, (!first || k > 0) ? 1u : 0u);
            }
            first = false;
            umma_commit_elect<1>(&empty[s]);
            if (++s == S) {
                s = 0;
                ph ^= 1;
            }
        }
        umma_commit_elect<1>(tdone);
    } else if (warp >= 4) {
        // warp e: TMEM lanes 32 (e - 4) .. +32 = tap (e - 4) / 2 of each pair, channels 32 ((e - 4) % 2) + lane
        const int quarter = warp - 4;
        uint8_t* stg = sStage + quarter * kStagingBytes;
        if (do_bias) wgrad_bias_sums(p, smem, sStage, full, empty, tile0, tile1, NK / 64, 0, sp, lane);
        mbar_wait(tdone, 0);
        tc_fence_after();
        const int csub = (quarter & 1) * 32;
        int nstore = 0;
        for (int q = 0; q < pairs; ++q) {
            const int tap = t0 + 2 * q + (quarter >> 1);
            const bool tap_ok = tap < t0 + taps_here && cg * 64 + csub < p.cs;
            for (int k0 = 0; k0 < NK; k0 += 32) {
                uint32_t r[32];
                tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + q * NK + k0, r);
                tmem_ld_wait();
                if (tile1 <= tile0) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) r[j] = 0u;
                }
                if (nstore > 0) bulk_wait_read<0>();
                __syncwarp();
                // transpose: staging row j (= output channel k0 + j) holds the 32 channels c (lanes)
                const uint32_t base = smem_u32(stg);
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    asm volatile("st.shared.b32 [%0], %1;" ::"r"(base + j * 128 + ((((lane >> 2) ^ (j & 7)) << 4) | ((lane & 3) << 2))),
                                 "r"(r[j])
                                 : "memory");
                fence_proxy_async_smem();
                __syncwarp();
                if (tap_ok && k0 < p.K) tma_store_3d_e(&p.tmWs, stg, tap * p.wcs + cg * 64 + csub, k0, sp);
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
