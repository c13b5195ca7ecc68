// Halo-tile implicit GEMM for stride-1 convolutions (fprop over x, bwd-data over dy).
//
// The im2col operand of tc_gemm_kernel (OP_IM2COL_K) re-reads every input pixel once per filter
// tap: a 5x5 bwd-data streams 25x its source from L2, and the L2 -> SM path (~6.3 KB/clk for the
// chip) then bounds the contraction well below the tensor pipe (AlexNet conv2 bwd-data: 1.66 GB
// of TMA loads per launch).  Here a 128-row M tile is a th x wr block of output pixels laid out
// with row stride wr (th * wr = 128), and ONE tiled TMA box per 64-channel block stages the
// (th + R - 1) x wr input halo of the whole tile (zero-filled outside the image = padding).  Tap
// (kh, kw) of the filter is then the same halo read from a start address shifted by kh*wr + kw
// 128-byte rows: the SWIZZLE_128B pattern is a function of the shared-memory address, so a
// row-shifted K-major descriptor reads the shifted matrix (tools/umma_shift_probe.cu checks every
// shift).  Output columns x0 + wv .. x0 + wr - 1 (wv = wr - (S - 1)) read wrapped halo rows and
// are junk: the 4-D TMA store writes only wv columns per row and clips at the image edge.
//
//   A: halo slot (2 slots, reused by all R*S taps of a channel block).  With ms = 2 a unit is two
//      vertically adjacent 128-row subtiles over one (2 th + R - 1)-row halo: every B k-block feeds
//      two MMAs (subtile 1 reads 128 rows further), halving the filter's L2 -> SM traffic per FLOP
//      for narrow N (AlexNet conv2 bwd-data: N = 96)
//   B: filter k-block (tap, channel block), K-major [Cout][R][S][cs] (fprop) or MN-major
//      [R][S][ks][cs] (bwd-data), ring of `stages` slots
//   D: TMEM accumulators (4, or 2 for BN = 256), epilogue as in tc_gemm_kernel (bias, ReLU,
//      ReLU-mask, alpha; bf16 or fp32), TMA store per output row segment
//
// Warp roles (384 threads): 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 4-11 epilogue.
#pragma once

#include <cuda_bf16.h>

#include "ptx.cuh"
#include "tc_gemm.cuh"

namespace tcb {

struct HaloParams {
    CUtensorMap tmA;  // 4-D tiled {cs, W, H, N} over the source, box {64, wr, hh, 1}, SW128
    CUtensorMap tmB;  // filter: K-major {K, rows} box {64, BN} or MN-major {rows, K} boxes {64, 64}
    CUtensorMap tmD;  // 4-D {N, Wo, Ho, images} store, box {128 B of columns, wst, 1, 1}, SW128
    int N;            // GEMM columns (output channel stride)
    int b_mn;         // B is MN-major
    int R, S, flip;   // flip: bwd-data (tap (kh, kw) reads halo offset (R-1-kh, S-1-kw))
    int ncb;          // 64-channel blocks of the source (the last may be partial: TMA zero-fills it)
    int k_last;       // 16-channel MMA steps of the last block (1..4): the zero-filled rest is not issued
    int ldk;          // B k coordinate of tap t, channel block cb: t * ldk + 64 * cb
    int wr, th, hh;   // halo row stride (pixels), output rows per 128-row subtile, halo rows
    int ms;           // 128-row subtiles per unit (1 or 2; 2 needs BN <= 128)
    int wv, wst;      // valid output columns per tile, store box width
    int xt, yt, nimg; // x tiles, y tiles per image, images
    int Ho, Wo;       // output image extent
    int lo_x, lo_y;   // halo origin relative to the tile's first output pixel
    int tiles_n, units;
    uint32_t halo_bytes;  // bytes per halo slot (1024-aligned, includes the over-read slack)
    uint32_t halo_tx;     // bytes one halo box delivers
    int stages;           // B ring slots
    uint32_t b_bytes;     // bytes per B slot: BN rows, or (K-major, one column tile) round16(N) rows
    int epi;              // EPI_BF16 / EPI_F32
    const float* bias;
    int n_bias;
    int relu;
    float alpha;
    const __nv_bfloat16* mask;  // ReLU-backward fold (bf16 out): forward ReLU output, D's pixel indexing
    long long mask_ld;
};

template <int BN>
struct HaloCfg {
    static constexpr int kBBytes = BN * BK * 2;
    static constexpr int kAcc = BN <= 128 ? 4 : 2;
    static constexpr uint32_t kTmemCols = kAcc * BN;
    static constexpr int kStaging = 8 * kStagingBytes;
};

struct HaloTile {
    int img, y0, x0, nt;
};
__device__ __forceinline__ HaloTile halo_tile(const HaloParams& p, int u) {
    HaloTile t;
    t.nt = u % p.tiles_n;
    int m = u / p.tiles_n;
    const int per_img = p.yt * p.xt;
    t.img = m / per_img;
    m -= t.img * per_img;
    const int ty = m / p.xt;
    t.y0 = ty * p.th * p.ms;
    t.x0 = (m - ty * p.xt) * p.wv;
    return t;
}

template <int BN, int MS>
__global__ void __launch_bounds__(kNumThreads, 1) tc_conv_halo_kernel(const __grid_constant__ HaloParams p) {
    using Cfg = HaloCfg<BN>;
    constexpr int NACC = Cfg::kAcc;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages;
    uint8_t* sHalo = smem;                                   // 2 slots
    uint8_t* sB = smem + 2 * p.halo_bytes;                   // S slots
    uint8_t* sStage = sB + S * p.b_bytes;                    // epilogue staging
    uint64_t* a_full = reinterpret_cast<uint64_t*>(sStage + Cfg::kStaging);
    uint64_t* a_empty = a_full + 2;
    uint64_t* b_full = a_empty + 2;
    uint64_t* b_empty = b_full + 8;
    uint64_t* tfull = b_empty + 8;
    uint64_t* tempty = tfull + NACC;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NACC);

    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    const int taps = p.R * p.S;
    constexpr int nbuf = NACC / MS;  // unit accumulator buffers (MS * BN TMEM columns each)

    if (warp == 0 && lane == 0) {
        tma_prefetch(&p.tmA);
        tma_prefetch(&p.tmB);
        tma_prefetch(&p.tmD);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&a_full[s], 1);
            mbar_init(&a_empty[s], 1);
        }
        for (int s = 0; s < S; ++s) {
            mbar_init(&b_full[s], 1);
            mbar_init(&b_empty[s], 1);
        }
        for (int b = 0; b < NACC; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 8);  // one arrival per epilogue warp
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
        // ---------------- TMA producer
        int ai = 0, bs = 0;
        uint32_t bph = 0;
        for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
            const HaloTile t = halo_tile(p, u);
            const int n0 = t.nt * BN;
            for (int cb = 0; cb < p.ncb; ++cb, ++ai) {
                const int as = ai & 1;
                mbar_wait(&a_empty[as], ((ai >> 1) & 1) ^ 1);
#if defined(TCB_EXP_NOLOAD) || defined(TCB_EXP_NOHALO)
                if (lane == 0) mbar_arrive(&a_full[as]);  // experiment: no halo loads
#else
                tma_load_4d_e(sHalo + as * p.halo_bytes, &p.tmA, smem_u32(&a_full[as]), cb * 64, t.x0 + p.lo_x,
                              t.y0 + p.lo_y, t.img);
                mbar_arrive_expect_tx_e(&a_full[as], p.halo_tx);
#endif
                for (int tap = 0; tap < taps; ++tap) {
                    const int s = bs;
                    mbar_wait(&b_empty[s], bph ^ 1);
                    if (++bs == S) {
                        bs = 0;
                        bph ^= 1;
                    }
                    uint8_t* b_dst = sB + s * p.b_bytes;
                    const int kc = tap * p.ldk + cb * 64;
#ifdef TCB_EXP_NOLOAD
                    if (lane == 0) mbar_arrive(&b_full[s]);  // experiment: no filter loads
                    continue;
#endif
                    if (p.b_mn) {
#pragma unroll
                        for (int a = 0; a < BN / 64; ++a)
                            tma_load_2d_e<1>(b_dst + a * BK * 128, &p.tmB, smem_u32(&b_full[s]), n0 + a * 64, kc);
                    } else {
                        tma_load_2d_e<1>(b_dst, &p.tmB, smem_u32(&b_full[s]), kc, n0);
                    }
                    mbar_arrive_expect_tx_e(&b_full[s], p.b_bytes);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        const uint32_t idesc_full = umma_idesc_bf16(BM, BN, 0u, p.b_mn ? 1u : 0u);
        const uint64_t a_desc0 = umma_desc_sw128(smem_u32(sHalo), 0, 1024);
        auto b_desc_at = [&](uint32_t base, int k) -> uint64_t {
            return p.b_mn ? umma_desc_sw128(base + k * 2048, BK * 128, 1024) : umma_desc_sw128(base + k * 32, 0, 1024);
        };
        const uint64_t b_desc0 = b_desc_at(smem_u32(sB), 0);
        uint64_t b_koff[BK / 16];
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) b_koff[k] = b_desc_at(smem_u32(sB), k) - b_desc0;
        int ai = 0, tc = 0, bs = 0;
        uint32_t bph = 0;
        uint64_t b_off = 0;
        const uint64_t b_step = p.b_bytes >> 4;
        // per tap +-1 row; at the end of a filter row +-(wr - S) more (descriptor units)
        const int64_t tap_step = p.flip ? -8 : 8;
        const int64_t row_step = (p.flip ? -8 : 8) * static_cast<int64_t>(p.wr - p.S);
        for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++tc) {
            const HaloTile t = halo_tile(p, u);
            const int buf = tc % nbuf;
            mbar_wait(&tempty[buf], ((tc / nbuf) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + buf * MS * BN;
            uint32_t idesc = idesc_full;
            const int n_left = p.N - t.nt * BN;
            if (n_left < BN) {
                const int gran = p.b_mn ? 64 : 16;
                idesc = umma_idesc_bf16(BM, static_cast<uint32_t>((n_left + gran - 1) / gran * gran), 0u, p.b_mn ? 1u : 0u);
            }
            for (int cb = 0; cb < p.ncb; ++cb, ++ai) {
                const int as = ai & 1;
                const int kn = cb == p.ncb - 1 ? p.k_last : BK / 16;
                mbar_wait(&a_full[as], (ai >> 1) & 1);
                tc_fence_after();
                // tap (kh, kw) reads the halo shifted by kh*wr + kw rows (bwd-data: (R-1-kh)*wr +
                // (S-1-kw)); walked incrementally, in 16-byte descriptor units (8 per row)
                uint64_t a_tap = a_desc0 + static_cast<uint64_t>((as * p.halo_bytes) >> 4) +
                                 static_cast<uint64_t>(p.flip ? ((p.R - 1) * p.wr + p.S - 1) * 8 : 0);
                int kw = 0;
                for (int tap = 0; tap < taps; ++tap) {
                    mbar_wait(&b_full[bs], bph);
                    tc_fence_after();
                    const uint64_t b_s = b_desc0 + b_off;
                    const bool first = cb == 0 && tap == 0;
#pragma unroll
                    for (int sub = 0; sub < MS; ++sub) {
                        const uint64_t a_sub = a_tap + static_cast<uint64_t>(sub * (BM * 128 >> 4));
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k)
                            if (k < kn)
                                umma_bf16_elect<1>(d_tmem + sub * BN, a_sub + static_cast<uint64_t>(k * 2),
                                                   b_s + b_koff[k], idesc, (!first || k > 0) ? 1u : 0u);
                    }
                    umma_commit_elect<1>(&b_empty[bs]);
                    if (++bs == S) {
                        bs = 0;
                        bph ^= 1;
                        b_off = 0;
                    } else {
                        b_off += b_step;
                    }
                    a_tap += tap_step;
                    if (++kw == p.S) {
                        kw = 0;
                        a_tap += row_step;
                    }
                }
                umma_commit_elect<1>(&a_empty[as]);
            }
            umma_commit_elect<1>(&tfull[buf]);
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: warp e reads TMEM lanes 32 (e % 4) .. +32 (its 32 tile rows)
        // and the 64-column chunks c0 = 64 (e / 4) + 128 i
        const int ew = warp - 4;
        const int quarter = ew & 3, grp = ew >> 2;
        uint8_t* stg = sStage + ew * kStagingBytes;
        const bool bf16_out = p.epi == EPI_BF16;
        int nstore = 0, tc = 0;
        // this warp's rows: tile row r = 32 quarter + lane -> output pixel (y0 + r / wr, x0 + r % wr)
        const int r = quarter * 32 + lane;
        const int ry = r / p.wr, rx = r - (r / p.wr) * p.wr;
        for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++tc) {
            const HaloTile t0 = halo_tile(p, u);
            const int buf = tc % nbuf;
            mbar_wait(&tfull[buf], (tc / nbuf) & 1);
            tc_fence_after();
            const int n0 = t0.nt * BN;
            if (grp * 64 >= BN) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[buf]);
                continue;
            }
          for (int sub = 0; sub < MS; ++sub) {
            HaloTile t = t0;
            t.y0 += sub * p.th;
            const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + (buf * MS + sub) * BN;
            const int oy = t.y0 + ry, ox = t.x0 + rx;
            const bool row_valid = rx < p.wv && oy < p.Ho && ox < p.Wo;
            for (int c0 = grp * 64; c0 < BN; c0 += 128) {
                uint32_t r0[32], r1[32];
                tmem_ld32(t_row + c0, r0);
                tmem_ld32(t_row + c0 + 32, r1);
                const int nb = n0 + c0;
                float b0 = 0.f, b1 = 0.f;
                if (p.bias) {
                    if (nb + lane < p.n_bias) b0 = __ldg(p.bias + nb + lane);
                    if (nb + 32 + lane < p.n_bias) b1 = __ldg(p.bias + nb + 32 + lane);
                }
                tmem_ld_wait();
                if (c0 + 128 >= BN && sub == MS - 1) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[buf]);
                }
                if (p.alpha != 1.f) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        r0[j] = __float_as_uint(__uint_as_float(r0[j]) * p.alpha);
                        r1[j] = __float_as_uint(__uint_as_float(r1[j]) * p.alpha);
                    }
                }
                if (p.mask) {
                    uint64_t mbits = 0;
                    if (row_valid) {
                        const long long pix = (static_cast<long long>(t.img) * p.Ho + oy) * p.Wo + ox;
                        const uint4* mp = reinterpret_cast<const uint4*>(p.mask + pix * p.mask_ld + nb);
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            if (nb + q * 8 >= p.N) break;
                            const uint4 m = __ldg(mp + q);
                            const uint32_t w[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
                            for (int h = 0; h < 8; ++h) {
                                const uint32_t b = (w[h >> 1] >> ((h & 1) * 16)) & 0xFFFFu;
                                if (!(b & 0x8000u) && (b & 0x7FFFu)) mbits |= 1ull << (q * 8 + h);
                            }
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if (!((mbits >> j) & 1)) r0[j] = 0u;
                        if (!((mbits >> (32 + j)) & 1)) r1[j] = 0u;
                    }
                }
                if (p.bias) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        r0[j] = __float_as_uint(__uint_as_float(r0[j]) + __shfl_sync(0xffffffffu, b0, j));
                        r1[j] = __float_as_uint(__uint_as_float(r1[j]) + __shfl_sync(0xffffffffu, b1, j));
                    }
                }
                if (p.relu) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        r0[j] = __float_as_uint(fmaxf(__uint_as_float(r0[j]), 0.f));
                        r1[j] = __float_as_uint(fmaxf(__uint_as_float(r1[j]), 0.f));
                    }
                }
                const int nrows = bf16_out ? 1 : 2;
                for (int sub = 0; sub < nrows; ++sub) {
                    uint32_t packed[32];
                    if (bf16_out) {
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            packed[j] = pack_bf16x2(__uint_as_float(r0[2 * j]), __uint_as_float(r0[2 * j + 1]));
                            packed[16 + j] = pack_bf16x2(__uint_as_float(r1[2 * j]), __uint_as_float(r1[2 * j + 1]));
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j) packed[j] = sub ? r1[j] : r0[j];
                    }
                    if (nstore > 0) bulk_wait_read<0>();  // the previous store has read the buffer
                    __syncwarp();
                    const uint32_t row_addr = smem_u32(stg);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        st_shared_v4(row_addr + sw128_off(lane, q), packed[4 * q], packed[4 * q + 1], packed[4 * q + 2],
                                     packed[4 * q + 3]);
                    fence_proxy_async_smem();
                    __syncwarp();
                    const int col = nb + sub * 32;
                    if (p.wr >= 32) {
                        // one output row segment: 32 pixels (wr = 32: the wv valid ones)
                        const int y = t.y0 + (quarter * 32) / p.wr;
                        const int x = t.x0 + (quarter * 32) % p.wr;
                        if (y < p.Ho) tma_store_4d_e(&p.tmD, stg, col, x, y, t.img);
                    } else {
                        // wr = 16: two output rows of 16 pixels (wv valid) per 32-row chunk
                        const int y = t.y0 + quarter * 2;
                        if (y < p.Ho) tma_store_4d_e(&p.tmD, stg, col, t.x0, y, t.img);
                        if (y + 1 < p.Ho) tma_store_4d_e(&p.tmD, stg + 16 * 128, col, t.x0, y + 1, t.img);
                    }
                    bulk_commit();
                    ++nstore;
                }
            }
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

}  // namespace tcb
