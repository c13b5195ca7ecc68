// tcgen05 implicit-GEMM core used by every contraction of the training step
// (Convolv fwd / bwd-data / bwd-filter and the FC MatMul forms).
//
//   D[m, n] = alpha * sum_k A[m, k] * B[n, k]   bf16 operands, fp32 accumulation in TMEM
//
// Operand sources (per operand, chosen at launch):
//   OP_TMA_K     row-major [rows, K]: TMA 2D box {64 K, rows} -> SW128 K-major smem
//   OP_TMA_MN    row-major [K, rows]: TMA 2D boxes {64 rows, 64 K} -> SW128 MN-major smem
//   OP_GATHER_K  implicit im2col rows of an NHWC activation (fprop: x, bwd-data: dy),
//                16-byte cp.async gathers with zero fill, written pre-swizzled (A only)
//   OP_GATHER_MN implicit im2col of x, transposed, for bwd-filter (B only)
//   OP_IM2COL_K  TMA im2col of an NHWC activation: one {64 channels x 128 pixels} box per
//                k-block = (filter tap, 64-channel block), tap passed as the im2col offset (A only)
//   OP_IM2COL_MN TMA im2col of x for bwd-filter: {64 channels x 64 pixels} boxes (B only)
//   OP_IM2COL32_K / OP_IM2COL32_MN  the same for channel strides that are multiples of 32
//                but not 64: 32-channel boxes in SWIZZLE_64B layout; a 64-wide k-block of A
//                is two 8 KB halves (each one (tap, 32-channel block)), B's columns come in
//                32-wide atoms
//
// Persistent, warp-specialised (384 threads, one CTA per SM):
//   warp 0      TMA producer (elected lane)
//   warp 1      MMA issuer: tcgen05.mma into one of two TMEM accumulators;
//               tcgen05.commit releases smem stages / publishes finished tiles
//   warp 2      TMEM allocator (2 x BN fp32 columns)
//   warps 4-7   epilogue: tcgen05.ld (warp%4 selects its 32 TMEM lanes), bias /
//               ReLU / alpha, bf16 or fp32 pack, swizzled smem staging, TMA store
//               (clipped at the tensor bounds); overlaps the next tile's main loop
//   warps 8-11  im2col gather producers (only for OP_GATHER_* operands)
// Work units are (m tile, n tile, k split) handed out round-robin to the CTAs.
#pragma once

#include <cuda_bf16.h>

#include "ptx.cuh"

namespace tcb {

enum OperandMode : int {
    OP_TMA_K = 0,
    OP_TMA_MN = 1,
    OP_GATHER_K = 2,
    OP_GATHER_MN = 3,
    OP_IM2COL_K = 4,
    OP_IM2COL_MN = 5,
    OP_IM2COL32_K = 6,
    OP_IM2COL32_MN = 7
};
enum GatherKind : int { GATHER_FPROP = 0, GATHER_DGRAD = 1 };
enum EpiMode : int { EPI_BF16 = 0, EPI_F32 = 1, EPI_SGD = 2 };

// Implicit-GEMM geometry.  Activations are NHWC with a channel stride that is a
// multiple of 8 (16-byte chunks never straddle two filter taps).
struct ConvGeom {
    int N, H, W, C;  // input image (fprop / wgrad source) or dx image (dgrad rows)
    int R, S, stride, pad;
    int Ho, Wo, Co;  // output image; Co = channel stride of dy (dgrad source)
};

struct GemmParams {
    CUtensorMap tmA;  // valid when a_mode is a TMA mode
    CUtensorMap tmB;  // valid when b_mode is a TMA mode
    CUtensorMap tmD;  // 3-D store map {N, M, splits}, SW128, box {128 B of columns, 32 rows, 1}
    int M, N, K;
    int a_mode, b_mode;
    int trans_out;   // host-side: the split-K reduce writes D[n][m] (swapped filter gradient)
    // EPI_SGD: the tile is a filter gradient; apply the momentum update to p / v (fp32, row
    // stride sgd_ld) and refresh the bf16 shadow instead of storing the gradient
    float* sgd_p;
    float* sgd_v;
    __nv_bfloat16* sgd_shadow;
    long long sgd_ld;
    float sgd_lr, sgd_mom, sgd_decay;
    int b_resident;  // 1: one N tile, no split-K, num_kb <= stages: B is loaded once per CTA into
                     // ring slot kb and reused by every later unit (only A streams)
    int gather_kind;            // GatherKind for OP_GATHER_K
    const __nv_bfloat16* gsrc;  // gather source tensor
    ConvGeom g;
    int num_kb;                 // total k-blocks
    int kb_per_split;           // k-blocks per split
    int splits;
    int tiles_m, tiles_n;
    int units;                  // tiles_m * tiles_n * splits
    int epi;                    // EpiMode of the stored tile
    const float* bias;          // per-column bias, may be null (never with splits > 1)
    int n_bias;                 // bias is read for n < n_bias (padded channels get 0)
    int relu;
    float alpha;
    // ReLU-backward folded into the epilogue (bf16 output, no split-K): D *= [mask > 0], mask is
    // the forward ReLU output, same row / column indexing as D with row stride mask_ld
    const __nv_bfloat16* mask;
    long long mask_ld;
    // TMA im2col operand: tmA (OP_IM2COL_K) or tmB (OP_IM2COL_MN) is a 4-D {c, w, h, n} im2col map
    int i2c_cpb;             // 64-channel (32 for OP_IM2COL32_K) blocks per filter tap (A side)
    int i2c_ldk;             // k coordinate of tap t in the other operand = t * i2c_ldk + 64 * block
    int i2c_lo_w, i2c_lo_h;  // first source pixel of output pixel (y, x) = (y * stride + lo_h, x * stride + lo_w)
    int i2c_flip;            // bwd-data: tap (kh, kw) is the offset (R-1-kh, S-1-kw)
    int i2c_P, i2c_Q;        // pixel grid the rows (A) / k-blocks (B) walk: P x Q per image
    // Folded bias gradient (CG = 1, MN-major TMA A: filter / FC-weight gradients, A = dy): warps
    // 2-3 sum every staged A tile of the units in column tile 0 over k and write the per-split
    // column sums bias_ws[split][M] (the final bias gradient when unsplit).  bias_out: host side.
    float* bias_ws;
    float* bias_out;
    int bias_src;  // 1: column sums of A (index m, length M); 2: of the MN-major TMA B (index n, length N)
};

constexpr int BK = 64;  // bf16 elements per k-block = one 128-byte swizzle row
constexpr int BM = 128;
constexpr int kNumThreads = 384;
constexpr int kStagingBytes = 4096;  // per epilogue warp per buffer: 32 rows x 128 B

// CG = 2: CTA pair (cta_group::2).  The pair computes a (2*BM) x BN tile: each CTA holds
// its BM rows of A and BN/2 rows (columns of D) of B; the leader issues the MMAs.
// SK = 1 (short-K): half the operand ring and 4x the epilogue staging (4 buffers per epilogue
// warp).  Measured neutral-to-slower on the short-K contractions of the configs (the store
// issue rate was not the limit once the accumulator release stopped fencing at GPU scope), so
// no launch path instantiates it; kept for experiments (launch_bn<BN, 1, 1>).
template <int BN, int CG = 1, int SK = 0>
struct TileCfg {
    static constexpr int kBNL = BN / CG;  // B rows held by one CTA
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = kBNL * BK * 2;
    static constexpr int kRing = SK ? 98304 : 196608;
    static constexpr int kStages = (kRing / (kABytes + kBBytes)) > 8 ? 8 : (kRing / (kABytes + kBBytes));
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStagingTotal = (SK ? 32 : 8) * kStagingBytes;
    static constexpr int kSmemBytes = kStages * kStageBytes + kStagingTotal + 1024 /*align*/ + 256 /*barriers*/;
    // TMEM accumulators: 4 for BN <= 128 (the MMA runs up to 3 tiles ahead of the epilogue
    // on short-K tiles), 2 for BN = 256; 512 columns at most
    static constexpr int kAcc = BN <= 128 ? 4 : 2;
    static constexpr uint32_t kTmemCols = kAcc * BN < 32 ? 32 : kAcc * BN;
    static constexpr int kLag = kStages - 2;                             // cp.async groups in flight
};

// Byte offset of 16B chunk `j` of row `r` inside a SW128 tile (1024B-aligned base).
__device__ __forceinline__ uint32_t sw128_off(int r, int j) {
    return static_cast<uint32_t>(r * 128 + ((j ^ (r & 7)) << 4));
}

struct Unit {
    int mt, nt, sp, kb0, kb1;
};

__device__ __forceinline__ Unit decode_unit(const GemmParams& p, int u) {
    Unit w;
    w.nt = u % p.tiles_n;
    const int r = u / p.tiles_n;
    w.mt = r % p.tiles_m;
    w.sp = r / p.tiles_m;
    w.kb0 = w.sp * p.kb_per_split;
    w.kb1 = min(p.num_kb, w.kb0 + p.kb_per_split);
    return w;
}

// Columns a CTA-pair tile issues (K-major B): all BN, or N left rounded up to 16 on the last
// column tile (M = 256 needs N % 16 == 0; each CTA then holds N/2 rows, a multiple of 8).
template <int BN>
__device__ __forceinline__ int pair_n_issue(const GemmParams& p, int nt) {
    const int n_left = p.N - nt * BN;
    return n_left >= BN ? BN : (n_left + 15) / 16 * 16;
}

// ---- A gather (K-major rows of an implicit im2col) --------------------------------
// Each of the 128 producer threads owns one tile row; its 8 chunks per k-block
// walk (kh, kw, c) incrementally (no division in the steady state).
struct RowGather {
    const __nv_bfloat16* base;  // image n of this row
    int ry, rx;                 // output (fprop) or input (dgrad) pixel of this row
    bool valid;
    int c[8], kw[8], kh[8], kk[8];
};

__device__ __forceinline__ void row_gather_init(const GemmParams& p, RowGather& rg, int m, int kb0) {
    const ConvGeom& g = p.g;
    const bool fprop = p.gather_kind == GATHER_FPROP;
    rg.valid = m < p.M;
    int n = 0;
    rg.ry = rg.rx = 0;
    if (rg.valid) {
        const int hw = fprop ? g.Ho * g.Wo : g.H * g.W;
        const int wd = fprop ? g.Wo : g.W;
        n = m / hw;
        const int rem = m - n * hw;
        rg.ry = rem / wd;
        rg.rx = rem - rg.ry * wd;
    }
    const int C = fprop ? g.C : g.Co;
    rg.base = p.gsrc + static_cast<long long>(n) * (fprop ? static_cast<long long>(g.H) * g.W * g.C
                                                            : static_cast<long long>(g.Ho) * g.Wo * g.Co);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int k = kb0 * BK + j * 8;
        const int tap = k / C;
        rg.c[j] = k - tap * C;
        rg.kh[j] = tap / g.S;
        rg.kw[j] = tap - rg.kh[j] * g.S;
        rg.kk[j] = k;
    }
}

// Source pixel of (row, tap) or null when the tap falls into padding / a stride hole.
__device__ __forceinline__ const __nv_bfloat16* tap_source(const GemmParams& p, const RowGather& rg, int kh, int kw) {
    const ConvGeom& g = p.g;
    if (p.gather_kind == GATHER_FPROP) {
        const int iy = rg.ry * g.stride - g.pad + kh;
        const int ix = rg.rx * g.stride - g.pad + kw;
        if (static_cast<unsigned>(iy) < static_cast<unsigned>(g.H) && static_cast<unsigned>(ix) < static_cast<unsigned>(g.W))
            return rg.base + (static_cast<long long>(iy) * g.W + ix) * g.C;
        return nullptr;
    }
    int oy = rg.ry + g.pad - kh, ox = rg.rx + g.pad - kw;
    if (oy < 0 || ox < 0) return nullptr;
    if (g.stride != 1) {
        const int qy = oy / g.stride, qx = ox / g.stride;
        if (qy * g.stride != oy || qx * g.stride != ox) return nullptr;
        oy = qy;
        ox = qx;
    }
    if (oy >= g.Ho || ox >= g.Wo) return nullptr;
    return rg.base + (static_cast<long long>(oy) * g.Wo + ox) * g.Co;
}

__device__ __forceinline__ void row_gather_issue(const GemmParams& p, RowGather& rg, uint32_t sA, int row) {
    const ConvGeom& g = p.g;
    const bool fprop = p.gather_kind == GATHER_FPROP;
    const int C = fprop ? g.C : g.Co;
    if (C % BK == 0) {
        // the whole k-block is one filter tap: one address, 128 contiguous bytes
        const __nv_bfloat16* src = (rg.valid && rg.kk[0] < p.K) ? tap_source(p, rg, rg.kh[0], rg.kw[0]) : nullptr;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            cp_async_16(sA + sw128_off(row, j), src ? src + rg.c[0] + j * 8 : p.gsrc, src ? 16u : 0u);
        rg.kk[0] += BK;
        rg.c[0] += BK;
        if (rg.c[0] >= C) {
            rg.c[0] = 0;
            if (++rg.kw[0] == g.S) {
                rg.kw[0] = 0;
                ++rg.kh[0];
            }
        }
        return;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const __nv_bfloat16* src = (rg.valid && rg.kk[j] < p.K) ? tap_source(p, rg, rg.kh[j], rg.kw[j]) : nullptr;
        cp_async_16(sA + sw128_off(row, j), src ? src + rg.c[j] : p.gsrc, src ? 16u : 0u);
        // advance this chunk by one k-block (64 channels along (kh, kw, c))
        rg.kk[j] += BK;
        rg.c[j] += BK;
        while (rg.c[j] >= C) {
            rg.c[j] -= C;
            if (++rg.kw[j] == g.S) {
                rg.kw[j] = 0;
                ++rg.kh[j];
            }
        }
    }
}

// ---- B gather for bwd-filter (MN-major): rows = output pixels (k), columns n = (kh, kw, c)
template <int BN>
struct ColGather {
    static constexpr int kChunks = BN / 16;  // 16-byte chunks per thread per k-block
    int code[kChunks];                       // c | kw << 12 | kh << 20, or -1 when n >= N
};

template <int BN>
__device__ __forceinline__ void col_gather_init(const GemmParams& p, ColGather<BN>& cg, int n0, int half) {
    const ConvGeom& g = p.g;
#pragma unroll
    for (int q = 0; q < ColGather<BN>::kChunks; ++q) {
        const int cc = half + 2 * q;
        const int n = n0 + (cc >> 3) * 64 + (cc & 7) * 8;
        if (n < p.N) {
            const int tap = n / g.C;
            const int c = n - tap * g.C;
            const int kh = tap / g.S;
            cg.code[q] = c | ((tap - kh * g.S) << 12) | (kh << 20);
        } else {
            cg.code[q] = -1;
        }
    }
}

template <int BN>
__device__ __forceinline__ void col_gather_issue(const GemmParams& p, const ColGather<BN>& cg, uint32_t sB, int kr,
                                                 int half, int kb) {
    const ConvGeom& g = p.g;
    const int pix = kb * BK + kr;
    const bool pv = pix < g.N * g.Ho * g.Wo;
    int rn = 0, oy = 0, ox = 0;
    if (pv) {
        rn = pix / (g.Ho * g.Wo);
        const int rem = pix - rn * g.Ho * g.Wo;
        oy = rem / g.Wo;
        ox = rem - oy * g.Wo;
    }
    const __nv_bfloat16* img = p.gsrc + static_cast<long long>(rn) * g.H * g.W * g.C;
#pragma unroll
    for (int q = 0; q < ColGather<BN>::kChunks; ++q) {
        const int cc = half + 2 * q;
        const void* src = p.gsrc;
        uint32_t bytes = 0;
        const int code = cg.code[q];
        if (pv && code >= 0) {
            const int c = code & 0xFFF, kw = (code >> 12) & 0xFF, kh = code >> 20;
            const int iy = oy * g.stride - g.pad + kh;
            const int ix = ox * g.stride - g.pad + kw;
            if (static_cast<unsigned>(iy) < static_cast<unsigned>(g.H) &&
                static_cast<unsigned>(ix) < static_cast<unsigned>(g.W)) {
                src = img + (static_cast<long long>(iy) * g.W + ix) * g.C + c;
                bytes = 16;
            }
        }
        cp_async_16(sB + (cc >> 3) * (BK * 128) + sw128_off(kr, cc & 7), src, bytes);
    }
}

// ---- channel-stride-4 gathers (first-layer convs, 3 real channels + 1 zero pad) ----
// One 8-byte chunk = one filter tap; a 64-element k-block = 16 taps.
struct RowGather4 {
    const __nv_bfloat16* base;  // tap (0, 0) of this output pixel (may lie outside the image)
    uint32_t rowmask, colmask;  // bit kh / kw: that filter row / column lands inside the image
    int kh, kw, tap, off;       // current tap and its element offset from base
    bool valid;
};

// Per-tap work is a mask test, a select and the copy: the image-bounds tests are folded into
// two per-pixel bit masks (R, S <= 32) and the tap address advances incrementally.
__device__ __forceinline__ void row_gather4_init(const GemmParams& p, RowGather4& rg, int m, int kb0) {
    const ConvGeom& g = p.g;
    rg.valid = m < p.M;
    int n = 0, ry = 0, rx = 0;
    if (rg.valid) {
        n = m / (g.Ho * g.Wo);
        const int rem = m - n * g.Ho * g.Wo;
        ry = rem / g.Wo;
        rx = rem - ry * g.Wo;
    }
    const int iy0 = ry * g.stride - g.pad, ix0 = rx * g.stride - g.pad;
    rg.rowmask = rg.colmask = 0;
    for (int k = 0; k < g.R; ++k)
        if (static_cast<unsigned>(iy0 + k) < static_cast<unsigned>(g.H)) rg.rowmask |= 1u << k;
    for (int k = 0; k < g.S; ++k)
        if (static_cast<unsigned>(ix0 + k) < static_cast<unsigned>(g.W)) rg.colmask |= 1u << k;
    rg.base = p.gsrc + (static_cast<long long>(n) * g.H * g.W + static_cast<long long>(iy0) * g.W + ix0) * 4;
    rg.tap = kb0 * (BK / 4);
    rg.kh = rg.tap / g.S;
    rg.kw = rg.tap - rg.kh * g.S;
    rg.off = (rg.kh * g.W + rg.kw) * 4;
}

__device__ __forceinline__ void row_gather4_issue(const GemmParams& p, RowGather4& rg, uint32_t sA, int row) {
    const ConvGeom& g = p.g;
    const int ntaps = g.R * g.S;
    const int wrap = (g.W - g.S) * 4;
#pragma unroll
    for (int jj = 0; jj < BK / 4; ++jj) {
        const bool v = rg.valid && rg.tap < ntaps && ((rg.rowmask >> rg.kh) & (rg.colmask >> rg.kw) & 1u);
        cp_async_8(sA + static_cast<uint32_t>(row * 128 + (((jj >> 1) ^ (row & 7)) << 4) + (jj & 1) * 8),
                   v ? static_cast<const void*>(rg.base + rg.off) : static_cast<const void*>(p.gsrc), v ? 8u : 0u);
        ++rg.tap;
        rg.off += 4;
        if (++rg.kw == g.S) {
            rg.kw = 0;
            ++rg.kh;
            rg.off += wrap;
        }
    }
}

template <int BN>
struct ColGather4 {
    static constexpr int kChunks = BN / 16;
    int code[kChunks][2];  // (kh << 8 | kw) of the two taps in a 16-byte chunk, -1 = beyond N
    int off[kChunks][2];   // element offset of that tap from the pixel's tap (0, 0)
};

template <int BN>
__device__ __forceinline__ void col_gather4_init(const GemmParams& p, ColGather4<BN>& cg, int n0, int half) {
    const ConvGeom& g = p.g;
#pragma unroll
    for (int q = 0; q < ColGather4<BN>::kChunks; ++q) {
        const int cc = half + 2 * q;
        const int n = n0 + (cc >> 3) * 64 + (cc & 7) * 8;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int nn = n + 4 * h;
            if (nn < p.N) {
                const int tap = nn >> 2;
                const int kh = tap / g.S;
                cg.code[q][h] = (kh << 8) | (tap - kh * g.S);
                cg.off[q][h] = (kh * g.W + (tap - kh * g.S)) * 4;
            } else {
                cg.code[q][h] = -1;
                cg.off[q][h] = 0;
            }
        }
    }
}

// One k-row (output pixel) per thread per k-block: its image-bounds tests become two bit
// masks, then every tap is a mask test, a select and the copy.
template <int BN>
__device__ __forceinline__ void col_gather4_issue(const GemmParams& p, const ColGather4<BN>& cg, uint32_t sB, int kr,
                                                  int half, int kb) {
    const ConvGeom& g = p.g;
    const int pix = kb * BK + kr;
    const bool pv = pix < g.N * g.Ho * g.Wo;
    int rn = 0, oy = 0, ox = 0;
    if (pv) {
        rn = pix / (g.Ho * g.Wo);
        const int rem = pix - rn * g.Ho * g.Wo;
        oy = rem / g.Wo;
        ox = rem - oy * g.Wo;
    }
    const int iy0 = oy * g.stride - g.pad, ix0 = ox * g.stride - g.pad;
    uint32_t rowmask = 0, colmask = 0;
    if (pv) {
        for (int k = 0; k < g.R; ++k)
            if (static_cast<unsigned>(iy0 + k) < static_cast<unsigned>(g.H)) rowmask |= 1u << k;
        for (int k = 0; k < g.S; ++k)
            if (static_cast<unsigned>(ix0 + k) < static_cast<unsigned>(g.W)) colmask |= 1u << k;
    }
    const __nv_bfloat16* base =
        p.gsrc + (static_cast<long long>(rn) * g.H * g.W + static_cast<long long>(iy0) * g.W + ix0) * 4;
#pragma unroll
    for (int q = 0; q < ColGather4<BN>::kChunks; ++q) {
        const int cc = half + 2 * q;
        const uint32_t dst = sB + (cc >> 3) * (BK * 128) + sw128_off(kr, cc & 7);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int code = cg.code[q][h];
            const bool v = code >= 0 && ((rowmask >> (code >> 8)) & (colmask >> (code & 0xFF)) & 1u);
            cp_async_8(dst + h * 8, v ? static_cast<const void*>(base + cg.off[q][h]) : static_cast<const void*>(p.gsrc),
                       v ? 8u : 0u);
        }
    }
}

template <int BN, int CG, int SK>
__global__ void __launch_bounds__(kNumThreads, 1) tc_gemm_kernel(const __grid_constant__ GemmParams p) {
    using Cfg = TileCfg<BN, CG, SK>;
    constexpr int S = Cfg::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + S * Cfg::kABytes;
    uint8_t* sStage = smem + S * Cfg::kStageBytes;  // epilogue staging (1024-aligned)
    uint64_t* full = reinterpret_cast<uint64_t*>(sStage + Cfg::kStagingTotal);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    constexpr int NACC = Cfg::kAcc;
    uint64_t* tempty = tfull + NACC;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NACC);

    // warp index broadcast from lane 0: provably warp-uniform, so the role branches below and
    // the loop state inside them can live in uniform registers
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    const bool a_gather = CG == 1 && p.a_mode == OP_GATHER_K;  // CTA pairs use TMA operands only
    const bool b_gather = CG == 1 && p.b_mode == OP_GATHER_MN;
    const bool any_gather = a_gather || b_gather;
    const int rank = CG == 2 ? static_cast<int>(cluster_ctarank()) : 0;  // 0 = MMA leader
    const int pair = blockIdx.x / CG, npairs = gridDim.x / CG;

    if (warp == 0 && lane == 0) {
        if (!a_gather) tma_prefetch(&p.tmA);
        if (!b_gather) tma_prefetch(&p.tmB);
        tma_prefetch(&p.tmD);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1 + (any_gather ? 128 : 0));
            mbar_init(&empty[s], 1 + (p.bias_ws != nullptr ? 2 : 0));  // + the bias warps 2-3
        }
        for (int b = 0; b < NACC; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], CG * (any_gather ? 4 : 8));  // one arrival per epilogue warp of the pair
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<CG>(tmem_slot, Cfg::kTmemCols);
    tc_fence_before();
    if constexpr (CG == 2)
        cluster_sync_all();  // peer barriers initialised before any remote arrive / complete_tx
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // PDL: the prologue above overlapped the previous kernel; no global access before this
    pdl_trigger();
    pdl_wait();

    if (warp == 0) {
        // ---------------- TMA producer (warp-converged; the issue helpers elect one lane)
        {
            uint32_t tx = 0;
#ifdef TCB_L2HINT
            const uint64_t pol_b = l2_policy_evict_last();
#endif
            if (!a_gather) tx += Cfg::kABytes;
            if (!b_gather) tx += Cfg::kBBytes;
            tx *= CG;  // the leader's barrier counts the bytes landing in both CTAs
            const ConvGeom& g = p.g;
            int it = 0;
            for (int u = pair; u < p.units; u += npairs) {
                const Unit w = decode_unit(p, u);
                // CTA pair with a K-major B: the last column tile issues only round16(N left)
                // columns, so the peer's B half starts at half of that (see the MMA issuer)
                const int n_half = CG == 2 && p.b_mode == OP_TMA_K ? pair_n_issue<BN>(p, w.nt) / 2 : Cfg::kBNL;
                const int m0 = w.mt * (BM * CG) + rank * BM, n0 = w.nt * BN + rank * n_half;
                const bool load_b = !p.b_resident || u == pair;  // resident B: first unit only
                const uint32_t tx_u = load_b || b_gather ? tx : tx - Cfg::kBBytes * CG;
                // im2col A: first pixel of this row tile
                int a_n = 0, a_y = 0, a_x = 0;
                if (p.a_mode == OP_IM2COL_K || p.a_mode == OP_IM2COL32_K) {
                    const int pq = p.i2c_P * p.i2c_Q;
                    a_n = m0 / pq;
                    const int rem = m0 - a_n * pq;
                    const int oy = rem / p.i2c_Q;
                    a_y = oy * g.stride + p.i2c_lo_h;
                    a_x = (rem - oy * p.i2c_Q) * g.stride + p.i2c_lo_w;
                }
                for (int kb = w.kb0; kb < w.kb1; ++kb, ++it) {
                    const int s = it % S;
                    mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
                    uint8_t* a_dst = sA + s * Cfg::kABytes;
                    uint8_t* b_dst = sB + (p.b_resident ? kb : s) * Cfg::kBBytes;
                    // transaction barrier: the leader CTA's full[s] (own barrier for CG = 1)
                    const uint32_t bar = CG == 2 ? mapa_shared(smem_u32(&full[s]), 0) : smem_u32(&full[s]);
                    int kc = kb * BK;  // k coordinate of this block in the plain-TMA operand
#ifdef TCB_EXP_NOLOAD
                    if (rank == 0 && lane == 0) mbar_arrive(&full[s]);  // experiment: MMA / epilogue pipeline without operand loads
                    continue;
#endif
                    if (p.a_mode == OP_TMA_K) {
                        tma_load_2d_e<CG>(a_dst, &p.tmA, bar, kc, m0);
                    } else if (p.a_mode == OP_TMA_MN) {
#pragma unroll
                        for (int a = 0; a < BM / 64; ++a)
                            tma_load_2d_e<CG>(a_dst + a * BK * 128, &p.tmA, bar, m0 + a * 64, kc);
                    } else if (p.a_mode == OP_IM2COL_MN) {
                        // A = im2col(x)^T (swapped filter gradient): rows m = tap * cs + c in
                        // 64-channel atoms, the 64 output pixels of this k-block along k
                        const int pq = p.i2c_P * p.i2c_Q;
                        const int pix = kb * BK;
                        const int an_img = pix / pq;
                        const int rem = pix - an_img * pq;
                        const int oy = rem / p.i2c_Q;
                        const int ay = oy * g.stride + p.i2c_lo_h;
                        const int ax = (rem - oy * p.i2c_Q) * g.stride + p.i2c_lo_w;
#pragma unroll
                        for (int row = 0; row < BM; row += 64) {
                            int m = m0 + row;
                            if (m >= p.M) m = 0;  // rows past M are clipped by the reduce; load finite data
                            const int tap = m / g.C, c = m - tap * g.C;
                            const int kh = tap / g.S, kw = tap - kh * g.S;
                            tma_load_im2col_4d_e<CG>(a_dst + row * BK * 2, &p.tmA, bar, c, ax, ay, an_img,
                                                     static_cast<uint16_t>(kw), static_cast<uint16_t>(kh));
                        }
                    } else if (p.a_mode == OP_IM2COL_K) {
                        const int tap = kb / p.i2c_cpb, cb = kb - tap * p.i2c_cpb;
                        const int kh = tap / g.S, kw = tap - kh * g.S;
                        const int ow = p.i2c_flip ? g.S - 1 - kw : kw, oh = p.i2c_flip ? g.R - 1 - kh : kh;
                        tma_load_im2col_4d_e<CG>(a_dst, &p.tmA, bar, cb * 64, a_x, a_y, a_n, static_cast<uint16_t>(ow),
                                           static_cast<uint16_t>(oh));
                        kc = tap * p.i2c_ldk + cb * 64;
                    } else if (p.a_mode == OP_IM2COL32_K) {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            int blk = kb * 2 + h;  // 32-wide k-block; past K: any valid block (B is zero there)
                            if (blk * 32 >= p.K) blk = 0;
                            const int tap = blk / p.i2c_cpb, cb = blk - tap * p.i2c_cpb;
                            const int kh = tap / g.S, kw = tap - kh * g.S;
                            const int ow = p.i2c_flip ? g.S - 1 - kw : kw, oh = p.i2c_flip ? g.R - 1 - kh : kh;
                            tma_load_im2col_4d_e<CG>(a_dst + h * (Cfg::kABytes / 2), &p.tmA, bar, cb * 32, a_x, a_y, a_n,
                                               static_cast<uint16_t>(ow), static_cast<uint16_t>(oh));
                        }
                    }
                    if (!load_b) {
                        // resident B: nothing to load for this k-block
                    } else if (p.b_mode == OP_TMA_K) {
#ifdef TCB_L2HINT
                        tma_load_2d_cg_hint<CG>(b_dst, &p.tmB, bar, kc, n0, pol_b);
#else
                        tma_load_2d_e<CG>(b_dst, &p.tmB, bar, kc, n0);
#endif
                    } else if (p.b_mode == OP_TMA_MN) {
#pragma unroll
                        for (int a = 0; a < Cfg::kBNL / 64; ++a)
#ifdef TCB_L2HINT
                            tma_load_2d_cg_hint<CG>(b_dst + a * BK * 128, &p.tmB, bar, n0 + a * 64, kc, pol_b);
#else
                            tma_load_2d_e<CG>(b_dst + a * BK * 128, &p.tmB, bar, n0 + a * 64, kc);
#endif
                    } else if (p.b_mode == OP_IM2COL_MN || p.b_mode == OP_IM2COL32_MN) {
                        // 64 output pixels of this k-block; columns n = tap * cs + c in 64-channel atoms
                        const int pq = p.i2c_P * p.i2c_Q;
                        const int pix = kb * BK;
                        const int bn_img = pix / pq;
                        const int rem = pix - bn_img * pq;
                        const int oy = rem / p.i2c_Q;
                        const int by = oy * g.stride + p.i2c_lo_h;
                        const int bx = (rem - oy * p.i2c_Q) * g.stride + p.i2c_lo_w;
                        const int box = p.b_mode == OP_IM2COL32_MN ? 32 : 64;  // columns per box
                        for (int col = 0; col < Cfg::kBNL; col += box) {
                            int n = n0 + col;
                            if (n >= p.N) n = 0;  // columns past N are clipped by the store; load finite data
                            const int tap = n / g.C, c = n - tap * g.C;
                            const int kh = tap / g.S, kw = tap - kh * g.S;
                            tma_load_im2col_4d_e<CG>(b_dst + col * BK * 2, &p.tmB, bar, c, bx, by, bn_img,
                                               static_cast<uint16_t>(kw), static_cast<uint16_t>(kh));
                        }
                    }
                    if (rank == 0) mbar_arrive_expect_tx_e(&full[s], tx_u);
                }
            }
        }
    } else if (warp == 1 && rank == 0) {
        // ---------------- MMA issuer (the leader CTA of a pair)
        const bool a_mn = p.a_mode == OP_TMA_MN || p.a_mode == OP_IM2COL_MN;
        const bool a_sw64 = p.a_mode == OP_IM2COL32_K;
        const bool b_sw64 = p.b_mode == OP_IM2COL32_MN;
        const bool b_mn = p.b_mode == OP_TMA_MN || p.b_mode == OP_GATHER_MN || p.b_mode == OP_IM2COL_MN || b_sw64;
        const uint32_t idesc_full = umma_idesc_bf16(BM * CG, BN, a_mn ? 1u : 0u, b_mn ? 1u : 0u);
        // Operand descriptors are built once: stage-0 bases plus per-k-step offsets (the start
        // address field is the low 14 bits in 16-byte units; every other field is fixed per
        // operand mode), so the issue loop is 4 MMAs and adds per k-block.
        //   K-major SW128: 32 bytes along the swizzled row per k-step; MN-major SW128: two 8-row
        //   k-groups (2 x 1024 B); SW64 K-major A: two 8 KB halves of 64-byte rows; SW64
        //   MN-major B: 32-column atoms of 64 k-rows (4 KB apart), 512-byte 8-row groups
        auto a_desc_at = [&](uint32_t base, int k) -> uint64_t {
            return a_mn ? umma_desc_sw128(base + k * 2048, BK * 128, 1024)
                   : a_sw64 ? umma_desc_sw64(base + (k >> 1) * (Cfg::kABytes / 2) + (k & 1) * 32, 0, 512)
                            : umma_desc_sw128(base + k * 32, 0, 1024);
        };
        auto b_desc_at = [&](uint32_t base, int k) -> uint64_t {
            return b_sw64 ? umma_desc_sw64(base + k * 1024, BK * 64, 512)
                   : b_mn ? umma_desc_sw128(base + k * 2048, BK * 128, 1024)
                          : umma_desc_sw128(base + k * 32, 0, 1024);
        };
        const uint64_t a_desc0 = a_desc_at(smem_u32(sA), 0), b_desc0 = b_desc_at(smem_u32(sB), 0);
        uint64_t a_koff[BK / 16], b_koff[BK / 16];
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
            a_koff[k] = a_desc_at(smem_u32(sA), k) - a_desc0;
            b_koff[k] = b_desc_at(smem_u32(sB), k) - b_desc0;
        }
        int it = 0, tc = 0;
        for (int u = pair; u < p.units; u += npairs, ++tc) {
            const Unit w = decode_unit(p, u);
            const int buf = tc % NACC;
            mbar_wait(&tempty[buf], ((tc / NACC) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + buf * BN;
            // the last column tile issues only the columns that exist (rounded to 16): N = 96 on
            // a 128-wide tile costs 96/128 of the MMA time (single-CTA tiles)
            uint32_t idesc = idesc_full;
            if (CG == 2 && p.b_mode == OP_TMA_K) {
                const int n_issue = pair_n_issue<BN>(p, w.nt);
                if (n_issue < BN) idesc = umma_idesc_bf16(BM * CG, static_cast<uint32_t>(n_issue), a_mn ? 1u : 0u, 0u);
            } else if (CG == 1) {
                // K-major B: any multiple of 16; MN-major B: whole swizzle atoms (64 / 32 columns)
                const int gran = b_sw64 ? 32 : b_mn ? 64 : 16;
                const int n_left = p.N - w.nt * BN;
                if (n_left < BN)
                    idesc = umma_idesc_bf16(BM, static_cast<uint32_t>((n_left + gran - 1) / gran * gran), a_mn ? 1u : 0u,
                                            b_mn ? 1u : 0u);
            }
            // warp-converged loop; the MMA / commit helpers elect the issuing lane
            for (int kb = w.kb0; kb < w.kb1; ++kb, ++it) {
                const int s = it % S;
                mbar_wait(&full[s], (it / S) & 1);
                tc_fence_after();
                // stage s descriptors = stage-0 descriptors + the stage offset in 16-byte units
                const uint64_t a_s = a_desc0 + static_cast<uint64_t>(s * (Cfg::kABytes >> 4));
                const uint64_t b_s = b_desc0 + static_cast<uint64_t>((p.b_resident ? kb : s) * (Cfg::kBBytes >> 4));
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                    umma_bf16_elect<CG>(d_tmem, a_s + a_koff[k], b_s + b_koff[k], idesc, (kb > w.kb0 || k > 0) ? 1u : 0u);
                umma_commit_elect<CG>(&empty[s]);
                if (kb == w.kb1 - 1) umma_commit_elect<CG>(&tfull[buf]);
            }
        }
    } else if ((warp == 2 || warp == 3) && p.bias_ws != nullptr && (CG == 1 || rank == 0)) {
        // ---------------- folded bias gradient: warp 2 / 3 sums A atom 0 / 1 (64 rows of M each)
        // of every stage over its 64 k rows; lane = (row group rg, 16-byte chunk kc), rows
        // rg + 4 i, so the row groups combine with two xor shuffles in a fixed order.  CTA pair:
        // the leader (whose full barrier counts both CTAs' bytes) also reads the peer's A rows
        // through DSMEM and releases the peer's stage with a remote arrive.
        const int a = warp - 2, kc = lane & 7, rg = lane >> 3;
        const bool from_b = p.bias_src == 2;
        const int natoms = from_b ? Cfg::kBNL / 64 : BM / 64;  // B: host keeps BN <= 128 (CG = 1)
        const int len = from_b ? p.N : p.M;
        int it = 0;
        for (int u = pair; u < p.units; u += npairs) {
            const Unit w = decode_unit(p, u);
            const bool need = (from_b ? w.mt == 0 : w.nt == 0) && a < natoms;
            float acc[CG][8];
#pragma unroll
            for (int h = 0; h < CG; ++h)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[h][j] = 0.f;
            for (int kb = w.kb0; kb < w.kb1; ++kb, ++it) {
                const int s = it % S;
                mbar_wait(&full[s], (it / S) & 1);
                if (need) {
                    const uint32_t local = smem_u32((from_b ? sB + s * Cfg::kBBytes : sA + s * Cfg::kABytes) + a * BK * 128);
#pragma unroll
                    for (int h = 0; h < CG; ++h) {
                        const uint32_t base = CG == 2 ? mapa_shared(local, h) : local;
#pragma unroll 4
                        for (int i = 0; i < 16; ++i) {
                            const int r = rg + 4 * i;
                            uint4 v;
                            if constexpr (CG == 2)
                                asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
                                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                                             : "r"(base + r * 128 + ((kc ^ (r & 7)) << 4))
                                             : "memory");
                            else
                                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                                             : "r"(base + r * 128 + ((kc ^ (r & 7)) << 4))
                                             : "memory");
                            const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const float2 f = __bfloat1622float2(hv[q]);
                                acc[h][2 * q] += f.x;
                                acc[h][2 * q + 1] += f.y;
                            }
                        }
                    }
                }
                // generic reads before the async-proxy refill of the stage (see wgrad_bias_sums)
                if constexpr (CG == 2)
                    asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
                else
                    fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&empty[s]);
                    if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(smem_u32(&empty[s]), 1));
                }
            }
            if (need) {
#pragma unroll
                for (int h = 0; h < CG; ++h) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        acc[h][j] += __shfl_xor_sync(0xffffffffu, acc[h][j], 8);
                        acc[h][j] += __shfl_xor_sync(0xffffffffu, acc[h][j], 16);
                    }
                    if (rg == 0) {
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const int m = (from_b ? w.nt * BN : w.mt * (BM * CG) + h * BM) + a * 64 + kc * 8 + j;
                            if (m < len) p.bias_ws[static_cast<long long>(w.sp) * len + m] = acc[h][j];
                        }
                    }
                }
            }
        }
    } else if (warp >= 8 && any_gather) {
        // ---------------- im2col gather producers (128 threads)
        if (any_gather) {
            constexpr int LAG = Cfg::kLag;
            const int t = threadIdx.x - 256;
            int it = 0;
            const bool c4 = p.g.C == 4;  // channel-stride-4 first-layer input (fprop A / wgrad B)
            for (int u = pair; u < p.units; u += npairs) {
                const Unit w = decode_unit(p, u);
                if (a_gather && c4) {
                    RowGather4 rg;
                    row_gather4_init(p, rg, w.mt * BM + t, w.kb0);
                    for (int kb = w.kb0; kb < w.kb1; ++kb, ++it) {
                        const int s = it % S;
                        mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
                        row_gather4_issue(p, rg, smem_u32(sA + s * Cfg::kABytes), t);
                        cp_async_commit();
                        if (it >= LAG) {
                            cp_async_wait<LAG>();
                            fence_proxy_async_smem();
                            mbar_arrive(&full[(it - LAG) % S]);
                        }
                    }
                } else if (b_gather && c4) {
                    ColGather4<BN> cg;
                    col_gather4_init<BN>(p, cg, w.nt * BN, t >> 6);
                    for (int kb = w.kb0; kb < w.kb1; ++kb, ++it) {
                        const int s = it % S;
                        mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
                        col_gather4_issue<BN>(p, cg, smem_u32(sB + s * Cfg::kBBytes), t & 63, t >> 6, kb);
                        cp_async_commit();
                        if (it >= LAG) {
                            cp_async_wait<LAG>();
                            fence_proxy_async_smem();
                            mbar_arrive(&full[(it - LAG) % S]);
                        }
                    }
                } else if (a_gather) {
                    RowGather rg;
                    row_gather_init(p, rg, w.mt * BM + t, w.kb0);
                    for (int kb = w.kb0; kb < w.kb1; ++kb, ++it) {
                        const int s = it % S;
                        mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
                        row_gather_issue(p, rg, smem_u32(sA + s * Cfg::kABytes), t);
                        cp_async_commit();
                        if (it >= LAG) {
                            cp_async_wait<LAG>();
                            fence_proxy_async_smem();
                            mbar_arrive(&full[(it - LAG) % S]);
                        }
                    }
                } else {
                    ColGather<BN> cg;
                    col_gather_init<BN>(p, cg, w.nt * BN, t >> 6);
                    for (int kb = w.kb0; kb < w.kb1; ++kb, ++it) {
                        const int s = it % S;
                        mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
                        col_gather_issue<BN>(p, cg, smem_u32(sB + s * Cfg::kBBytes), t & 63, t >> 6, kb);
                        cp_async_commit();
                        if (it >= LAG) {
                            cp_async_wait<LAG>();
                            fence_proxy_async_smem();
                            mbar_arrive(&full[(it - LAG) % S]);
                        }
                    }
                }
            }
            cp_async_wait<0>();
            fence_proxy_async_smem();
            for (int i = max(0, it - LAG); i < it; ++i) mbar_arrive(&full[i % S]);
        }
    } else if (warp >= 4) {
        // ---------------- epilogue (TMEM -> regs -> swizzled smem -> TMA store)
        // Without im2col gathers, warps 8-11 join the epilogue: warp e (0..7) reads TMEM lane
        // quarter e % 4 (tile rows [32 (e % 4), +32)) and the 64-column chunks of its group
        // e / 4; the 8 staging buffers are then one per warp instead of two.
        const int ew = warp - 4;
        const int quarter = ew & 3, grp = ew >> 2;
        const int ngrp = any_gather ? 1 : 2;
        constexpr int kBufs8 = Cfg::kStagingTotal / kStagingBytes / 8;  // buffers per warp with 8 warps
        const int nbuf = kBufs8 * 2 / ngrp;
        uint8_t* stage_base = sStage + ew * nbuf * kStagingBytes;
        const bool bf16_out = p.epi == EPI_BF16;
        int nstore = 0;
        int tc = 0;
        // accumulator release goes to the leader's tempty (remote arrive from the peer CTA).  A
        // single CTA arrives locally: the cluster-scope release compiles to a GPU-scope MEMBAR
        // that measured ~18% of the stall samples of short-K GEMMs.
        auto release_accum = [&](uint32_t remote, uint64_t* local) {
            if constexpr (CG == 2)
                mbar_arrive_cluster(remote);
            else
                mbar_arrive(local);
        };
        uint32_t tempty_addr[NACC];
#pragma unroll
        for (int b = 0; b < NACC; ++b)
            tempty_addr[b] = CG == 2 ? mapa_shared(smem_u32(&tempty[b]), 0) : smem_u32(&tempty[b]);
        // BN = 64 with two warp groups: the groups take alternate tiles (one 64-column chunk
        // each) instead of group 1 idling, so two tiles drain concurrently
        const bool alternate = BN == 64 && ngrp == 2;
        for (int u = pair; u < p.units; u += npairs, ++tc) {
            const Unit w = decode_unit(p, u);
            const int buf = tc % NACC;
            mbar_wait(&tfull[buf], (tc / NACC) & 1);
            tc_fence_after();
            const int m0 = w.mt * (BM * CG) + rank * BM, n0 = w.nt * BN;
            const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + buf * BN;
            if (alternate ? grp != (tc & 1) : grp * 64 >= BN) {  // no chunk of this tile for this warp
                tc_fence_before();
                __syncwarp();
                if (lane == 0) release_accum(tempty_addr[buf], &tempty[buf]);
                continue;
            }
            // One staging row = 128 B (64 bf16 or 32 fp32 columns).  The two TMEM reads of a
            // 64-column chunk are issued back to back and waited once; the chunk's bias values
            // are fetched one per lane meanwhile and broadcast with shuffles.
            for (int c0 = alternate ? 0 : grp * 64; c0 < BN; c0 += 64 * ngrp) {
                uint32_t r0[32], r1[32];
#ifdef TCB_EXP_NOTMEM
#pragma unroll
                for (int j = 0; j < 32; ++j) r0[j] = r1[j] = j + c0;
#else
                tmem_ld32(t_row + c0, r0);
                tmem_ld32(t_row + c0 + 32, r1);
#endif
                const int nb = n0 + c0;
                float b0 = 0.f, b1 = 0.f;
                if (p.bias) {
                    if (nb + lane < p.n_bias) b0 = __ldg(p.bias + nb + lane);
                    if (nb + 32 + lane < p.n_bias) b1 = __ldg(p.bias + nb + 32 + lane);
                }
                tmem_ld_wait();
                if (c0 + 64 * ngrp >= BN) {
                    // this warp's TMEM reads of the accumulator are done: hand it back to the MMA warp
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) release_accum(tempty_addr[buf], &tempty[buf]);
                }
                uint64_t mbits = ~0ull;  // bit j: column nb + j passes the ReLU mask
                if (p.mask) {
                    mbits = 0;
                    const int row = m0 + quarter * 32 + lane;
                    if (row < p.M) {
                        const uint4* mp = reinterpret_cast<const uint4*>(p.mask + row * p.mask_ld + nb);
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
                }
                // each optional stage is one warp-uniform branch around a fully unrolled pass (no
                // per-element branches: the plain store path is just the pack)
                if (p.alpha != 1.f) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        r0[j] = __float_as_uint(__uint_as_float(r0[j]) * p.alpha);
                        r1[j] = __float_as_uint(__uint_as_float(r1[j]) * p.alpha);
                    }
                }
                if (p.mask) {
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
                if (p.epi == EPI_SGD) {
                    // fused update.  The accumulator arrives one parameter row per lane; it is
                    // transposed through this warp's staging buffer (32 rows x 32 fp32 columns per
                    // pass, SW128 chunk order) so that eight lanes cover one 128-byte row segment and
                    // the p / v / shadow traffic is fully coalesced.  All eight row groups' loads
                    // are issued before the first update (memory-level parallelism).
                    const uint32_t stg = smem_u32(stage_base);
                    const int rsub = lane >> 3, j = lane & 7;
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        const uint32_t* src = half ? r1 : r0;
                        __syncwarp();  // the previous pass's reads of the buffer are done
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            st_shared_v4(stg + sw128_off(lane, q), src[4 * q], src[4 * q + 1], src[4 * q + 2],
                                         src[4 * q + 3]);
                        __syncwarp();
                        const int col = nb + half * 32 + 4 * j;
                        if (col >= p.N) continue;  // N % 4 == 0: a float4 never straddles N
                        float4 P4[8], V4[8];
#pragma unroll
                        for (int it = 0; it < 8; ++it) {
                            const int row = m0 + quarter * 32 + it * 4 + rsub;
                            if (row < p.M) {
                                P4[it] = *reinterpret_cast<const float4*>(p.sgd_p + row * p.sgd_ld + col);
                                V4[it] = *reinterpret_cast<const float4*>(p.sgd_v + row * p.sgd_ld + col);
                            }
                        }
#pragma unroll
                        for (int it = 0; it < 8; ++it) {
                            const int rr = it * 4 + rsub, row = m0 + quarter * 32 + rr;
                            if (row >= p.M) continue;
                            uint32_t g0, g1, g2, g3;
                            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                         : "=r"(g0), "=r"(g1), "=r"(g2), "=r"(g3)
                                         : "r"(stg + sw128_off(rr, j)));
                            float4 P = P4[it], V = V4[it];
                            sgd_update1(P.x, V.x, __uint_as_float(g0), p.sgd_mom, p.sgd_lr, p.sgd_decay);
                            sgd_update1(P.y, V.y, __uint_as_float(g1), p.sgd_mom, p.sgd_lr, p.sgd_decay);
                            sgd_update1(P.z, V.z, __uint_as_float(g2), p.sgd_mom, p.sgd_lr, p.sgd_decay);
                            sgd_update1(P.w, V.w, __uint_as_float(g3), p.sgd_mom, p.sgd_lr, p.sgd_decay);
                            const long long o = row * p.sgd_ld + col;
                            *reinterpret_cast<float4*>(p.sgd_p + o) = P;
                            *reinterpret_cast<float4*>(p.sgd_v + o) = V;
                            *reinterpret_cast<uint2*>(p.sgd_shadow + o) =
                                make_uint2(pack_bf16x2(P.x, P.y), pack_bf16x2(P.z, P.w));
                        }
                    }
                    continue;
                }
                const int nrows = bf16_out ? 1 : 2;  // 128-byte staging rows in this chunk
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
                    // staging buffer reuse: the TMA store issued two stores ago must have read it
                    uint8_t* stg = stage_base + (nstore % nbuf) * kStagingBytes;
                    if (nstore >= nbuf) {  // every lane: only the issuing lane has groups
                        if (nbuf >= 8) bulk_wait_read<7>();
                        else if (nbuf >= 4) bulk_wait_read<3>();
                        else if (nbuf == 2) bulk_wait_read<1>();
                        else bulk_wait_read<0>();
                    }
                    __syncwarp();
                    const uint32_t row_addr = smem_u32(stg);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        st_shared_v4(row_addr + sw128_off(lane, q), packed[4 * q], packed[4 * q + 1],
                                     packed[4 * q + 2], packed[4 * q + 3]);
                    fence_proxy_async_smem();
                    __syncwarp();
#ifndef TCB_EXP_NOSTORE
                    tma_store_3d_e(&p.tmD, stg, nb + sub * 32, m0 + quarter * 32, w.sp);
#endif
                    bulk_commit();
                    ++nstore;
                }
            }
        }
        bulk_wait<0>();
        __syncwarp();
    }

    tc_fence_before();
    if constexpr (CG == 2)
        cluster_sync_all();  // the leader's MMAs and both epilogues are done with both TMEMs
    else
        __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<CG>(tmem_base, Cfg::kTmemCols);
    }
}

}  // namespace tcb
