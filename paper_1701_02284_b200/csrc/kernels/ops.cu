// Bandwidth-bound kernels of the training step.  See ops.cuh for layouts.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "ops.cuh"
#include "ptx.cuh"
#include "tc_philox.h"

namespace tcb {

namespace {

constexpr int kThreads = 256;

inline int grid_for(long long work, int per_block = kThreads) {
    const long long b = (work + per_block - 1) / per_block;
    return static_cast<int>(std::max<long long>(1, std::min<long long>(b, static_cast<long long>(num_sms()) * 32)));
}

__device__ __forceinline__ void unpack8(const uint4& q, float (&f)[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 t = __bfloat1622float2(h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
    uint4 q;
    q.x = pack_bf16x2(f[0], f[1]);
    q.y = pack_bf16x2(f[2], f[3]);
    q.z = pack_bf16x2(f[4], f[5]);
    q.w = pack_bf16x2(f[6], f[7]);
    return q;
}

// Storage-type generic access: activations are bf16 (default) or fp32 (the parity precision
// mode); every kernel computes in fp32 and touches 8 consecutive elements per access.
__device__ __forceinline__ float to_f(bf16 v) { return __bfloat162float(v); }
__device__ __forceinline__ float to_f(float v) { return v; }
template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
__device__ __forceinline__ void ld8(const bf16* p, float (&f)[8]) {
    const uint4 q = *reinterpret_cast<const uint4*>(p);  // one 16-byte load (unpack8 reads through a reference)
    unpack8(q, f);
}
__device__ __forceinline__ void ld8(const float* p, float (&f)[8]) {
    const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
    f[0] = a.x, f[1] = a.y, f[2] = a.z, f[3] = a.w, f[4] = b.x, f[5] = b.y, f[6] = b.z, f[7] = b.w;
}
// raw (packed) 8-element registers, unpacked later: keeps loads in flight without widening
template <typename T>
struct Raw8 {
    uint4 q;
};
template <>
struct Raw8<float> {
    float4 a, b;
};
__device__ __forceinline__ Raw8<bf16> ld_raw8cs(const bf16* p) { return Raw8<bf16>{__ldcs(reinterpret_cast<const uint4*>(p))}; }
__device__ __forceinline__ Raw8<float> ld_raw8cs(const float* p) {
    return Raw8<float>{__ldcs(reinterpret_cast<const float4*>(p)), __ldcs(reinterpret_cast<const float4*>(p) + 1)};
}
__device__ __forceinline__ Raw8<bf16> ld_raw8(const bf16* p) { return Raw8<bf16>{*reinterpret_cast<const uint4*>(p)}; }
__device__ __forceinline__ Raw8<float> ld_raw8(const float* p) {
    return Raw8<float>{reinterpret_cast<const float4*>(p)[0], reinterpret_cast<const float4*>(p)[1]};
}
template <typename T>
__device__ __forceinline__ Raw8<T> raw8_zero() {
    Raw8<T> r;
    if constexpr (sizeof(T) == 2) r.q = make_uint4(0, 0, 0, 0);
    else r.a = r.b = make_float4(0.f, 0.f, 0.f, 0.f);
    return r;
}
__device__ __forceinline__ void unpack_raw(const Raw8<bf16>& r, float (&f)[8]) { unpack8(r.q, f); }
__device__ __forceinline__ void unpack_raw(const Raw8<float>& r, float (&f)[8]) {
    f[0] = r.a.x, f[1] = r.a.y, f[2] = r.a.z, f[3] = r.a.w, f[4] = r.b.x, f[5] = r.b.y, f[6] = r.b.z, f[7] = r.b.w;
}
__device__ __forceinline__ void st8(bf16* p, const float (&f)[8]) { *reinterpret_cast<uint4*>(p) = pack8(f); }
__device__ __forceinline__ void st8(float* p, const float (&f)[8]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(f[0], f[1], f[2], f[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(f[4], f[5], f[6], f[7]);
}

// ---------------------------------------------------------------- elementwise (8 elements per thread)
template <typename T>
__global__ void k_relu_fwd(const T* __restrict__ x, T* __restrict__ y, long long n8) {
    pdl_wait();
    pdl_trigger();
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n8;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        float f[8];
        ld8(x + i * 8, f);
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = fmaxf(f[j], 0.f);
        st8(y + i * 8, f);
    }
}

template <typename T>
__global__ void k_relu_bwd(const T* __restrict__ dy, const T* __restrict__ y, T* __restrict__ dx, long long n8) {
    pdl_wait();
    pdl_trigger();
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n8;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        float g[8], f[8];
        ld8(dy + i * 8, g);
        ld8(y + i * 8, f);
#pragma unroll
        for (int j = 0; j < 8; ++j) g[j] = f[j] > 0.f ? g[j] : 0.f;
        st8(dx + i * 8, g);
    }
}

template <typename T>
// relu: forward y = max(a + b, 0); relu_y (may be null): a folded in-place ReLU backward behind
// an adjoint sum, y = [relu_y > 0] (a + b) (relu_y is the forward ReLU output)
__global__ void k_add(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ y, long long n8, int relu,
                      const T* __restrict__ relu_y) {
    pdl_wait();
    pdl_trigger();
    const long long S = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long i0 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i0 < n8; i0 += 2 * S) {
        float p[2][8], q[2][8], r[2][8];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (i0 + u * S < n8) {
                ld8(a + (i0 + u * S) * 8, p[u]);
                ld8(b + (i0 + u * S) * 8, q[u]);
                if (relu_y) ld8(relu_y + (i0 + u * S) * 8, r[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (i0 + u * S >= n8) break;
#pragma unroll
            for (int j = 0; j < 8; ++j) p[u][j] = relu ? fmaxf(p[u][j] + q[u][j], 0.f) : p[u][j] + q[u][j];
            if (relu_y) {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (!(r[u][j] > 0.f)) p[u][j] = 0.f;
            }
            st8(y + (i0 + u * S) * 8, p[u]);
        }
    }
}

// relu_y (may be null): a folded in-place ReLU backward behind the dropout backward product,
// y *= [relu_y > 0] (relu_y is the forward ReLU output)
template <typename T>
__global__ void k_mask_mul(const T* __restrict__ x, const uint2* __restrict__ keep, float scale, T* __restrict__ y,
                           long long n8, const T* __restrict__ relu_y) {
    pdl_wait();
    pdl_trigger();
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n8;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        float f[8];
        ld8(x + i * 8, f);
        const uint2 m = keep[i];
        const uint8_t* mb = reinterpret_cast<const uint8_t*>(&m);
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = mb[j] ? f[j] * scale : 0.f;
        if (relu_y) {
            float r[8];
            ld8(relu_y + i * 8, r);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (!(r[j] > 0.f)) f[j] = 0.f;
        }
        st8(y + i * 8, f);
    }
}

// Dropout forward in one pass: the keep mask of k_dropout_mask (same Philox stream, element by
// element) written for the backward, and y = x * keep * scale.
template <typename T>
__global__ void k_dropout_apply(const T* __restrict__ x, uint8_t* __restrict__ keep, T* __restrict__ y, int N, int H,
                                int W, int C, int cs, float rate, float scale, uint64_t seed, uint32_t var,
                                const uint32_t* iter_n0) {
    pdl_wait();
    pdl_trigger();
    const uint32_t iter = iter_n0[0], n0 = iter_n0[1];
    const long long n8 = static_cast<long long>(N) * H * W * cs / 8;
    for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < n8;
         q += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long i0 = q * 8;
        const int c0 = static_cast<int>(i0 % cs);  // cs % 8 == 0: the 8 elements share the pixel
        long long pix = i0 / cs;
        const int w = static_cast<int>(pix % W);
        pix /= W;
        const int h = static_cast<int>(pix % H);
        const int n = static_cast<int>(pix / H);
        float f[8];
        ld8(x + i0, f);
        uint8_t kb[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = c0 + j;
            uint8_t k = 0;
            if (c < C) {
                const uint32_t e = static_cast<uint32_t>((static_cast<long long>(c) * H + h) * W + w);
                k = tcp_dropout_value(seed, var, n0 + n, iter, e, rate) != 0.f;
            }
            kb[j] = k;
            f[j] = k ? f[j] * scale : 0.f;
        }
        *reinterpret_cast<uint2*>(keep + i0) = *reinterpret_cast<const uint2*>(kb);
        st8(y + i0, f);
    }
}

// keep mask for every stored element of an NHWC (or [N][Fs] with H=W=1) tensor.
__global__ void k_dropout_mask(uint8_t* __restrict__ keep, int N, int H, int W, int C, int cs, float rate,
                               uint64_t seed, uint32_t var, const uint32_t* iter_n0) {
    pdl_wait();
    pdl_trigger();
    const uint32_t iter = iter_n0[0], n0 = iter_n0[1];
    const long long total = static_cast<long long>(N) * H * W * cs;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i % cs);
        long long pix = i / cs;
        const int w = static_cast<int>(pix % W);
        pix /= W;
        const int h = static_cast<int>(pix % H);
        const int n = static_cast<int>(pix / H);
        uint8_t k = 0;
        if (c < C) {
            const uint32_t e = static_cast<uint32_t>((static_cast<long long>(c) * H + h) * W + w);
            k = tcp_dropout_value(seed, var, n0 + n, iter, e, rate) != 0.f;
        }
        keep[i] = k;
    }
}

// ---------------------------------------------------------------- pooling (NHWC, 8 channels per thread)
// Max pooling stores the argmax as a 1-byte window-local position r*k + s (255 =
// empty window); the flat NCHW index the reference reports is
// reconstructed from it on download (tc_pool_indices_download), so the index
// stream costs 1 B per output instead of 4.
// IT: index type of the element loop (int when the tensor has < 2^31 chunks: 64-bit
// division is ~4x the cost of 32-bit on this path)
template <typename T, typename IT>
__global__ void k_pool_fwd(const T* __restrict__ x, Act4 xi, T* __restrict__ y, Act4 yo,
                           uint8_t* __restrict__ idx, int k, int stride, int pad, int is_max, int flag_nonpos) {
    pdl_wait();
    pdl_trigger();
    const int cg = xi.cs / 8;
    const IT total = static_cast<IT>(yo.pixels() * cg);
    for (IT t = blockIdx.x * static_cast<IT>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<IT>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(t % cg);
        IT p = t / cg;
        const int ow = static_cast<int>(p % yo.W);
        p /= yo.W;
        const int oh = static_cast<int>(p % yo.H);
        const int n = static_cast<int>(p / yo.H);
        float best[8], sum[8];
        int bi[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            best[j] = 0.f;
            sum[j] = 0.f;
            bi[j] = 255;
        }
        const T* img = x + static_cast<long long>(n) * xi.H * xi.W * xi.cs + g * 8;
        for (int r = 0; r < k; ++r) {
            const int ih = oh * stride - pad + r;
            if (ih < 0 || ih >= xi.H) continue;
            for (int s = 0; s < k; ++s) {
                const int iw = ow * stride - pad + s;
                if (iw < 0 || iw >= xi.W) continue;
                float f[8];
                ld8(img + (static_cast<long long>(ih) * xi.W + iw) * xi.cs, f);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    sum[j] += f[j];
                    if (bi[j] == 255 || f[j] > best[j]) {  // first maximum in row-major window order
                        best[j] = f[j];
                        bi[j] = r * k + s;
                    }
                }
            }
        }
        const long long o = ((static_cast<long long>(n) * yo.H + oh) * yo.W + ow) * yo.cs + g * 8;
        float out[8];
        const float inv = 1.f / static_cast<float>(k * k);
#pragma unroll
        for (int j = 0; j < 8; ++j) out[j] = is_max ? best[j] : sum[j] * inv;
        st8(y + o, out);
        if (idx) {
            if (flag_nonpos) {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (!(best[j] > 0.f)) bi[j] |= 0x80;
            }
            uint2 q;
            q.x = static_cast<uint32_t>(bi[0]) | static_cast<uint32_t>(bi[1]) << 8 | static_cast<uint32_t>(bi[2]) << 16 |
                  static_cast<uint32_t>(bi[3]) << 24;
            q.y = static_cast<uint32_t>(bi[4]) | static_cast<uint32_t>(bi[5]) << 8 | static_cast<uint32_t>(bi[6]) << 16 |
                  static_cast<uint32_t>(bi[7]) << 24;
            *reinterpret_cast<uint2*>(idx + o) = q;
        }
    }
}

// Fixed-window max pooling on bf16 storage (K x K window, stride S known at compile time): the
// K*K taps are unrolled so all loads are in flight together, and the compare / select runs on
// packed bf16 pairs (one HGT2 mask + two LOP3 per channel pair and tap instead of ~5 fp32
// instructions per channel).  The argmax half-words track the first maximum in row-major
// window order exactly like k_pool_fwd; the max of bf16 values is one of them, so y is
// bit-identical to the fp32-compare path.
// One output pixel x 8 channels of a fixed-window max pool (see the kernels below).
template <int K, int S>
__device__ __forceinline__ void maxpool_fwd_px(const bf16* __restrict__ x, const Act4& xi, bf16* __restrict__ y,
                                               const Act4& yo, uint8_t* __restrict__ idx, int pad, int flag_nonpos,
                                               int n, int oh, int ow, int g) {
    {
        const int ih0 = oh * S - pad, iw0 = ow * S - pad;
        const bf16* img = x + static_cast<long long>(n) * xi.H * xi.W * xi.cs + g * 8;
        uint4 v[K * K];
#pragma unroll
        for (int r = 0; r < K; ++r)
#pragma unroll
            for (int s = 0; s < K; ++s) {
                const int ih = ih0 + r, iw = iw0 + s;
                if (ih >= 0 && ih < xi.H && iw >= 0 && iw < xi.W)
                    v[r * K + s] = *reinterpret_cast<const uint4*>(img + (static_cast<long long>(ih) * xi.W + iw) * xi.cs);
                else
                    v[r * K + s] = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);  // -inf: never wins
            }
        // Start from the first in-bounds tap (a window always holds one), then keep strict maxima.
        const int r0 = ih0 < 0 ? -ih0 : 0, s0 = iw0 < 0 ? -iw0 : 0;
        uint32_t best[4], bi[4];
        const uint32_t first = static_cast<uint32_t>(r0 * K + s0) * 0x10001u;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            best[i] = 0xFF80FF80u;
            bi[i] = first;
        }
#pragma unroll
        for (int tap = 0; tap < K * K; ++tap) {
            const uint32_t tid = static_cast<uint32_t>(tap) * 0x10001u;
            const uint32_t* f = reinterpret_cast<const uint32_t*>(&v[tap]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t m = __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&f[i]),
                                               *reinterpret_cast<const __nv_bfloat162*>(&best[i]));
                best[i] = (f[i] & m) | (best[i] & ~m);
                bi[i] = (tid & m) | (bi[i] & ~m);
            }
        }
        const long long o = ((static_cast<long long>(n) * yo.H + oh) * yo.W + ow) * yo.cs + g * 8;
        *reinterpret_cast<uint4*>(y + o) = make_uint4(best[0], best[1], best[2], best[3]);
        if (idx) {
            if (flag_nonpos) {  // folded ReLU backward: a window whose maximum is <= 0 passes no gradient
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    bi[i] |= ~__hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&best[i]), __float2bfloat162_rn(0.f)) &
                             0x00800080u;
            }
            *reinterpret_cast<uint2*>(idx + o) =
                make_uint2(__byte_perm(bi[0], bi[1], 0x6420), __byte_perm(bi[2], bi[3], 0x6420));
        }
    }
}

template <typename IT, int K, int S>
__global__ void k_maxpool_fwd_bf16(const bf16* __restrict__ x, Act4 xi, bf16* __restrict__ y, Act4 yo,
                                   uint8_t* __restrict__ idx, int pad, int flag_nonpos) {
    pdl_wait();
    pdl_trigger();
    const int cg = xi.cs / 8;
    const IT total = static_cast<IT>(yo.pixels() * cg);
    for (IT t = blockIdx.x * static_cast<IT>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<IT>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(t % cg);
        IT p = t / cg;
        const int ow = static_cast<int>(p % yo.W);
        p /= yo.W;
        const int oh = static_cast<int>(p % yo.H);
        const int n = static_cast<int>(p / yo.H);
        maxpool_fwd_px<K, S>(x, xi, y, yo, idx, pad, flag_nonpos, n, oh, ow, g);
    }
}

// Stride-1 K x K max pool over column strips: a thread owns one output column x 8 channels for
// R consecutive output rows and keeps the horizontal (max, first column) of the last K input rows
// in a register ring, so each input row is loaded once per strip (K loads per output instead of
// K*K).  Row-major first-strict-max is preserved: the row pass keeps the first column reaching the
// row maximum, the column pass the first row whose maximum strictly exceeds the earlier ones, and
// a window of -inf / NaN keeps the first in-bounds tap exactly as maxpool_fwd_px does.
template <int K, int R>
__global__ void k_maxpool_fwd_strip(const bf16* __restrict__ x, Act4 xi, bf16* __restrict__ y, Act4 yo,
                                    uint8_t* __restrict__ idx, int pad, int flag_nonpos) {
    pdl_wait();
    pdl_trigger();
    const int cg = xi.cs / 8;
    const int strips = (yo.H + R - 1) / R;
    long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (t >= static_cast<long long>(yo.N) * strips * yo.W * cg) return;
    const int g = static_cast<int>(t % cg);
    t /= cg;
    const int ow = static_cast<int>(t % yo.W);
    t /= yo.W;
    const int oh0 = static_cast<int>(t % strips) * R;
    const int n = static_cast<int>(t / strips);
    const int iw0 = ow - pad;
    const int s0 = iw0 < 0 ? -iw0 : 0;
    const bf16* img = x + static_cast<long long>(n) * xi.H * xi.W * xi.cs + g * 8;
    uint32_t hm[K][4], hv[K][4];  // ring slot = input row mod K
    auto load_row = [&](int ih, uint32_t (&m)[4], uint32_t (&vi)[4]) {
        uint4 v[K];
#pragma unroll
        for (int c = 0; c < K; ++c) {
            const int iw = iw0 + c;
            if (ih >= 0 && ih < xi.H && iw >= 0 && iw < xi.W)
                v[c] = *reinterpret_cast<const uint4*>(img + (static_cast<long long>(ih) * xi.W + iw) * xi.cs);
            else
                v[c] = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            m[i] = 0xFF80FF80u;
            vi[i] = static_cast<uint32_t>(s0) * 0x10001u;
        }
#pragma unroll
        for (int c = 0; c < K; ++c) {
            const uint32_t* f = reinterpret_cast<const uint32_t*>(&v[c]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t mk = __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&f[i]),
                                                *reinterpret_cast<const __nv_bfloat162*>(&m[i]));
                m[i] = (f[i] & mk) | (m[i] & ~mk);
                vi[i] = ((static_cast<uint32_t>(c) * 0x10001u) & mk) | (vi[i] & ~mk);
            }
        }
    };
#pragma unroll
    for (int u = 0; u < K - 1; ++u) load_row(oh0 - pad + u, hm[u], hv[u]);
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int oh = oh0 + j;
        if (oh >= yo.H) break;
        load_row(oh - pad + K - 1, hm[(j + K - 1) % K], hv[(j + K - 1) % K]);
        const int r0 = oh - pad < 0 ? pad - oh : 0;
        uint32_t best[4], bi[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            best[i] = 0xFF80FF80u;
            bi[i] = static_cast<uint32_t>(r0 * K + s0) * 0x10001u;
        }
#pragma unroll
        for (int u = 0; u < K; ++u) {
            const int sl = (j + u) % K;
            const uint32_t rowid = static_cast<uint32_t>(u * K) * 0x10001u;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t mk = __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&hm[sl][i]),
                                                *reinterpret_cast<const __nv_bfloat162*>(&best[i]));
                best[i] = (hm[sl][i] & mk) | (best[i] & ~mk);
                bi[i] = ((rowid + hv[sl][i]) & mk) | (bi[i] & ~mk);
            }
        }
        const long long o = ((static_cast<long long>(n) * yo.H + oh) * yo.W + ow) * yo.cs + g * 8;
        *reinterpret_cast<uint4*>(y + o) = make_uint4(best[0], best[1], best[2], best[3]);
        if (idx) {
            if (flag_nonpos) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    bi[i] |= ~__hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&best[i]), __float2bfloat162_rn(0.f)) &
                             0x00800080u;
            }
            *reinterpret_cast<uint2*>(idx + o) =
                make_uint2(__byte_perm(bi[0], bi[1], 0x6420), __byte_perm(bi[2], bi[3], 0x6420));
        }
    }
}

// Fixed-window max-pool backward, patch formulation.  Input rows r = a*S - pad + u (0 <= u < S)
// of patch a are covered exactly by the windows oh = a - (NW-1) + da, 0 <= da < NW = ceil(K/S),
// and the window-local tap of (u, da) is u + (NW-1-da)*S: a compile-time constant.  One thread
// owns an S x S patch x 8 channels: it loads the NW x NW covering windows' dy / argmax once and
// sends every pixel its matching taps, accumulating in the (oh, ow)-ascending order of
// k_pool_bwd (bit-identical sums).  An argmax byte with bit 7 set (flagged forward) matches no
// tap, which is how a folded ReLU backward is applied without reading the ReLU output.
template <typename T, int K, int S>
__device__ __forceinline__ void maxpool_bwd_patch_px(const T* __restrict__ dy, const Act4& yo,
                                                     const uint8_t* __restrict__ idx, T* __restrict__ dx,
                                                     const Act4& xi, int pad, const T* __restrict__ relu_y, int n,
                                                     int pa, int pb, int g) {
    constexpr int NW = (K + S - 1) / S;
    {
        const long long obase = static_cast<long long>(n) * yo.H * yo.W * yo.cs + g * 8;
        Raw8<T> d[NW * NW];
        uint2 q[NW * NW];
#pragma unroll
        for (int da = 0; da < NW; ++da)
#pragma unroll
            for (int db = 0; db < NW; ++db) {
                const int oh = pa - (NW - 1) + da, ow = pb - (NW - 1) + db;
                if (oh >= 0 && oh < yo.H && ow >= 0 && ow < yo.W) {
                    const long long o = obase + (static_cast<long long>(oh) * yo.W + ow) * yo.cs;
                    d[da * NW + db] = ld_raw8(dy + o);
                    q[da * NW + db] = __ldg(reinterpret_cast<const uint2*>(idx + o));
                } else {
                    q[da * NW + db] = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);  // matches no tap
                    d[da * NW + db] = raw8_zero<T>();
                }
            }
#pragma unroll
        for (int u = 0; u < S; ++u) {
            const int ih = pa * S - pad + u;
            if (ih < 0 || ih >= xi.H) continue;
#pragma unroll
            for (int v = 0; v < S; ++v) {
                const int iw = pb * S - pad + v;
                if (iw < 0 || iw >= xi.W) continue;
                float acc[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[j] = 0.f;
#pragma unroll
                for (int da = 0; da < NW; ++da) {
                    const int tr = u + (NW - 1 - da) * S;
                    if (tr >= K) continue;
#pragma unroll
                    for (int db = 0; db < NW; ++db) {
                        const int tc = v + (NW - 1 - db) * S;
                        if (tc >= K) continue;
                        const uint32_t mm = static_cast<uint32_t>(tr * K + tc) * 0x01010101u;
                        const uint32_t e0 = __vcmpeq4(q[da * NW + db].x, mm), e1 = __vcmpeq4(q[da * NW + db].y, mm);
                        float f[8];
                        unpack_raw(d[da * NW + db], f);
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            if ((((j < 4 ? e0 : e1) >> (8 * (j & 3))) & 1u) != 0u) acc[j] += f[j];
                    }
                }
                const long long o = ((static_cast<long long>(n) * xi.H + ih) * xi.W + iw) * xi.cs + g * 8;
                if (relu_y) {
                    float m[8];
                    ld8(relu_y + o, m);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (!(m[j] > 0.f)) acc[j] = 0.f;
                }
                st8(dx + o, acc);
            }
        }
    }
}

template <typename T, int K, int S>
__global__ void k_maxpool_bwd_patch(const T* __restrict__ dy, Act4 yo, const uint8_t* __restrict__ idx,
                                    T* __restrict__ dx, Act4 xi, int pad, const T* __restrict__ relu_y) {
    pdl_wait();
    pdl_trigger();
    const int cg = xi.cs / 8;
    const int PA = (xi.H + pad + S - 1) / S, PB = (xi.W + pad + S - 1) / S;
    const int total = xi.N * PA * PB * cg;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const int g = t % cg;
        int p = t / cg;
        const int pb = p % PB;
        p /= PB;
        const int pa = p % PA;
        const int n = p / PA;
        maxpool_bwd_patch_px<T, K, S>(dy, yo, idx, dx, xi, pad, relu_y, n, pa, pb, g);
    }
}

// Stride-1 backward over column strips: a thread owns one input column x 8 channels for R
// consecutive input rows; the K covering window rows (K columns each, gradient + argmax bytes)
// sit in a register ring, so each window is loaded once per strip instead of K*K times.  The
// per-pixel sums run in the same (oh, ow)-ascending order as maxpool_bwd_patch_px.
template <typename T, int K, int R>
__global__ void k_maxpool_bwd_strip(const T* __restrict__ dy, Act4 yo, const uint8_t* __restrict__ idx,
                                    T* __restrict__ dx, Act4 xi, int pad, const T* __restrict__ relu_y) {
    pdl_wait();
    pdl_trigger();
    const int cg = xi.cs / 8;
    const int strips = (xi.H + R - 1) / R;
    long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (t >= static_cast<long long>(xi.N) * strips * xi.W * cg) return;
    const int g = static_cast<int>(t % cg);
    t /= cg;
    const int iw = static_cast<int>(t % xi.W);
    t /= xi.W;
    const int ih0 = static_cast<int>(t % strips) * R;
    const int n = static_cast<int>(t / strips);
    const long long obase = static_cast<long long>(n) * yo.H * yo.W * yo.cs + g * 8;
    const int ow0 = iw + pad - (K - 1);
    Raw8<T> d[K][K];
    uint2 q[K][K];
    auto load_row = [&](int oh, Raw8<T> (&dr)[K], uint2 (&qr)[K]) {
#pragma unroll
        for (int c = 0; c < K; ++c) {
            const int ow = ow0 + c;
            if (oh >= 0 && oh < yo.H && ow >= 0 && ow < yo.W) {
                const long long o = obase + (static_cast<long long>(oh) * yo.W + ow) * yo.cs;
                dr[c] = ld_raw8(dy + o);
                qr[c] = __ldg(reinterpret_cast<const uint2*>(idx + o));
            } else {
                qr[c] = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
                dr[c] = raw8_zero<T>();
            }
        }
    };
#pragma unroll
    for (int da = 0; da < K - 1; ++da) load_row(ih0 + pad - (K - 1) + da, d[da], q[da]);
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int ih = ih0 + j;
        if (ih >= xi.H) break;
        load_row(ih + pad, d[(j + K - 1) % K], q[(j + K - 1) % K]);
        float acc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll
        for (int da = 0; da < K; ++da) {
            const int sl = (j + da) % K;
            const int tr = K - 1 - da;
#pragma unroll
            for (int db = 0; db < K; ++db) {
                const int tc = K - 1 - db;
                const uint32_t mm = static_cast<uint32_t>(tr * K + tc) * 0x01010101u;
                const uint32_t e0 = __vcmpeq4(q[sl][db].x, mm), e1 = __vcmpeq4(q[sl][db].y, mm);
                float f[8];
                unpack_raw(d[sl][db], f);
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    if ((((e < 4 ? e0 : e1) >> (8 * (e & 3))) & 1u) != 0u) acc[e] += f[e];
            }
        }
        const long long o = ((static_cast<long long>(n) * xi.H + ih) * xi.W + iw) * xi.cs + g * 8;
        if (relu_y) {
            float m[8];
            ld8(relu_y + o, m);
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (!(m[e] > 0.f)) acc[e] = 0.f;
        }
        st8(dx + o, acc);
    }
}

// Gather formulation: each input element sums the windows that selected it
// (no atomics; fixed window order, deterministic).
template <typename T, typename IT>
__global__ void k_pool_bwd(const T* __restrict__ dy, Act4 yo, const uint8_t* __restrict__ idx,
                           T* __restrict__ dx, Act4 xi, int k, int stride, int pad, int is_max,
                           const T* __restrict__ relu_y) {
    pdl_wait();
    pdl_trigger();
    const int cg = xi.cs / 8;
    const IT total = static_cast<IT>(xi.pixels() * cg);
    const float inv = 1.f / static_cast<float>(k * k);
    for (IT t = blockIdx.x * static_cast<IT>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<IT>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(t % cg);
        IT p = t / cg;
        const int iw = static_cast<int>(p % xi.W);
        p /= xi.W;
        const int ih = static_cast<int>(p % xi.H);
        const int n = static_cast<int>(p / xi.H);
        const int nh = ih + pad - k + 1, nw = iw + pad - k + 1;
        const int oh0 = nh <= 0 ? 0 : (nh + stride - 1) / stride;
        const int ow0 = nw <= 0 ? 0 : (nw + stride - 1) / stride;
        const int oh1 = min(yo.H - 1, (ih + pad) / stride);
        const int ow1 = min(yo.W - 1, (iw + pad) / stride);
        float acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.f;
        const long long obase = static_cast<long long>(n) * yo.H * yo.W * yo.cs + g * 8;
        for (int oh = oh0; oh <= oh1; ++oh)
            for (int ow = ow0; ow <= ow1; ++ow) {
                const long long o = obase + (static_cast<long long>(oh) * yo.W + ow) * yo.cs;
                float d[8];
                ld8(dy + o, d);
                if (is_max) {
                    const uint32_t me = static_cast<uint32_t>((ih - (oh * stride - pad)) * k + (iw - (ow * stride - pad)));
                    const uint2 q = __ldg(reinterpret_cast<const uint2*>(idx + o));
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const uint32_t w = ((j < 4 ? q.x : q.y) >> (8 * (j & 3))) & 0xFFu;
                        if (w == me) acc[j] += d[j];
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[j] += d[j] * inv;
                }
            }
        const long long o = ((static_cast<long long>(n) * xi.H + ih) * xi.W + iw) * xi.cs + g * 8;
        if (relu_y) {  // folded ReLU backward: relu_y is the ReLU output (= the pooling input)
            float m[8];
            ld8(relu_y + o, m);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (!(m[j] > 0.f)) acc[j] = 0.f;
        }
        st8(dx + o, acc);
    }
}

// ---------------------------------------------------------------- LRN (across channels, one warp per pixel)
template <typename T>
__global__ void k_lrn_fwd(const T* __restrict__ x, T* __restrict__ y, Act4 a, int size, float alpha, float beta,
                          float kk) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ float sm[];
    const int warps = blockDim.x / 32, wid = threadIdx.x / 32, lane = threadIdx.x % 32;
    float* sq = sm + wid * a.cs;
    const int half = size / 2;
    const float an = alpha / static_cast<float>(size);
    for (long long p = blockIdx.x * static_cast<long long>(warps) + wid; p < a.pixels();
         p += static_cast<long long>(gridDim.x) * warps) {
        const T* xp = x + p * a.cs;
        for (int c = lane; c < a.cs; c += 32) {
            const float v = to_f(xp[c]);
            sq[c] = v * v;
        }
        __syncwarp();
        for (int c = lane; c < a.cs; c += 32) {
            float out = 0.f;
            if (c < a.C) {
                float s = 0.f;
                for (int cc = max(0, c - half); cc <= min(a.C - 1, c + half); ++cc) s += sq[cc];
                const float scale = kk + an * s;
                out = to_f(xp[c]) * powf(scale, -beta);
            }
            y[p * a.cs + c] = from_f<T>(out);
        }
        __syncwarp();
    }
}

template <typename T>
__global__ void k_lrn_bwd(const T* __restrict__ dy, const T* __restrict__ x, const T* __restrict__ y,
                          T* __restrict__ dx, Act4 a, int size, float alpha, float beta, float kk, int relu) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ float sm[];
    const int warps = blockDim.x / 32, wid = threadIdx.x / 32, lane = threadIdx.x % 32;
    float* sq = sm + wid * 3 * a.cs;
    float* sc = sq + a.cs;
    float* tt = sc + a.cs;
    const int half = size / 2;
    const float an = alpha / static_cast<float>(size);
    const float coef = 2.f * alpha * beta / static_cast<float>(size);
    for (long long p = blockIdx.x * static_cast<long long>(warps) + wid; p < a.pixels();
         p += static_cast<long long>(gridDim.x) * warps) {
        const long long o = p * a.cs;
        for (int c = lane; c < a.cs; c += 32) {
            const float v = to_f(x[o + c]);
            sq[c] = v * v;
        }
        __syncwarp();
        for (int c = lane; c < a.C; c += 32) {
            float s = 0.f;
            for (int cc = max(0, c - half); cc <= min(a.C - 1, c + half); ++cc) s += sq[cc];
            sc[c] = kk + an * s;
            tt[c] = to_f(dy[o + c]) * to_f(y[o + c]) / sc[c];
        }
        __syncwarp();
        for (int c = lane; c < a.cs; c += 32) {
            float out = 0.f;
            if (c < a.C) {
                float s = 0.f;
                for (int cc = max(0, c - half); cc <= min(a.C - 1, c + half); ++cc) s += tt[cc];
                out = to_f(dy[o + c]) * powf(sc[c], -beta) - coef * to_f(x[o + c]) * s;
                if (relu && !(to_f(x[o + c]) > 0.f)) out = 0.f;
            }
            dx[o + c] = from_f<T>(out);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- softmax / loss head (fp32)
template <typename T>
__global__ void k_softmax_fwd(const T* __restrict__ x, long long ld, float* __restrict__ y, int rows, int F) {
    pdl_wait();
    pdl_trigger();
    const int warps = blockDim.x / 32, wid = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int r = blockIdx.x * warps + wid; r < rows; r += gridDim.x * warps) {
        const T* xr = x + r * ld;
        float m = -INFINITY;
        for (int j = lane; j < F; j += 32) m = fmaxf(m, to_f(xr[j]));
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float s = 0.f;
        for (int j = lane; j < F; j += 32) s += expf(to_f(xr[j]) - m);
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const float inv = 1.f / s;
        for (int j = lane; j < F; j += 32) y[static_cast<long long>(r) * F + j] = expf(to_f(xr[j]) - m) * inv;
    }
}

template <typename T>
__global__ void k_softmax_bwd(const float* __restrict__ dy, const float* __restrict__ y, T* __restrict__ dx,
                              long long ld, int rows, int F) {
    pdl_wait();
    pdl_trigger();
    const int warps = blockDim.x / 32, wid = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int r = blockIdx.x * warps + wid; r < rows; r += gridDim.x * warps) {
        const long long o = static_cast<long long>(r) * F;
        float d = 0.f;
        for (int j = lane; j < F; j += 32) d = __fmaf_rn(dy[o + j], y[o + j], d);
        for (int s = 16; s; s >>= 1) d += __shfl_xor_sync(0xffffffffu, d, s);
        for (int j = lane; j < ld; j += 32)
            dx[r * ld + j] = from_f<T>(j < F ? y[o + j] * (dy[o + j] - d) : 0.f);
    }
}

// Softmax log-loss head in one pass per row (warp per row), the same operations in the same order
// as k_softmax_fwd, k_f32_ew (Log / Recip / Scale / Mul), k_onehot and k_softmax_bwd, so the
// result is bit-identical to the separate statements:
//   S = softmax(z); L = log(max(S, 1e-30)); R = 1 / max(S, 1e-30); G = (Y * c) * R;
//   dz = S * (G - sum_j G_j S_j)   (pad columns of dz up to ld are 0)
template <typename T>
__global__ void k_softmax_xent(const T* __restrict__ z, long long ld, const int32_t* __restrict__ labels, float c,
                               float* __restrict__ L, float* __restrict__ Y, T* __restrict__ dz, int rows, int F) {
    pdl_wait();
    pdl_trigger();
    const int warps = blockDim.x / 32, wid = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int r = blockIdx.x * warps + wid; r < rows; r += gridDim.x * warps) {
        const T* zr = z + r * ld;
        const int lab = labels[r];
        float m = -INFINITY;
        for (int j = lane; j < F; j += 32) m = fmaxf(m, to_f(zr[j]));
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float s = 0.f;
        for (int j = lane; j < F; j += 32) s += expf(to_f(zr[j]) - m);
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const float inv = 1.f / s;
        const long long o = static_cast<long long>(r) * F;
        float d = 0.f;
        for (int j = lane; j < F; j += 32) {
            const float sj = expf(to_f(zr[j]) - m) * inv;
            const float yj = lab == j ? 1.f : 0.f;
            L[o + j] = logf(fmaxf(sj, 1e-30f));
            if (Y) Y[o + j] = yj;
            const float g = (yj * c) * (1.f / fmaxf(sj, 1e-30f));
            d = __fmaf_rn(g, sj, d);
        }
        for (int k = 16; k; k >>= 1) d += __shfl_xor_sync(0xffffffffu, d, k);
        for (int j = lane; j < ld; j += 32) {
            float v = 0.f;
            if (j < F) {
                const float sj = expf(to_f(zr[j]) - m) * inv;
                const float g = ((lab == j ? 1.f : 0.f) * c) * (1.f / fmaxf(sj, 1e-30f));
                v = sj * (g - d);
            }
            dz[r * ld + j] = from_f<T>(v);
        }
    }
}

__global__ void k_f32_ew(int op, const float* __restrict__ a, const float* __restrict__ b, float scale,
                         float* __restrict__ y, long long n) {
    pdl_wait();
    pdl_trigger();
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const float v = a[i];
        float r;
        switch (op) {
            case F32_LOG: r = logf(fmaxf(v, 1e-30f)); break;  // clamp before Log
            case F32_RECIP: r = 1.f / fmaxf(v, 1e-30f); break;
            case F32_SCALE: r = v * scale; break;
            case F32_MUL: r = v * b[i]; break;
            default: r = v + b[i]; break;
        }
        y[i] = r;
    }
}

__global__ void k_onehot(const int32_t* __restrict__ labels, float* __restrict__ y, int N, int K) {
    pdl_wait();
    pdl_trigger();
    const long long total = static_cast<long long>(N) * K;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        y[i] = labels[i / K] == static_cast<int>(i % K) ? 1.f : 0.f;
}

struct LossArgs {
    const float* a[4];
    const float* b[4];
    long long n[4];
    double coef[4];
    int nterms;
};

// One block, fixed strided partition + fixed tree: deterministic.
// Deterministic two-level reduction in one launch: kLossBlocks blocks write fp64
// partials; the last block to finish (ticket counter) sums them in block order and
// resets the counter for the next step (graph replays).
constexpr int kLossBlocks = 128;
__global__ void __launch_bounds__(256) k_loss(LossArgs args, float* out, double* partial, unsigned* ticket) {
    pdl_wait();
    pdl_trigger();
    __shared__ double red[256];
    __shared__ bool last;
    double acc = 0.0;
    for (int t = 0; t < args.nterms; ++t) {
        double s = 0.0;
        for (long long i = blockIdx.x * 256ll + threadIdx.x; i < args.n[t]; i += 256ll * gridDim.x)
            s += static_cast<double>(args.a[t][i]) * static_cast<double>(args.b[t][i]);
        acc += args.coef[t] * s;
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = 128; s; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        partial[blockIdx.x] = red[0];
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        double tot = 0.0;
        for (int b = 0; b < static_cast<int>(gridDim.x); ++b) tot += static_cast<volatile double*>(partial)[b];
        *out = static_cast<float>(tot);
        *ticket = 0;
    }
}

// Test body: precision = fraction of rows whose argmax (first maximum in
// column order, as std::max_element) equals the label.  One warp per row; integer hit count.
template <typename T>
__global__ void k_argmax_hits(const T* __restrict__ logits, long long ld, int N, int C,
                              const int32_t* __restrict__ labels, unsigned* hits) {
    pdl_wait();
    pdl_trigger();
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= N) return;
    const T* row = logits + static_cast<long long>(warp) * ld;
    float best = -INFINITY;
    int bi = C;
    for (int j = lane; j < C; j += 32) {
        const float v = static_cast<float>(row[j]);
        if (v > best || bi == C) {
            best = v;
            bi = j;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const float ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
        }
    }
    if (lane == 0 && bi == labels[warp]) atomicAdd(hits, 1u);
}

// ---------------------------------------------------------------- channel reductions
// Column (channel) sums over the rows (pixels) of an NHWC / [rows][ld] bf16 matrix.
// Stage 1: grid (channel tiles, row splits); each thread owns 8 channels (one
// 16-byte load per row) and strides over its split's rows; the row slots of a
// block are combined in shared memory in a fixed order and written as one partial
// per (split, channel).  Stage 2 sums the partials of a channel in split order.
// Deterministic for a fixed shape (the partition depends only on rows / ld).
//   RED_SUM   a = sum x
//   RED_STATS a = sum (x - x0), b = sum (x - x0)^2   (x0 = row 0: shifted single pass)
//   RED_BNBWD a = sum dy,       b = sum dy * (x - mean)   (x istd in the final stage)
enum RedMode { RED_SUM = 0, RED_STATS = 1, RED_BNBWD = 2 };
constexpr int kRedThreads = 256;

// Blocks of one channel tile are grouped in clusters of kRedCluster along the split axis; the
// cluster combines its blocks' sums through distributed shared memory and writes ONE partial,
// so the final kernel reads 4x fewer partials (it is latency-bound on them).
constexpr int kRedCluster = 4;
#ifndef TCB_RED_BPS
#define TCB_RED_BPS 3
#endif
#ifndef TCB_RED_U
#define TCB_RED_U 8
#endif
constexpr int kRedBlocksPerSm = TCB_RED_BPS;  // __launch_bounds__ minimum: <= 85 registers per thread

struct RedPlan {
    int ct;        // channels per tile (multiple of 8, <= 512)
    int tiles;     // channel tiles
    int splits;    // row splits (blocks along y, a multiple of kRedCluster)
    int parts;     // partials per channel = splits / kRedCluster
    long long rps; // rows per split
};

// max_clusters: co-resident clusters of the kernel (cudaOccupancyMaxActiveClusters); clusters
// are placed per GPC, so the one-wave block count is max_clusters * kRedCluster, which is below
// SMs * blocks-per-SM (a second partial wave costs ~40% of the kernel).
RedPlan red_plan(long long rows, int ld, int max_clusters) {
    RedPlan r;
    r.ct = std::min(ld, 512);
    r.tiles = (ld + r.ct - 1) / r.ct;
    const int rpi = kRedThreads / (r.ct / 8);
    const long long target = static_cast<long long>(max_clusters) * kRedCluster;  // one wave
    long long sp = std::max<long long>(1, target / r.tiles / kRedCluster * kRedCluster);
    sp = std::min<long long>(sp, std::max<long long>(1, rows / (8LL * rpi)));  // >= 8 rows per thread
    sp = std::min<long long>(sp, 1024);
    r.rps = (rows + sp - 1) / sp;
    const int used = static_cast<int>((rows + r.rps - 1) / r.rps);
    r.splits = (used + kRedCluster - 1) / kRedCluster * kRedCluster;  // trailing blocks see no rows
    r.parts = r.splits / kRedCluster;
    return r;
}

template <int MODE, typename T>
__global__ void __launch_bounds__(kRedThreads, kRedBlocksPerSm) k_chan_reduce(const T* __restrict__ x, const T* __restrict__ x2,
                                                             const float* __restrict__ stats, long long rows, int C,
                                                             int ld, int ct, long long rps, int splits,
                                                             float* __restrict__ part) {
    pdl_wait();
    pdl_trigger();
    __shared__ __align__(16) float sm[(MODE == RED_SUM ? 1 : 2) * kRedThreads * 8];
    const int tpr = ct >> 3;
    const int rpi = kRedThreads / tpr;
    const int tr = threadIdx.x / tpr, tc = threadIdx.x - tr * tpr;
    const int c0 = blockIdx.x * ct + tc * 8;
    float a[8], b[8], m[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = b[j] = m[j] = 0.f;
    const bool live = tr < rpi && c0 < ld;
    if (live) {
        if (MODE == RED_STATS) {
            ld8(x + c0, m);
        } else if (MODE == RED_BNBWD) {
#pragma unroll
            for (int j = 0; j < 8; ++j) m[j] = stats[min(c0 + j, C - 1)];
        }
        const long long r0 = blockIdx.y * rps, r1 = min(rows, r0 + rps);
        const T* px = x + r0 * ld + c0;
        const T* p2 = MODE == RED_BNBWD ? x2 + r0 * ld + c0 : nullptr;
        constexpr int U = (MODE == RED_BNBWD ? TCB_RED_U / 2 : TCB_RED_U) * 2 / static_cast<int>(sizeof(T));  // 64 B / tensor in flight
        for (long long rb = tr; r0 + rb < r1; rb += U * rpi) {
            Raw8<T> q[U], q2[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long r = rb + u * rpi;
                const bool ok = r0 + r < r1;
                q[u] = ok ? ld_raw8cs(px + r * ld) : raw8_zero<T>();
                if (MODE == RED_BNBWD) q2[u] = ok ? ld_raw8cs(p2 + r * ld) : raw8_zero<T>();
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (r0 + rb + u * rpi >= r1) break;
                float f[8];
                unpack_raw(q[u], f);
                if (MODE == RED_SUM) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) a[j] += f[j];
                } else if (MODE == RED_STATS) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float d = f[j] - m[j];
                        a[j] += d;
                        b[j] = fmaf(d, d, b[j]);
                    }
                } else {
                    float g[8];
                    unpack_raw(q2[u], g);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        a[j] += f[j];
                        b[j] = fmaf(f[j], g[j] - m[j], b[j]);  // x istd applied in the final stage
                    }
                }
            }
        }
    }
    // row-slot tr, channel offset tc*8 within the tile: sm[tr][ct]
    constexpr int NB = MODE == RED_SUM ? 1 : 2;
    auto put = [&](int slot, const float (&v)[8], int which) {
        float4* d = reinterpret_cast<float4*>(sm + which * kRedThreads * 8 + slot * ct + tc * 8);
        d[0] = make_float4(v[0], v[1], v[2], v[3]);
        d[1] = make_float4(v[4], v[5], v[6], v[7]);
    };
    if (tr < rpi) {
        put(tr, a, 0);
        if (NB == 2) put(tr, b, 1);
    }
    __syncthreads();
    // fixed pairwise tree over the row slots (deterministic for a given shape)
    int span = 1;
    while (span < rpi) span <<= 1;
    for (int h = span >> 1; h > 0; h >>= 1) {
        if (tr < h && tr + h < rpi) {
#pragma unroll
            for (int w = 0; w < NB; ++w) {
                float4* d = reinterpret_cast<float4*>(sm + w * kRedThreads * 8 + tr * ct + tc * 8);
                const float4* e = reinterpret_cast<const float4*>(sm + w * kRedThreads * 8 + (tr + h) * ct + tc * 8);
                const float4 d0 = d[0], d1 = d[1], e0 = e[0], e1 = e[1];
                d[0] = make_float4(d0.x + e0.x, d0.y + e0.y, d0.z + e0.z, d0.w + e0.w);
                d[1] = make_float4(d1.x + e1.x, d1.y + e1.y, d1.z + e1.z, d1.w + e1.w);
            }
        }
        __syncthreads();
    }
    // cluster combine: rank 0 sums the kRedCluster blocks' slot-0 rows in rank order
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (rank == 0) {
        const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
        for (int cc = threadIdx.x; cc < ct; cc += kRedThreads) {
            const int c = blockIdx.x * ct + cc;
            if (c >= C) continue;
            float sa = 0.f, sb = 0.f;
#pragma unroll
            for (int r = 0; r < kRedCluster; ++r) {
                uint32_t ra, rb;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(base + cc * 4), "r"(r));
                float va, vb = 0.f;
                asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(va) : "r"(ra));
                if (NB == 2) {
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                                 : "=r"(rb)
                                 : "r"(base + (kRedThreads * 8 + cc) * 4), "r"(r));
                    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(vb) : "r"(rb));
                }
                sa += va;
                sb += vb;
            }
            const int q = blockIdx.y / kRedCluster;
            part[static_cast<long long>(q) * C + c] = sa;
            if (MODE != RED_SUM) part[static_cast<long long>(splits / kRedCluster + q) * C + c] = sb;
        }
    }
    // keep every block's shared memory alive until rank 0 has read it
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Stage 2.  RED_SUM: out[c] = scale * sum.  RED_STATS: stats = (mean, istd), coef =
// (gamma * istd, beta - mean * gamma * istd).  RED_BNBWD: out = (sum dy, sum dy*xhat) and, when
// gamma is given, the data-gradient coefficients (k1, k2, k3) at out + 2C, with `beta` = the
// forward statistics (mean, istd) and `scale` = 1 / rows:
//   dx = gamma*istd*(dy - sum(dy)/M - xhat*sum(dy*xhat)/M) = k1*dy + k2*x + k3
template <int MODE, typename T>
__global__ void __launch_bounds__(256) k_chan_final(const float* __restrict__ part, int splits, int C, float scale,
                                                    float* __restrict__ out, const T* __restrict__ x, long long rows,
                                                    float eps, const float* __restrict__ gamma,
                                                    const float* __restrict__ beta, float* __restrict__ coef) {
    pdl_wait();
    pdl_trigger();
    // one warp per channel: lane l sums splits l, l+32, ...; the warp combines the 32 lane sums
    // with a fixed xor tree (deterministic)
    const int lane = threadIdx.x & 31;
    const int c = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (c >= C) return;
    float sa = 0.f, sb = 0.f;
#pragma unroll 4
    for (int q = lane; q < splits; q += 32) {
        sa += part[static_cast<long long>(q) * C + c];
        if (MODE != RED_SUM) sb += part[static_cast<long long>(splits + q) * C + c];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        sa += __shfl_xor_sync(0xffffffffu, sa, o);
        if (MODE != RED_SUM) sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
    if (lane != 0) return;
    if (MODE == RED_SUM) {
        out[c] = sa * scale;
    } else if (MODE == RED_STATS) {
        const float inv = 1.f / static_cast<float>(rows);
        const float m1 = sa * inv;
        const float mean = to_f(x[c]) + m1;
        const float var = fmaxf(sb * inv - m1 * m1, 0.f);
        const float istd = rsqrtf(var + eps);
        out[c] = mean;
        out[C + c] = istd;
        const float g = gamma[c] * istd;
        coef[c] = g;
        coef[C + c] = beta[c] - mean * g;
    } else {
        sb *= beta[C + c];  // sum dy*(x - mean) -> sum dy*xhat
        out[c] = sa;
        out[C + c] = sb;
        if (gamma) {
            const float is = beta[C + c], mean = beta[c];
            const float g = gamma[c] * is;
            const float t = sb * scale * is;  // sum(dy*xhat)/M * istd
            out[2 * C + c] = g;
            out[3 * C + c] = -g * t;
            out[4 * C + c] = -g * sa * scale + g * t * mean;
        }
    }
}

// 8 per-channel coefficients starting at channel c0 (a multiple of 8): two 16-byte loads when
// the array offset is 16-byte aligned and all 8 channels exist, else guarded scalars.
__device__ __forceinline__ void ld_coef8(const float* __restrict__ a, int c0, int C, float (&v)[8]) {
    if (c0 + 8 <= C && (reinterpret_cast<uintptr_t>(a + c0) & 15) == 0) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(a + c0)), y = __ldg(reinterpret_cast<const float4*>(a + c0) + 1);
        v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w, v[4] = y.x, v[5] = y.y, v[6] = y.z, v[7] = y.w;
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = c0 + j < C ? __ldg(a + c0 + j) : 0.f;
    }
}

// y = x * coef[c] + coef[C + c] over 8 channels per thread; pad channels -> 0.
template <typename T>
__global__ void k_chan_affine(const T* __restrict__ x, const float* __restrict__ coef, T* __restrict__ y,
                              long long n8, int ld8, int C, int relu, const T* __restrict__ res) {
    pdl_wait();
    pdl_trigger();
    const long long S = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long i0 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i0 < n8; i0 += 2 * S) {
        Raw8<T> q[2], rq[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            q[u] = i0 + u * S < n8 ? ld_raw8cs(x + (i0 + u * S) * 8) : raw8_zero<T>();
            if (res) rq[u] = i0 + u * S < n8 ? ld_raw8cs(res + (i0 + u * S) * 8) : raw8_zero<T>();
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const long long i = i0 + u * S;
            if (i >= n8) break;
            const int c0 = static_cast<int>(n8 < (1ll << 31) ? static_cast<int>(i) % ld8 : i % ld8) * 8;
            float f[8], a[8], b[8];
            unpack_raw(q[u], f);
            ld_coef8(coef, c0, C, a);
            ld_coef8(coef + C, c0, C, b);
            if (res) {
                // folded residual add: the BN output is rounded to the storage type first, exactly
                // as the separate add would have read it
                float r[8];
                unpack_raw(rq[u], r);
#pragma unroll
                for (int j = 0; j < 8; ++j) f[j] = to_f(from_f<T>(fmaf(f[j], a[j], b[j]))) + r[j];
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) f[j] = fmaf(f[j], a[j], b[j]);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                f[j] = c0 + j < C ? f[j] : 0.f;
                if (relu) f[j] = fmaxf(f[j], 0.f);
            }
            st8(y + i * 8, f);
        }
    }
}

// dx = k1*dy + k2*x + k3 per channel (coefficients from k_chan_final<RED_BNBWD>)
template <typename T>
__global__ void k_bn_bwd_apply(const T* __restrict__ dy, const T* __restrict__ x, const float* __restrict__ k,
                               T* __restrict__ dx, long long n8, int ld8, int C) {
    pdl_wait();
    pdl_trigger();
    const long long S = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long i0 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i0 < n8; i0 += 2 * S) {
        Raw8<T> q[2], r[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const bool ok = i0 + u * S < n8;
            q[u] = ok ? ld_raw8cs(dy + (i0 + u * S) * 8) : raw8_zero<T>();
            r[u] = ok ? ld_raw8cs(x + (i0 + u * S) * 8) : raw8_zero<T>();
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const long long i = i0 + u * S;
            if (i >= n8) break;
            const int c0 = static_cast<int>(n8 < (1ll << 31) ? static_cast<int>(i) % ld8 : i % ld8) * 8;
            float f[8], g[8], k1[8], k2[8], k3[8];
            unpack_raw(q[u], f);
            unpack_raw(r[u], g);
            ld_coef8(k, c0, C, k1);
            ld_coef8(k + C, c0, C, k2);
            ld_coef8(k + 2 * C, c0, C, k3);
#pragma unroll
            for (int j = 0; j < 8; ++j) f[j] = c0 + j < C ? fmaf(k1[j], f[j], fmaf(k2[j], g[j], k3[j])) : 0.f;
            st8(dx + i * 8, f);
        }
    }
}

template <typename T>
__global__ void k_bias_add(const T* __restrict__ x, const float* __restrict__ b, T* __restrict__ y, long long rows,
                           int cols, long long ld, int relu) {
    pdl_wait();
    pdl_trigger();
    const long long total = rows * ld;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i % ld);
        float v = c < cols ? to_f(x[i]) + b[c] : 0.f;
        if (relu) v = fmaxf(v, 0.f);
        y[i] = from_f<T>(v);
    }
}

template <typename T>
__global__ void k_channel_copy(const T* __restrict__ src, int src_cs, T* __restrict__ dst, int dst_cs, int off,
                               int c, long long pixels) {
    pdl_wait();
    pdl_trigger();
    const long long total = pixels * c;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long p = i / c;
        const int ch = static_cast<int>(i - p * c);
        dst[p * dst_cs + off + ch] = src[p * src_cs + ch];
    }
}

// 8-channel chunks when strides, offset and width are multiples of 8 (every GoogLeNet concat)
template <typename T>
// relu_y (may be null, dst layout): a folded in-place ReLU backward of the copied gradient slice
__global__ void k_channel_copy8(const T* __restrict__ src, int src_cs, T* __restrict__ dst, int dst_cs, int off, int c8,
                                long long pixels, const T* __restrict__ relu_y) {
    pdl_wait();
    pdl_trigger();
    const long long total = pixels * c8;
    const bool i32 = total < (1ll << 31);
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long p = i32 ? static_cast<long long>(static_cast<int>(t) / c8) : t / c8;
        const int g = static_cast<int>(t - p * c8);
        float f[8];
        ld8(src + p * src_cs + g * 8, f);
        if (relu_y) {
            float r[8];
            ld8(relu_y + p * dst_cs + off + g * 8, r);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (!(r[j] > 0.f)) f[j] = 0.f;
        }
        st8(dst + p * dst_cs + off + g * 8, f);
    }
}


// ---------------------------------------------------------------- LRN v2: thread per (pixel, 8 channels)
// Window sums over channels [c - n/2, c + n/2] read the neighbouring 16-byte
// chunks of the same pixel (L1 hits); n <= 9 so chunks g-1 .. g+1 suffice.
// v[8..16) = channels g*8..g*8+7 and NEED channels either side (zero beyond the tensor).
// NEED <= 4 reads the neighbours with 8-byte loads, otherwise whole neighbour chunks.
template <int NEED, typename T>
__device__ __forceinline__ void load_chunk3(const T* __restrict__ p, int g, int ng, float (&v)[24]) {
    static_assert(NEED <= 8, "LRN window too wide");
    float f[8];
    ld8(p + g * 8, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[8 + j] = f[j];
    if constexpr (NEED <= 4 && sizeof(T) == 4) {
        float4 lo = make_float4(0.f, 0.f, 0.f, 0.f), hi = lo;
        if (g > 0) lo = *reinterpret_cast<const float4*>(p + g * 8 - 4);
        if (g + 1 < ng) hi = *reinterpret_cast<const float4*>(p + g * 8 + 8);
        v[4] = lo.x, v[5] = lo.y, v[6] = lo.z, v[7] = lo.w;
        v[16] = hi.x, v[17] = hi.y, v[18] = hi.z, v[19] = hi.w;
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = v[20 + j] = 0.f;
    } else if constexpr (NEED <= 4) {
        uint2 lo = make_uint2(0, 0), hi = make_uint2(0, 0);
        if (g > 0) lo = *reinterpret_cast<const uint2*>(p + g * 8 - 4);
        if (g + 1 < ng) hi = *reinterpret_cast<const uint2*>(p + g * 8 + 8);
        const __nv_bfloat162* l2 = reinterpret_cast<const __nv_bfloat162*>(&lo);
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&hi);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const float2 a = __bfloat1622float2(l2[i]), b = __bfloat1622float2(h2[i]);
            v[4 + 2 * i] = a.x;
            v[5 + 2 * i] = a.y;
            v[16 + 2 * i] = b.x;
            v[17 + 2 * i] = b.y;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = v[20 + j] = 0.f;
    } else {
        float lo[8], hi[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) lo[j] = hi[j] = 0.f;
        if (g > 0) ld8(p + g * 8 - 8, lo);
        if (g + 1 < ng) ld8(p + g * 8 + 8, hi);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            v[j] = lo[j];
            v[16 + j] = hi[j];
        }
    }
}

// Two chunks per thread (g2, g2 + 1; ng even): v[8..24) = channels g2*8 .. g2*8+15 and NEED <= 4
// channels either side read with 8-byte loads (zero beyond the tensor): 4 loads per 16 channels
// instead of v2's 6.
template <int NEED, typename T>
__device__ __forceinline__ void load_chunk2x(const T* __restrict__ p, int g2, int ng, float (&v)[32]) {
    static_assert(NEED <= 4 && sizeof(T) == 2, "two-chunk LRN loads: bf16, window <= 9");
    float f[8];
    ld8(p + g2 * 8, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[8 + j] = f[j];
    ld8(p + g2 * 8 + 8, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[16 + j] = f[j];
    uint2 lo = make_uint2(0, 0), hi = make_uint2(0, 0);
    if (g2 > 0) lo = *reinterpret_cast<const uint2*>(p + g2 * 8 - 4);
    if (g2 + 2 < ng) hi = *reinterpret_cast<const uint2*>(p + g2 * 8 + 16);
    const __nv_bfloat162* l2 = reinterpret_cast<const __nv_bfloat162*>(&lo);
    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&hi);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float2 a = __bfloat1622float2(l2[i]), b = __bfloat1622float2(h2[i]);
        v[4 + 2 * i] = a.x;
        v[5 + 2 * i] = a.y;
        v[24 + 2 * i] = b.x;
        v[25 + 2 * i] = b.y;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = v[28 + j] = 0.f;
}

// LRN scale terms are >= k > 0 and far from the denormal range: pow / reciprocal straight on the
// MUFU approximations (the same lg2 / ex2 / rcp __powf and __fdividef use, minus their
// denormal-range fix-ups and branches).
__device__ __forceinline__ float pow_pos(float x, float e) {
    float l, r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(x));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(l * e));
    return r;
}
__device__ __forceinline__ float rcp_pos(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// HALF = n/2 is a template parameter so every window loop unrolls and the
// per-thread channel windows stay in registers.
template <int HALF, typename T, typename IT>
__global__ void k_lrn2_fwd(const T* __restrict__ x, T* __restrict__ y, Act4 a, float alpha, float beta,
                           float kk) {
    pdl_wait();
    pdl_trigger();
    const int ng = a.cs / 8;
    const long long total = a.pixels() * ng;
    const float an = alpha / static_cast<float>(2 * HALF + 1);
    for (IT t = blockIdx.x * static_cast<IT>(blockDim.x) + threadIdx.x; t < static_cast<IT>(total);
         t += static_cast<IT>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(t % ng);
        const T* px = x + static_cast<long long>(t / ng) * a.cs;
        float v[24];
        load_chunk3<HALF>(px, g, ng, v);
        // channels outside [0, C) contribute nothing (pads are zero, neighbours beyond the tensor loaded as 0)
        float out[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float s = 0.f;
#pragma unroll
            for (int d = -HALF; d <= HALF; ++d) s += v[8 + j + d] * v[8 + j + d];
            out[j] = (a.C == a.cs || (g * 8 + j) < a.C) ? v[8 + j] * pow_pos(kk + an * s, -beta) : 0.f;
        }
        st8(y + static_cast<long long>(t) * 8, out);
    }
}

template <int HALF, typename T, typename IT>
__global__ void k_lrn2_bwd(const T* __restrict__ dy, const T* __restrict__ x, const T* __restrict__ y,
                           T* __restrict__ dx, Act4 a, float alpha, float beta, float kk, int relu) {
    pdl_wait();
    pdl_trigger();
    const int ng = a.cs / 8;
    const long long total = a.pixels() * ng;
    const float an = alpha / static_cast<float>(2 * HALF + 1);
    const float coef = 2.f * alpha * beta / static_cast<float>(2 * HALF + 1);
    constexpr int L = 8 - HALF, U = 16 + HALF;  // window of channels g*8-HALF .. g*8+7+HALF
    const bool full = a.C == a.cs;                // no pad channels: skip the per-channel test
    for (IT t = blockIdx.x * static_cast<IT>(blockDim.x) + threadIdx.x; t < static_cast<IT>(total);
         t += static_cast<IT>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(t % ng);
        const long long base = static_cast<long long>(t / ng) * a.cs;
        float xv[24], dv[24], yv[24];
        load_chunk3<2 * HALF>(x + base, g, ng, xv);
        load_chunk3<HALF>(dy + base, g, ng, dv);
        load_chunk3<HALF>(y + base, g, ng, yv);
        float sc[24], tt[24];
#pragma unroll
        for (int i = L; i < U; ++i) {
            float s = 0.f;
#pragma unroll
            for (int d = -HALF; d <= HALF; ++d) s += xv[i + d] * xv[i + d];
            sc[i] = kk + an * s;
            // zero for channels outside [0, C): dy and y are zero there
            tt[i] = dv[i] * yv[i] * rcp_pos(sc[i]);  // MUFU reciprocal
        }
        float out[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float s = 0.f;
#pragma unroll
            for (int d = -HALF; d <= HALF; ++d) s += tt[8 + j + d];
            out[j] = (full || (g * 8 + j) < a.C) ? dv[8 + j] * pow_pos(sc[8 + j], -beta) - coef * xv[8 + j] * s : 0.f;
            if (relu && !(xv[8 + j] > 0.f)) out[j] = 0.f;  // folded ReLU backward: x is the ReLU output
        }
        st8(dx + base + g * 8, out);
    }
}

// v2 with two 8-channel chunks per thread (bf16, window <= 5 so the backward's x window stays
// within 4 channels): the same per-channel arithmetic, a third fewer load instructions.
template <int HALF, typename IT>
__global__ void k_lrn2x_fwd(const bf16* __restrict__ x, bf16* __restrict__ y, Act4 a, float alpha, float beta,
                            float kk) {
    pdl_wait();
    pdl_trigger();
    const int ng = a.cs / 8, nh = ng / 2;
    const long long total = a.pixels() * nh;
    const float an = alpha / static_cast<float>(2 * HALF + 1);
    for (IT t = blockIdx.x * static_cast<IT>(blockDim.x) + threadIdx.x; t < static_cast<IT>(total);
         t += static_cast<IT>(gridDim.x) * blockDim.x) {
        const int g2 = static_cast<int>(t % nh) * 2;
        const bf16* px = x + static_cast<long long>(t / nh) * a.cs;
        float v[32];
        load_chunk2x<HALF>(px, g2, ng, v);
        float out[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            float s = 0.f;
#pragma unroll
            for (int d = -HALF; d <= HALF; ++d) s += v[8 + j + d] * v[8 + j + d];
            out[j] = (a.C == a.cs || (g2 * 8 + j) < a.C) ? v[8 + j] * pow_pos(kk + an * s, -beta) : 0.f;
        }
        bf16* py = y + static_cast<long long>(t / nh) * a.cs + g2 * 8;
        st8(py, *reinterpret_cast<float(*)[8]>(out));
        st8(py + 8, *reinterpret_cast<float(*)[8]>(out + 8));
    }
}

template <int HALF, typename IT>
__global__ void k_lrn2x_bwd(const bf16* __restrict__ dy, const bf16* __restrict__ x, const bf16* __restrict__ y,
                            bf16* __restrict__ dx, Act4 a, float alpha, float beta, float kk, int relu) {
    pdl_wait();
    pdl_trigger();
    const int ng = a.cs / 8, nh = ng / 2;
    const long long total = a.pixels() * nh;
    const float an = alpha / static_cast<float>(2 * HALF + 1);
    const float coef = 2.f * alpha * beta / static_cast<float>(2 * HALF + 1);
    constexpr int L = 8 - HALF, U = 24 + HALF;  // window of channels g2*8-HALF .. g2*8+15+HALF
    const bool full = a.C == a.cs;
    for (IT t = blockIdx.x * static_cast<IT>(blockDim.x) + threadIdx.x; t < static_cast<IT>(total);
         t += static_cast<IT>(gridDim.x) * blockDim.x) {
        const int g2 = static_cast<int>(t % nh) * 2;
        const long long base = static_cast<long long>(t / nh) * a.cs;
        float xv[32], dv[32], yv[32];
        load_chunk2x<2 * HALF>(x + base, g2, ng, xv);
        load_chunk2x<HALF>(dy + base, g2, ng, dv);
        load_chunk2x<HALF>(y + base, g2, ng, yv);
        float sc[32], tt[32];
#pragma unroll
        for (int i = L; i < U; ++i) {
            float s = 0.f;
#pragma unroll
            for (int d = -HALF; d <= HALF; ++d) s += xv[i + d] * xv[i + d];
            sc[i] = kk + an * s;
            tt[i] = dv[i] * yv[i] * rcp_pos(sc[i]);
        }
        float out[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            float s = 0.f;
#pragma unroll
            for (int d = -HALF; d <= HALF; ++d) s += tt[8 + j + d];
            out[j] = (full || (g2 * 8 + j) < a.C) ? dv[8 + j] * pow_pos(sc[8 + j], -beta) - coef * xv[8 + j] * s : 0.f;
            if (relu && !(xv[8 + j] > 0.f)) out[j] = 0.f;
        }
        st8(dx + base + g2 * 8, *reinterpret_cast<float(*)[8]>(out));
        st8(dx + base + g2 * 8 + 8, *reinterpret_cast<float(*)[8]>(out + 8));
    }
}

// ---------------------------------------------------------------- LRN v3: pixel-aligned warps
// ng = cs/8 <= 32 lanes own one pixel's channel chunks (32/ng pixels per warp, the spare lanes
// idle); every lane loads only its own 8 channels and takes the HALF channels either side from
// the neighbouring lanes with shuffles (zero at the pixel's first / last chunk).  Compared with
// v2 this drops the neighbour loads and, in the backward, the 1.5x-redundant scale / t terms of
// the window margin (each lane computes them for its own channels only).  Same arithmetic and
// summation order as v2.
struct LrnLanes {
    int ng, ppw;
    long long pix;
    bool active;
    int g;
};
__device__ __forceinline__ LrnLanes lrn_lanes(const Act4& a, long long warp, int lane) {
    LrnLanes r;
    r.ng = a.cs / 8;
    r.ppw = 32 / r.ng;
    const int pl = lane / r.ng;
    r.g = lane - pl * r.ng;
    r.pix = warp * r.ppw + pl;
    r.active = pl < r.ppw && r.pix < a.pixels();
    return r;
}
// w[HALF + j] = v[j]; w[0..HALF) from the previous chunk, w[HALF+8..) from the next one
template <int HALF>
__device__ __forceinline__ void lrn_window(const float (&v)[8], int g, int ng, float (&w)[8 + 2 * HALF]) {
#pragma unroll
    for (int i = 0; i < HALF; ++i) {
        const float l = __shfl_up_sync(0xffffffffu, v[8 - HALF + i], 1);
        const float r = __shfl_down_sync(0xffffffffu, v[i], 1);
        w[i] = g > 0 ? l : 0.f;
        w[HALF + 8 + i] = g + 1 < ng ? r : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) w[HALF + j] = v[j];
}

template <int HALF, typename T>
__global__ void k_lrn3_fwd(const T* __restrict__ x, T* __restrict__ y, Act4 a, float alpha, float beta, float kk) {
    pdl_wait();
    pdl_trigger();
    const float an = alpha / static_cast<float>(2 * HALF + 1);
    const int lane = threadIdx.x & 31;
    const long long nw = (a.pixels() + 32 / (a.cs / 8) - 1) / (32 / (a.cs / 8));
    for (long long w = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5; w < nw;
         w += (static_cast<long long>(gridDim.x) * blockDim.x) >> 5) {
        const LrnLanes L = lrn_lanes(a, w, lane);
        const long long o = L.pix * a.cs + L.g * 8;
        float xv[8], q[8];
        if (L.active)
            ld8(x + o, xv);
        else
#pragma unroll
            for (int j = 0; j < 8; ++j) xv[j] = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) q[j] = xv[j] * xv[j];
        float qw[8 + 2 * HALF];
        lrn_window<HALF>(q, L.g, L.ng, qw);
        float out[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float s = 0.f;
#pragma unroll
            for (int d = 0; d <= 2 * HALF; ++d) s += qw[j + d];
            // pad channels (>= C) hold x = 0, so the product is already zero there
            out[j] = xv[j] * pow_pos(kk + an * s, -beta);
        }
        if (L.active) st8(y + o, out);
    }
}

template <int HALF, typename T>
__global__ void k_lrn3_bwd(const T* __restrict__ dy, const T* __restrict__ x, const T* __restrict__ y,
                           T* __restrict__ dx, Act4 a, float alpha, float beta, float kk, int relu) {
    pdl_wait();
    pdl_trigger();
    const float an = alpha / static_cast<float>(2 * HALF + 1);
    const float coef = 2.f * alpha * beta / static_cast<float>(2 * HALF + 1);
    const int lane = threadIdx.x & 31;
    const long long nw = (a.pixels() + 32 / (a.cs / 8) - 1) / (32 / (a.cs / 8));
    for (long long w = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5; w < nw;
         w += (static_cast<long long>(gridDim.x) * blockDim.x) >> 5) {
        const LrnLanes L = lrn_lanes(a, w, lane);
        const long long o = L.pix * a.cs + L.g * 8;
        float xv[8], dv[8], yv[8];
        if (L.active) {
            ld8(x + o, xv);
            ld8(dy + o, dv);
            ld8(y + o, yv);
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) xv[j] = dv[j] = yv[j] = 0.f;
        }
        float q[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) q[j] = xv[j] * xv[j];
        float qw[8 + 2 * HALF];
        lrn_window<HALF>(q, L.g, L.ng, qw);
        float sc[8], tt[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float s = 0.f;
#pragma unroll
            for (int d = 0; d <= 2 * HALF; ++d) s += qw[j + d];
            sc[j] = kk + an * s;
            tt[j] = dv[j] * yv[j] * rcp_pos(sc[j]);  // zero outside [0, C): dy and y are zero there
        }
        float tw[8 + 2 * HALF];
        lrn_window<HALF>(tt, L.g, L.ng, tw);
        float out[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float s = 0.f;
#pragma unroll
            for (int d = 0; d <= 2 * HALF; ++d) s += tw[j + d];
            out[j] = dv[j] * pow_pos(sc[j], -beta) - coef * xv[j] * s;  // zero on pad channels (dy = x = 0)
            if (relu && !(xv[j] > 0.f)) out[j] = 0.f;  // folded ReLU backward: x is the ReLU output
        }
        if (L.active) st8(dx + o, out);
    }
}

// ---------------------------------------------------------------- input staging
// Source coordinates of staged element i; false for padding (channel pad or outside the image).
__device__ __forceinline__ bool stage_src(const StageLayout& L, long long i, int& n, int& c, int& h, int& w) {
    if (!L.s2d) {
        c = static_cast<int>(i % L.cs);
        long long p = i / L.cs;
        w = static_cast<int>(p % L.W);
        p /= L.W;
        h = static_cast<int>(p % L.H);
        n = static_cast<int>(p / L.H);
        return c < L.C;
    }
    const int cc = L.s2d * L.s2d * L.cs;
    const int ch = static_cast<int>(i % cc);
    long long p = i / cc;
    const int Q = static_cast<int>(p % L.Ws);
    p /= L.Ws;
    const int P = static_cast<int>(p % L.Hs);
    n = static_cast<int>(p / L.Hs);
    c = ch % L.cs;
    const int ij = ch / L.cs;
    h = P * L.s2d + ij / L.s2d - L.pad;
    w = Q * L.s2d + ij % L.s2d - L.pad;
    return c < L.C && h >= 0 && h < L.H && w >= 0 && w < L.W;
}

// Row-tiled staging: block (n, output row) reads the source rows it needs coalesced into
// shared memory ([c][row][w] fp32, zero outside the image), then writes the output row as
// 16-byte chunks.  Output row = image row h (NHWC) or space-to-depth row P (rows s*P - pad + i).
template <typename T, typename SRC>
__global__ void __launch_bounds__(256) k_stage_rows(const SRC* __restrict__ x, T* __restrict__ y, StageLayout L,
                                                    int log2_cs, int log2_s) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ float tile[];
    const int rows_out = L.s2d ? L.Hs : L.H;
    const int n = blockIdx.x / rows_out, r = blockIdx.x - n * rows_out;
    const int s = 1 << log2_s;
    const int h0 = L.s2d ? r * s - L.pad : r;
    const int C = L.C, W = L.W;
    constexpr int VW = 16 / sizeof(SRC);  // source elements per 16-byte load
    if (W % VW == 0) {
        // tile row (c, i) = source row h0 + i of channel c; all 16-byte loads of the block in flight
        const int wv = W / VW, total = C * s * wv;
#pragma unroll 4
        for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
            const int ci = idx / wv, w = (idx - ci * wv) * VW;
            const int c = ci >> log2_s, h = h0 + (ci & (s - 1));
            float f[VW];
            if (h >= 0 && h < L.H) {
                const uint4 v = __ldcs(reinterpret_cast<const uint4*>(x + ((static_cast<long long>(n) * C + c) * L.H + h) * W + w));
                const SRC* e = reinterpret_cast<const SRC*>(&v);
#pragma unroll
                for (int j = 0; j < VW; ++j) f[j] = to_f(e[j]);
            } else {
#pragma unroll
                for (int j = 0; j < VW; ++j) f[j] = 0.f;
            }
#pragma unroll
            for (int j = 0; j < VW; ++j) tile[ci * W + w + j] = f[j];
        }
    } else {
        for (int ci = 0; ci < C * s; ++ci) {
            const int c = ci >> log2_s, h = h0 + (ci & (s - 1));
            const bool ok = h >= 0 && h < L.H;
            const SRC* src = x + ((static_cast<long long>(n) * C + c) * L.H + h) * W;
            for (int w = threadIdx.x; w < W; w += blockDim.x) tile[ci * W + w] = ok ? to_f(__ldcs(src + w)) : 0.f;
        }
    }
    __syncthreads();
    const int log2_cc = 2 * log2_s + log2_cs;  // output channels per output pixel = s*s*cs
    const int wout = L.s2d ? L.Ws : L.W;
    const int chunks = (wout << log2_cc) >> 3;
    T* out = y + (static_cast<long long>(n) * rows_out + r) * (static_cast<long long>(wout) << log2_cc);
    for (int q = threadIdx.x; q < chunks; q += blockDim.x) {
        const int e0 = q << 3;
        float f[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int Q = (e0 + j) >> log2_cc, ch = (e0 + j) & ((1 << log2_cc) - 1);
            const int c = ch & ((1 << log2_cs) - 1), ij = ch >> log2_cs;
            const int i = ij >> log2_s, jj = ij & (s - 1);
            const int w = L.s2d ? (Q << log2_s) + jj - L.pad : Q;
            f[j] = (c < C && w >= 0 && w < W) ? tile[((c << log2_s) + i) * W + w] : 0.f;
        }
        st8(out + q * 8, f);
    }
}

// Direct staging for 4-channel strides (cs = 4, C <= 4): every staged 8-element chunk is two
// horizontally adjacent source positions x 4 channels (a pixel pair, or with space-to-depth two
// neighbouring taps of one pixel), so a thread reads one 8-byte pair per real channel straight
// from the NCHW rows (each input element is used once: no shared-memory tile) and writes 16 B.
template <typename T>
__global__ void k_stage_direct(const float* __restrict__ x, T* __restrict__ y, StageLayout L, int log2_s) {
    pdl_wait();
    pdl_trigger();
    const long long chunks = L.elems() / 8;
    const int s = 1 << log2_s;
    for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < chunks;
         q += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long e0 = q * 8;
        int n, h, w0;
        if (L.s2d) {
            const int lcc = 2 * log2_s + 2;  // channels per staged pixel = s * s * 4
            const long long pix = e0 >> lcc;
            const int ij0 = static_cast<int>(e0 & ((1 << lcc) - 1)) >> 2;
            const int Q = static_cast<int>(pix % L.Ws);
            const long long t = pix / L.Ws;
            const int P = static_cast<int>(t % L.Hs);
            n = static_cast<int>(t / L.Hs);
            h = P * s + (ij0 >> log2_s) - L.pad;
            w0 = Q * s + (ij0 & (s - 1)) - L.pad;
        } else {
            const long long pix = e0 >> 2;
            w0 = static_cast<int>(pix % L.W);
            const long long t = pix / L.W;
            h = static_cast<int>(t % L.H);
            n = static_cast<int>(t / L.H);
        }
        float f[8];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            float a = 0.f, b = 0.f;
            if (c < L.C && h >= 0 && h < L.H) {
                const float* row = x + ((static_cast<long long>(n) * L.C + c) * L.H + h) * L.W;
                if (w0 >= 0 && w0 + 1 < L.W && ((reinterpret_cast<uintptr_t>(row + w0) & 7) == 0)) {
                    const float2 v = __ldcs(reinterpret_cast<const float2*>(row + w0));
                    a = v.x, b = v.y;
                } else {
                    if (w0 >= 0 && w0 < L.W) a = __ldcs(row + w0);
                    if (w0 + 1 >= 0 && w0 + 1 < L.W) b = __ldcs(row + w0 + 1);
                }
            }
            f[c] = a;
            f[4 + c] = b;
        }
        st8(y + e0, f);
    }
}

template <typename T, typename SRC>
__global__ void k_nchw_to_nhwc(const SRC* __restrict__ x, T* __restrict__ y, StageLayout L) {
    pdl_wait();
    pdl_trigger();
    const long long total = L.elems();
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        int n, c, h, w;
        const bool ok = stage_src(L, i, n, c, h, w);
        y[i] = from_f<T>(ok ? to_f(x[((static_cast<long long>(n) * L.C + c) * L.H + h) * L.W + w]) : 0.f);
    }
}

template <typename T>
__global__ void k_synth(T* __restrict__ x, int32_t* __restrict__ labels, StageLayout L, int classes, uint64_t seed,
                        uint32_t iter, uint32_t n0) {
    pdl_wait();
    pdl_trigger();
    const long long total = L.elems();
    const long long per_img = total / L.N;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        int n, c, h, w;
        const bool ok = stage_src(L, i, n, c, h, w);
        const uint32_t ng = n0 + n;
        const uint32_t y = tcp_label(seed, ng, iter, classes);
        if (i % per_img == 0) labels[n] = static_cast<int32_t>(y);
        float v = 0.f;
        if (ok) {
            const uint32_t e = static_cast<uint32_t>((static_cast<long long>(c) * L.H + h) * L.W + w);
            float u1, u2;
            tcp_uniform_pair(seed, ng, iter, e, &u1, &u2);
            const double r = sqrt(-2.0 * log(static_cast<double>(u1)));
            const double t = 6.283185307179586 * static_cast<double>(u2);
            const double z = (e & 1) ? r * sin(t) : r * cos(t);
            v = static_cast<float>(static_cast<double>(tcp_centroid(seed, y, e)) + 0.1 * z);
        }
        x[i] = from_f<T>(v);
    }
}

// bf16 filter shadow [K][RS][cs] (row stride ld) -> K-major bwd-data operand [cs][RS][ks]: one 32 x 32
// (k, c) tile of one filter tap per block, transposed through shared memory (coalesced both ways).
__global__ void __launch_bounds__(256) k_krsc_to_crsk(const bf16* __restrict__ src, int K, int RS, int cs, long long ld,
                                                      bf16* __restrict__ dst, int ks) {
    pdl_wait();
    pdl_trigger();
    __shared__ bf16 tile[32][33];
    const int c0 = blockIdx.x * 32, k0 = blockIdx.y * 32, rs = blockIdx.z;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
    for (int y = 0; y < 32; y += 8) {
        const int k = k0 + ty + y, c = c0 + tx;
        tile[ty + y][tx] = k < K && c < cs ? src[k * ld + static_cast<long long>(rs) * cs + c] : __float2bfloat16(0.f);
    }
    __syncthreads();
#pragma unroll
    for (int y = 0; y < 32; y += 8) {
        const int c = c0 + ty + y, k = k0 + tx;
        if (c < cs && k < K) dst[(static_cast<long long>(c) * RS + rs) * ks + k] = tile[tx][ty + y];
    }
}

__global__ void k_s2d_mask_grad(float* __restrict__ g, int K, long long ld, int Rp, int s, int cs, int R, int S) {
    pdl_wait();
    pdl_trigger();
    const int cols = Rp * Rp * s * s * cs;
    const long long total = static_cast<long long>(K) * cols;
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int col = static_cast<int>(t % cols);
        const int k = static_cast<int>(t / cols);
        const int ab = col / (s * s * cs), ij = (col / cs) % (s * s);
        const int kh = (ab / Rp) * s + ij / s, kw = (ab % Rp) * s + ij % s;
        if (kh >= R || kw >= S) g[k * ld + col] = 0.f;
    }
}

// ---------------------------------------------------------------- fp32 parity mode: bf16 split
// x = hi + mid + lo (hi = bf16(x), mid = bf16(x - hi), lo = bf16(x - hi - mid): 24-bit
// mantissa).  A contraction over fp32 operands runs as one bf16 contraction over kSplitN
// operand copies whose products hi*hi + hi*mid + mid*hi + hi*lo + mid*mid + lo*hi are the
// terms of the fp32 product down to 2^-24; the copies sit side by side along the contraction
// index (channels / columns: SPLIT_COLS) or stacked along it (rows / images: SPLIT_ROWS).
// parts: 2 bits per copy (0 hi, 1 mid, 2 lo).
__device__ __forceinline__ float split_part(float v, int part) {
    const float hi = __bfloat162float(__float2bfloat16_rn(v));
    if (part == 0) return hi;
    const float mid = __bfloat162float(__float2bfloat16_rn(v - hi));
    return part == 1 ? mid : v - hi - mid;
}
// src [rows_src][ld_src] (L used columns, rows >= rows_src read as 0) ->
//   SPLIT_COLS: dst [R][n*L]      dst[r][j*L + e]
//   SPLIT_ROWS: dst [n*R][L]      dst[j*R + r][e]
__global__ void k_splitn(const float* __restrict__ src, long long rows_src, long long ld_src, bf16* __restrict__ dst,
                         long long R, int L, int rows_mode, int n, int parts) {
    pdl_wait();
    pdl_trigger();
    const long long total = n * R * L;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        long long r;
        int j, e;
        if (rows_mode) {
            const long long jr = i / L;
            e = static_cast<int>(i - jr * L);
            j = static_cast<int>(jr / R);
            r = jr - static_cast<long long>(j) * R;
        } else {
            r = i / (static_cast<long long>(n) * L);
            const int je = static_cast<int>(i - r * n * L);
            j = je / L;
            e = je - j * L;
        }
        const float v = r < rows_src ? src[r * ld_src + e] : 0.f;
        dst[i] = __float2bfloat16_rn(split_part(v, (parts >> (2 * j)) & 3));
    }
}
// conv filter p [K][RS][cs] (row stride ld) -> bwd-data operand [RS][n ks][cs]:
//   dst[(rs*n*ks + j*ks + k)*cs + c] = part_j(p[k][rs][c])  (k >= K: 0)
__global__ void k_splitn_rskc(const float* __restrict__ p, long long ld, int K, int RS, int cs, int ks,
                              bf16* __restrict__ dst, int n, int parts) {
    pdl_wait();
    pdl_trigger();
    const long long total = static_cast<long long>(RS) * n * ks * cs;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i % cs);
        const long long q = i / cs;
        const int kk = static_cast<int>(q % (n * ks));
        const int rs = static_cast<int>(q / (n * ks));
        const int j = kk / ks, k = kk - j * ks;
        const float v = k < K ? p[k * ld + static_cast<long long>(rs) * cs + c] : 0.f;
        dst[i] = __float2bfloat16_rn(split_part(v, (parts >> (2 * j)) & 3));
    }
}

// ---------------------------------------------------------------- SGD
__global__ void k_set_iter(uint32_t* d, uint32_t iter, uint32_t n0) {
    pdl_wait();
    pdl_trigger();
    d[0] = iter;
    d[1] = n0;
}

// Multi-tensor momentum SGD: one launch updates a whole gradient bucket.  Work is
// split into 4-element units (float4 p / v / g, 8-byte bf16 shadow stores); unit u
// belongs to the tensor whose prefix range [start4[t], start4[t+1]) holds it.
constexpr int kMaxSgd = 48;
struct SgdBatch {
    SgdTensor t[kMaxSgd];
    long long start4[kMaxSgd + 1];
    int nt;
};

__device__ __forceinline__ void sgd_scalar(const SgdTensor& t, long long i) {
    float np = t.p[i], v = t.v[i];
    if (t.gscale) sgd_update1_scaled(np, v, t.g[i], t.momentum, t.lr_alpha, t.decay, *t.gscale);
    else sgd_update1(np, v, t.g[i], t.momentum, t.lr_alpha, t.decay);
    t.v[i] = v;
    t.p[i] = np;
    const bf16 b = __float2bfloat16_rn(np);
    if (t.shadow) t.shadow[i] = b;
    if (t.shadow_rskc) {
        const int c = static_cast<int>(i % t.cs);
        const long long q = i / t.cs;
        const int rs = static_cast<int>(q % t.RS);
        const int k = static_cast<int>(q / t.RS);
        if (t.rskc_kmajor)
            t.shadow_rskc[(static_cast<long long>(c) * t.RS + rs) * t.ks + k] = b;
        else
            t.shadow_rskc[(static_cast<long long>(rs) * t.ks + k) * t.cs + c] = b;
    }
}

__global__ void __launch_bounds__(256) k_sgd(const __grid_constant__ SgdBatch b) {
    pdl_wait();
    pdl_trigger();
    const long long total = b.start4[b.nt];
    for (long long u = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; u < total;
         u += static_cast<long long>(gridDim.x) * blockDim.x) {
        int lo = 0, hi = b.nt - 1;  // last t with start4[t] <= u
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (b.start4[mid] <= u) lo = mid; else hi = mid - 1;
        }
        const SgdTensor& t = b.t[lo];
        const long long i = (u - b.start4[lo]) * 4;
        if (i + 4 > t.n) {
            for (long long j = i; j < t.n; ++j) sgd_scalar(t, j);
            continue;
        }
        float4 np = *reinterpret_cast<const float4*>(t.p + i);
        const float4 g = __ldcs(reinterpret_cast<const float4*>(t.g + i));
        float4 v = *reinterpret_cast<const float4*>(t.v + i);
        if (t.gscale) {  // global-L2 gradient clipping: g' = scale * (g + decay p)
            const float sc = *t.gscale;
            sgd_update1_scaled(np.x, v.x, g.x, t.momentum, t.lr_alpha, t.decay, sc);
            sgd_update1_scaled(np.y, v.y, g.y, t.momentum, t.lr_alpha, t.decay, sc);
            sgd_update1_scaled(np.z, v.z, g.z, t.momentum, t.lr_alpha, t.decay, sc);
            sgd_update1_scaled(np.w, v.w, g.w, t.momentum, t.lr_alpha, t.decay, sc);
        } else {
            sgd_update1(np.x, v.x, g.x, t.momentum, t.lr_alpha, t.decay);
            sgd_update1(np.y, v.y, g.y, t.momentum, t.lr_alpha, t.decay);
            sgd_update1(np.z, v.z, g.z, t.momentum, t.lr_alpha, t.decay);
            sgd_update1(np.w, v.w, g.w, t.momentum, t.lr_alpha, t.decay);
        }
        *reinterpret_cast<float4*>(t.v + i) = v;
        *reinterpret_cast<float4*>(t.p + i) = np;
        if (t.shadow || t.shadow_rskc) {
            uint2 h;
            h.x = pack_bf16x2(np.x, np.y);
            h.y = pack_bf16x2(np.z, np.w);
            if (t.shadow) *reinterpret_cast<uint2*>(t.shadow + i) = h;
            if (t.shadow_rskc) {  // 4 consecutive channels share (k, rs): cs is a multiple of 8 here
                const unsigned ui = static_cast<unsigned>(i);
                const unsigned c = ui % static_cast<unsigned>(t.cs);
                const unsigned q = ui / static_cast<unsigned>(t.cs);
                const unsigned rs = q % static_cast<unsigned>(t.RS);
                const unsigned k = q / static_cast<unsigned>(t.RS);
                if (t.rskc_kmajor) {  // [c][rs][k]: the 4 channels are RS*ks apart
                    const long long row = static_cast<long long>(t.RS) * t.ks;
                    bf16* d = t.shadow_rskc + static_cast<long long>(c) * row + static_cast<long long>(rs) * t.ks + k;
                    d[0] = __ushort_as_bfloat16(static_cast<unsigned short>(h.x & 0xFFFFu));
                    d[row] = __ushort_as_bfloat16(static_cast<unsigned short>(h.x >> 16));
                    d[2 * row] = __ushort_as_bfloat16(static_cast<unsigned short>(h.y & 0xFFFFu));
                    d[3 * row] = __ushort_as_bfloat16(static_cast<unsigned short>(h.y >> 16));
                } else {
                    *reinterpret_cast<uint2*>(t.shadow_rskc + (static_cast<long long>(rs) * t.ks + k) * t.cs + c) = h;
                }
            }
        }
    }
}

// Global L2 norm of the regularised gradient g' = g + decay * p over every parameter
// (SPEC.md:323, 361 clipping).  Fixed grid-stride partition per launch, fp64 block
// partials in a fixed slot per (launch, block); k_clip_scale sums them in slot order:
// deterministic.
constexpr int kClipBlocks = 148;
__global__ void __launch_bounds__(256) k_sgd_sumsq(const __grid_constant__ SgdBatch b, double* partial) {
    pdl_wait();
    pdl_trigger();
    __shared__ double red[256];
    const long long total = b.start4[b.nt];
    double acc = 0.0;
    for (long long u = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; u < total;
         u += static_cast<long long>(gridDim.x) * blockDim.x) {
        int lo = 0, hi = b.nt - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (b.start4[mid] <= u) lo = mid; else hi = mid - 1;
        }
        const SgdTensor& t = b.t[lo];
        const long long i0 = (u - b.start4[lo]) * 4;
        for (long long i = i0; i < i0 + 4 && i < t.n; ++i) {
            const float gr = __fmaf_rn(t.decay, t.p[i], t.g[i]);
            acc += static_cast<double>(gr) * gr;
        }
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int k = 128; k; k >>= 1) {
        if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}
__global__ void k_clip_scale(const double* partial, int n, float clip, float* scale) {
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x != 0) return;
    double tot = 0.0;
    for (int i = 0; i < n; ++i) tot += partial[i];
    const double norm = sqrt(tot);
    scale[0] = norm > clip ? static_cast<float>(clip / norm) : 1.f;
    scale[1] = static_cast<float>(norm);
}

}  // namespace

// ================================================================ launchers
#define EW_GRID(n) grid_for((n)), kThreads, 0, st

template <typename T>
tc_status launch_relu_fwd(const T* x, T* y, long long n, cudaStream_t st) {
    TCB_LAUNCH(k_relu_fwd<T>, EW_GRID(n / 8), x, y, n / 8);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
template <typename T>
tc_status launch_relu_bwd(const T* dy, const T* y, T* dx, long long n, cudaStream_t st) {
    TCB_LAUNCH(k_relu_bwd<T>, EW_GRID(n / 8), dy, y, dx, n / 8);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
template <typename T>
tc_status launch_add(const T* a, const T* b, T* y, long long n, int relu, cudaStream_t st, const T* relu_y) {
    TCB_LAUNCH(k_add<T>, EW_GRID(n / 8), a, b, y, n / 8, relu, relu_y);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
template <typename T>
tc_status launch_mask_mul(const T* x, const uint8_t* keep, float scale, T* y, long long n, cudaStream_t st,
                          const T* relu_y) {
    TCB_LAUNCH(k_mask_mul<T>, EW_GRID(n / 8), x, reinterpret_cast<const uint2*>(keep), scale, y, n / 8, relu_y);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
template <typename T>
tc_status launch_dropout_apply(const T* x, uint8_t* keep, T* y, int N, int H, int W, int C, int cs, float rate,
                               uint64_t seed, uint32_t var, const uint32_t* iter_n0, cudaStream_t st) {
    if (cs % 8) return fail(TC_INVALID_ARG, "dropout apply: channel stride must be a multiple of 8");
    const long long n = static_cast<long long>(N) * H * W * cs;
    TCB_LAUNCH(k_dropout_apply<T>, EW_GRID(n / 8), x, keep, y, N, H, W, C, cs, rate, 1.f / (1.f - rate), seed, var,
               iter_n0);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
template tc_status launch_dropout_apply<bf16>(const bf16*, uint8_t*, bf16*, int, int, int, int, int, float, uint64_t,
                                              uint32_t, const uint32_t*, cudaStream_t);
template tc_status launch_dropout_apply<float>(const float*, uint8_t*, float*, int, int, int, int, int, float, uint64_t,
                                               uint32_t, const uint32_t*, cudaStream_t);
tc_status launch_dropout_mask(uint8_t* keep, int N, int H, int W, int C, int cs, float rate, uint64_t seed,
                              uint32_t var, const uint32_t* iter_n0, cudaStream_t st) {
    const long long n = static_cast<long long>(N) * H * W * cs;
    TCB_LAUNCH(k_dropout_mask, EW_GRID(n), keep, N, H, W, C, cs, rate, seed, var, iter_n0);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
// TCB_FIXED_POOL=0 routes every pooling through the generic runtime-window kernels (A/B switch).
long long patch_threads(const Act4& xi, int pad, int S) {
    return static_cast<long long>(xi.N) * ((xi.H + pad + S - 1) / S) * ((xi.W + pad + S - 1) / S) * (xi.cs / 8);
}
// Rows per strip of the stride-1 3x3 max-pool kernels: TCB_POOL_STRIP = 4 | 8 (default),
// 0 = one thread per pixel (A/B)
static int pool_strip() {
    const char* e = std::getenv("TCB_POOL_STRIP");
    const int v = e ? std::atoi(e) : 8;
    return v == 0 || v == 4 ? v : 8;
}
bool fixed_pool_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("TCB_FIXED_POOL");
        return !(e && e[0] == '0');
    }();
    return on;
}
template <typename T>
tc_status launch_pool_fwd(const T* x, Act4 xi, T* y, Act4 yo, uint8_t* idx, int k, int stride, int pad, int is_max,
                          int flag_nonpos, cudaStream_t st) {
    if (idx && k * k > 255) return fail(TC_INVALID_ARG, "max pooling: window too large for 1-byte argmax");
    if (flag_nonpos && k * k > 127) return fail(TC_INVALID_ARG, "max pooling: window too large for a flagged argmax");
    const long long n = yo.pixels() * (xi.cs / 8);
    if constexpr (std::is_same<T, bf16>::value) {
        if (is_max && n < (1ll << 31) && fixed_pool_enabled()) {
            if (k == 3 && stride == 2) {
                TCB_LAUNCH((k_maxpool_fwd_bf16<int, 3, 2>), EW_GRID(n), x, xi, y, yo, idx, pad, flag_nonpos);
                TCB_LAUNCH_CHECK();
                return TC_OK;
            }
            if (k == 2 && stride == 2) {
                TCB_LAUNCH((k_maxpool_fwd_bf16<int, 2, 2>), EW_GRID(n), x, xi, y, yo, idx, pad, flag_nonpos);
                TCB_LAUNCH_CHECK();
                return TC_OK;
            }
            if (k == 3 && stride == 1) {
                if (const int R = pool_strip()) {
                    const long long th = static_cast<long long>(yo.N) * ((yo.H + R - 1) / R) * yo.W * (xi.cs / 8);
                    const int blocks = static_cast<int>((th + 255) / 256);
                    if (R == 4) TCB_LAUNCH((k_maxpool_fwd_strip<3, 4>), blocks, 256, 0, st, x, xi, y, yo, idx, pad, flag_nonpos);
                    else TCB_LAUNCH((k_maxpool_fwd_strip<3, 8>), blocks, 256, 0, st, x, xi, y, yo, idx, pad, flag_nonpos);
                } else {
                    TCB_LAUNCH((k_maxpool_fwd_bf16<int, 3, 1>), EW_GRID(n), x, xi, y, yo, idx, pad, flag_nonpos);
                }
                TCB_LAUNCH_CHECK();
                return TC_OK;
            }
        }
    }
    if (n < (1ll << 31))
        TCB_LAUNCH((k_pool_fwd<T, int>), EW_GRID(n), x, xi, y, yo, idx, k, stride, pad, is_max, flag_nonpos);
    else
        TCB_LAUNCH((k_pool_fwd<T, long long>), EW_GRID(n), x, xi, y, yo, idx, k, stride, pad, is_max, flag_nonpos);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
template <typename T>
tc_status launch_pool_bwd(const T* dy, Act4 yo, const uint8_t* idx, T* dx, Act4 xi, int k, int stride, int pad,
                          int is_max, const T* relu_y, cudaStream_t st) {
    const long long n = xi.pixels() * (xi.cs / 8);
    if (is_max && n < (1ll << 31) && fixed_pool_enabled()) {
        if (k == 3 && stride == 2) {
            TCB_LAUNCH((k_maxpool_bwd_patch<T, 3, 2>), EW_GRID(patch_threads(xi, pad, 2)), dy, yo, idx, dx, xi, pad, relu_y);
            TCB_LAUNCH_CHECK();
            return TC_OK;
        }
        if (k == 2 && stride == 2) {
            TCB_LAUNCH((k_maxpool_bwd_patch<T, 2, 2>), EW_GRID(patch_threads(xi, pad, 2)), dy, yo, idx, dx, xi, pad, relu_y);
            TCB_LAUNCH_CHECK();
            return TC_OK;
        }
        if (k == 3 && stride == 1) {
            if (const int R = pool_strip()) {
                const long long th = static_cast<long long>(xi.N) * ((xi.H + R - 1) / R) * xi.W * (xi.cs / 8);
                const int blocks = static_cast<int>((th + 255) / 256);
                if (R == 4) TCB_LAUNCH((k_maxpool_bwd_strip<T, 3, 4>), blocks, 256, 0, st, dy, yo, idx, dx, xi, pad, relu_y);
                else TCB_LAUNCH((k_maxpool_bwd_strip<T, 3, 8>), blocks, 256, 0, st, dy, yo, idx, dx, xi, pad, relu_y);
            } else {
                TCB_LAUNCH((k_maxpool_bwd_patch<T, 3, 1>), EW_GRID(patch_threads(xi, pad, 1)), dy, yo, idx, dx, xi, pad,
                           relu_y);
            }
            TCB_LAUNCH_CHECK();
            return TC_OK;
        }
    }
    if (n < (1ll << 31))
        TCB_LAUNCH((k_pool_bwd<T, int>), EW_GRID(n), dy, yo, idx, dx, xi, k, stride, pad, is_max, relu_y);
    else
        TCB_LAUNCH((k_pool_bwd<T, long long>), EW_GRID(n), dy, yo, idx, dx, xi, k, stride, pad, is_max, relu_y);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
// TCB_LRN3: 0 = v2 (neighbour-load) kernels only, 1 (default) = v3 backward where lanes tile
// pixels exactly, 2 = v3 everywhere (A/B switch).
int lrn3_mode() {
    static const int m = [] {
        const char* e = std::getenv("TCB_LRN3");
        return e ? std::atoi(e) : 1;
    }();
    return m;
}
// two chunks per thread (k_lrn2x_*): bf16, windows 3 / 5, an even chunk count; TCB_LRN2X=0: v2 (A/B)
static bool lrn2x_ok(const Act4& a, int size) {
    const char* e = std::getenv("TCB_LRN2X");
    return !(e && e[0] == '0') && (size == 3 || size == 5) && a.cs % 16 == 0;
}
template <typename T>
tc_status launch_lrn_fwd(const T* x, T* y, Act4 a, int size, float alpha, float beta, float k, cudaStream_t st) {
    const long long n = a.pixels() * (a.cs / 8);
    // measured (AlexNet b128): the v3 forward is no faster than v2 for 32 % ng == 0 and 16% slower
    // with idle lanes, so it is opt-in (TCB_LRN3=2)
    if (a.cs / 8 <= 32 && lrn3_mode() == 2) {
        const long long threads = (a.pixels() + 32 / (a.cs / 8) - 1) / (32 / (a.cs / 8)) * 32;
        bool done = true;
        switch (size) {
            case 3: TCB_LAUNCH((k_lrn3_fwd<1, T>), EW_GRID(threads), x, y, a, alpha, beta, k); break;
            case 5: TCB_LAUNCH((k_lrn3_fwd<2, T>), EW_GRID(threads), x, y, a, alpha, beta, k); break;
            case 7: TCB_LAUNCH((k_lrn3_fwd<3, T>), EW_GRID(threads), x, y, a, alpha, beta, k); break;
            case 9: TCB_LAUNCH((k_lrn3_fwd<4, T>), EW_GRID(threads), x, y, a, alpha, beta, k); break;
            default: done = false;
        }
        if (done) {
            TCB_LAUNCH_CHECK();
            return TC_OK;
        }
    }
    if constexpr (sizeof(T) == 2) {
        if (lrn2x_ok(a, size)) {
            const long long n2 = n / 2;
            if (size == 3) TCB_LAUNCH((k_lrn2x_fwd<1, long long>), EW_GRID(n2), x, y, a, alpha, beta, k);
            else TCB_LAUNCH((k_lrn2x_fwd<2, long long>), EW_GRID(n2), x, y, a, alpha, beta, k);
            TCB_LAUNCH_CHECK();
            return TC_OK;
        }
    }
    switch (size) {  // odd windows up to 9: register-resident template kernels
        case 3: if (n < (1ll << 31)) TCB_LAUNCH((k_lrn2_fwd<1, T, int>), EW_GRID(n), x, y, a, alpha, beta, k); else TCB_LAUNCH((k_lrn2_fwd<1, T, long long>), EW_GRID(n), x, y, a, alpha, beta, k); break;
        case 5: if (n < (1ll << 31)) TCB_LAUNCH((k_lrn2_fwd<2, T, int>), EW_GRID(n), x, y, a, alpha, beta, k); else TCB_LAUNCH((k_lrn2_fwd<2, T, long long>), EW_GRID(n), x, y, a, alpha, beta, k); break;
        case 7: if (n < (1ll << 31)) TCB_LAUNCH((k_lrn2_fwd<3, T, int>), EW_GRID(n), x, y, a, alpha, beta, k); else TCB_LAUNCH((k_lrn2_fwd<3, T, long long>), EW_GRID(n), x, y, a, alpha, beta, k); break;
        case 9: if (n < (1ll << 31)) TCB_LAUNCH((k_lrn2_fwd<4, T, int>), EW_GRID(n), x, y, a, alpha, beta, k); else TCB_LAUNCH((k_lrn2_fwd<4, T, long long>), EW_GRID(n), x, y, a, alpha, beta, k); break;
        default: {  // general path: warp per pixel with the channel vector in shared memory
            const int warps = 8;
            TCB_LAUNCH(k_lrn_fwd<T>, grid_for(a.pixels(), warps), warps * 32, warps * a.cs * sizeof(float), st, x, y, a, size,
                                                                                                     alpha, beta, k);
        }
    }
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
template <typename T>
tc_status launch_lrn_bwd(const T* dy, const T* x, const T* y, T* dx, Act4 a, int size, float alpha, float beta,
                         float k, int relu, cudaStream_t st) {
    const long long n = a.pixels() * (a.cs / 8);
    // v3 backward when the pixel's chunks tile the warp exactly (no idle lanes): -7% vs v2 at C=256
    if (a.cs / 8 <= 32 && (lrn3_mode() == 2 || (lrn3_mode() == 1 && 32 % (a.cs / 8) == 0))) {
        const long long threads = (a.pixels() + 32 / (a.cs / 8) - 1) / (32 / (a.cs / 8)) * 32;
        bool done = true;
        switch (size) {
            case 3: TCB_LAUNCH((k_lrn3_bwd<1, T>), EW_GRID(threads), dy, x, y, dx, a, alpha, beta, k, relu); break;
            case 5: TCB_LAUNCH((k_lrn3_bwd<2, T>), EW_GRID(threads), dy, x, y, dx, a, alpha, beta, k, relu); break;
            case 7: TCB_LAUNCH((k_lrn3_bwd<3, T>), EW_GRID(threads), dy, x, y, dx, a, alpha, beta, k, relu); break;
            case 9: TCB_LAUNCH((k_lrn3_bwd<4, T>), EW_GRID(threads), dy, x, y, dx, a, alpha, beta, k, relu); break;
            default: done = false;
        }
        if (done) {
            TCB_LAUNCH_CHECK();
            return TC_OK;
        }
    }
    if constexpr (sizeof(T) == 2) {
        if (lrn2x_ok(a, size)) {
            const long long n2 = n / 2;
            if (size == 3) TCB_LAUNCH((k_lrn2x_bwd<1, long long>), EW_GRID(n2), dy, x, y, dx, a, alpha, beta, k, relu);
            else TCB_LAUNCH((k_lrn2x_bwd<2, long long>), EW_GRID(n2), dy, x, y, dx, a, alpha, beta, k, relu);
            TCB_LAUNCH_CHECK();
            return TC_OK;
        }
    }
    switch (size) {
        case 3: if (n < (1ll << 31)) TCB_LAUNCH((k_lrn2_bwd<1, T, int>), EW_GRID(n), dy, x, y, dx, a, alpha, beta, k, relu); else TCB_LAUNCH((k_lrn2_bwd<1, T, long long>), EW_GRID(n), dy, x, y, dx, a, alpha, beta, k, relu); break;
        case 5: if (n < (1ll << 31)) TCB_LAUNCH((k_lrn2_bwd<2, T, int>), EW_GRID(n), dy, x, y, dx, a, alpha, beta, k, relu); else TCB_LAUNCH((k_lrn2_bwd<2, T, long long>), EW_GRID(n), dy, x, y, dx, a, alpha, beta, k, relu); break;
        case 7: if (n < (1ll << 31)) TCB_LAUNCH((k_lrn2_bwd<3, T, int>), EW_GRID(n), dy, x, y, dx, a, alpha, beta, k, relu); else TCB_LAUNCH((k_lrn2_bwd<3, T, long long>), EW_GRID(n), dy, x, y, dx, a, alpha, beta, k, relu); break;
        case 9: if (n < (1ll << 31)) TCB_LAUNCH((k_lrn2_bwd<4, T, int>), EW_GRID(n), dy, x, y, dx, a, alpha, beta, k, relu); else TCB_LAUNCH((k_lrn2_bwd<4, T, long long>), EW_GRID(n), dy, x, y, dx, a, alpha, beta, k, relu); break;
        default: {
            const int warps = 8;
            TCB_LAUNCH(k_lrn_bwd<T>, grid_for(a.pixels(), warps), warps * 32, warps * 3 * a.cs * sizeof(float), st, 
                dy, x, y, dx, a, size, alpha, beta, k, relu);
        }
    }
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
template <typename T>
tc_status launch_softmax_fwd(const T* x, long long in_ld, float* y, int rows, int F, cudaStream_t st) {
    TCB_LAUNCH(k_softmax_fwd<T>, grid_for(rows, 8), 256, 0, st, x, in_ld, y, rows, F);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
template <typename T>
tc_status launch_softmax_bwd(const float* dy, const float* y, T* dx, long long out_ld, int rows, int F,
                             cudaStream_t st) {
    TCB_LAUNCH(k_softmax_bwd<T>, grid_for(rows, 8), 256, 0, st, dy, y, dx, out_ld, rows, F);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
template <typename T>
tc_status launch_softmax_xent(const T* z, long long ld, const int32_t* labels, float c, float* L, float* Y, T* dz,
                              int rows, int F, cudaStream_t st) {
    // one warp per block: every row's warp on its own SM (the head is latency-bound: 128 rows of
    // 1000 classes on 16 blocks of 8 warps measured 15.9 us)
    TCB_LAUNCH(k_softmax_xent<T>, rows, 32, 0, st, z, ld, labels, c, L, Y, dz, rows, F);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
template tc_status launch_softmax_xent<bf16>(const bf16*, long long, const int32_t*, float, float*, float*, bf16*, int,
                                             int, cudaStream_t);
template tc_status launch_softmax_xent<float>(const float*, long long, const int32_t*, float, float*, float*, float*,
                                              int, int, cudaStream_t);
tc_status launch_f32_ew(int op, const float* a, const float* b, float scale, float* y, long long n, cudaStream_t st) {
    TCB_LAUNCH(k_f32_ew, EW_GRID(n), op, a, b, scale, y, n);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
template <typename T>
tc_status launch_argmax_hits(const T* logits, long long ld, int N, int C, const int32_t* labels, unsigned* hits,
                             cudaStream_t st) {
    TCB_CUDA_CHECK(cudaMemsetAsync(hits, 0, sizeof(unsigned), st));
    TCB_LAUNCH(k_argmax_hits<T>, (N + 7) / 8, 256, 0, st, logits, ld, N, C, labels, hits);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
template tc_status launch_argmax_hits<bf16>(const bf16*, long long, int, int, const int32_t*, unsigned*, cudaStream_t);
template tc_status launch_argmax_hits<float>(const float*, long long, int, int, const int32_t*, unsigned*, cudaStream_t);
tc_status launch_onehot(const int32_t* labels, float* y, int N, int K, cudaStream_t st) {
    TCB_LAUNCH(k_onehot, EW_GRID(static_cast<long long>(N) * K), labels, y, N, K);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_loss(const float* const* a, const float* const* b, const long long* n, const double* coef, int nterms,
                      float* out, cudaStream_t st) {
    if (nterms < 1 || nterms > 4) return fail(TC_INVALID_ARG, "loss: 1..4 terms");
    LossArgs args{};
    args.nterms = nterms;
    for (int t = 0; t < nterms; ++t) {
        args.a[t] = a[t];
        args.b[t] = b[t];
        args.n[t] = n[t];
        args.coef[t] = coef[t];
    }
    // out[0] = loss; out + 16 holds kLossBlocks fp64 partials, then the ticket counter (zero-initialised)
    double* partial = reinterpret_cast<double*>(out + 16);
    unsigned* ticket = reinterpret_cast<unsigned*>(partial + kLossBlocks);
    TCB_LAUNCH(k_loss, kLossBlocks, 256, 0, st, args, out, partial, ticket);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
size_t colsum_partials_floats(int cols) {
    // 2 accumulators x splits x C, with splits * tiles <= 4 * SMs and ct >= min(C, 512)
    const int ld = std::max(8, (cols + 7) / 8 * 8);
    const int tiles = (ld + 511) / 512;
    const size_t n = 2ull * (static_cast<size_t>(num_sms()) * 4 / tiles + 1) * ld + 3ull * ld + 64;
    return (n + 63) / 64 * 64;  // keeps the coefficient area behind the partials 16-byte aligned
}

template <int MODE, typename T>
static tc_status chan_reduce(const T* x, const T* x2, const float* stats, long long rows, int C, long long ld,
                             float* part, int max_partials, cudaStream_t st, RedPlan* out_plan) {
    if ((ld & 7) || (reinterpret_cast<uintptr_t>(x) & 15) || (x2 && (reinterpret_cast<uintptr_t>(x2) & 15)))
        return fail(TC_INVALID_ARG, "channel reduction: misaligned operand");
    static const int max_clusters = [] {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(1, kRedCluster * 64);
        cfg.blockDim = dim3(kRedThreads);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 1;
        attr[0].val.clusterDim.y = kRedCluster;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k_chan_reduce<MODE, T>, &cfg) != cudaSuccess || n <= 0) {
            cudaGetLastError();
            n = num_sms() * kRedBlocksPerSm / kRedCluster * 7 / 8;
        }
        return n;
    }();
    RedPlan rp = red_plan(rows, static_cast<int>(ld), max_clusters);
    if (2ll * rp.parts * C > max_partials) return fail(TC_INTERNAL, "channel reduction: scratch too small");
    dim3 grid(rp.tiles, rp.splits);
    TCB_CUDA_CHECK(launch_kernel_cluster((k_chan_reduce<MODE, T>), grid, dim3(kRedThreads), 0, st, dim3(1, kRedCluster, 1),
                                         x, x2, stats, rows, C, static_cast<int>(ld), rp.ct, rp.rps, rp.splits, part));
    TCB_LAUNCH_CHECK();
    *out_plan = rp;
    return TC_OK;
}

template <typename T>
tc_status launch_colsum(const T* x, long long rows, int cols, long long ld, float* out, float* partials,
                        int max_partials, cudaStream_t st) {
    RedPlan rp;
    tc_status s = chan_reduce<RED_SUM, T>(x, nullptr, nullptr, rows, cols, ld, partials, max_partials, st, &rp);
    if (s != TC_OK) return s;
    TCB_LAUNCH((k_chan_final<RED_SUM, T>), (cols + 7) / 8, 256, 0, st, partials, rp.parts, cols, 1.f, out,
               static_cast<const T*>(nullptr), rows, 0.f,
                                                               nullptr, nullptr, nullptr);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
template <typename T>
tc_status launch_bias_add(const T* x, const float* b, T* y, long long rows, int cols, long long ld, int relu,
                          cudaStream_t st) {
    TCB_LAUNCH(k_bias_add<T>, EW_GRID(rows * ld), x, b, y, rows, cols, ld, relu);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
template <typename T>
tc_status launch_channel_copy(const T* src, int src_cs, T* dst, int dst_cs, int off, int c, long long pixels,
                              cudaStream_t st, const T* relu_y) {
    if ((src_cs | dst_cs | off | c) % 8 == 0 && (reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) % 16 == 0) {
        TCB_LAUNCH(k_channel_copy8<T>, EW_GRID(pixels * (c / 8)), src, src_cs, dst, dst_cs, off, c / 8, pixels, relu_y);
        TCB_LAUNCH_CHECK();
        return TC_OK;
    }
    if (relu_y) return fail(TC_INTERNAL, "channel copy: folded ReLU backward needs 8-channel alignment");
    TCB_LAUNCH(k_channel_copy<T>, EW_GRID(pixels * c), src, src_cs, dst, dst_cs, off, c, pixels);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_zero(void* p, size_t bytes, cudaStream_t st) {
    TCB_CUDA_CHECK(cudaMemsetAsync(p, 0, bytes, st));
    return TC_OK;
}

template <typename T>
tc_status launch_bn_fwd(const T* x, const float* gamma, const float* beta, T* y, float* stats, long long pixels, int C,
                        int cs, float eps, int relu, const T* res, float* partials, int max_partials, cudaStream_t st) {
    RedPlan rp;
    float* coef = partials + max_partials;  // caller sizes partials to max_partials + 3*C
    tc_status s = chan_reduce<RED_STATS, T>(x, nullptr, nullptr, pixels, C, cs, partials, max_partials, st, &rp);
    if (s != TC_OK) return s;
    TCB_LAUNCH((k_chan_final<RED_STATS, T>), (C + 7) / 8, 256, 0, st, partials, rp.parts, C, 1.f, stats, x, pixels, eps, gamma,
                                                              beta, coef);
    TCB_LAUNCH_CHECK();
    const long long n8 = pixels * cs / 8;
    TCB_LAUNCH(k_chan_affine<T>, EW_GRID(n8), x, coef, y, n8, cs / 8, C, relu, res);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}

template <typename T>
tc_status launch_bn_bwd_reduce(const T* dy, const T* x, const float* gamma, const float* stats, float* sums,
                               long long pixels, int C, int cs, float* partials, int max_partials, cudaStream_t st) {
    RedPlan rp;
    tc_status s = chan_reduce<RED_BNBWD, T>(dy, x, stats, pixels, C, cs, partials, max_partials, st, &rp);
    if (s != TC_OK) return s;
    TCB_LAUNCH((k_chan_final<RED_BNBWD, T>), (C + 7) / 8, 256, 0, st, partials, rp.parts, C,
               1.f / static_cast<float>(pixels), sums, static_cast<const T*>(nullptr), pixels, 0.f, gamma, stats,
               static_cast<float*>(nullptr));
    TCB_LAUNCH_CHECK();
    return TC_OK;
}

template <typename T>
tc_status launch_bn_bwd_apply(const T* dy, const T* x, const float* k, T* dx, long long pixels, int C, int cs,
                              cudaStream_t st) {
    const long long n8 = pixels * cs / 8;
    TCB_LAUNCH(k_bn_bwd_apply<T>, EW_GRID(n8), dy, x, k, dx, n8, cs / 8, C);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}

template <typename T, typename SRC>
tc_status launch_nchw_to_nhwc(const SRC* x, T* y, StageLayout L, cudaStream_t st) {
    const int s = L.s2d ? L.s2d : 1;
    if constexpr (std::is_same_v<SRC, float>) {
        const char* e = std::getenv("TCB_STAGE_DIRECT");  // 0: the row-tiled kernel (A/B)
        const int ls = (s & (s - 1)) == 0 ? __builtin_ctz(static_cast<unsigned>(s)) : -1;
        if (!(e && e[0] == '0') && L.cs == 4 && L.C <= 4 && ls >= 0 && (L.s2d || L.W % 2 == 0)) {
            const long long chunks = L.elems() / 8;
            TCB_LAUNCH((k_stage_direct<T>), static_cast<int>(std::min<long long>((chunks + 255) / 256, num_sms() * 16LL)),
                       256, 0, st, static_cast<const float*>(x), y, L, ls);
            TCB_LAUNCH_CHECK();
            return TC_OK;
        }
    }
    const size_t smem = static_cast<size_t>(L.C) * s * L.W * sizeof(float);
    const int wout = L.s2d ? L.Ws : L.W;
    auto log2i = [](int v) { int l = 0; while ((1 << l) < v) ++l; return (1 << l) == v ? l : -1; };
    const int lcs = log2i(L.cs), ls = log2i(s);
    if (smem <= 48 * 1024 && lcs >= 0 && ls >= 0 && (static_cast<long long>(wout) * s * s * L.cs) % 8 == 0 &&
        (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
        TCB_LAUNCH((k_stage_rows<T, SRC>), L.N * (L.s2d ? L.Hs : L.H), 256, smem, st, x, y, L, lcs, ls);
        TCB_LAUNCH_CHECK();
        return TC_OK;
    }
    TCB_LAUNCH((k_nchw_to_nhwc<T, SRC>), EW_GRID(L.elems()), x, y, L);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
template <typename T>
tc_status launch_synth_batch(T* x, int32_t* labels, StageLayout L, int classes, uint64_t seed, uint32_t iter,
                             uint32_t n0, cudaStream_t st) {
    TCB_LAUNCH(k_synth<T>, EW_GRID(L.elems()), x, labels, L, classes, seed, iter, n0);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_krsc_to_crsk(const bf16* src, int K, int RS, int cs, long long ld, bf16* dst, int ks, cudaStream_t st) {
    LowPriorityScope low;  // runs beside the update on the side stream
    TCB_LAUNCH(k_krsc_to_crsk, dim3(ceil_div(cs, 32), ceil_div(K, 32), RS), 256, 0, st, src, K, RS, cs, ld, dst, ks);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_s2d_mask_grad(float* g, int K, long long ld, int Rp, int s, int cs, int R, int S, cudaStream_t st) {
    TCB_LAUNCH(k_s2d_mask_grad, EW_GRID(static_cast<long long>(K) * Rp * Rp * s * s * cs), g, K, ld, Rp, s, cs, R, S);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_sgd(const SgdTensor* ts, int nt, SgdTensor*, cudaStream_t st) {
    LowPriorityScope low;  // yields SMs to the step's kernels (see launch_priority)
    for (int base = 0; base < nt; base += kMaxSgd) {
        SgdBatch b;
        b.nt = std::min(kMaxSgd, nt - base);
        b.start4[0] = 0;
        for (int i = 0; i < b.nt; ++i) {
            const SgdTensor& t = ts[base + i];
            if ((reinterpret_cast<uintptr_t>(t.p) | reinterpret_cast<uintptr_t>(t.v) | reinterpret_cast<uintptr_t>(t.g)) & 15)
                return fail(TC_INVALID_ARG, "sgd: p / v / g must be 16-byte aligned");
            if (t.shadow_rskc && (t.cs % 4 || t.n >= (1ll << 31)))
                return fail(TC_INVALID_ARG, "sgd: RSKC shadow needs cs % 4 == 0 and n < 2^31");
            b.t[i] = t;
            b.start4[i + 1] = b.start4[i] + (t.n + 3) / 4;
        }
        // TCB_SGD_SHORT=1: one 4-element unit per thread (many short blocks the scheduler can
        // interleave with step kernels) instead of a grid-stride grid of SMs x 32 blocks
        static const bool short_blocks = [] {
            const char* e = std::getenv("TCB_SGD_SHORT");
            return e && e[0] == '1';
        }();
        const long long units = b.start4[b.nt];
        const int blocks = short_blocks ? static_cast<int>(std::min<long long>((units + kThreads - 1) / kThreads, 1ll << 30))
                                        : grid_for(units);
        TCB_LAUNCH(k_sgd, blocks, kThreads, 0, st, b);
        TCB_LAUNCH_CHECK();
    }
    return TC_OK;
}

tc_status launch_clip_scale(const SgdTensor* ts, int nt, float clip, double* partials, float* scale, cudaStream_t st) {
    int launches = 0;
    for (int base = 0; base < nt; base += kMaxSgd, ++launches) {
        SgdBatch b;
        b.nt = std::min(kMaxSgd, nt - base);
        b.start4[0] = 0;
        for (int i = 0; i < b.nt; ++i) {
            b.t[i] = ts[base + i];
            b.start4[i + 1] = b.start4[i] + (b.t[i].n + 3) / 4;
        }
        TCB_LAUNCH(k_sgd_sumsq, kClipBlocks, kThreads, 0, st, b, partials + static_cast<long long>(launches) * kClipBlocks);
        TCB_LAUNCH_CHECK();
    }
    TCB_LAUNCH(k_clip_scale, 1, 32, 0, st, partials, launches * kClipBlocks, clip, scale);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
size_t clip_partials_doubles(int nt) { return static_cast<size_t>((nt + kMaxSgd - 1) / kMaxSgd + 1) * kClipBlocks; }

tc_status launch_set_iter(uint32_t* d_iter, uint32_t iter, uint32_t n0, cudaStream_t st) {
    TCB_LAUNCH(k_set_iter, 1, 1, 0, st, d_iter, iter, n0);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}

tc_status launch_split(const float* src, long long rows_src, long long ld_src, bf16* dst, long long R, int L,
                       int rows_mode, int parts, cudaStream_t st) {
    TCB_LAUNCH(k_splitn, EW_GRID(kSplitN * R * L), src, rows_src, ld_src, dst, R, L, rows_mode, kSplitN, parts);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_split_rskc(const float* p, long long ld, int K, int RS, int cs, int ks, bf16* dst, int parts,
                            cudaStream_t st) {
    TCB_LAUNCH(k_splitn_rskc, EW_GRID(static_cast<long long>(RS) * kSplitN * ks * cs), p, ld, K, RS, cs, ks, dst, kSplitN,
               parts);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}

// storage types: bf16 (default) and fp32 (parity precision mode)
template tc_status launch_relu_fwd<bf16>(const bf16*, bf16*, long long, cudaStream_t);
template tc_status launch_relu_bwd<bf16>(const bf16*, const bf16*, bf16*, long long, cudaStream_t);
template tc_status launch_add<bf16>(const bf16*, const bf16*, bf16*, long long, int, cudaStream_t, const bf16*);
template tc_status launch_mask_mul<bf16>(const bf16*, const uint8_t*, float, bf16*, long long, cudaStream_t, const bf16*);
template tc_status launch_pool_fwd<bf16>(const bf16*, Act4, bf16*, Act4, uint8_t*, int, int, int, int, int, cudaStream_t);
template tc_status launch_pool_bwd<bf16>(const bf16*, Act4, const uint8_t*, bf16*, Act4, int, int, int, int,
                                         const bf16*, cudaStream_t);
template tc_status launch_lrn_fwd<bf16>(const bf16*, bf16*, Act4, int, float, float, float, cudaStream_t);
template tc_status launch_lrn_bwd<bf16>(const bf16*, const bf16*, const bf16*, bf16*, Act4, int, float, float, float,
                                        int, cudaStream_t);
template tc_status launch_softmax_fwd<bf16>(const bf16*, long long, float*, int, int, cudaStream_t);
template tc_status launch_softmax_bwd<bf16>(const float*, const float*, bf16*, long long, int, int, cudaStream_t);
template tc_status launch_colsum<bf16>(const bf16*, long long, int, long long, float*, float*, int, cudaStream_t);
template tc_status launch_bias_add<bf16>(const bf16*, const float*, bf16*, long long, int, long long, int, cudaStream_t);
template tc_status launch_channel_copy<bf16>(const bf16*, int, bf16*, int, int, int, long long, cudaStream_t, const bf16*);
template tc_status launch_bn_fwd<bf16>(const bf16*, const float*, const float*, bf16*, float*, long long, int, int, float, int, const bf16*,
                                     float*, int, cudaStream_t);
template tc_status launch_bn_bwd_reduce<bf16>(const bf16*, const bf16*, const float*, const float*, float*, long long,
                                            int, int, float*, int, cudaStream_t);
template tc_status launch_bn_bwd_apply<bf16>(const bf16*, const bf16*, const float*, bf16*, long long, int, int,
                                           cudaStream_t);
template tc_status launch_nchw_to_nhwc<bf16, float>(const float*, bf16*, StageLayout, cudaStream_t);
template tc_status launch_nchw_to_nhwc<bf16, bf16>(const bf16*, bf16*, StageLayout, cudaStream_t);
template tc_status launch_synth_batch<bf16>(bf16*, int32_t*, StageLayout, int, uint64_t, uint32_t, uint32_t, cudaStream_t);
template tc_status launch_relu_fwd<float>(const float*, float*, long long, cudaStream_t);
template tc_status launch_relu_bwd<float>(const float*, const float*, float*, long long, cudaStream_t);
template tc_status launch_add<float>(const float*, const float*, float*, long long, int, cudaStream_t, const float*);
template tc_status launch_mask_mul<float>(const float*, const uint8_t*, float, float*, long long, cudaStream_t, const float*);
template tc_status launch_pool_fwd<float>(const float*, Act4, float*, Act4, uint8_t*, int, int, int, int, int, cudaStream_t);
template tc_status launch_pool_bwd<float>(const float*, Act4, const uint8_t*, float*, Act4, int, int, int, int,
                                         const float*, cudaStream_t);
template tc_status launch_lrn_fwd<float>(const float*, float*, Act4, int, float, float, float, cudaStream_t);
template tc_status launch_lrn_bwd<float>(const float*, const float*, const float*, float*, Act4, int, float, float, float,
                                        int, cudaStream_t);
template tc_status launch_softmax_fwd<float>(const float*, long long, float*, int, int, cudaStream_t);
template tc_status launch_softmax_bwd<float>(const float*, const float*, float*, long long, int, int, cudaStream_t);
template tc_status launch_colsum<float>(const float*, long long, int, long long, float*, float*, int, cudaStream_t);
template tc_status launch_bias_add<float>(const float*, const float*, float*, long long, int, long long, int, cudaStream_t);
template tc_status launch_channel_copy<float>(const float*, int, float*, int, int, int, long long, cudaStream_t, const float*);
template tc_status launch_bn_fwd<float>(const float*, const float*, const float*, float*, float*, long long, int, int, float, int, const float*,
                                     float*, int, cudaStream_t);
template tc_status launch_bn_bwd_reduce<float>(const float*, const float*, const float*, const float*, float*, long long,
                                            int, int, float*, int, cudaStream_t);
template tc_status launch_bn_bwd_apply<float>(const float*, const float*, const float*, float*, long long, int, int,
                                           cudaStream_t);
template tc_status launch_nchw_to_nhwc<float, float>(const float*, float*, StageLayout, cudaStream_t);
template tc_status launch_synth_batch<float>(float*, int32_t*, StageLayout, int, uint64_t, uint32_t, uint32_t, cudaStream_t);

}  // namespace tcb
