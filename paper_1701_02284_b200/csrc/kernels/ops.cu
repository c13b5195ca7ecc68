// Bandwidth-bound kernels of the training step.  See ops.cuh for layouts.
#include <algorithm>
#include <cmath>

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

// ---------------------------------------------------------------- elementwise (8 x bf16 per thread)
__global__ void k_relu_fwd(const uint4* __restrict__ x, uint4* __restrict__ y, long long n8) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n8;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        float f[8];
        unpack8(x[i], f);
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = fmaxf(f[j], 0.f);
        y[i] = pack8(f);
    }
}

__global__ void k_relu_bwd(const uint4* __restrict__ dy, const uint4* __restrict__ y, uint4* __restrict__ dx,
                           long long n8) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n8;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        float g[8], f[8];
        unpack8(dy[i], g);
        unpack8(y[i], f);
#pragma unroll
        for (int j = 0; j < 8; ++j) g[j] = f[j] > 0.f ? g[j] : 0.f;
        dx[i] = pack8(g);
    }
}

__global__ void k_add(const uint4* __restrict__ a, const uint4* __restrict__ b, uint4* __restrict__ y, long long n8) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n8;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        float p[8], q[8];
        unpack8(a[i], p);
        unpack8(b[i], q);
#pragma unroll
        for (int j = 0; j < 8; ++j) p[j] += q[j];
        y[i] = pack8(p);
    }
}

__global__ void k_mask_mul(const uint4* __restrict__ x, const uint2* __restrict__ keep, float scale,
                           uint4* __restrict__ y, long long n8) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n8;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        float f[8];
        unpack8(x[i], f);
        const uint2 m = keep[i];
        const uint8_t* mb = reinterpret_cast<const uint8_t*>(&m);
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = mb[j] ? f[j] * scale : 0.f;
        y[i] = pack8(f);
    }
}

// keep mask for every stored element of an NHWC (or [N][Fs] with H=W=1) tensor.
__global__ void k_dropout_mask(uint8_t* __restrict__ keep, int N, int H, int W, int C, int cs, float rate,
                               uint64_t seed, uint32_t var, const uint32_t* iter_n0) {
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
__global__ void k_pool_fwd(const bf16* __restrict__ x, Act4 xi, bf16* __restrict__ y, Act4 yo,
                           int32_t* __restrict__ idx, int k, int stride, int pad, int is_max) {
    const int cg = xi.cs / 8;
    const long long total = yo.pixels() * cg;
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(t % cg);
        long long p = t / cg;
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
            bi[j] = -1;
        }
        for (int r = 0; r < k; ++r) {
            const int ih = oh * stride - pad + r;
            if (ih < 0 || ih >= xi.H) continue;
            for (int s = 0; s < k; ++s) {
                const int iw = ow * stride - pad + s;
                if (iw < 0 || iw >= xi.W) continue;
                float f[8];
                unpack8(*reinterpret_cast<const uint4*>(x + ((static_cast<long long>(n) * xi.H + ih) * xi.W + iw) * xi.cs + g * 8), f);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    sum[j] += f[j];
                    if (bi[j] < 0 || f[j] > best[j]) {  // first maximum in row-major window order
                        best[j] = f[j];
                        bi[j] = ih * xi.W + iw;
                    }
                }
            }
        }
        const long long o = ((static_cast<long long>(n) * yo.H + oh) * yo.W + ow) * yo.cs + g * 8;
        float out[8];
        const float inv = 1.f / static_cast<float>(k * k);
#pragma unroll
        for (int j = 0; j < 8; ++j) out[j] = is_max ? best[j] : sum[j] * inv;
        *reinterpret_cast<uint4*>(y + o) = pack8(out);
        if (idx) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int c = g * 8 + j;
                // flat NCHW input index: layout independent, compared bit-exactly with the oracle
                idx[o + j] = (c < xi.C && bi[j] >= 0)
                                 ? static_cast<int32_t>((static_cast<long long>(n) * xi.C + c) * xi.H * xi.W + bi[j])
                                 : -1;
            }
        }
    }
}

// Gather formulation: each input element sums the windows that selected it.
__global__ void k_pool_bwd(const bf16* __restrict__ dy, Act4 yo, const int32_t* __restrict__ idx,
                           bf16* __restrict__ dx, Act4 xi, int k, int stride, int pad, int is_max) {
    const int cg = xi.cs / 8;
    const long long total = xi.pixels() * cg;
    const float inv = 1.f / static_cast<float>(k * k);
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(t % cg);
        long long p = t / cg;
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
        for (int oh = oh0; oh <= oh1; ++oh)
            for (int ow = ow0; ow <= ow1; ++ow) {
                const long long o = ((static_cast<long long>(n) * yo.H + oh) * yo.W + ow) * yo.cs + g * 8;
                float d[8];
                unpack8(*reinterpret_cast<const uint4*>(dy + o), d);
                if (is_max) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int c = g * 8 + j;
                        const int me = static_cast<int>((static_cast<long long>(n) * xi.C + c) * xi.H * xi.W + ih * xi.W + iw);
                        if (c < xi.C && idx[o + j] == me) acc[j] += d[j];
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[j] += d[j] * inv;
                }
            }
        *reinterpret_cast<uint4*>(dx + ((static_cast<long long>(n) * xi.H + ih) * xi.W + iw) * xi.cs + g * 8) = pack8(acc);
    }
}

// ---------------------------------------------------------------- LRN (across channels, one warp per pixel)
__global__ void k_lrn_fwd(const bf16* __restrict__ x, bf16* __restrict__ y, Act4 a, int size, float alpha, float beta,
                          float kk) {
    extern __shared__ float sm[];
    const int warps = blockDim.x / 32, wid = threadIdx.x / 32, lane = threadIdx.x % 32;
    float* sq = sm + wid * a.cs;
    const int half = size / 2;
    const float an = alpha / static_cast<float>(size);
    for (long long p = blockIdx.x * static_cast<long long>(warps) + wid; p < a.pixels();
         p += static_cast<long long>(gridDim.x) * warps) {
        const bf16* xp = x + p * a.cs;
        for (int c = lane; c < a.cs; c += 32) {
            const float v = __bfloat162float(xp[c]);
            sq[c] = v * v;
        }
        __syncwarp();
        for (int c = lane; c < a.cs; c += 32) {
            float out = 0.f;
            if (c < a.C) {
                float s = 0.f;
                for (int cc = max(0, c - half); cc <= min(a.C - 1, c + half); ++cc) s += sq[cc];
                const float scale = kk + an * s;
                out = __bfloat162float(xp[c]) * powf(scale, -beta);
            }
            y[p * a.cs + c] = __float2bfloat16_rn(out);
        }
        __syncwarp();
    }
}

__global__ void k_lrn_bwd(const bf16* __restrict__ dy, const bf16* __restrict__ x, const bf16* __restrict__ y,
                          bf16* __restrict__ dx, Act4 a, int size, float alpha, float beta, float kk) {
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
            const float v = __bfloat162float(x[o + c]);
            sq[c] = v * v;
        }
        __syncwarp();
        for (int c = lane; c < a.C; c += 32) {
            float s = 0.f;
            for (int cc = max(0, c - half); cc <= min(a.C - 1, c + half); ++cc) s += sq[cc];
            sc[c] = kk + an * s;
            tt[c] = __bfloat162float(dy[o + c]) * __bfloat162float(y[o + c]) / sc[c];
        }
        __syncwarp();
        for (int c = lane; c < a.cs; c += 32) {
            float out = 0.f;
            if (c < a.C) {
                float s = 0.f;
                for (int cc = max(0, c - half); cc <= min(a.C - 1, c + half); ++cc) s += tt[cc];
                out = __bfloat162float(dy[o + c]) * powf(sc[c], -beta) - coef * __bfloat162float(x[o + c]) * s;
            }
            dx[o + c] = __float2bfloat16_rn(out);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- softmax / loss head (fp32)
__global__ void k_softmax_fwd(const bf16* __restrict__ x, long long ld, float* __restrict__ y, int rows, int F) {
    const int warps = blockDim.x / 32, wid = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int r = blockIdx.x * warps + wid; r < rows; r += gridDim.x * warps) {
        const bf16* xr = x + r * ld;
        float m = -INFINITY;
        for (int j = lane; j < F; j += 32) m = fmaxf(m, __bfloat162float(xr[j]));
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float s = 0.f;
        for (int j = lane; j < F; j += 32) s += expf(__bfloat162float(xr[j]) - m);
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const float inv = 1.f / s;
        for (int j = lane; j < F; j += 32) y[static_cast<long long>(r) * F + j] = expf(__bfloat162float(xr[j]) - m) * inv;
    }
}

__global__ void k_softmax_bwd(const float* __restrict__ dy, const float* __restrict__ y, bf16* __restrict__ dx,
                              long long ld, int rows, int F) {
    const int warps = blockDim.x / 32, wid = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int r = blockIdx.x * warps + wid; r < rows; r += gridDim.x * warps) {
        const long long o = static_cast<long long>(r) * F;
        float d = 0.f;
        for (int j = lane; j < F; j += 32) d += dy[o + j] * y[o + j];
        for (int s = 16; s; s >>= 1) d += __shfl_xor_sync(0xffffffffu, d, s);
        for (int j = lane; j < ld; j += 32)
            dx[r * ld + j] = __float2bfloat16_rn(j < F ? y[o + j] * (dy[o + j] - d) : 0.f);
    }
}

__global__ void k_f32_ew(int op, const float* __restrict__ a, const float* __restrict__ b, float scale,
                         float* __restrict__ y, long long n) {
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
__global__ void k_loss(LossArgs args, float* out) {
    __shared__ double red[1024];
    double acc = 0.0;
    for (int t = 0; t < args.nterms; ++t) {
        double s = 0.0;
        for (long long i = threadIdx.x; i < args.n[t]; i += blockDim.x)
            s += static_cast<double>(args.a[t][i]) * static_cast<double>(args.b[t][i]);
        acc += args.coef[t] * s;
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = static_cast<float>(red[0]);
}

// ---------------------------------------------------------------- column reductions
// Stage 1: block b sums rows [b*rpb, (b+1)*rpb) for every column, 8 columns per thread.
__global__ void k_colsum_partial(const bf16* __restrict__ x, long long rows, int cols, long long ld, long long rpb,
                                 float* __restrict__ part, const float* __restrict__ center, int mode) {
    // mode 0: sum x ; mode 1: sum (x - center)^2
    extern __shared__ float sm[];
    const int tpr = (cols + 7) / 8;             // threads per row
    const int rpi = max(1, blockDim.x / tpr);   // rows per iteration
    const int tr = threadIdx.x / tpr, tc = threadIdx.x % tpr;
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    const long long r0 = blockIdx.x * rpb, r1 = min(rows, r0 + rpb);
    if (tr < rpi) {
        for (long long r = r0 + tr; r < r1; r += rpi) {
            float f[8];
            unpack8(*reinterpret_cast<const uint4*>(x + r * ld + tc * 8), f);
            if (mode == 1) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int c = tc * 8 + j;
                    const float d = f[j] - (c < cols ? center[c] : 0.f);
                    f[j] = d * d;
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] += f[j];
        }
    }
    // reduce over the rpi row-slots in a fixed order
    const int width = tpr * 8;
    for (int i = threadIdx.x; i < rpi * width; i += blockDim.x) sm[i] = 0.f;
    __syncthreads();
    if (tr < rpi)
#pragma unroll
        for (int j = 0; j < 8; ++j) sm[tr * width + tc * 8 + j] = acc[j];
    __syncthreads();
    for (int c = threadIdx.x; c < cols; c += blockDim.x) {
        float s = 0.f;
        for (int q = 0; q < rpi; ++q) s += sm[q * width + c];
        part[blockIdx.x * static_cast<long long>(cols) + c] = s;
    }
}

__global__ void k_colsum_final(const float* __restrict__ part, int nparts, int cols, float* __restrict__ out, float scale) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += gridDim.x * blockDim.x) {
        float s = 0.f;
        for (int b = 0; b < nparts; ++b) s += part[b * static_cast<long long>(cols) + c];
        out[c] = s * scale;
    }
}

int colsum_blocks(long long rows, int cols, int max_partials) {
    const long long by_rows = (rows + 255) / 256;
    long long b = std::min<long long>(by_rows, static_cast<long long>(num_sms()) * 4);
    b = std::min<long long>(b, std::max(1, max_partials / std::max(1, cols)));
    return static_cast<int>(std::max<long long>(1, b));
}

tc_status colsum_run(const bf16* x, long long rows, int cols, long long ld, float* out, float* partials, int max_partials,
                     const float* center, int mode, float scale, cudaStream_t st) {
    if ((ld & 7) || (reinterpret_cast<uintptr_t>(x) & 15)) return fail(TC_INVALID_ARG, "colsum: misaligned operand");
    const int nb = colsum_blocks(rows, cols, max_partials);
    const long long rpb = (rows + nb - 1) / nb;
    const int tpr = (cols + 7) / 8;
    const int threads = std::min(1024, std::max(kThreads, ((tpr + 31) / 32) * 32));
    const int rpi = std::max(1, threads / tpr);
    const size_t smem = static_cast<size_t>(rpi) * tpr * 8 * sizeof(float);
    k_colsum_partial<<<nb, threads, smem, st>>>(x, rows, cols, ld, rpb, partials, center, mode);
    TCB_LAUNCH_CHECK();
    k_colsum_final<<<(cols + 255) / 256, 256, 0, st>>>(partials, nb, cols, out, scale);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}

__global__ void k_bias_add(const bf16* __restrict__ x, const float* __restrict__ b, bf16* __restrict__ y, long long rows,
                           int cols, long long ld, int relu) {
    const long long total = rows * ld;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i % ld);
        float v = c < cols ? __bfloat162float(x[i]) + b[c] : 0.f;
        if (relu) v = fmaxf(v, 0.f);
        y[i] = __float2bfloat16_rn(v);
    }
}

__global__ void k_channel_copy(const bf16* __restrict__ src, int src_cs, bf16* __restrict__ dst, int dst_cs, int off,
                               int c, long long pixels) {
    const long long total = pixels * c;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long p = i / c;
        const int ch = static_cast<int>(i - p * c);
        dst[p * dst_cs + off + ch] = src[p * src_cs + ch];
    }
}

// ---------------------------------------------------------------- batch norm
__global__ void k_bn_finish_stats(const float* __restrict__ mean, const float* __restrict__ var, float* stats, int C,
                                  float eps) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < C) {
        stats[c] = mean[c];
        stats[C + c] = rsqrtf(var[c] + eps);
    }
}

__global__ void k_bn_apply(const bf16* __restrict__ x, const float* __restrict__ gamma, const float* __restrict__ beta,
                           const float* __restrict__ stats, bf16* __restrict__ y, long long pixels, int C, int cs) {
    const long long total = pixels * cs;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i % cs);
        float v = 0.f;
        if (c < C) v = gamma[c] * (__bfloat162float(x[i]) - stats[c]) * stats[C + c] + beta[c];
        y[i] = __float2bfloat16_rn(v);
    }
}

// dx = g*istd*(dy - sum(dy)/M - xhat*sum(dy*xhat)/M)
__global__ void k_bn_bwd_apply(const bf16* __restrict__ dy, const bf16* __restrict__ x, const float* __restrict__ gamma,
                               const float* __restrict__ stats, const float* __restrict__ sdy,
                               const float* __restrict__ sdyx, bf16* __restrict__ dx, long long pixels, int C, int cs) {
    const long long total = pixels * cs;
    const float invm = 1.f / static_cast<float>(pixels);
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i % cs);
        float v = 0.f;
        if (c < C) {
            const float is = stats[C + c];
            const float xh = (__bfloat162float(x[i]) - stats[c]) * is;
            v = gamma[c] * is * (__bfloat162float(dy[i]) - sdy[c] * invm - xh * sdyx[c] * invm);
        }
        dx[i] = __float2bfloat16_rn(v);
    }
}

// sum(dy * xhat) per channel, partial stage (fixed partition)
__global__ void k_bn_dyx_partial(const bf16* __restrict__ dy, const bf16* __restrict__ x, const float* __restrict__ stats,
                                 long long pixels, int C, int cs, long long rpb, float* __restrict__ part) {
    const long long r0 = blockIdx.x * rpb, r1 = min(pixels, r0 + rpb);
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        float s = 0.f;
        const float m = stats[c], is = stats[C + c];
        for (long long r = r0; r < r1; ++r)
            s += __bfloat162float(dy[r * cs + c]) * (__bfloat162float(x[r * cs + c]) - m) * is;
        part[blockIdx.x * static_cast<long long>(C) + c] = s;
    }
}

// ---------------------------------------------------------------- dense im2col (small-C first layers)
__global__ void k_im2col(const bf16* __restrict__ x, Act4 xi, int R, int S, int stride, int pad, int Ho, int Wo,
                         int Kp, bf16* __restrict__ col) {
    const int groups = Kp / 8;
    const long long total = static_cast<long long>(xi.N) * Ho * Wo * groups;
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(t % groups);
        long long m = t / groups;
        const int ow = static_cast<int>(m % Wo);
        long long q = m / Wo;
        const int oh = static_cast<int>(q % Ho);
        const int n = static_cast<int>(q / Ho);
        __align__(16) bf16 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int kk = g * 8 + j;
            bf16 val = __float2bfloat16_rn(0.f);
            if (kk < R * S * xi.C) {
                const int c = kk % xi.C;
                const int rs = kk / xi.C;
                const int r = rs / S, s = rs - (rs / S) * S;
                const int ih = oh * stride - pad + r, iw = ow * stride - pad + s;
                if (ih >= 0 && ih < xi.H && iw >= 0 && iw < xi.W)
                    val = x[((static_cast<long long>(n) * xi.H + ih) * xi.W + iw) * xi.cs + c];
            }
            v[j] = val;
        }
        *reinterpret_cast<uint4*>(col + m * Kp + g * 8) = *reinterpret_cast<const uint4*>(v);
    }
}

// ---------------------------------------------------------------- LRN v2: thread per (pixel, 8 channels)
// Window sums over channels [c - n/2, c + n/2] read the neighbouring 16-byte
// chunks of the same pixel (L1 hits); n <= 9 so chunks g-1 .. g+1 suffice.
__device__ __forceinline__ void load_chunk3(const bf16* __restrict__ p, int g, int ng, float (&v)[24]) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const int gg = g - 1 + q;
        float f[8];
        if (gg >= 0 && gg < ng) {
            unpack8(*reinterpret_cast<const uint4*>(p + gg * 8), f);
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) f[j] = 0.f;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) v[q * 8 + j] = f[j];
    }
}

// HALF = n/2 is a template parameter so every window loop unrolls and the
// per-thread channel windows stay in registers.
template <int HALF>
__global__ void k_lrn2_fwd(const bf16* __restrict__ x, bf16* __restrict__ y, Act4 a, float alpha, float beta,
                           float kk) {
    const int ng = a.cs / 8;
    const long long total = a.pixels() * ng;
    const float an = alpha / static_cast<float>(2 * HALF + 1);
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(t % ng);
        const bf16* px = x + (t / ng) * a.cs;
        float v[24];
        load_chunk3(px, g, ng, v);
        // channels outside [0, C) contribute nothing (pads are zero, neighbours beyond the tensor loaded as 0)
        float out[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float s = 0.f;
#pragma unroll
            for (int d = -HALF; d <= HALF; ++d) s += v[8 + j + d] * v[8 + j + d];
            out[j] = (g * 8 + j) < a.C ? v[8 + j] * __powf(kk + an * s, -beta) : 0.f;
        }
        *reinterpret_cast<uint4*>(y + t * 8) = pack8(out);
    }
}

template <int HALF>
__global__ void k_lrn2_bwd(const bf16* __restrict__ dy, const bf16* __restrict__ x, const bf16* __restrict__ y,
                           bf16* __restrict__ dx, Act4 a, float alpha, float beta, float kk) {
    const int ng = a.cs / 8;
    const long long total = a.pixels() * ng;
    const float an = alpha / static_cast<float>(2 * HALF + 1);
    const float coef = 2.f * alpha * beta / static_cast<float>(2 * HALF + 1);
    constexpr int L = 8 - HALF, U = 16 + HALF;  // window of channels g*8-HALF .. g*8+7+HALF
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(t % ng);
        const long long base = (t / ng) * a.cs;
        float xv[24], dv[24], yv[24];
        load_chunk3(x + base, g, ng, xv);
        load_chunk3(dy + base, g, ng, dv);
        load_chunk3(y + base, g, ng, yv);
        float sc[24], tt[24];
#pragma unroll
        for (int i = L; i < U; ++i) {
            float s = 0.f;
#pragma unroll
            for (int d = -HALF; d <= HALF; ++d) s += xv[i + d] * xv[i + d];
            sc[i] = kk + an * s;
            // zero for channels outside [0, C): dy and y are zero there
            tt[i] = dv[i] * yv[i] * __frcp_rn(sc[i]);
        }
        float out[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float s = 0.f;
#pragma unroll
            for (int d = -HALF; d <= HALF; ++d) s += tt[8 + j + d];
            out[j] = (g * 8 + j) < a.C ? dv[8 + j] * __powf(sc[8 + j], -beta) - coef * xv[8 + j] * s : 0.f;
        }
        *reinterpret_cast<uint4*>(dx + base + g * 8) = pack8(out);
    }
}

// ---------------------------------------------------------------- input staging
__global__ void k_nchw_to_nhwc(const float* __restrict__ x, bf16* __restrict__ y, int N, int C, int H, int W, int cs) {
    const long long total = static_cast<long long>(N) * H * W * cs;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i % cs);
        long long p = i / cs;
        const int w = static_cast<int>(p % W);
        p /= W;
        const int h = static_cast<int>(p % H);
        const int n = static_cast<int>(p / H);
        y[i] = __float2bfloat16_rn(c < C ? x[((static_cast<long long>(n) * C + c) * H + h) * W + w] : 0.f);
    }
}

__global__ void k_synth(bf16* __restrict__ x, int32_t* __restrict__ labels, int N, int C, int H, int W, int cs,
                        int classes, uint64_t seed, uint32_t iter, uint32_t n0) {
    const long long total = static_cast<long long>(N) * H * W * cs;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i % cs);
        long long p = i / cs;
        const int w = static_cast<int>(p % W);
        p /= W;
        const int h = static_cast<int>(p % H);
        const int n = static_cast<int>(p / H);
        const uint32_t ng = n0 + n;
        const uint32_t y = tcp_label(seed, ng, iter, classes);
        if (c == 0 && h == 0 && w == 0) labels[n] = static_cast<int32_t>(y);
        float v = 0.f;
        if (c < C) {
            const uint32_t e = static_cast<uint32_t>((static_cast<long long>(c) * H + h) * W + w);
            float u1, u2;
            tcp_uniform_pair(seed, ng, iter, e, &u1, &u2);
            const double r = sqrt(-2.0 * log(static_cast<double>(u1)));
            const double t = 6.283185307179586 * static_cast<double>(u2);
            const double z = (e & 1) ? r * sin(t) : r * cos(t);
            v = static_cast<float>(static_cast<double>(tcp_centroid(seed, y, e)) + 0.1 * z);
        }
        x[i] = __float2bfloat16_rn(v);
    }
}

// ---------------------------------------------------------------- SGD
__global__ void k_sgd(SgdTensor t) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < t.n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const float p = t.p[i];
        const float v = t.momentum * t.v[i] + t.lr_alpha * (t.g[i] + t.decay * p);
        const float np = p + v;
        t.v[i] = v;
        t.p[i] = np;
        const bf16 b = __float2bfloat16_rn(np);
        if (t.shadow) t.shadow[i] = b;
        if (t.shadow_rskc) {
            const int c = static_cast<int>(i % t.cs);
            const long long q = i / t.cs;
            const int rs = static_cast<int>(q % t.RS);
            const int k = static_cast<int>(q / t.RS);
            t.shadow_rskc[(static_cast<long long>(rs) * t.ks + k) * t.cs + c] = b;
        }
    }
}

}  // namespace

// ================================================================ launchers
#define EW_GRID(n) grid_for((n)), kThreads, 0, st

tc_status launch_relu_fwd(const bf16* x, bf16* y, long long n, cudaStream_t st) {
    k_relu_fwd<<<EW_GRID(n / 8)>>>(reinterpret_cast<const uint4*>(x), reinterpret_cast<uint4*>(y), n / 8);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_relu_bwd(const bf16* dy, const bf16* y, bf16* dx, long long n, cudaStream_t st) {
    k_relu_bwd<<<EW_GRID(n / 8)>>>(reinterpret_cast<const uint4*>(dy), reinterpret_cast<const uint4*>(y),
                                    reinterpret_cast<uint4*>(dx), n / 8);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_add_bf16(const bf16* a, const bf16* b, bf16* y, long long n, cudaStream_t st) {
    k_add<<<EW_GRID(n / 8)>>>(reinterpret_cast<const uint4*>(a), reinterpret_cast<const uint4*>(b),
                               reinterpret_cast<uint4*>(y), n / 8);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_mask_mul(const bf16* x, const uint8_t* keep, float scale, bf16* y, long long n, cudaStream_t st) {
    k_mask_mul<<<EW_GRID(n / 8)>>>(reinterpret_cast<const uint4*>(x), reinterpret_cast<const uint2*>(keep), scale,
                                    reinterpret_cast<uint4*>(y), n / 8);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_dropout_mask(uint8_t* keep, int N, int H, int W, int C, int cs, float rate, uint64_t seed,
                              uint32_t var, const uint32_t* iter_n0, cudaStream_t st) {
    const long long n = static_cast<long long>(N) * H * W * cs;
    k_dropout_mask<<<EW_GRID(n)>>>(keep, N, H, W, C, cs, rate, seed, var, iter_n0);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_pool_fwd(const bf16* x, Act4 xi, bf16* y, Act4 yo, int32_t* idx, int k, int stride, int pad,
                          int is_max, cudaStream_t st) {
    k_pool_fwd<<<EW_GRID(yo.pixels() * (xi.cs / 8))>>>(x, xi, y, yo, idx, k, stride, pad, is_max);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_pool_bwd(const bf16* dy, Act4 yo, const int32_t* idx, bf16* dx, Act4 xi, int k, int stride, int pad,
                          int is_max, cudaStream_t st) {
    k_pool_bwd<<<EW_GRID(xi.pixels() * (xi.cs / 8))>>>(dy, yo, idx, dx, xi, k, stride, pad, is_max);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_lrn_fwd(const bf16* x, bf16* y, Act4 a, int size, float alpha, float beta, float k, cudaStream_t st) {
    const long long n = a.pixels() * (a.cs / 8);
    switch (size) {  // odd windows up to 9: register-resident template kernels
        case 3: k_lrn2_fwd<1><<<EW_GRID(n)>>>(x, y, a, alpha, beta, k); break;
        case 5: k_lrn2_fwd<2><<<EW_GRID(n)>>>(x, y, a, alpha, beta, k); break;
        case 7: k_lrn2_fwd<3><<<EW_GRID(n)>>>(x, y, a, alpha, beta, k); break;
        case 9: k_lrn2_fwd<4><<<EW_GRID(n)>>>(x, y, a, alpha, beta, k); break;
        default: {  // general path: warp per pixel with the channel vector in shared memory
            const int warps = 8;
            k_lrn_fwd<<<grid_for(a.pixels(), warps), warps * 32, warps * a.cs * sizeof(float), st>>>(x, y, a, size,
                                                                                                     alpha, beta, k);
        }
    }
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_lrn_bwd(const bf16* dy, const bf16* x, const bf16* y, bf16* dx, Act4 a, int size, float alpha,
                         float beta, float k, cudaStream_t st) {
    const long long n = a.pixels() * (a.cs / 8);
    switch (size) {
        case 3: k_lrn2_bwd<1><<<EW_GRID(n)>>>(dy, x, y, dx, a, alpha, beta, k); break;
        case 5: k_lrn2_bwd<2><<<EW_GRID(n)>>>(dy, x, y, dx, a, alpha, beta, k); break;
        case 7: k_lrn2_bwd<3><<<EW_GRID(n)>>>(dy, x, y, dx, a, alpha, beta, k); break;
        case 9: k_lrn2_bwd<4><<<EW_GRID(n)>>>(dy, x, y, dx, a, alpha, beta, k); break;
        default: {
            const int warps = 8;
            k_lrn_bwd<<<grid_for(a.pixels(), warps), warps * 32, warps * 3 * a.cs * sizeof(float), st>>>(
                dy, x, y, dx, a, size, alpha, beta, k);
        }
    }
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_im2col(const bf16* x, Act4 xi, int R, int S, int stride, int pad, int Ho, int Wo, int Kp, bf16* col,
                        cudaStream_t st) {
    if (Kp % 8) return fail(TC_INVALID_ARG, "im2col: Kp must be a multiple of 8");
    k_im2col<<<EW_GRID(static_cast<long long>(xi.N) * Ho * Wo * (Kp / 8))>>>(x, xi, R, S, stride, pad, Ho, Wo, Kp, col);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_softmax_fwd(const bf16* x, long long in_ld, float* y, int rows, int F, cudaStream_t st) {
    k_softmax_fwd<<<grid_for(rows, 8), 256, 0, st>>>(x, in_ld, y, rows, F);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_softmax_bwd(const float* dy, const float* y, bf16* dx, long long out_ld, int rows, int F,
                             cudaStream_t st) {
    k_softmax_bwd<<<grid_for(rows, 8), 256, 0, st>>>(dy, y, dx, out_ld, rows, F);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_f32_ew(int op, const float* a, const float* b, float scale, float* y, long long n, cudaStream_t st) {
    k_f32_ew<<<EW_GRID(n)>>>(op, a, b, scale, y, n);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_onehot(const int32_t* labels, float* y, int N, int K, cudaStream_t st) {
    k_onehot<<<EW_GRID(static_cast<long long>(N) * K)>>>(labels, y, N, K);
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
    k_loss<<<1, 1024, 0, st>>>(args, out);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
size_t colsum_partials_floats(int cols) { return static_cast<size_t>(num_sms()) * 4 * std::max(cols, 8) + 64; }
tc_status launch_colsum(const bf16* x, long long rows, int cols, long long ld, float* out, float* partials,
                        int max_partials, cudaStream_t st) {
    return colsum_run(x, rows, cols, ld, out, partials, max_partials, nullptr, 0, 1.f, st);
}
tc_status launch_bias_add(const bf16* x, const float* b, bf16* y, long long rows, int cols, long long ld, int relu,
                          cudaStream_t st) {
    k_bias_add<<<EW_GRID(rows * ld)>>>(x, b, y, rows, cols, ld, relu);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_channel_copy(const bf16* src, int src_cs, bf16* dst, int dst_cs, int off, int c, long long pixels,
                              cudaStream_t st) {
    k_channel_copy<<<EW_GRID(pixels * c)>>>(src, src_cs, dst, dst_cs, off, c, pixels);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_zero(void* p, size_t bytes, cudaStream_t st) {
    TCB_CUDA_CHECK(cudaMemsetAsync(p, 0, bytes, st));
    return TC_OK;
}

tc_status launch_bn_fwd(const bf16* x, const float* gamma, const float* beta, bf16* y, float* stats, long long pixels,
                        int C, int cs, float eps, float* partials, int max_partials, cudaStream_t st) {
    // two-pass statistics: mean, then mean of squared deviations (biased variance)
    float* mean = partials + max_partials;  // caller sizes partials to max_partials + 2*C
    float* var = mean + C;
    tc_status s = colsum_run(x, pixels, C, cs, mean, partials, max_partials, nullptr, 0, 1.f / pixels, st);
    if (s != TC_OK) return s;
    s = colsum_run(x, pixels, C, cs, var, partials, max_partials, mean, 1, 1.f / pixels, st);
    if (s != TC_OK) return s;
    k_bn_finish_stats<<<(C + 255) / 256, 256, 0, st>>>(mean, var, stats, C, eps);
    TCB_LAUNCH_CHECK();
    k_bn_apply<<<EW_GRID(pixels * cs)>>>(x, gamma, beta, stats, y, pixels, C, cs);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}

tc_status launch_bn_bwd(const bf16* dy, const bf16* x, const float* gamma, const float* stats, bf16* dx, float* dgamma,
                        float* dbeta, long long pixels, int C, int cs, float* partials, int max_partials,
                        cudaStream_t st) {
    float* sdy = partials + max_partials;
    float* sdyx = sdy + C;
    tc_status s = colsum_run(dy, pixels, C, cs, sdy, partials, max_partials, nullptr, 0, 1.f, st);
    if (s != TC_OK) return s;
    const int nb = colsum_blocks(pixels, C, max_partials);
    const long long rpb = (pixels + nb - 1) / nb;
    k_bn_dyx_partial<<<nb, 256, 0, st>>>(dy, x, stats, pixels, C, cs, rpb, partials);
    TCB_LAUNCH_CHECK();
    k_colsum_final<<<(C + 255) / 256, 256, 0, st>>>(partials, nb, C, sdyx, 1.f);
    TCB_LAUNCH_CHECK();
    if (dgamma) TCB_CUDA_CHECK(cudaMemcpyAsync(dgamma, sdyx, C * sizeof(float), cudaMemcpyDeviceToDevice, st));
    if (dbeta) TCB_CUDA_CHECK(cudaMemcpyAsync(dbeta, sdy, C * sizeof(float), cudaMemcpyDeviceToDevice, st));
    if (dx) {
        k_bn_bwd_apply<<<EW_GRID(pixels * cs)>>>(dy, x, gamma, stats, sdy, sdyx, dx, pixels, C, cs);
        TCB_LAUNCH_CHECK();
    }
    return TC_OK;
}

tc_status launch_nchw_to_nhwc(const float* x, bf16* y, int N, int C, int H, int W, int cs, cudaStream_t st) {
    k_nchw_to_nhwc<<<EW_GRID(static_cast<long long>(N) * H * W * cs)>>>(x, y, N, C, H, W, cs);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_synth_batch(bf16* x, int32_t* labels, int N, int C, int H, int W, int cs, int classes, uint64_t seed,
                             uint32_t iter, uint32_t n0, cudaStream_t st) {
    k_synth<<<EW_GRID(static_cast<long long>(N) * H * W * cs)>>>(x, labels, N, C, H, W, cs, classes, seed, iter, n0);
    TCB_LAUNCH_CHECK();
    return TC_OK;
}
tc_status launch_sgd(const SgdTensor* ts, int nt, SgdTensor*, cudaStream_t st) {
    for (int i = 0; i < nt; ++i) {
        k_sgd<<<EW_GRID(ts[i].n)>>>(ts[i]);
        TCB_LAUNCH_CHECK();
    }
    return TC_OK;
}

}  // namespace tcb
