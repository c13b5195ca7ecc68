// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see tc_oracle.h).
//
// Restates the reference runtime on the host: NCHW tensors,
// fp32 or fp64, deterministic OpenMP (static partitions, every output element
// reduced in a fixed order by one thread).  Each kernel cites the SPEC / paper
// line it follows.
#include "tc_oracle.h"

#include <immintrin.h>
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "tc_philox.h"

namespace {

using i64 = int64_t;

// ----------------------------------------------------------------- GEMM
// C[M,N] (+)= op(A)[M,K] * op(B)[K,N]; row-major.  Every C element sums k in
// ascending order (k-blocks in order, k in order inside a block) whatever the
// thread count, so results are deterministic.  Packed panels + a 6 x (2 vector)
// register micro-kernel (AVX2 FMA): fast enough that the oracle runs the
// BASELINE shapes (AlexNet b128 steps) in seconds; the arithmetic is the plain
// dot product of the SPEC contraction.
template <class T>
struct Vec;
template <>
struct Vec<float> {
    using V = __m256;
    static constexpr int L = 8;
    static V zero() { return _mm256_setzero_ps(); }
    static V load(const float* p) { return _mm256_loadu_ps(p); }
    static void store(float* p, V v) { _mm256_storeu_ps(p, v); }
    static V bcast(float a) { return _mm256_set1_ps(a); }
    static V fma(V a, V b, V c) { return _mm256_fmadd_ps(a, b, c); }
};
template <>
struct Vec<double> {
    using V = __m256d;
    static constexpr int L = 4;
    static V zero() { return _mm256_setzero_pd(); }
    static V load(const double* p) { return _mm256_loadu_pd(p); }
    static void store(double* p, V v) { _mm256_storeu_pd(p, v); }
    static V bcast(double a) { return _mm256_set1_pd(a); }
    static V fma(V a, V b, V c) { return _mm256_fmadd_pd(a, b, c); }
};

constexpr int GEMM_MR = 6;

// acc[MR][NR] over kc steps of packed A (MR-interleaved) and packed B (NR-interleaved).
template <class T>
inline void micro_kernel(int kc, const T* ap, const T* bp, T* c, i64 ldc, int mr, int nr, bool load_c) {
    using VT = Vec<T>;
    using V = typename VT::V;
    constexpr int L = VT::L, NR = 2 * L;
    V acc[GEMM_MR][2];
    T buf[GEMM_MR][NR];
    if (load_c) {
        for (int i = 0; i < GEMM_MR; ++i)
            for (int j = 0; j < NR; ++j) buf[i][j] = (i < mr && j < nr) ? c[i * ldc + j] : T(0);
        for (int i = 0; i < GEMM_MR; ++i) {
            acc[i][0] = VT::load(&buf[i][0]);
            acc[i][1] = VT::load(&buf[i][L]);
        }
    } else {
        for (int i = 0; i < GEMM_MR; ++i) acc[i][0] = acc[i][1] = VT::zero();
    }
    for (int k = 0; k < kc; ++k) {
        const V b0 = VT::load(bp), b1 = VT::load(bp + L);
        for (int i = 0; i < GEMM_MR; ++i) {
            const V a = VT::bcast(ap[i]);
            acc[i][0] = VT::fma(a, b0, acc[i][0]);
            acc[i][1] = VT::fma(a, b1, acc[i][1]);
        }
        ap += GEMM_MR;
        bp += NR;
    }
    if (mr == GEMM_MR && nr == NR) {
        for (int i = 0; i < GEMM_MR; ++i) {
            VT::store(c + i * ldc, acc[i][0]);
            VT::store(c + i * ldc + L, acc[i][1]);
        }
        return;
    }
    for (int i = 0; i < GEMM_MR; ++i) {
        VT::store(&buf[i][0], acc[i][0]);
        VT::store(&buf[i][L], acc[i][1]);
    }
    for (int i = 0; i < mr; ++i)
        for (int j = 0; j < nr; ++j) c[i * ldc + j] = buf[i][j];
}

template <class T>
void gemm(int M, int N, int K, const T* A, i64 lda, bool ta, const T* B, i64 ldb, bool tb, T* C, i64 ldc, bool acc) {
    constexpr int NR = 2 * Vec<T>::L;
    constexpr int MB = 16 * GEMM_MR, NB = 128, KB = 256;
    const int nmb = (M + MB - 1) / MB, nnb = (N + NB - 1) / NB;
    if (K == 0) {
        if (!acc)
            for (int i = 0; i < M; ++i)
                for (int j = 0; j < N; ++j) C[i * ldc + j] = T(0);
        return;
    }
#pragma omp parallel
    {
        std::vector<T> ap(static_cast<size_t>(MB) * KB), bp(static_cast<size_t>(NB) * KB);
#pragma omp for collapse(2) schedule(static)
        for (int mb = 0; mb < nmb; ++mb)
            for (int nb = 0; nb < nnb; ++nb) {
                const int i0 = mb * MB, i1 = std::min(M, i0 + MB), j0 = nb * NB, j1 = std::min(N, j0 + NB);
                for (int k0 = 0; k0 < K; k0 += KB) {
                    const int kc = std::min(K, k0 + KB) - k0;
                    // pack B[k0:k0+kc, j0:j1] as NR-wide strips (zero padded), reading B contiguously
                    const int jw = (j1 - j0 + NR - 1) / NR * NR, iw = (i1 - i0 + GEMM_MR - 1) / GEMM_MR * GEMM_MR;
                    auto bslot = [&](int j, int k) -> T& { return bp[static_cast<i64>(j / NR) * kc * NR + k * NR + j % NR]; };
                    auto aslot = [&](int i, int k) -> T& { return ap[static_cast<i64>(i / GEMM_MR) * kc * GEMM_MR + k * GEMM_MR + i % GEMM_MR]; };
                    if (tb) {
                        for (int j = 0; j < jw; ++j) {
                            const T* col = B + static_cast<i64>(j0 + j) * ldb + k0;
                            for (int k = 0; k < kc; ++k) bslot(j, k) = j0 + j < j1 ? col[k] : T(0);
                        }
                    } else {
                        for (int k = 0; k < kc; ++k) {
                            const T* row = B + static_cast<i64>(k0 + k) * ldb + j0;
                            for (int j = 0; j < jw; ++j) bslot(j, k) = j0 + j < j1 ? row[j] : T(0);
                        }
                    }
                    // pack A[i0:i1, k0:k0+kc] as MR-tall strips (zero padded)
                    if (ta) {
                        for (int k = 0; k < kc; ++k) {
                            const T* row = A + static_cast<i64>(k0 + k) * lda + i0;
                            for (int i = 0; i < iw; ++i) aslot(i, k) = i0 + i < i1 ? row[i] : T(0);
                        }
                    } else {
                        for (int i = 0; i < iw; ++i) {
                            const T* row = A + static_cast<i64>(i0 + i) * lda + k0;
                            for (int k = 0; k < kc; ++k) aslot(i, k) = i0 + i < i1 ? row[k] : T(0);
                        }
                    }
                    const bool load_c = acc || k0 > 0;
                    for (int ir = i0; ir < i1; ir += GEMM_MR)
                        for (int jr = j0; jr < j1; jr += NR)
                            micro_kernel<T>(kc, ap.data() + static_cast<i64>(ir - i0) * kc,
                                            bp.data() + static_cast<i64>(jr - j0) * kc, C + ir * ldc + jr, ldc,
                                            std::min(GEMM_MR, i1 - ir), std::min(NR, j1 - jr), load_c);
                }
            }
    }
}

// ----------------------------------------------------------------- convolution
// Lowered to GEMM over im2col columns, a chunk of G images per
// GEMM so small feature maps still fill the machine: col[(c,r,s)][g*HWo + p].
template <class T>
void im2col(const T* x, T* col, int G, int C, int H, int W, int R, int S, int stride, int pad, int Ho, int Wo) {
    const i64 HWo = static_cast<i64>(Ho) * Wo, ld = G * HWo;
#pragma omp parallel for collapse(2) schedule(static)
    for (int g = 0; g < G; ++g)
        for (int c = 0; c < C; ++c) {
            const T* xc = x + (static_cast<i64>(g) * C + c) * H * W;
            for (int r = 0; r < R; ++r)
                for (int s = 0; s < S; ++s) {
                    T* dst = col + static_cast<i64>((c * R + r) * S + s) * ld + g * HWo;
                    for (int oh = 0; oh < Ho; ++oh) {
                        const int ih = oh * stride - pad + r;
                        for (int ow = 0; ow < Wo; ++ow) {
                            const int iw = ow * stride - pad + s;
                            dst[oh * Wo + ow] = (ih >= 0 && ih < H && iw >= 0 && iw < W) ? xc[static_cast<i64>(ih) * W + iw] : T(0);
                        }
                    }
                }
        }
}

// dx[g, c, ih, iw] = sum over (r, s, oh, ow) that read it of col[(c,r,s)][g*HWo + oh*Wo + ow], fixed order.
template <class T>
void col2im(const T* col, T* dx, int G, int C, int H, int W, int R, int S, int stride, int pad, int Ho, int Wo) {
    const i64 HWo = static_cast<i64>(Ho) * Wo, ld = G * HWo;
#pragma omp parallel for collapse(2) schedule(static)
    for (int g = 0; g < G; ++g)
        for (int c = 0; c < C; ++c) {
            T* xc = dx + (static_cast<i64>(g) * C + c) * H * W;
            std::fill(xc, xc + static_cast<i64>(H) * W, T(0));
            for (int r = 0; r < R; ++r)
                for (int s = 0; s < S; ++s) {
                    const T* src = col + static_cast<i64>((c * R + r) * S + s) * ld + g * HWo;
                    for (int oh = 0; oh < Ho; ++oh) {
                        const int ih = oh * stride - pad + r;
                        if (ih < 0 || ih >= H) continue;
                        for (int ow = 0; ow < Wo; ++ow) {
                            const int iw = ow * stride - pad + s;
                            if (iw >= 0 && iw < W) xc[static_cast<i64>(ih) * W + iw] += src[oh * Wo + ow];
                        }
                    }
                }
        }
}

// Grow-only scratch buffers reused across calls (no page-fault churn per call).
template <class T>
T* scratch(int slot, i64 n) {
    static std::vector<T> bufs[4];
    if (static_cast<i64>(bufs[slot].size()) < n) bufs[slot].resize(n);
    return bufs[slot].data();
}

// Images per GEMM: >= ~16k columns, im2col buffer <= 64M elements.
inline int conv_chunk(i64 CRS, i64 HWo, int N) {
    const i64 want = (16384 + HWo - 1) / HWo;
    const i64 cap = std::max<i64>(1, (static_cast<i64>(64) << 20) / std::max<i64>(1, CRS * HWo));
    return static_cast<int>(std::max<i64>(1, std::min<i64>({want, cap, static_cast<i64>(N)})));
}

// [n][K][HWo] <-> [K][g*HWo] for a chunk of G images
template <class T>
void nk_to_kn(const T* src, T* dst, int G, int K, i64 HWo) {
#pragma omp parallel for collapse(2) schedule(static)
    for (int g = 0; g < G; ++g)
        for (int k = 0; k < K; ++k)
            std::memcpy(dst + static_cast<i64>(k) * G * HWo + g * HWo, src + (static_cast<i64>(g) * K + k) * HWo, sizeof(T) * HWo);
}

template <class T>
void conv_fwd(const T* x, const T* w, const T* b, T* y, int N, int C, int H, int W, int K, int R, int S, int stride,
              int pad, bool direct) {
    const int Ho = (H + 2 * pad - R) / stride + 1, Wo = (W + 2 * pad - S) / stride + 1;
    const i64 CRS = static_cast<i64>(C) * R * S, HWo = static_cast<i64>(Ho) * Wo;
    if (direct) {  // no im2col workspace
#pragma omp parallel for collapse(2) schedule(static)
        for (int n = 0; n < N; ++n)
            for (int k = 0; k < K; ++k)
                for (int oh = 0; oh < Ho; ++oh)
                    for (int ow = 0; ow < Wo; ++ow) {
                        T acc = T(0);
                        for (int c = 0; c < C; ++c)
                            for (int r = 0; r < R; ++r) {
                                const int ih = oh * stride - pad + r;
                                if (ih < 0 || ih >= H) continue;
                                for (int s = 0; s < S; ++s) {
                                    const int iw = ow * stride - pad + s;
                                    if (iw < 0 || iw >= W) continue;
                                    acc += x[((static_cast<i64>(n) * C + c) * H + ih) * W + iw] *
                                           w[((static_cast<i64>(k) * C + c) * R + r) * S + s];
                                }
                            }
                        y[((static_cast<i64>(n) * K + k) * Ho + oh) * Wo + ow] = acc + (b ? b[k] : T(0));
                    }
        return;
    }
    const int G = conv_chunk(CRS, HWo, N);
    T* col = scratch<T>(0, CRS * G * HWo);
    T* out = scratch<T>(1, static_cast<i64>(K) * G * HWo);
    for (int n0 = 0; n0 < N; n0 += G) {
        const int g = std::min(G, N - n0);
        const i64 ld = g * HWo;
        im2col(x + static_cast<i64>(n0) * C * H * W, col, g, C, H, W, R, S, stride, pad, Ho, Wo);
        gemm<T>(K, static_cast<int>(ld), static_cast<int>(CRS), w, CRS, false, col, ld, false, out, ld, false);
#pragma omp parallel for collapse(2) schedule(static)
        for (int i = 0; i < g; ++i)
            for (int k = 0; k < K; ++k) {
                T* yk = y + ((static_cast<i64>(n0) + i) * K + k) * HWo;
                const T* ok = out + static_cast<i64>(k) * ld + i * HWo;
                const T bk = b ? b[k] : T(0);
                for (i64 p = 0; p < HWo; ++p) yk[p] = b ? ok[p] + bk : ok[p];
            }
    }
}

// dx = col2im(W^T dy): dcol[(c,r,s)][g*HWo+p] = sum_k w[k,(c,r,s)] dy[g,k,p]
template <class T>
void conv_bwd_data(const T* dy, const T* w, T* dx, int N, int C, int H, int W, int K, int R, int S, int stride, int pad) {
    const int Ho = (H + 2 * pad - R) / stride + 1, Wo = (W + 2 * pad - S) / stride + 1;
    const i64 CRS = static_cast<i64>(C) * R * S, HWo = static_cast<i64>(Ho) * Wo;
    const int G = conv_chunk(CRS, HWo, N);
    T* dcol = scratch<T>(0, CRS * G * HWo);
    T* dyk = scratch<T>(1, static_cast<i64>(K) * G * HWo);
    for (int n0 = 0; n0 < N; n0 += G) {
        const int g = std::min(G, N - n0);
        const i64 ld = g * HWo;
        nk_to_kn(dy + static_cast<i64>(n0) * K * HWo, dyk, g, K, HWo);
        gemm<T>(static_cast<int>(CRS), static_cast<int>(ld), K, w, CRS, true, dyk, ld, false, dcol, ld, false);
        col2im(dcol, dx + static_cast<i64>(n0) * C * H * W, g, C, H, W, R, S, stride, pad, Ho, Wo);
    }
}

// dw[K, CRS] = sum over images and pixels (ascending) of dy[n,k,p] col[(c,r,s), p]
template <class T>
void conv_bwd_filter(const T* dy, const T* x, T* dw, int N, int C, int H, int W, int K, int R, int S, int stride, int pad) {
    const int Ho = (H + 2 * pad - R) / stride + 1, Wo = (W + 2 * pad - S) / stride + 1;
    const i64 CRS = static_cast<i64>(C) * R * S, HWo = static_cast<i64>(Ho) * Wo;
    const int G = conv_chunk(CRS, HWo, N);
    T* col = scratch<T>(0, CRS * G * HWo);
    T* dyk = scratch<T>(1, static_cast<i64>(K) * G * HWo);
    for (int n0 = 0; n0 < N; n0 += G) {
        const int g = std::min(G, N - n0);
        const i64 ld = g * HWo;
        im2col(x + static_cast<i64>(n0) * C * H * W, col, g, C, H, W, R, S, stride, pad, Ho, Wo);
        nk_to_kn(dy + static_cast<i64>(n0) * K * HWo, dyk, g, K, HWo);
        gemm<T>(K, static_cast<int>(CRS), static_cast<int>(ld), dyk, ld, false, col, ld, true, dw, CRS, n0 > 0);
    }
}

template <class T>
void conv_bwd_bias(const T* dy, T* db, int N, int K, i64 HW) {
#pragma omp parallel for schedule(static)
    for (int k = 0; k < K; ++k) {
        T acc = T(0);
        for (int n = 0; n < N; ++n)
            for (i64 i = 0; i < HW; ++i) acc += dy[(static_cast<i64>(n) * K + k) * HW + i];
        db[k] = acc;
    }
}

// ----------------------------------------------------------------- pooling
// Max: the first maximum in row-major window order wins (strict >); padded
// cells never win.  idx = flat NCHW input index (layout independent).
// Avg: window sum / (k*k) (padded cells count as zeros).
template <class T>
void pool_fwd(const T* x, T* y, int32_t* idx, int N, int C, int H, int W, int k, int stride, int pad, bool is_max) {
    const int Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
#pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < N; ++n)
        for (int c = 0; c < C; ++c) {
            const i64 base = (static_cast<i64>(n) * C + c) * H * W;
            for (int oh = 0; oh < Ho; ++oh)
                for (int ow = 0; ow < Wo; ++ow) {
                    T best = T(0), sum = T(0);
                    i64 bi = -1;
                    for (int r = 0; r < k; ++r) {
                        const int ih = oh * stride - pad + r;
                        if (ih < 0 || ih >= H) continue;
                        for (int s = 0; s < k; ++s) {
                            const int iw = ow * stride - pad + s;
                            if (iw < 0 || iw >= W) continue;
                            const T v = x[base + static_cast<i64>(ih) * W + iw];
                            sum += v;
                            if (bi < 0 || v > best) {
                                best = v;
                                bi = base + static_cast<i64>(ih) * W + iw;
                            }
                        }
                    }
                    const i64 o = ((static_cast<i64>(n) * C + c) * Ho + oh) * Wo + ow;
                    y[o] = is_max ? best : sum / static_cast<T>(k * k);
                    if (idx) idx[o] = static_cast<int32_t>(bi);
                }
        }
}

template <class T>
void pool_bwd(const T* dy, const T* x, T* dx, int N, int C, int H, int W, int k, int stride, int pad, bool is_max) {
    const int Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
    std::vector<int32_t> idx;
    if (is_max) {
        idx.resize(static_cast<size_t>(N) * C * Ho * Wo);
        std::vector<T> tmp(idx.size());
        pool_fwd(x, tmp.data(), idx.data(), N, C, H, W, k, stride, pad, true);
    }
    std::fill(dx, dx + static_cast<i64>(N) * C * H * W, T(0));
    // Each (n, c) plane is independent; windows are visited in a fixed order.
#pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < N; ++n)
        for (int c = 0; c < C; ++c) {
            const i64 ob = (static_cast<i64>(n) * C + c) * Ho * Wo;
            const i64 ib = (static_cast<i64>(n) * C + c) * H * W;
            for (int oh = 0; oh < Ho; ++oh)
                for (int ow = 0; ow < Wo; ++ow) {
                    const i64 o = ob + static_cast<i64>(oh) * Wo + ow;
                    if (is_max) {
                        dx[idx[o]] += dy[o];
                        continue;
                    }
                    const T g = dy[o] / static_cast<T>(k * k);
                    for (int r = 0; r < k; ++r) {
                        const int ih = oh * stride - pad + r;
                        if (ih < 0 || ih >= H) continue;
                        for (int s = 0; s < k; ++s) {
                            const int iw = ow * stride - pad + s;
                            if (iw >= 0 && iw < W) dx[ib + static_cast<i64>(ih) * W + iw] += g;
                        }
                    }
                }
        }
}

// ----------------------------------------------------------------- LRN (Caffe ACROSS_CHANNELS)
//   scale_c = k + alpha/n * sum_{c' in [c - n/2, c + n/2]} a_{c'}^2 ;  b_c = a_c * scale_c^-beta
template <class T>
void lrn_scale(const T* x, std::vector<T>& sc, int N, int C, i64 HW, int size, double alpha, double k) {
    sc.resize(static_cast<size_t>(N) * C * HW);
    const int half = size / 2;
#pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < N; ++n)
        for (i64 p = 0; p < HW; ++p)
            for (int c = 0; c < C; ++c) {
                T acc = T(0);
                for (int cc = std::max(0, c - half); cc <= std::min(C - 1, c + half); ++cc) {
                    const T v = x[(static_cast<i64>(n) * C + cc) * HW + p];
                    acc += v * v;
                }
                sc[(static_cast<i64>(n) * C + c) * HW + p] = static_cast<T>(k) + static_cast<T>(alpha / size) * acc;
            }
}

template <class T>
void lrn_fwd(const T* x, T* y, int N, int C, i64 HW, int size, double alpha, double beta, double k) {
    std::vector<T> sc;
    lrn_scale(x, sc, N, C, HW, size, alpha, k);
    const i64 n_el = static_cast<i64>(N) * C * HW;
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < n_el; ++i) y[i] = x[i] * std::pow(sc[i], static_cast<T>(-beta));
}

// dx_c = dy_c * s_c^-b  -  (2 a b / n) * x_c * sum_{c': c in window(c')} dy_c' * y_c' / s_c'
template <class T>
void lrn_bwd(const T* dy, const T* x, const T* y, T* dx, int N, int C, i64 HW, int size, double alpha, double beta,
             double k) {
    std::vector<T> sc;
    lrn_scale(x, sc, N, C, HW, size, alpha, k);
    const int half = size / 2;
    const T coef = static_cast<T>(2.0 * alpha * beta / size);
#pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < N; ++n)
        for (i64 p = 0; p < HW; ++p)
            for (int c = 0; c < C; ++c) {
                T acc = T(0);
                for (int cc = std::max(0, c - half); cc <= std::min(C - 1, c + half); ++cc) {
                    const i64 j = (static_cast<i64>(n) * C + cc) * HW + p;
                    acc += dy[j] * y[j] / sc[j];
                }
                const i64 i = (static_cast<i64>(n) * C + c) * HW + p;
                dx[i] = dy[i] * std::pow(sc[i], static_cast<T>(-beta)) - coef * x[i] * acc;
            }
}

// ----------------------------------------------------------------- softmax
template <class T>
void softmax_fwd(const T* x, T* y, int rows, int cols) {
#pragma omp parallel for schedule(static)
    for (int r = 0; r < rows; ++r) {
        const T* xr = x + static_cast<i64>(r) * cols;
        T* yr = y + static_cast<i64>(r) * cols;
        T m = xr[0];
        for (int j = 1; j < cols; ++j) m = std::max(m, xr[j]);
        T s = T(0);
        for (int j = 0; j < cols; ++j) s += (yr[j] = std::exp(xr[j] - m));
        for (int j = 0; j < cols; ++j) yr[j] /= s;
    }
}

template <class T>
void softmax_bwd(const T* dy, const T* y, T* dx, int rows, int cols) {
#pragma omp parallel for schedule(static)
    for (int r = 0; r < rows; ++r) {
        const i64 o = static_cast<i64>(r) * cols;
        T d = T(0);
        for (int j = 0; j < cols; ++j) d += dy[o + j] * y[o + j];
        for (int j = 0; j < cols; ++j) dx[o + j] = y[o + j] * (dy[o + j] - d);
    }
}

// ----------------------------------------------------------------- batch norm
// Training-mode batch statistics, biased variance, channel affine.
template <class T>
void bn_stats(const T* x, int N, int C, i64 HW, std::vector<T>& mean, std::vector<T>& istd, double eps) {
    mean.assign(C, T(0));
    istd.assign(C, T(0));
    const T cnt = static_cast<T>(static_cast<i64>(N) * HW);
#pragma omp parallel for schedule(static)
    for (int c = 0; c < C; ++c) {
        T s = T(0);
        for (int n = 0; n < N; ++n)
            for (i64 p = 0; p < HW; ++p) s += x[(static_cast<i64>(n) * C + c) * HW + p];
        const T m = s / cnt;
        T v = T(0);
        for (int n = 0; n < N; ++n)
            for (i64 p = 0; p < HW; ++p) {
                const T d = x[(static_cast<i64>(n) * C + c) * HW + p] - m;
                v += d * d;
            }
        mean[c] = m;
        istd[c] = T(1) / std::sqrt(v / cnt + static_cast<T>(eps));
    }
}

template <class T>
void bn_fwd(const T* x, const T* g, const T* b, T* y, int N, int C, i64 HW, double eps) {
    std::vector<T> mean, istd;
    bn_stats(x, N, C, HW, mean, istd, eps);
#pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < N; ++n)
        for (int c = 0; c < C; ++c)
            for (i64 p = 0; p < HW; ++p) {
                const i64 i = (static_cast<i64>(n) * C + c) * HW + p;
                y[i] = g[c] * (x[i] - mean[c]) * istd[c] + b[c];
            }
}

template <class T>
void bn_bwd(const T* dy, const T* x, const T* g, T* dx, T* dg, T* db, int N, int C, i64 HW, double eps) {
    std::vector<T> mean, istd;
    bn_stats(x, N, C, HW, mean, istd, eps);
    const T cnt = static_cast<T>(static_cast<i64>(N) * HW);
#pragma omp parallel for schedule(static)
    for (int c = 0; c < C; ++c) {
        T sdy = T(0), sdyx = T(0);
        for (int n = 0; n < N; ++n)
            for (i64 p = 0; p < HW; ++p) {
                const i64 i = (static_cast<i64>(n) * C + c) * HW + p;
                sdy += dy[i];
                sdyx += dy[i] * (x[i] - mean[c]) * istd[c];
            }
        if (dg) dg[c] = sdyx;
        if (db) db[c] = sdy;
        if (dx) {
            const T gs = (g ? g[c] : T(1)) * istd[c];
            for (int n = 0; n < N; ++n)
                for (i64 p = 0; p < HW; ++p) {
                    const i64 i = (static_cast<i64>(n) * C + c) * HW + p;
                    const T xh = (x[i] - mean[c]) * istd[c];
                    dx[i] = gs * (dy[i] - sdy / cnt - xh * sdyx / cnt);
                }
        }
    }
}

// ================================================================= plan execution
struct PoolSim {  // best-fit pool, reuse or dealloc mode
    bool reuse = false;
    std::multimap<i64, int> free_blocks;  // bytes -> block id
    std::unordered_map<int, std::pair<int, i64>> held;  // storage -> (block, bytes)
    int next_block = 0;
    orc_pool_stats st{};
    void acquire(int storage, i64 bytes) {
        if (reuse) {
            auto it = free_blocks.lower_bound(bytes);
            if (it != free_blocks.end()) {
                held[storage] = {it->second, it->first};
                free_blocks.erase(it);
                st.reuses++;
                st.live_bytes += bytes;
                st.peak_bytes = std::max(st.peak_bytes, st.live_bytes);
                return;
            }
        }
        held[storage] = {next_block++, bytes};
        st.allocs_from_os++;
        st.os_bytes += bytes;
        st.live_bytes += bytes;
        st.peak_bytes = std::max(st.peak_bytes, st.live_bytes);
    }
    void release(int storage) {
        auto it = held.find(storage);
        if (it == held.end()) return;
        st.releases++;
        st.live_bytes -= it->second.second;
        if (reuse) free_blocks.emplace(it->second.second, it->second.first);
        else st.os_bytes -= it->second.second;
        held.erase(it);
    }
};

i64 count_of(const int64_t* d, int rank) {
    i64 n = 1;
    for (int i = 0; i < rank; ++i) n *= d[i];
    return n;
}

struct Dims {
    int rank = 0;
    int64_t d[4] = {1, 1, 1, 1};
    i64 count() const { return count_of(d, rank); }
    i64 hw() const { return rank == 4 ? d[2] * d[3] : 1; }
};

class CtxBase {
public:
    virtual ~CtxBase() = default;
};

template <class T>
class Exec : public CtxBase {
public:
    Exec(const tc_plan* p, uint64_t seed) : plan_(p), seed_(seed) {
        params_.resize(p->nparams);
        vel_.resize(p->nparams);
        grads_.resize(p->nparams);
        for (int i = 0; i < p->nparams; ++i) {
            const i64 n = count_of(p->params[i].dims, p->params[i].rank);
            params_[i].assign(n, T(0));
            vel_[i].assign(n, T(0));
        }
        for (int i = 0; i < p->nvars; ++i) {
            Dims d;
            d.rank = p->vars[i].rank;
            for (int j = 0; j < d.rank; ++j) d.d[j] = p->vars[i].dims[j];
            vdims_[p->vars[i].id] = d;
        }
        for (int i = 0; i < p->nstmts; ++i)
            if (p->stmts[i].kind == TC_STMT_LET) var_storage_[p->stmts[i].var] = p->stmts[i].storage;
        pool_.reuse = p->mode == TC_MODE_REUSE;
    }

    const tc_plan* plan_;
    uint64_t seed_;
    std::vector<std::vector<T>> params_, vel_, grads_;
    std::unordered_map<int, Dims> vdims_;
    std::unordered_map<int, int> var_storage_;
    std::unordered_map<int, std::vector<T>> store_;
    std::vector<float> bx_;
    std::vector<int32_t> by_;
    bool have_batch_ = false;
    PoolSim pool_;
    std::vector<i64> trace_;
    double ws_cap_mb_ = -1.0;
    int iter_ = 0, n0_ = 0;
    bool prof_ = std::getenv("ORC_PROFILE") != nullptr;  // per-op seconds to stderr at destruction
    double prof_t_[TC_OP_COUNT] = {};
    ~Exec() override {
        if (!prof_) return;
        for (int i = 0; i < TC_OP_COUNT; ++i)
            if (prof_t_[i] > 0) std::fprintf(stderr, "orc op %2d: %.3f s\n", i, prof_t_[i]);
    }
    bool bf16_ = false;  // emulate the device's bf16 activation storage and bf16 GEMM weight operands
    std::unordered_map<int, bool> f32_var_;  // vars the device keeps in fp32 / as masks (not rounded)

    static T round_bf16(T v) {
        float f = static_cast<float>(v);
        uint32_t u;
        std::memcpy(&u, &f, 4);
        if ((u & 0x7f800000u) != 0x7f800000u) u += 0x7fffu + ((u >> 16) & 1u);
        u &= 0xffff0000u;
        std::memcpy(&f, &u, 4);
        return static_cast<T>(f);
    }

    // Device dtype rule (runtime.cu analyze_layouts): loss-head tensors fp32, masks u8, rest bf16.
    void classify_vars() {
        std::unordered_map<int, int> dt;  // 0 bf16, 1 f32, 2 mask
        for (int i = 0; i < plan_->nstmts; ++i) {
            const tc_stmt& s = plan_->stmts[i];
            if (s.kind != TC_STMT_LET) continue;
            int d = 0;
            if (s.op == TC_OP_LOAD_Y || s.op == TC_OP_SOFTMAX_FWD || s.op == TC_OP_LOG || s.op == TC_OP_RECIP) d = 1;
            if (s.op == TC_OP_DROPOUT_MASK) d = 2;
            if (s.op == TC_OP_SCALE || s.op == TC_OP_MUL || s.op == TC_OP_ADD)
                for (int k = 0; k < s.nin; ++k)
                    if (s.in[k].kind == TC_REF_VAR && dt[s.in[k].index] == 1) d = 1;
            dt[s.var] = d;
            f32_var_[s.var] = d != 0;  // not rounded to bf16
        }
    }

    void init_params() {
        for (int i = 0; i < plan_->nparams; ++i) {
            const tc_param_desc& pd = plan_->params[i];
            std::vector<T>& w = params_[i];
            if (pd.init_kind == TC_INIT_CONSTANT) {
                std::fill(w.begin(), w.end(), static_cast<T>(static_cast<float>(pd.init_value)));
            } else if (pd.init_kind == TC_INIT_XAVIER) {
                const double a = std::sqrt(6.0 / static_cast<double>(pd.fan_in + pd.fan_out));
                for (size_t j = 0; j < w.size(); ++j)
                    w[j] = static_cast<T>(static_cast<float>((2.0 * tcp_param_uniform(seed_, i, static_cast<uint32_t>(j)) - 1.0) * a));
            } else {
                for (size_t j = 0; j < w.size(); ++j) {
                    const double u1 = tcp_param_uniform(seed_, i, static_cast<uint32_t>(2 * j));
                    const double u2 = tcp_param_uniform(seed_, i, static_cast<uint32_t>(2 * j + 1));
                    w[j] = static_cast<T>(static_cast<float>(pd.sigma * std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2)));
                }
            }
            std::fill(vel_[i].begin(), vel_[i].end(), T(0));
        }
    }

    std::vector<std::vector<T>> wq_;  // bf16-rounded GEMM weight operands (bf16 emulation)

    const T* get(const tc_ref& r, Dims* d = nullptr) {
        if (r.kind == TC_REF_PARAM) {
            const tc_param_desc& pd = plan_->params[r.index];
            if (d) {
                d->rank = pd.rank;
                for (int j = 0; j < pd.rank; ++j) d->d[j] = pd.dims[j];
            }
            if (bf16_ && pd.rank >= 2) return wq_[r.index].data();
            return params_[r.index].data();
        }
        if (d) *d = vdims_.at(r.index);
        auto it = store_.find(var_storage_.at(r.index));
        if (it == store_.end()) throw std::runtime_error("oracle: read of freed/undefined var X" + std::to_string(r.index));
        return it->second.data();
    }

    // Evaluate the right-hand side of a Let / Update into `out` (shape `od`).
    void eval(const tc_stmt& s, std::vector<T>& out, const Dims& od) {
        out.assign(od.count(), T(0));
        T* y = out.data();
        Dims a, b, c;
        switch (s.op) {
            case TC_OP_LOAD_X:
#pragma omp parallel for schedule(static)
                for (i64 i = 0; i < od.count(); ++i) y[i] = static_cast<T>(bx_[i]);
                return;
            case TC_OP_LOAD_Y:
                for (int n = 0; n < od.d[0]; ++n) y[static_cast<i64>(n) * od.d[1] + by_[n]] = T(1);
                return;
            case TC_OP_CONV_FWD: {
                const T* x = get(s.in[0], &a);
                const T* w = get(s.in[1], &b);
                const T* bias = s.nin > 2 ? get(s.in[2]) : nullptr;
                bool direct = false;
                if (ws_cap_mb_ >= 0) {
                    const double col_mb = 4.0 * a.d[0] * a.d[1] * b.d[2] * b.d[3] * od.d[2] * od.d[3] / 1e6;
                    direct = col_mb > ws_cap_mb_;  // SPEC.md:525 workspace fallback
                }
                conv_fwd(x, w, bias, y, a.d[0], a.d[1], a.d[2], a.d[3], b.d[0], b.d[2], b.d[3], s.stride, s.pad, direct);
                return;
            }
            case TC_OP_CONV_BWD_DATA: {
                const T* dy = get(s.in[0], &a);
                const T* w = get(s.in[1], &b);
                conv_bwd_data(dy, w, y, od.d[0], od.d[1], od.d[2], od.d[3], b.d[0], b.d[2], b.d[3], s.stride, s.pad);
                return;
            }
            case TC_OP_CONV_BWD_FILTER: {
                const T* dy = get(s.in[0], &a);
                const T* x = get(s.in[1], &b);
                conv_bwd_filter(dy, x, y, b.d[0], b.d[1], b.d[2], b.d[3], a.d[1], od.d[2], od.d[3], s.stride, s.pad);
                return;
            }
            case TC_OP_CONV_BWD_BIAS: {
                const T* dy = get(s.in[0], &a);
                conv_bwd_bias(dy, y, a.d[0], a.d[1], a.hw());
                return;
            }
            case TC_OP_POOL_FWD: {
                const T* x = get(s.in[0], &a);
                pool_fwd<T>(x, y, nullptr, a.d[0], a.d[1], a.d[2], a.d[3], s.k, s.stride, s.pad, s.max_pool);
                return;
            }
            case TC_OP_POOL_BWD: {
                const T* dy = get(s.in[0]);
                const T* x = get(s.in[2], &c);
                pool_bwd(dy, x, y, c.d[0], c.d[1], c.d[2], c.d[3], s.k, s.stride, s.pad, s.max_pool);
                return;
            }
            case TC_OP_RELU_FWD: {
                const T* x = get(s.in[0]);
#pragma omp parallel for schedule(static)
                for (i64 i = 0; i < od.count(); ++i) y[i] = x[i] > T(0) ? x[i] : T(0);
                return;
            }
            case TC_OP_RELU_BWD: {
                const T* dy = get(s.in[0]);
                const T* fy = get(s.in[1]);
#pragma omp parallel for schedule(static)
                for (i64 i = 0; i < od.count(); ++i) y[i] = fy[i] > T(0) ? dy[i] : T(0);
                return;
            }
            case TC_OP_SOFTMAX_FWD: softmax_fwd(get(s.in[0]), y, od.d[0], od.d[1]); return;
            case TC_OP_SOFTMAX_BWD: softmax_bwd(get(s.in[0]), get(s.in[1]), y, od.d[0], od.d[1]); return;
            case TC_OP_LRN_FWD: {
                const T* x = get(s.in[0], &a);
                lrn_fwd(x, y, a.d[0], a.d[1], a.hw(), s.lrn_size, s.alpha, s.beta, s.lrn_k);
                return;
            }
            case TC_OP_LRN_BWD: {
                const T* dy = get(s.in[0]);
                const T* fy = get(s.in[1]);
                const T* x = get(s.in[2], &a);
                lrn_bwd(dy, x, fy, y, a.d[0], a.d[1], a.hw(), s.lrn_size, s.alpha, s.beta, s.lrn_k);
                return;
            }
            case TC_OP_DROPOUT_MASK: {
                const i64 per = od.count() / od.d[0];
                for (int n = 0; n < od.d[0]; ++n)
                    for (i64 e = 0; e < per; ++e)
                        y[n * per + e] = static_cast<T>(tcp_dropout_value(seed_, static_cast<uint32_t>(s.var),
                                                                          static_cast<uint32_t>(n0_ + n),
                                                                          static_cast<uint32_t>(iter_),
                                                                          static_cast<uint32_t>(e), static_cast<float>(s.rate)));
                return;
            }
            case TC_OP_MUL: {
                const T* p = get(s.in[0]);
                const T* q = get(s.in[1]);
#pragma omp parallel for schedule(static)
                for (i64 i = 0; i < od.count(); ++i) y[i] = p[i] * q[i];
                return;
            }
            case TC_OP_ADD: {
                const T* p = get(s.in[0]);
                const T* q = get(s.in[1]);
#pragma omp parallel for schedule(static)
                for (i64 i = 0; i < od.count(); ++i) y[i] = p[i] + q[i];
                return;
            }
            case TC_OP_SCALE: {
                const T* p = get(s.in[0]);
#pragma omp parallel for schedule(static)
                for (i64 i = 0; i < od.count(); ++i) y[i] = p[i] * static_cast<T>(s.scale);
                return;
            }
            case TC_OP_LOG: {  // clamp at 1e-30 before Log
                const T* p = get(s.in[0]);
#pragma omp parallel for schedule(static)
                for (i64 i = 0; i < od.count(); ++i) y[i] = std::log(std::max(p[i], static_cast<T>(1e-30)));
                return;
            }
            case TC_OP_RECIP: {
                const T* p = get(s.in[0]);
#pragma omp parallel for schedule(static)
                for (i64 i = 0; i < od.count(); ++i) y[i] = T(1) / std::max(p[i], static_cast<T>(1e-30));
                return;
            }
            case TC_OP_MATMUL_FWD: {  // Y[N,out] = A[N,in] W[out,in]^T
                const T* A = get(s.in[0], &a);
                const T* W = get(s.in[1], &b);
                const int in = static_cast<int>(b.d[1]);
                gemm<T>(static_cast<int>(od.d[0]), static_cast<int>(od.d[1]), in, A, in, false, W, in, true, y, od.d[1], false);
                return;
            }
            case TC_OP_MATMUL_BWD_DATA: {  // dA[N,in] = up[N,out] W[out,in]
                const T* up = get(s.in[0], &a);
                const T* W = get(s.in[1], &b);
                gemm<T>(static_cast<int>(a.d[0]), static_cast<int>(b.d[1]), static_cast<int>(b.d[0]), up, a.d[1], false, W,
                        b.d[1], false, y, b.d[1], false);
                return;
            }
            case TC_OP_MATMUL_BWD_W: {  // dW[out,in] = up[N,out]^T A[N,in]
                const T* up = get(s.in[0], &a);
                const T* A = get(s.in[1], &b);
                const i64 in = b.count() / b.d[0];
                gemm<T>(static_cast<int>(a.d[1]), static_cast<int>(in), static_cast<int>(a.d[0]), up, a.d[1], true, A, in,
                        false, y, in, false);
                return;
            }
            case TC_OP_BIAS_ADD: {
                const T* x = get(s.in[0], &a);
                const T* bb = get(s.in[1]);
                const i64 C = a.d[1], hw = a.hw();
#pragma omp parallel for schedule(static)
                for (i64 i = 0; i < od.count(); ++i) y[i] = x[i] + bb[(i / hw) % C];
                return;
            }
            case TC_OP_BIAS_GRAD: {
                const T* up = get(s.in[0], &a);
                conv_bwd_bias(up, y, static_cast<int>(a.d[0]), static_cast<int>(a.d[1]), a.hw());
                return;
            }
            case TC_OP_CONCAT: {
                i64 off = 0;
                for (int t = 0; t < s.nin; ++t) {
                    const T* p = get(s.in[t], &a);
                    const i64 C = a.d[1], hw = a.hw();
                    for (int n = 0; n < od.d[0]; ++n)
                        std::memcpy(y + (n * od.d[1] + off) * hw, p + n * C * hw, sizeof(T) * C * hw);
                    off += C;
                }
                return;
            }
            case TC_OP_CONCAT_BWD: {
                const T* up = get(s.in[0], &a);
                const i64 hw = a.hw();
                for (int n = 0; n < od.d[0]; ++n)
                    std::memcpy(y + n * s.extent * hw, up + (n * a.d[1] + s.offset) * hw, sizeof(T) * s.extent * hw);
                return;
            }
            case TC_OP_BN_FWD: {
                const T* x = get(s.in[0], &a);
                bn_fwd(x, get(s.in[1]), get(s.in[2]), y, a.d[0], a.d[1], a.hw(), s.eps);
                return;
            }
            case TC_OP_BN_BWD_DATA: {
                const T* up = get(s.in[0]);
                const T* x = get(s.in[1], &a);
                bn_bwd<T>(up, x, get(s.in[2]), y, nullptr, nullptr, a.d[0], a.d[1], a.hw(), s.eps);
                return;
            }
            case TC_OP_BN_BWD_GAMMA: {
                const T* up = get(s.in[0]);
                const T* x = get(s.in[1], &a);
                bn_bwd<T>(up, x, nullptr, nullptr, y, nullptr, a.d[0], a.d[1], a.hw(), s.eps);
                return;
            }
            case TC_OP_BN_BWD_BETA: {
                const T* up = get(s.in[0], &a);
                conv_bwd_bias(up, y, static_cast<int>(a.d[0]), static_cast<int>(a.d[1]), a.hw());
                return;
            }
            default: throw std::runtime_error("oracle: unsupported op " + std::to_string(s.op));
        }
    }

    double step(int iter, int n0, bool update, bool keep) {
        iter_ = iter;
        n0_ = n0;
        if (!have_batch_) synth(iter, n0);
        have_batch_ = false;
        store_.clear();
        pool_.held.clear();
        pool_.st.live_bytes = 0;
        trace_.clear();
        if (bf16_) {
            if (f32_var_.empty()) classify_vars();
            wq_.assign(params_.size(), {});
            for (size_t i = 0; i < params_.size(); ++i)
                if (plan_->params[i].rank >= 2) {
                    wq_[i] = params_[i];
                    for (auto& v : wq_[i]) v = round_bf16(v);
                }
        }
        double loss = 0.0;
        std::vector<T> tmp;
        std::vector<const tc_stmt*> clipped;
        for (int i = 0; i < plan_->nstmts; ++i) {
            const tc_stmt& s = plan_->stmts[i];
            switch (s.kind) {
                case TC_STMT_LET: {
                    Dims od;
                    od.rank = s.rank;
                    for (int j = 0; j < s.rank; ++j) od.d[j] = s.dims[j];
                    const double t0 = prof_ ? omp_get_wtime() : 0.0;
                    eval(s, tmp, od);
                    if (prof_) prof_t_[s.op] += omp_get_wtime() - t0;
                    if (bf16_ && !f32_var_[s.var])
                        for (auto& v : tmp) v = round_bf16(v);
                    if (!s.inplace) pool_.acquire(s.storage, od.count() * 4);
                    store_[s.storage].swap(tmp);  // in place: same storage, new contents
                    break;
                }
                case TC_STMT_DEALLOC:
                    if (!keep) store_.erase(s.storage);
                    pool_.release(s.storage);
                    break;
                case TC_STMT_UPDATE: {
                    const tc_param_desc& pd = plan_->params[s.param];
                    Dims od;
                    od.rank = pd.rank;
                    for (int j = 0; j < pd.rank; ++j) od.d[j] = pd.dims[j];
                    const double t0 = prof_ ? omp_get_wtime() : 0.0;
                    eval(s, tmp, od);
                    if (prof_) prof_t_[s.op] += omp_get_wtime() - t0;
                    grads_[s.param] = tmp;
                    if (update && plan_->clip > 0) {
                        clipped.push_back(&s);  // applied after the whole gradient is known
                    } else if (update) {
                        // v = momentum*v + lr_alpha*(g + decay*p); p = p + v
                        std::vector<T>& p = params_[s.param];
                        std::vector<T>& v = vel_[s.param];
                        for (size_t j = 0; j < p.size(); ++j) {
                            v[j] = static_cast<T>(s.momentum) * v[j] + static_cast<T>(s.lr_alpha) * (tmp[j] + static_cast<T>(s.decay) * p[j]);
                            p[j] += v[j];
                        }
                    }
                    break;
                }
                case TC_STMT_PRINT: {
                    double l = 0.0;
                    for (int t = 0; t < s.nterms; ++t) {
                        Dims d;
                        const T* yv = get(s.in[2 * t], &d);
                        const T* lv = get(s.in[2 * t + 1]);
                        double dot = 0.0;
                        for (i64 j = 0; j < d.count(); ++j) dot += static_cast<double>(yv[j]) * static_cast<double>(lv[j]);
                        l += s.coef[t] * dot;
                    }
                    loss = l;
                    break;
                }
            }
            trace_.push_back(pool_.st.live_bytes);
        }
        if (!clipped.empty()) {
            // g' = clip(g + decay p), clip = global L2-norm scaling over the
            // concatenated gradient: g' *= min(1, clip / ||g'||_2)
            double ss = 0.0;
            for (const tc_stmt* u : clipped) {
                const std::vector<T>& g = grads_[u->param];
                const std::vector<T>& p = params_[u->param];
                for (size_t j = 0; j < p.size(); ++j) {
                    const double gr = static_cast<double>(g[j] + static_cast<T>(u->decay) * p[j]);
                    ss += gr * gr;
                }
            }
            const double norm = std::sqrt(ss);
            const T sc = norm > plan_->clip ? static_cast<T>(plan_->clip / norm) : T(1);
            last_clip_norm_ = norm;
            for (const tc_stmt* u : clipped) {
                const std::vector<T>& g = grads_[u->param];
                std::vector<T>& p = params_[u->param];
                std::vector<T>& v = vel_[u->param];
                for (size_t j = 0; j < p.size(); ++j) {
                    v[j] = static_cast<T>(u->momentum) * v[j] + static_cast<T>(u->lr_alpha) * (sc * (g[j] + static_cast<T>(u->decay) * p[j]));
                    p[j] += v[j];
                }
            }
        }
        return loss;
    }
    double last_clip_norm_ = 0.0;

    double test(int iter, int n0) {
        iter_ = iter;
        n0_ = n0;
        if (!have_batch_) synth(iter, n0);
        have_batch_ = false;
        store_.clear();
        std::vector<T> tmp;
        for (int i = 0; i < plan_->ntest; ++i) {
            const tc_stmt& s = plan_->test_stmts[i];
            Dims od;
            od.rank = s.rank;
            for (int j = 0; j < s.rank; ++j) od.d[j] = s.dims[j];
            if (s.op == TC_OP_DROPOUT_MASK) {  // test-mode dropout = identity
                tmp.assign(od.count(), T(1));
            } else {
                eval(s, tmp, od);
            }
            store_[s.storage].swap(tmp);
        }
        Dims d;
        const T* lg = get(tc_ref{TC_REF_VAR, plan_->logits_var}, &d);
        int hit = 0;
        for (int n = 0; n < d.d[0]; ++n) {
            const T* r = lg + n * d.d[1];
            const int am = static_cast<int>(std::max_element(r, r + d.d[1]) - r);
            hit += am == by_[n];
        }
        return static_cast<double>(hit) / static_cast<double>(d.d[0]);
    }

    void synth(int iter, int n0) {
        const i64 per = plan_->input_dims[1] * plan_->input_dims[2] * plan_->input_dims[3];
        bx_.resize(plan_->batch * per);
        by_.resize(plan_->batch);
        orc_synth_batch(plan_, seed_, iter, n0, bx_.data(), by_.data());
    }
};

struct Holder {
    std::unique_ptr<Exec<float>> f;
    std::unique_ptr<Exec<double>> d;
};

}  // namespace

struct orc_ctx {
    Holder h;
};

template <class Fn>
static auto with(orc_ctx* c, Fn&& fn) {
    return c->h.f ? fn(*c->h.f) : fn(*c->h.d);
}

extern "C" {

#define ORC_DEF(T, sfx)                                                                                          \
    void orc_conv_fwd_##sfx(const T* x, const T* w, const T* b, T* y, int N, int C, int H, int W, int K, int R,   \
                            int S, int stride, int pad, int direct) {                                            \
        conv_fwd(x, w, b, y, N, C, H, W, K, R, S, stride, pad, direct != 0);                                     \
    }                                                                                                            \
    void orc_conv_bwd_data_##sfx(const T* dy, const T* w, T* dx, int N, int C, int H, int W, int K, int R, int S, \
                                 int stride, int pad) {                                                          \
        conv_bwd_data(dy, w, dx, N, C, H, W, K, R, S, stride, pad);                                              \
    }                                                                                                            \
    void orc_conv_bwd_filter_##sfx(const T* dy, const T* x, T* dw, int N, int C, int H, int W, int K, int R,      \
                                   int S, int stride, int pad) {                                                 \
        conv_bwd_filter(dy, x, dw, N, C, H, W, K, R, S, stride, pad);                                            \
    }                                                                                                            \
    void orc_conv_bwd_bias_##sfx(const T* dy, T* db, int N, int K, int HW) { conv_bwd_bias(dy, db, N, K, HW); }   \
    void orc_pool_fwd_##sfx(const T* x, T* y, int32_t* idx, int N, int C, int H, int W, int k, int stride,        \
                            int pad, int is_max) {                                                               \
        pool_fwd(x, y, idx, N, C, H, W, k, stride, pad, is_max != 0);                                            \
    }                                                                                                            \
    void orc_pool_bwd_##sfx(const T* dy, const T* x, T* dx, int N, int C, int H, int W, int k, int stride,        \
                            int pad, int is_max) {                                                               \
        pool_bwd(dy, x, dx, N, C, H, W, k, stride, pad, is_max != 0);                                            \
    }                                                                                                            \
    void orc_lrn_fwd_##sfx(const T* x, T* y, int N, int C, int HW, int size, double alpha, double beta,          \
                           double k) {                                                                           \
        lrn_fwd(x, y, N, C, HW, size, alpha, beta, k);                                                           \
    }                                                                                                            \
    void orc_lrn_bwd_##sfx(const T* dy, const T* x, const T* y, T* dx, int N, int C, int HW, int size,           \
                           double alpha, double beta, double k) {                                                \
        lrn_bwd(dy, x, y, dx, N, C, HW, size, alpha, beta, k);                                                   \
    }                                                                                                            \
    void orc_softmax_fwd_##sfx(const T* x, T* y, int rows, int cols) { softmax_fwd(x, y, rows, cols); }           \
    void orc_softmax_bwd_##sfx(const T* dy, const T* y, T* dx, int rows, int cols) {                              \
        softmax_bwd(dy, y, dx, rows, cols);                                                                      \
    }                                                                                                            \
    void orc_bn_fwd_##sfx(const T* x, const T* g, const T* b, T* y, int N, int C, int HW, double eps) {          \
        bn_fwd(x, g, b, y, N, C, HW, eps);                                                                       \
    }                                                                                                            \
    void orc_bn_bwd_##sfx(const T* dy, const T* x, const T* g, T* dx, T* dg, T* dbeta, int N, int C, int HW,      \
                          double eps) {                                                                          \
        bn_bwd(dy, x, g, dx, dg, dbeta, N, C, HW, eps);                                                          \
    }                                                                                                            \
    void orc_matmul_##sfx(const T* A, const T* B, T* C, int M, int N, int K, int ta, int tb) {                   \
        gemm<T>(M, N, K, A, ta ? M : K, ta != 0, B, tb ? K : N, tb != 0, C, N, false);                            \
    }

ORC_DEF(float, f32)
ORC_DEF(double, f64)
#undef ORC_DEF

struct LoadedPlan {
    tc_plan plan{};
    std::string name;
    std::vector<tc_param_desc> params;
    std::vector<tc_stmt> stmts, test;
    std::vector<tc_var_desc> vars;
};

tc_plan* orc_plan_load(const char* path) {
    FILE* f = std::fopen(path, "rb");
    if (!f) {
        std::fprintf(stderr, "orc_plan_load: cannot open %s\n", path);
        return nullptr;
    }
    auto lp = std::make_unique<LoadedPlan>();
    bool ok = true;
    auto get = [&](void* d, size_t n) { ok = ok && std::fread(d, 1, n, f) == n; };
    uint32_t hdr[6] = {};
    get(hdr, sizeof hdr);
    if (!ok || hdr[0] != 0x4c504354u || hdr[1] != 1u || hdr[2] != sizeof(tc_stmt) || hdr[3] != sizeof(tc_param_desc) ||
        hdr[4] != sizeof(tc_var_desc) || hdr[5] != TC_MAX_IN) {
        std::fprintf(stderr, "orc_plan_load: %s is not a TCPL v1 plan of this ABI\n", path);
        std::fclose(f);
        return nullptr;
    }
    char name[64];
    get(name, sizeof name);
    name[63] = 0;
    lp->name = name;
    int64_t head[6];
    get(head, sizeof head);
    int32_t counts[7];
    get(counts, sizeof counts);
    double solver[4];
    get(solver, sizeof solver);
    if (!ok || counts[0] < 0 || counts[1] < 0 || counts[2] < 0 || counts[4] < 0) {
        std::fclose(f);
        return nullptr;
    }
    lp->params.resize(counts[0]);
    lp->stmts.resize(counts[1]);
    lp->test.resize(counts[2]);
    lp->vars.resize(counts[4]);
    get(lp->params.data(), sizeof(tc_param_desc) * lp->params.size());
    get(lp->stmts.data(), sizeof(tc_stmt) * lp->stmts.size());
    get(lp->test.data(), sizeof(tc_stmt) * lp->test.size());
    get(lp->vars.data(), sizeof(tc_var_desc) * lp->vars.size());
    std::fclose(f);
    if (!ok) {
        std::fprintf(stderr, "orc_plan_load: %s is truncated\n", path);
        return nullptr;
    }
    tc_plan& p = lp->plan;
    p.name = lp->name.c_str();
    p.batch = head[0];
    p.classes = head[1];
    for (int i = 0; i < 4; ++i) p.input_dims[i] = head[2 + i];
    p.nparams = counts[0];
    p.params = lp->params.data();
    p.nstmts = counts[1];
    p.stmts = lp->stmts.data();
    p.ntest = counts[2];
    p.test_stmts = lp->test.data();
    p.logits_var = counts[3];
    p.nvars = counts[4];
    p.vars = lp->vars.data();
    p.max_var = counts[5];
    p.mode = counts[6];
    p.lr = solver[0];
    p.momentum = solver[1];
    p.decay = solver[2];
    p.clip = solver[3];
    return &lp.release()->plan;  // plan is the first member: orc_plan_free recovers the owner
}

void orc_plan_free(tc_plan* plan) { delete reinterpret_cast<LoadedPlan*>(plan); }
int orc_plan_param_dims(const tc_plan* plan, int i, int64_t* out) {
    if (i < 0 || i >= plan->nparams) return -1;
    for (int j = 0; j < 4; ++j) out[j] = j < plan->params[i].rank ? plan->params[i].dims[j] : 1;
    return plan->params[i].rank;
}
void orc_plan_input_dims(const tc_plan* plan, int64_t* out) {
    for (int j = 0; j < 4; ++j) out[j] = plan->input_dims[j];
}

orc_ctx* orc_create(const tc_plan* plan, uint64_t seed, int f64, int threads) {
    if (threads > 0) omp_set_num_threads(threads);
    auto* c = new orc_ctx;
    if (f64) c->h.d = std::make_unique<Exec<double>>(plan, seed);
    else c->h.f = std::make_unique<Exec<float>>(plan, seed);
    return c;
}
void orc_destroy(orc_ctx* c) { delete c; }

void orc_init_params(orc_ctx* c) {
    with(c, [](auto& e) { e.init_params(); return 0; });
}
void orc_param_get(orc_ctx* c, int i, float* out) {
    with(c, [&](auto& e) { for (size_t j = 0; j < e.params_[i].size(); ++j) out[j] = static_cast<float>(e.params_[i][j]); return 0; });
}
void orc_param_set(orc_ctx* c, int i, const float* in) {
    with(c, [&](auto& e) { for (size_t j = 0; j < e.params_[i].size(); ++j) e.params_[i][j] = in[j]; return 0; });
}
void orc_param_get_f64(orc_ctx* c, int i, double* out) {
    with(c, [&](auto& e) { for (size_t j = 0; j < e.params_[i].size(); ++j) out[j] = static_cast<double>(e.params_[i][j]); return 0; });
}
void orc_param_set_f64(orc_ctx* c, int i, const double* in) {
    with(c, [&](auto& e) {
        using T = typename std::decay_t<decltype(e.params_[0])>::value_type;
        for (size_t j = 0; j < e.params_[i].size(); ++j) e.params_[i][j] = static_cast<T>(in[j]);
        return 0;
    });
}
void orc_velocity_get(orc_ctx* c, int i, float* out) {
    with(c, [&](auto& e) { for (size_t j = 0; j < e.vel_[i].size(); ++j) out[j] = static_cast<float>(e.vel_[i][j]); return 0; });
}

void orc_synth_batch(const tc_plan* plan, uint64_t seed, int iter, int n0, float* x, int32_t* labels) {
    const i64 per = plan->input_dims[1] * plan->input_dims[2] * plan->input_dims[3];
    const uint32_t K = static_cast<uint32_t>(plan->classes);
#pragma omp parallel for schedule(static)
    for (int n = 0; n < static_cast<int>(plan->batch); ++n) {
        const uint32_t ng = static_cast<uint32_t>(n0 + n);
        const uint32_t y = tcp_label(seed, ng, static_cast<uint32_t>(iter), K);
        labels[n] = static_cast<int32_t>(y);
        for (i64 e = 0; e < per; ++e) {
            float u1, u2;
            tcp_uniform_pair(seed, ng, static_cast<uint32_t>(iter), static_cast<uint32_t>(e), &u1, &u2);
            const double r = std::sqrt(-2.0 * std::log(static_cast<double>(u1)));
            const double t = 6.283185307179586 * static_cast<double>(u2);
            const double z = (e & 1) ? r * std::sin(t) : r * std::cos(t);
            x[n * per + e] = static_cast<float>(static_cast<double>(tcp_centroid(seed, y, static_cast<uint32_t>(e))) + 0.1 * z);
        }
    }
}

void orc_set_batch(orc_ctx* c, const float* x, const int32_t* labels) {
    with(c, [&](auto& e) {
        const i64 per = e.plan_->input_dims[1] * e.plan_->input_dims[2] * e.plan_->input_dims[3];
        e.bx_.assign(x, x + e.plan_->batch * per);
        e.by_.assign(labels, labels + e.plan_->batch);
        e.have_batch_ = true;
        return 0;
    });
}

double orc_step(orc_ctx* c, int iter, int n0, int update, int keep) {
    try {
        return with(c, [&](auto& e) { return e.step(iter, n0, update != 0, keep != 0); });
    } catch (const std::exception& ex) {
        std::fprintf(stderr, "orc_step: %s\n", ex.what());
        return std::nan("");
    }
}
double orc_test(orc_ctx* c, int iter, int n0) {
    return with(c, [&](auto& e) { return e.test(iter, n0); });
}

int orc_var_get(orc_ctx* c, int var, float* out, int64_t max_elems) {
    return with(c, [&](auto& e) -> int {
        auto si = e.var_storage_.find(var);
        if (si == e.var_storage_.end()) return -1;
        auto it = e.store_.find(si->second);
        if (it == e.store_.end()) return -2;
        const i64 n = std::min<i64>(max_elems, static_cast<i64>(it->second.size()));
        for (i64 j = 0; j < n; ++j) out[j] = static_cast<float>(it->second[j]);
        return static_cast<int>(n);
    });
}

int orc_grad_get(orc_ctx* c, int index, double* out, int64_t max_elems) {
    return with(c, [&](auto& e) -> int {
        const auto& g = e.grads_[index];
        const i64 n = std::min<i64>(max_elems, static_cast<i64>(g.size()));
        for (i64 j = 0; j < n; ++j) out[j] = static_cast<double>(g[j]);
        return static_cast<int>(n);
    });
}

void orc_pool_stats_get(orc_ctx* c, orc_pool_stats* s) {
    with(c, [&](auto& e) { *s = e.pool_.st; return 0; });
}

int orc_live_trace(orc_ctx* c, int64_t* out, int max) {
    return with(c, [&](auto& e) -> int {
        const int n = std::min<int>(max, static_cast<int>(e.trace_.size()));
        for (int j = 0; j < n; ++j) out[j] = e.trace_[j];
        return n;
    });
}

void orc_set_workspace_cap(orc_ctx* c, double mb) {
    with(c, [&](auto& e) { e.ws_cap_mb_ = mb; return 0; });
}

void orc_set_bf16_storage(orc_ctx* c, int on) {
    with(c, [&](auto& e) { e.bf16_ = on != 0; return 0; });
}

}  // extern "C"
