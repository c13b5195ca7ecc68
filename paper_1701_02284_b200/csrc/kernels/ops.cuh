// Bandwidth-bound kernels of the training step (everything that is not a
// contraction).  Device layouts (tc_abi.h): 4-D activations NHWC bf16 with
// channel stride cs (multiple of 8, pad channels kept at zero); 2-D
// activations [N][Fs] bf16 (Fs = ceil8(F)); loss-head tensors fp32 [N][F];
// dropout keep-masks uint8.  Every kernel is deterministic: reductions use a
// fixed partition and a fixed summation order.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "tc_abi.h"

namespace tcb {

using bf16 = __nv_bfloat16;

struct Act4 {  // NHWC activation view
    int N, H, W, C, cs;
    __host__ __device__ long long pixels() const { return static_cast<long long>(N) * H * W; }
    __host__ __device__ long long elems() const { return pixels() * cs; }
};

tc_status launch_relu_fwd(const bf16* x, bf16* y, long long n, cudaStream_t st);
tc_status launch_relu_bwd(const bf16* dy, const bf16* y, bf16* dx, long long n, cudaStream_t st);
// y = a + b (then max(y, 0) when relu: a residual add followed by an in-place ReLU)
tc_status launch_add_bf16(const bf16* a, const bf16* b, bf16* y, long long n, int relu, cudaStream_t st);
// y = x * keep * scale (inverted dropout; keep is a 0/1 byte mask)
tc_status launch_mask_mul(const bf16* x, const uint8_t* keep, float scale, bf16* y, long long n, cudaStream_t st);
// keep[n, e] for every stored element; e = NCHW element index within the sample (tc_philox.h)
tc_status launch_dropout_mask(uint8_t* keep, int N, int H, int W, int C, int cs, float rate, uint64_t seed,
                              uint32_t var, const uint32_t* iter_n0, cudaStream_t st);

// Max pooling argmax: 1 byte per output element, window-local position r*k + s (255 = empty).
tc_status launch_pool_fwd(const bf16* x, Act4 xi, bf16* y, Act4 yo, uint8_t* idx, int k, int stride, int pad,
                          int is_max, cudaStream_t st);
tc_status launch_pool_bwd(const bf16* dy, Act4 yo, const uint8_t* idx, bf16* dx, Act4 xi, int k, int stride, int pad,
                          int is_max, cudaStream_t st);
tc_status launch_lrn_fwd(const bf16* x, bf16* y, Act4 a, int size, float alpha, float beta, float k, cudaStream_t st);
tc_status launch_lrn_bwd(const bf16* dy, const bf16* x, const bf16* y, bf16* dx, Act4 a, int size, float alpha,
                         float beta, float k, cudaStream_t st);

// rows x F, input bf16 with row stride in_ld -> fp32 out (stride F)
tc_status launch_softmax_fwd(const bf16* x, long long in_ld, float* y, int rows, int F, cudaStream_t st);
// dx (bf16, stride out_ld, pad columns zeroed) = y * (dy - sum(dy*y))
tc_status launch_softmax_bwd(const float* dy, const float* y, bf16* dx, long long out_ld, int rows, int F,
                             cudaStream_t st);

enum F32Op { F32_LOG = 0, F32_RECIP = 1, F32_SCALE = 2, F32_MUL = 3, F32_ADD = 4 };
tc_status launch_f32_ew(int op, const float* a, const float* b, float scale, float* y, long long n, cudaStream_t st);
tc_status launch_onehot(const int32_t* labels, float* y, int N, int K, cudaStream_t st);
// loss = sum_t coef[t] * dot(a[t], b[t]) over n[t] elements -> *out (fp32 device scalar).
// `out` must point at >= 512 zero-initialised bytes (reduction partials + ticket follow the scalar).
tc_status launch_loss(const float* const* a, const float* const* b, const long long* n, const double* coef, int nterms,
                      float* out, cudaStream_t st);

// Column sums of a [rows][ld] bf16 matrix over its first `cols` columns -> out[cols] fp32 (deterministic).
tc_status launch_colsum(const bf16* x, long long rows, int cols, long long ld, float* out, float* partials,
                        int max_partials, cudaStream_t st);
size_t colsum_partials_floats(int cols);
tc_status launch_bias_add(const bf16* x, const float* b, bf16* y, long long rows, int cols, long long ld, int relu,
                          cudaStream_t st);

// Concat: copy `c` channels of src (stride src_cs) into dst channel offset `off` (stride dst_cs).
tc_status launch_channel_copy(const bf16* src, int src_cs, bf16* dst, int dst_cs, int off, int c, long long pixels,
                              cudaStream_t st);
tc_status launch_zero(void* p, size_t bytes, cudaStream_t st);

// BatchNorm over NHWC [pixels][cs] (training-mode batch statistics, biased variance):
// stats = (mean[C], istd[C]); y = gamma * (x - mean) * istd + beta (then max(y, 0) when relu: the
// in-place ReLU that follows a BN is folded into the apply pass).
// `partials` holds max_partials floats of reduction scratch plus 3*C coefficient floats.
tc_status launch_bn_fwd(const bf16* x, const float* gamma, const float* beta, bf16* y, float* stats, long long pixels,
                        int C, int cs, float eps, int relu, float* partials, int max_partials, cudaStream_t st);
// sums = (sum dy[C], sum dy * xhat[C]) — shared by dgamma (= sum dy*xhat), dbeta (= sum dy) and dx
tc_status launch_bn_bwd_reduce(const bf16* dy, const bf16* x, const float* stats, float* sums, long long pixels, int C,
                               int cs, float* partials, int max_partials, cudaStream_t st);
tc_status launch_bn_bwd_apply(const bf16* dy, const bf16* x, const float* gamma, const float* stats, const float* sums,
                              bf16* dx, long long pixels, int C, int cs, float* partials, int max_partials,
                              cudaStream_t st);

// Dense im2col for small-channel (first-layer) convolutions: col[m][kk], m = (n, oh, ow),
// kk = (kh, kw, c) over the REAL channels C, zero-padded to Kp (multiple of 8).
tc_status launch_im2col(const bf16* x, Act4 xi, int R, int S, int stride, int pad, int Ho, int Wo, int Kp, bf16* col,
                        cudaStream_t st);

// Device layout of the staged input image.  s2d = 0: NHWC bf16 with channel stride cs.
// s2d = s > 0 (space-to-depth for a stride-s first-layer conv): [N][Hs][Ws][s*s*cs] with
// element (P, Q, (i*s + j)*cs + c) = x(n, c, s*P + i - pad, s*Q + j - pad) (0 outside).
struct StageLayout {
    int N, C, H, W, cs;
    int s2d, pad, Hs, Ws;
    __host__ __device__ long long elems() const {
        return s2d ? static_cast<long long>(N) * Hs * Ws * s2d * s2d * cs : static_cast<long long>(N) * H * W * cs;
    }
};
// Input staging: NCHW fp32 -> the staged layout (bf16, pads zero).
tc_status launch_nchw_to_nhwc(const float* x, bf16* y, StageLayout L, cudaStream_t st);
// Synthetic batch generated on the device (identical law to oracle/tc_philox.h).
tc_status launch_synth_batch(bf16* x, int32_t* labels, StageLayout L, int classes, uint64_t seed, uint32_t iter,
                             uint32_t n0, cudaStream_t st);
// Space-to-depth filter gradient [K][ld]: zero the taps outside the original R x S window
// (column (a*Rp + b)*s*s*cs + (i*s + j)*cs + c is tap (s*a + i, s*b + j)).
tc_status launch_s2d_mask_grad(float* g, int K, long long ld, int Rp, int s, int cs, int R, int S, cudaStream_t st);

// Momentum SGD: v = mom*v + lr_alpha*(g + decay*p); p += v;
// refreshes the bf16 shadow(s) used as GEMM operands.
struct SgdTensor {
    float* p;
    float* v;
    const float* g;
    long long n;
    bf16* shadow;        // same layout as p (may be null)
    bf16* shadow_rskc;   // conv filters: [R][S][ks][cs] copy for bwd-data (may be null)
    int K, RS, cs, ks;   // shape info for the RSKC scatter (p is [K][RS][cs])
    float lr_alpha, momentum, decay;
};
tc_status launch_sgd(const SgdTensor* ts, int nt, SgdTensor* dev_scratch, cudaStream_t st);

// d_iter[0] = iter, d_iter[1] = n0 (kernel arguments travel with the launch: no host sync)
tc_status launch_set_iter(uint32_t* d_iter, uint32_t iter, uint32_t n0, cudaStream_t st);

}  // namespace tcb
