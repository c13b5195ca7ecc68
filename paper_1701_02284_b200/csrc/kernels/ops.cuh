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

// Activation launchers are templates on the storage type T: bf16 (default) or float (the fp32
// parity precision mode); both are instantiated in ops.cu.
template <typename T>
tc_status launch_relu_fwd(const T* x, T* y, long long n, cudaStream_t st);
template <typename T>
tc_status launch_relu_bwd(const T* dy, const T* y, T* dx, long long n, cudaStream_t st);
// y = a + b (then max(y, 0) when relu: a residual add followed by an in-place ReLU)
template <typename T>
tc_status launch_add(const T* a, const T* b, T* y, long long n, int relu, cudaStream_t st, const T* relu_y = nullptr);
// y = x * keep * scale (inverted dropout; keep is a 0/1 byte mask)
template <typename T>
tc_status launch_mask_mul(const T* x, const uint8_t* keep, float scale, T* y, long long n, cudaStream_t st,
                          const T* relu_y = nullptr);
// mask + product in one pass (the DropoutMask statement folded into its forward product)
template <typename T>
tc_status launch_dropout_apply(const T* x, uint8_t* keep, T* y, int N, int H, int W, int C, int cs, float rate,
                               uint64_t seed, uint32_t var, const uint32_t* iter_n0, cudaStream_t st);
// keep[n, e] for every stored element; e = NCHW element index within the sample (tc_philox.h)
tc_status launch_dropout_mask(uint8_t* keep, int N, int H, int W, int C, int cs, float rate, uint64_t seed,
                              uint32_t var, const uint32_t* iter_n0, cudaStream_t st);

// Max pooling argmax: 1 byte per output element, window-local position r*k + s (255 = empty).
// flag_nonpos (k*k <= 127): the pooling input is a ReLU output whose backward is folded into the
// pooling backward; a window whose maximum is <= 0 gets bit 7 set, so it routes no gradient
// (the ReLU mask at the argmax) and the backward never reads the ReLU output.
template <typename T>
tc_status launch_pool_fwd(const T* x, Act4 xi, T* y, Act4 yo, uint8_t* idx, int k, int stride, int pad, int is_max,
                          int flag_nonpos, cudaStream_t st);
// relu_y (may be null): the ReLU output feeding the pooling; dx *= [relu_y > 0] (ReLU backward folded in)
template <typename T>
tc_status launch_pool_bwd(const T* dy, Act4 yo, const uint8_t* idx, T* dx, Act4 xi, int k, int stride, int pad,
                          int is_max, const T* relu_y, cudaStream_t st);
template <typename T>
tc_status launch_lrn_fwd(const T* x, T* y, Act4 a, int size, float alpha, float beta, float k, cudaStream_t st);
// relu != 0: x is a ReLU output and the ReLU backward is folded in (dx *= [x > 0])
template <typename T>
tc_status launch_lrn_bwd(const T* dy, const T* x, const T* y, T* dx, Act4 a, int size, float alpha, float beta,
                         float k, int relu, cudaStream_t st);

// rows x F, input bf16 with row stride in_ld -> fp32 out (stride F)
template <typename T>
tc_status launch_softmax_fwd(const T* x, long long in_ld, float* y, int rows, int F, cudaStream_t st);
// dx (bf16, stride out_ld, pad columns zeroed) = y * (dy - sum(dy*y))
template <typename T>
tc_status launch_softmax_bwd(const float* dy, const float* y, T* dx, long long out_ld, int rows, int F,
                             cudaStream_t st);

enum F32Op { F32_LOG = 0, F32_RECIP = 1, F32_SCALE = 2, F32_MUL = 3, F32_ADD = 4 };
tc_status launch_f32_ew(int op, const float* a, const float* b, float scale, float* y, long long n, cudaStream_t st);
// fused softmax log-loss head: L = log S, Y = onehot (if Y != null), dz = softmax_bwd((Y c) / S, S)
template <typename T>
tc_status launch_softmax_xent(const T* z, long long ld, const int32_t* labels, float c, float* L, float* Y, T* dz,
                              int rows, int F, cudaStream_t st);
tc_status launch_onehot(const int32_t* labels, float* y, int N, int K, cudaStream_t st);
// hits = #rows whose first-maximum argmax equals the label (test body precision)
template <typename T>
tc_status launch_argmax_hits(const T* logits, long long ld, int N, int C, const int32_t* labels, unsigned* hits,
                             cudaStream_t st);
// loss = sum_t coef[t] * dot(a[t], b[t]) over n[t] elements -> *out (fp32 device scalar).
// `out` must point at >= 512 zero-initialised bytes (reduction partials + ticket follow the scalar).
tc_status launch_loss(const float* const* a, const float* const* b, const long long* n, const double* coef, int nterms,
                      float* out, cudaStream_t st);

// Column sums of a [rows][ld] bf16 matrix over its first `cols` columns -> out[cols] fp32 (deterministic).
template <typename T>
tc_status launch_colsum(const T* x, long long rows, int cols, long long ld, float* out, float* partials,
                        int max_partials, cudaStream_t st);
size_t colsum_partials_floats(int cols);
template <typename T>
tc_status launch_bias_add(const T* x, const float* b, T* y, long long rows, int cols, long long ld, int relu,
                          cudaStream_t st);

// Concat: copy `c` channels of src (stride src_cs) into dst channel offset `off` (stride dst_cs).
template <typename T>
tc_status launch_channel_copy(const T* src, int src_cs, T* dst, int dst_cs, int off, int c, long long pixels,
                              cudaStream_t st, const T* relu_y = nullptr);
tc_status launch_zero(void* p, size_t bytes, cudaStream_t st);

// BatchNorm over NHWC [pixels][cs] (training-mode batch statistics, biased variance):
// stats = (mean[C], istd[C]); y = gamma * (x - mean) * istd + beta (then max(y, 0) when relu: the
// in-place ReLU that follows a BN is folded into the apply pass).
// `partials` holds max_partials floats of reduction scratch plus 3*C coefficient floats.
template <typename T>
// res (may be null): a residual added to the (storage-rounded) BN output before the optional ReLU
tc_status launch_bn_fwd(const T* x, const float* gamma, const float* beta, T* y, float* stats, long long pixels, int C,
                        int cs, float eps, int relu, const T* res, float* partials, int max_partials, cudaStream_t st);
// sums[0..2C) = (sum dy, sum dy * xhat) — shared by dgamma (= sum dy*xhat), dbeta (= sum dy) —
// and sums[2C..5C) = the data-gradient coefficients (k1, k2, k3) from gamma and the forward stats
template <typename T>
tc_status launch_bn_bwd_reduce(const T* dy, const T* x, const float* gamma, const float* stats, float* sums,
                               long long pixels, int C, int cs, float* partials, int max_partials, cudaStream_t st);
// dx = k1*dy + k2*x + k3 per channel, k = sums + 2C of launch_bn_bwd_reduce
template <typename T>
tc_status launch_bn_bwd_apply(const T* dy, const T* x, const float* k, T* dx, long long pixels, int C, int cs,
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
template <typename T, typename SRC>
tc_status launch_nchw_to_nhwc(const SRC* x, T* y, StageLayout L, cudaStream_t st);
// Synthetic batch generated on the device (identical law to oracle/tc_philox.h).
template <typename T>
tc_status launch_synth_batch(T* x, int32_t* labels, StageLayout L, int classes, uint64_t seed, uint32_t iter,
                             uint32_t n0, cudaStream_t st);
// Space-to-depth filter gradient [K][ld]: zero the taps outside the original R x S window
// (column (a*Rp + b)*s*s*cs + (i*s + j)*cs + c is tap (s*a + i, s*b + j)).
tc_status launch_s2d_mask_grad(float* g, int K, long long ld, int Rp, int s, int cs, int R, int S, cudaStream_t st);
// [K][RS][cs] bf16 filter shadow (row stride ld) -> [cs][RS][ks] (K-major bwd-data filter operand)
tc_status launch_krsc_to_crsk(const bf16* src, int K, int RS, int cs, long long ld, bf16* dst, int ks, cudaStream_t st);

// Momentum SGD: v = mom*v + lr_alpha*(g + decay*p); p += v;
// refreshes the bf16 shadow(s) used as GEMM operands.
struct SgdTensor {
    float* p;
    float* v;
    const float* g;
    long long n;
    bf16* shadow;        // same layout as p (may be null)
    bf16* shadow_rskc;   // conv filters: copy for bwd-data (may be null): [R][S][ks][cs], or
                         // [cs][R][S][ks] (K-major bwd-data operand) when rskc_kmajor
    int K, RS, cs, ks;   // shape info for the RSKC scatter (p is [K][RS][cs])
    int rskc_kmajor;
    float lr_alpha, momentum, decay;
    const float* gscale;  // device scalar: global-L2 clip factor applied to g + decay p (null = 1)
};
tc_status launch_sgd(const SgdTensor* ts, int nt, SgdTensor* dev_scratch, cudaStream_t st);
// scale[0] = min(1, clip / ||g + decay p||_2) over all tensors (scale[1] = the norm)
tc_status launch_clip_scale(const SgdTensor* ts, int nt, float clip, double* partials, float* scale, cudaStream_t st);
size_t clip_partials_doubles(int nt);
// tc_gemm_bf16 with the momentum update of `sgd` (may be null) fused into the epilogue
// bias_out: also the column sums of the MN-major A operand over k (the bias gradient of a weight
// gradient whose A is dy), when gemm_bias_foldable(a)
tc_status gemm_args_ex(const tc_gemm_args* a, const SgdTensor* sgd, void* stream, float* bias_out = nullptr);
bool gemm_bias_foldable(const tc_gemm_args* a);

// fp32 parity mode: bf16 operand splits (see ops.cu).  kSplitN copies per operand; the part
// (0 hi, 1 mid, 2 lo) of copy j is (parts >> 2j) & 3.  A-side and B-side part lists pair up as
// hi*hi, hi*mid, mid*hi, hi*lo, mid*mid, lo*hi.
constexpr int kSplitN = 6;
enum { SPLIT_COLS = 0, SPLIT_ROWS = 1, SPLIT_A = 0x910, SPLIT_B = 0x184 };
tc_status launch_split(const float* src, long long rows_src, long long ld_src, bf16* dst, long long R, int L,
                       int rows_mode, int parts, cudaStream_t st);
tc_status launch_split_rskc(const float* p, long long ld, int K, int RS, int cs, int ks, bf16* dst, int parts,
                            cudaStream_t st);

// Convolv fprop / bwd-data with an fp32 output (y_f32 / dx_f32 = 1) — gemm.cu
tc_status conv_fwd_ex(const tc_conv_desc* d, const void* x, const void* w, const float* bias, int relu, void* y,
                      int y_f32, void* ws, size_t ws_bytes, void* stream);
// relu_mask: bf16 [N*H*W][cs] forward ReLU output; dx *= [mask > 0] in the epilogue (may be null)
tc_status conv_bwd_data_ex(const tc_conv_desc* d, const void* dy, const void* w_rskc, void* dx, int dx_f32, void* ws,
                           size_t ws_bytes, void* stream, const void* relu_mask = nullptr, int w_kmajor = 0);
// Filter gradient that also writes the bias gradient (sum of dy over the pixels) when dbias is
// non-null; only for convs where wgrad_bias_foldable() holds (the halo filter-gradient kernel).
tc_status conv_bwd_filter_ex(const tc_conv_desc* d, const void* dy, const void* x, float* dw, float* dbias, void* ws,
                             size_t ws_bytes, void* stream);
bool wgrad_bias_foldable(const tc_conv_desc* d);

// d_iter[0] = iter, d_iter[1] = n0 (kernel arguments travel with the launch: no host sync)
tc_status launch_set_iter(uint32_t* d_iter, uint32_t iter, uint32_t n0, cudaStream_t st);

}  // namespace tcb
