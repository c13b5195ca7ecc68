/*
 * tc_abi.h — C ABI of the B200 execution backend for the DeepDSL/tensorc
 * training step (arXiv 1701.02284).
 *
 * The cut is the one the reference spec draws between the plan producers and
 * the runtime (SPEC.md:291-302 IrProgram, SPEC.md:472-480 exec(stmt, env),
 * SPEC.md:481-483 pool_acquire/pool_release, SPEC.md:497 train).  Everything
 * above it (network definition, gradient derivation, SSA/CSE/schedule/dealloc,
 * memplan) stays host C++ (libtcb200 host part, see tc_plan.h); everything
 * below it is sm_100a CUDA behind these entry points.
 *
 * Conventions
 *  - No exceptions cross this boundary.  Every entry returns tc_status; the
 *    message of the last failure on the calling thread is tc_last_error().
 *    The codes mirror the reference diagnostics: CompileError kinds
 *    (diag.hpp:22-35), IoError / FormatError (diag.hpp:50-59) and the runtime
 *    faults ShapeFault / PoolExhausted.
 *  - Pointers passed to per-kernel entries are device pointers; `stream` is a
 *    cudaStream_t (NULL = legacy default stream).  All calls are asynchronous.
 *  - Activations on the device are NHWC with the channel extent padded to a
 *    multiple of 8 ("channel stride", cs); the reference layout is NCHW
 *    (shape.hpp:12) and the permutation happens only at upload / download.
 *  - bf16 storage for activations and their gradients; fp32 master
 *    parameters, velocities and parameter gradients.
 */
#ifndef TC_ABI_H
#define TC_ABI_H

#include <stddef.h>
#include <stdint.h>

#ifndef TC_API
#define TC_API __attribute__((visibility("default")))
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum tc_status {
    TC_OK = 0,
    TC_SHAPE_FAULT = 1,     /* SPEC.md:475 ShapeFault */
    TC_POOL_EXHAUSTED = 2,  /* SPEC.md:475 PoolExhausted */
    TC_INVALID_ARG = 3,
    TC_CUDA_ERROR = 4,
    TC_NCCL_ERROR = 5,
    TC_IO_ERROR = 6,        /* diag.hpp:50 IoError */
    TC_FORMAT_ERROR = 7,    /* diag.hpp:56 FormatError */
    TC_INTERNAL = 8,
    TC_COMPILE_ERROR = 9    /* diag.hpp:41 CompileError (kind in the message) */
} tc_status;

/* Message of the last non-OK status returned on this thread ("" if none). */
TC_API const char* tc_last_error(void);
/* Library build identification (arch, compiler). */
TC_API const char* tc_build_info(void);
/* Number of this library's kernels launched since process start (evidence counter). */
TC_API unsigned long long tc_kernel_launch_count(void);

/* ------------------------------------------------------------------ GEMM */
/* Operand layouts: TC_LAYOUT_K  = row-major [rows, K] (K contiguous),
 *                  TC_LAYOUT_MN = row-major [K, rows] (rows contiguous).   */
enum { TC_LAYOUT_K = 0, TC_LAYOUT_MN = 1 };
enum { TC_DTYPE_BF16 = 0, TC_DTYPE_F32 = 1 };

typedef struct tc_gemm_args {
    int M, N, K;
    int a_layout, b_layout;
    const void* A; long long lda;   /* bf16; leading stride in elements */
    const void* B; long long ldb;   /* bf16 */
    void* D; long long ldd;         /* bf16 or fp32 */
    int d_dtype;
    const float* bias;              /* per-column (N) bias, may be NULL */
    int relu;
    float alpha, beta;              /* D = alpha*A.B^T (+ beta*D, fp32 only) */
    int splits;                     /* split-K factor, 0 = auto */
    void* workspace; size_t workspace_bytes;  /* fp32 partials for split-K */
    int bias_n;                     /* bias[n] read for n < bias_n (0 = N); columns beyond get 0 */
    int b_rows;                     /* rows of B that exist (0 = N); D columns >= b_rows come out 0 */
    const void* relu_mask;          /* bf16 [M][mask_ld], may be NULL: D *= [relu_mask > 0] (ReLU backward
                                       folded into the epilogue; bf16 D, no split-K / beta) */
    long long mask_ld;
} tc_gemm_args;

/* D[M,N] = alpha * sum_k A[m,k] B[n,k] (+bias[n]) (relu), tcgen05 kind::f16. */
TC_API tc_status tc_gemm_bf16(const tc_gemm_args* args, void* stream);
/* Workspace bytes tc_gemm_bf16 needs for these args (0 when no split-K). */
TC_API size_t tc_gemm_workspace_bytes(const tc_gemm_args* args);

/* ------------------------------------------------------------ Convolution */
/* Convolv(s,p)(X, W, B).  NHWC activations with
 * channel stride cs (input) / ks (output); filters KRSC with channel stride cs. */
typedef struct tc_conv_desc {
    int N, C, H, W;      /* input */
    int K, R, S;         /* output channels, kernel */
    int stride, pad;
    int Ho, Wo;          /* output spatial (floor((H+2p-R)/s)+1) */
    int cs, ks;          /* channel strides of x and y: multiples of 8, or cs = 4 for a
                            first-layer input (fwd / bwd-filter only, 8-byte gathers) */
    int wld;             /* filter row stride in elements (0 = R*S*cs); multiple of 8 */
} tc_conv_desc;

TC_API tc_status tc_conv2d_fwd(const tc_conv_desc* d, const void* x, const void* w_krsc, const float* bias, int relu,
                        void* y, void* workspace, size_t ws_bytes, void* stream);
/* d_Convolv(s,p)(W)/d_X: w_rskc is the filter stored [R][S][K][cs]. */
TC_API tc_status tc_conv2d_bwd_data(const tc_conv_desc* d, const void* dy, const void* w_rskc, void* dx,
                             void* workspace, size_t ws_bytes, void* stream);
/* d_Convolv(s,p)(X)/d_W: dw fp32 [K][R][S][cs]. */
TC_API tc_status tc_conv2d_bwd_filter(const tc_conv_desc* d, const void* dy, const void* x, float* dw,
                               void* workspace, size_t ws_bytes, void* stream);
TC_API size_t tc_conv2d_workspace_bytes(const tc_conv_desc* d, int which /*0 fwd,1 data,2 filter*/);

#ifdef __cplusplus
}
#endif

#endif /* TC_ABI_H */
