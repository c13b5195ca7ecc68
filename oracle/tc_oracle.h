/*
 * tc_oracle.h — CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * A plain C++ restatement of the reference runtime's exec semantics
 * (exec kernels :474, best-fit MemoryPool :462-465/:481-488,
 * train :497-504) used to check the B200 backend.  It is imported only by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm; the product library never links or calls it.
 *
 * Parity pinning: the reference (/root/reference) contains no executable
 * runtime, so this oracle is pinned against the paper's
 * Fig. 2 memory table (via the shared plan), the SPEC `examples:` lines, the
 * hand-stepped solver and f64 finite differences
 * (SPEC.md:567).  Kernel arithmetic that lived in cuDNN in the paper's system
 * is "parity unpinned" beyond those checks.
 */
#ifndef TC_ORACLE_H
#define TC_ORACLE_H

#include <stdint.h>

#include "tc_plan.h"

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_API __attribute__((visibility("default")))

/* ---- per-op kernels, NCHW, fp32 (_f32) and fp64 (_f64) ------------------- */
#define ORC_DECL(T, sfx)                                                                                        \
    ORC_API void orc_conv_fwd_##sfx(const T* x, const T* w, const T* b, T* y, int N, int C, int H, int W, int K, \
                                    int R, int S, int stride, int pad, int direct);                             \
    ORC_API void orc_conv_bwd_data_##sfx(const T* dy, const T* w, T* dx, int N, int C, int H, int W, int K,      \
                                         int R, int S, int stride, int pad);                                    \
    ORC_API void orc_conv_bwd_filter_##sfx(const T* dy, const T* x, T* dw, int N, int C, int H, int W, int K,    \
                                           int R, int S, int stride, int pad);                                  \
    ORC_API void orc_conv_bwd_bias_##sfx(const T* dy, T* db, int N, int K, int HW);                             \
    ORC_API void orc_pool_fwd_##sfx(const T* x, T* y, int32_t* idx, int N, int C, int H, int W, int k,          \
                                    int stride, int pad, int is_max);                                           \
    ORC_API void orc_pool_bwd_##sfx(const T* dy, const T* x, T* dx, int N, int C, int H, int W, int k,          \
                                    int stride, int pad, int is_max);                                           \
    ORC_API void orc_lrn_fwd_##sfx(const T* x, T* y, int N, int C, int HW, int size, double alpha, double beta, \
                                   double k);                                                                   \
    ORC_API void orc_lrn_bwd_##sfx(const T* dy, const T* x, const T* y, T* dx, int N, int C, int HW, int size,  \
                                   double alpha, double beta, double k);                                        \
    ORC_API void orc_softmax_fwd_##sfx(const T* x, T* y, int rows, int cols);                                   \
    ORC_API void orc_softmax_bwd_##sfx(const T* dy, const T* y, T* dx, int rows, int cols);                     \
    ORC_API void orc_bn_fwd_##sfx(const T* x, const T* g, const T* b, T* y, int N, int C, int HW, double eps);  \
    ORC_API void orc_bn_bwd_##sfx(const T* dy, const T* x, const T* g, T* dx, T* dg, T* dbeta, int N, int C,    \
                                  int HW, double eps);                                                          \
    ORC_API void orc_matmul_##sfx(const T* A, const T* B, T* C, int M, int N, int K, int ta, int tb);

ORC_DECL(float, f32)
ORC_DECL(double, f64)
#undef ORC_DECL

/* ---- whole-plan execution -------------------------------------------------- */
typedef struct orc_ctx orc_ctx;
typedef struct orc_pool_stats {
    int64_t allocs_from_os, reuses, releases, live_bytes, peak_bytes, os_bytes;
} orc_pool_stats;

/* f64 != 0 runs every kernel in double (finite-difference checks). */
/* A plan serialized by tc_plan_save ("TCPL" v1), loaded without the product library (bench.py's
 * reference arm).  NULL on a missing / malformed file (message on stderr). */
ORC_API tc_plan* orc_plan_load(const char* path);
ORC_API void orc_plan_free(tc_plan* plan);
/* Shape queries on a plan: rank of parameter i (dims into out[4]); input dims into out[4]. */
ORC_API int orc_plan_param_dims(const tc_plan* plan, int i, int64_t* out);
ORC_API void orc_plan_input_dims(const tc_plan* plan, int64_t* out);
ORC_API orc_ctx* orc_create(const tc_plan* plan, uint64_t seed, int f64, int threads);
ORC_API void orc_destroy(orc_ctx* c);
/* Parameters in the reference layout (NCHW / (out,in)), fp32. */
ORC_API void orc_param_get(orc_ctx* c, int index, float* out);
ORC_API void orc_param_set(orc_ctx* c, int index, const float* in);
ORC_API void orc_param_get_f64(orc_ctx* c, int index, double* out);
ORC_API void orc_param_set_f64(orc_ctx* c, int index, const double* in);
ORC_API void orc_velocity_get(orc_ctx* c, int index, float* out);
/* Initialise parameters exactly as the device runtime does (tc_philox.h). */
ORC_API void orc_init_params(orc_ctx* c);
/* Synthetic batch of iteration `iter` for global samples [n0, n0+batch). */
ORC_API void orc_synth_batch(const tc_plan* plan, uint64_t seed, int iter, int n0, float* x, int32_t* labels);
/* Provide the next batch explicitly (NULL = synthesise for `iter`). */
ORC_API void orc_set_batch(orc_ctx* c, const float* x, const int32_t* labels);
/* One training iteration (train body).  update != 0 applies the Updates;
 * keep != 0 keeps every var (no Dealloc) so tests can inspect it.  Returns loss. */
ORC_API double orc_step(orc_ctx* c, int iter, int n0, int update, int keep);
/* Forward-only test body; writes argmax-match fraction. */
ORC_API double orc_test(orc_ctx* c, int iter, int n0);
ORC_API int orc_var_get(orc_ctx* c, int var, float* out, int64_t max_elems);
/* Gradient of the last step for parameter `index` (as fed to its Update). */
ORC_API int orc_grad_get(orc_ctx* c, int index, double* out, int64_t max_elems);
ORC_API void orc_pool_stats_get(orc_ctx* c, orc_pool_stats* s);
/* Per-statement live-bytes trace of the last step (dealloc mode), one entry per stmt. */
ORC_API int orc_live_trace(orc_ctx* c, int64_t* out, int max);
ORC_API void orc_set_workspace_cap(orc_ctx* c, double mb);
/* Emulate the device's storage precision: round every bf16-stored activation
 * to bf16 after each statement and use bf16-rounded weights as contraction
 * operands.  Used to measure the rounding envelope of the step. */
ORC_API void orc_set_bf16_storage(orc_ctx* c, int on);

#ifdef __cplusplus
}
#endif

#endif /* TC_ORACLE_H */
