/*
 * tc_runtime.h — the sm_100a executor behind the boundary.
 *
 * Replaces the reference runtime's exec(stmt, env) / pool_acquire /
 * pool_release / train: a tc_ctx owns one GPU's device
 * arena (static offsets from the plan's liveness, zero allocation in the
 * step), the persistent parameter slab (fp32 master weights, velocities,
 * gradient buffers, bf16 operand shadows) and, for data parallelism, an NCCL
 * communicator (one process per GPU).
 *
 * Ownership: the context owns every device buffer; host
 * pointers are borrowed for the duration of a call.  Threading: one owning
 * host thread at a time.  All work is enqueued on the context stream; only
 * tc_loss / tc_*_download / tc_sync block.
 */
#ifndef TC_RUNTIME_H
#define TC_RUNTIME_H

#include "tc_plan.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tc_ctx tc_ctx;

typedef struct tc_ctx_desc {
    int device;              /* CUDA device ordinal */
    int rank, world;         /* data-parallel rank / size (world 1 = no NCCL) */
    const void* nccl_id;     /* 128-byte ncclUniqueId from rank 0 (world > 1) */
    uint64_t seed;           /* TENSORC_SEED, default 42 */
    int use_graph;           /* capture the step in a CUDA graph after the first run */
    int keep;                /* parity mode: every storage gets its own arena range */
    int precision;           /* TC_PREC_BF16 (default): bf16 activations, bf16 tensor-core operands;
                                TC_PREC_F32: fp32 activations, every contraction as a 3-part bf16 split
                                of each operand, 6 cross terms (hi*hi, hi*mid, mid*hi, hi*lo, mid*mid,
                                lo*hi) accumulated in fp32 on the same tcgen05 kernels */
} tc_ctx_desc;

enum { TC_PREC_BF16 = 0, TC_PREC_F32 = 1 };

typedef struct tc_rt_memory {
    int64_t arena_bytes;       /* activation arena (per-step peak, device dtypes) */
    int64_t arena_keep_bytes;  /* what the arena would be without lifetime sharing */
    int64_t param_bytes;       /* fp32 params + velocities + grads + bf16 shadows */
    int64_t workspace_bytes;   /* split-K / reduction scratch */
    int64_t input_bytes;       /* staged batch */
    int64_t device_used_bytes; /* cudaMemGetInfo high-water (total - free) after setup */
} tc_rt_memory;

TC_API tc_status tc_ctx_create(const tc_plan* plan, const tc_ctx_desc* desc, tc_ctx** out);
TC_API void tc_ctx_destroy(tc_ctx* ctx);
TC_API void* tc_ctx_stream(tc_ctx* ctx);

/* Parameters in the reference layout (NCHW / (out,in)), fp32 host memory. */
TC_API tc_status tc_param_upload(tc_ctx* ctx, int index, const float* host);
TC_API tc_status tc_param_download(tc_ctx* ctx, int index, float* host);
TC_API tc_status tc_velocity_download(tc_ctx* ctx, int index, float* host);
TC_API tc_status tc_grad_download(tc_ctx* ctx, int index, float* host);
TC_API tc_status tc_velocity_upload(tc_ctx* ctx, int index, const float* host);
/* The plan a context executes (borrowed). */
TC_API const tc_plan* tc_ctx_plan(tc_ctx* ctx);

/* Snapshot / resume: one file per parameter, `<dir>/<name>.ddt`
 * = "DDSL" | u32 version 1 | u32 rank | u32 dims[rank] | f32 payload (little endian), in the
 * reference layout; velocities go to `<dir>/<name>.velocity.ddt` (momentum state, so a resumed
 * run continues bit-exactly).  Load matches by name: a missing file keeps the current value and
 * is counted in *missing (with a warning on stderr); extra files are ignored.  Errors:
 * TC_IO_ERROR (unreadable / unwritable), TC_FORMAT_ERROR (bad magic / version / dims, naming the file). */
TC_API tc_status tc_snapshot_save(tc_ctx* ctx, const char* dir);
TC_API tc_status tc_snapshot_load(tc_ctx* ctx, const char* dir, int* loaded, int* missing);
/* Xavier / constant init from the shared counter RNG (tc_philox.h); identical to the oracle. */
TC_API tc_status tc_init_params(tc_ctx* ctx);

/* Stage a batch: x NCHW fp32 (batch, C, H, W) and int32 labels, host memory.  Asynchronous
 * input pipeline: the H2D copy runs on the context's copy stream into one of two device
 * staging slots (overlapping a running step when the host memory is pinned); the next
 * tc_step / tc_exec_stmt converts it to the device layout.  The host buffers are borrowed
 * until tc_sync() or until the step after the consuming one has been enqueued. */
TC_API tc_status tc_stage_batch(tc_ctx* ctx, const float* x_host, const int32_t* labels_host);
/* Bytes one tc_stage_batch moves host -> device (images + labels): the images cross as bf16 when
 * the context rounds them on the host (bf16 precision, TCB_HOST_BF16 unset or 1), else fp32. */
TC_API int64_t tc_stage_bytes(const tc_ctx* ctx);
/* Generate the synthetic batch of `iter` on the device (global samples [n0, n0+batch)). */
TC_API tc_status tc_stage_synthetic(tc_ctx* ctx, int iter, int n0);
/* One training iteration over the staged batch (train body; update != 0 applies Updates). */
TC_API tc_status tc_step(tc_ctx* ctx, int iter, int n0, int update);
/* Execute a single train statement (interpreter / generated-code callers). */
TC_API tc_status tc_exec_stmt(tc_ctx* ctx, int index, int iter, int n0);
/* Test body over the staged batch: the forward Lets the main logits depend
 * on, test-mode dropout = identity; precision = fraction of rows whose first-maximum
 * argmax equals the label (blocks on the stream).  Reference: oracle orc_test / Exec::test. */
TC_API tc_status tc_test(tc_ctx* ctx, int iter, int n0, double* precision);
/* Loss of the last step (blocks on the stream). */
TC_API tc_status tc_loss(tc_ctx* ctx, double* loss);
/* Loss of the step before the last one enqueued, waiting for that step only (a training loop
 * that logs every step's loss one step late keeps the device busy); needs two steps. */
TC_API tc_status tc_loss_prev(tc_ctx* ctx, double* loss);
/* Var contents after a step (keep mode), converted to the reference layout, fp32. */
TC_API tc_status tc_var_download(tc_ctx* ctx, int var, float* host, int64_t max_elems);
/* Pool-forward argmax indices of a pooling output var (flat NCHW input index). */
TC_API tc_status tc_pool_indices_download(tc_ctx* ctx, int var, int32_t* host, int64_t max_elems);
TC_API tc_status tc_sync(tc_ctx* ctx);
TC_API tc_status tc_memory(tc_ctx* ctx, tc_rt_memory* out);
/* Kernels this context launched per step (counted at the first execution). */
TC_API int tc_launches_per_step(tc_ctx* ctx);

/* One eager step with a CUDA event after every statement: per-statement device ms. */
TC_API tc_status tc_profile_step(tc_ctx* ctx, int iter, int n0, int update, float* stmt_ms, int max);
/* Kernels each statement launched in the last tc_profile_step (0 = folded into its producer). */
TC_API int tc_profile_launches(tc_ctx* ctx, int* out, int max);
/* Device ms of the bucket all-reduce + momentum update that statement i completed in the last
 * tc_profile_step (0 for statements that complete no bucket; not included in stmt_ms). */
TC_API int tc_profile_updates(tc_ctx* ctx, float* out, int max);

/* NCCL bootstrap: rank 0 creates the id, the caller broadcasts it (torch.distributed). */
TC_API tc_status tc_nccl_unique_id(void* out128);

#ifdef __cplusplus
}
#endif

#endif /* TC_RUNTIME_H */
