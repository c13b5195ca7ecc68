/*
 * tc_plan.h — the memory-scheduled execution plan as plain C data.
 *
 * This is IrProgram flattened for consumers below the
 * boundary: the sm_100a runtime (tc_runtime.h) and the CPU oracle
 * (oracle/, test infrastructure).  One tc_stmt per IrStmt; operand kinds and
 * op codes are the exec vocabulary of SPEC.md:474 / Fig. 2.
 *
 * Shapes are in the reference layout (NCHW, shape.hpp:12).  Var ids are the
 * SSA numbers (Xn) of the compiler; storage ids name alias chains produced by
 * inline_inplace.
 */
#ifndef TC_PLAN_H
#define TC_PLAN_H

#include <stddef.h>
#include <stdint.h>

#include "tc_abi.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef enum tc_op {
    TC_OP_NONE = 0,
    TC_OP_LOAD_X = 1,          /* Cuda(X)                         */
    TC_OP_LOAD_Y = 2,          /* Cuda(Indicator(Y, K))           */
    TC_OP_CONV_FWD = 3,        /* Convolv(s,p)(x, W[, B])          in: x, W, B        */
    TC_OP_CONV_BWD_DATA = 4,   /* up * d_Convolv(s,p)(W)/d_x       in: up, W          */
    TC_OP_CONV_BWD_FILTER = 5, /* up * d_Convolv(s,p)(x)/d_W       in: up, x          */
    TC_OP_CONV_BWD_BIAS = 6,   /* up * d_Convolv(s,p)()/d_B        in: up             */
    TC_OP_POOL_FWD = 7,        /* Pooling(k,s,p,max)(x)            in: x              */
    TC_OP_POOL_BWD = 8,        /* up * d_Pooling(..)(y,x)/d_x      in: up, y, x       */
    TC_OP_RELU_FWD = 9,
    TC_OP_RELU_BWD = 10,       /* in: up, y */
    TC_OP_SOFTMAX_FWD = 11,
    TC_OP_SOFTMAX_BWD = 12,    /* in: up, y */
    TC_OP_LRN_FWD = 13,
    TC_OP_LRN_BWD = 14,        /* in: up, y, x */
    TC_OP_DROPOUT_MASK = 15,   /* in: x (shape only) */
    TC_OP_MUL = 16,            /* elementwise a * b */
    TC_OP_ADD = 17,            /* elementwise a + b (adjoint accumulation / residual) */
    TC_OP_MATMUL_FWD = 18,     /* (A)(i|@) * (W)(j|@) = A W^T      in: A, W           */
    TC_OP_MATMUL_BWD_DATA = 19,/* up W                             in: up, W          */
    TC_OP_MATMUL_BWD_W = 20,   /* up^T A                           in: up, A          */
    TC_OP_BIAS_ADD = 21,       /* (x + (i) => b)                   in: x, b           */
    TC_OP_BIAS_GRAD = 22,      /* column sum                       in: up             */
    TC_OP_LOG = 23,
    TC_OP_RECIP = 24,
    TC_OP_SCALE = 25,
    TC_OP_CONCAT = 26,         /* channel concat                   in: parts...       */
    TC_OP_CONCAT_BWD = 27,     /* channel slice [offset, offset+extent) in: up        */
    TC_OP_BN_FWD = 28,         /* in: x, gamma, beta */
    TC_OP_BN_BWD_DATA = 29,    /* in: up, x, gamma */
    TC_OP_BN_BWD_GAMMA = 30,   /* in: up, x */
    TC_OP_BN_BWD_BETA = 31,    /* in: up */
    TC_OP_PRINT_LOSS = 32,     /* loss = sum_t coef[t] * dot(in[2t], in[2t+1]) */
    TC_OP_COUNT = 33
} tc_op;

enum { TC_STMT_LET = 0, TC_STMT_DEALLOC = 1, TC_STMT_UPDATE = 2, TC_STMT_PRINT = 3 };
enum { TC_REF_NONE = 0, TC_REF_VAR = 1, TC_REF_PARAM = 2 };
enum { TC_INIT_XAVIER = 0, TC_INIT_CONSTANT = 1, TC_INIT_GAUSSIAN = 2 };
enum { TC_MODE_REUSE = 0, TC_MODE_DEALLOC = 1 };

#define TC_MAX_IN 8

typedef struct tc_ref {
    int kind;   /* TC_REF_* */
    int index;  /* var id or parameter index */
} tc_ref;

typedef struct tc_stmt {
    int kind;       /* TC_STMT_* */
    int op;         /* tc_op (Let, Update: the gradient op) */
    int var;        /* Let / Dealloc: SSA var id */
    int storage;    /* storage id (alias root) */
    int inplace;    /* Let writes into the storage of its overwritten operand */
    int param;      /* Update: parameter index */
    int nin;
    tc_ref in[TC_MAX_IN];
    int rank;
    int64_t dims[4];  /* Let result shape, NCHW */
    int64_t bytes;    /* bytes newly allocated (fp32 accounting), Dealloc: bytes freed */
    /* hyper-parameters */
    int k, stride, pad, max_pool, has_bias, lrn_size, slot;
    double alpha, beta, lrn_k, rate, scale, eps;
    int64_t offset, extent;
    /* Update: v = momentum*v + lr_alpha*(g + decay*p); p = p + v */
    double lr_alpha, momentum, decay;
    /* Print */
    int nterms;
    double coef[4];
} tc_stmt;

typedef struct tc_param_desc {
    char name[64];
    int rank;
    int64_t dims[4];
    int init_kind;
    double init_value, sigma, lr_mult, decay_mult;
    int64_t fan_in, fan_out;   /* Xavier fans (Cin*k^2, Cout*k^2) */
} tc_param_desc;

typedef struct tc_var_desc {
    int id;
    int rank;
    int64_t dims[4];
} tc_var_desc;

typedef struct tc_plan {
    const char* name;
    int64_t batch, classes;
    int64_t input_dims[4];
    int nparams;
    const tc_param_desc* params;
    int nstmts;
    const tc_stmt* stmts;          /* train-loop body */
    int ntest;
    const tc_stmt* test_stmts;     /* test body (forward to the main logits) */
    int logits_var;
    int nvars;
    const tc_var_desc* vars;
    int max_var;                   /* every var id < max_var */
    double lr, momentum, decay, clip;
    int mode;                      /* TC_MODE_* */
} tc_plan;

typedef struct tc_mem_summary {
    double peak_dealloc_mb, peak_reuse_mb, param_mb, workspace_mb;
    int64_t peak_dealloc_bytes, peak_reuse_bytes, param_bytes, workspace_bytes;
} tc_mem_summary;

typedef struct tc_compile_opts {
    double lr, momentum, decay, clip;   /* solver (PAPER.md:126 defaults 0.01, 0.9, 0.0005, 0) */
    int mode;                           /* TC_MODE_* */
    double workspace_cap_mb;            /* < 0: unlimited */
    int greedy_schedule;
    int64_t global_batch;               /* loss cardinality |N| (data parallel: G*B); 0 = batch */
    int no_cse;                         /* 1: skip common sub-expression elimination */
} tc_compile_opts;

typedef struct tc_net tc_net;  /* a compiled network (plan producer output) */

/* Network definition + gradient derivation + memory-scheduled plan
 * (expr.hpp network builders).  name: lenet | alexnet |
 * vgg16 | googlenet | resnet50 | inception. */
TC_API tc_status tc_net_compile(const char* name, int64_t batch, const tc_compile_opts* opts, tc_net** out);
/* A network from its text description (the reference's netspec-frontend; grammar
 * in csrc/host/netspec.hpp): data / net / solver sections, layer kinds conv, maxpool, avgpool, relu,
 * full, flatten, softmax, dropout, lrn, concat (+ batchnorm, residual), `.` composition, weighted
 * logloss terms.  batch > 0 overrides the data section; opts != NULL overrides its solver section.
 * Errors: TC_COMPILE_ERROR with "<ErrKind> at line:col: message" (diag.hpp kinds). */
TC_API tc_status tc_net_compile_spec(const char* text, int64_t batch, const tc_compile_opts* opts, tc_net** out);
/* Data source seed and solver iteration counts of a spec-compiled network. */
TC_API tc_status tc_net_spec_info(const tc_net* net, uint64_t* seed, int64_t* iters, int64_t* test_iters);
TC_API void tc_net_destroy(tc_net* net);
/* Codegen (PAPER.md 5): a standalone C++ training program (one compilation unit)
 * that embeds this plan and calls the runtime library only -- one tc_exec_stmt per IR statement,
 * the statement's Fig. 2 text as the comment above it, a one-line memory-mode flag, snapshot
 * load / save and a test procedure.  mode: TC_MODE_*; iters / test_iters <= 0 / < 0: the spec's
 * solver (or 1000 / 10).  Deterministic; the text lives until the next call on this net. */
TC_API const char* tc_net_codegen(tc_net* net, int mode, int64_t iters, int64_t test_iters);
/* Write a plan to `path` ("TCPL" v1: header of record sizes, name, batch / classes / input dims,
 * counts, solver, then the params / train stmts / test stmts / vars arrays as raw records). */
TC_API tc_status tc_plan_save(const tc_plan* plan, const char* path);
TC_API const tc_plan* tc_net_plan(const tc_net* net);
/* Fig. 2 style IR dump / memory table (text or csv), verifier message ("" = valid). */
TC_API const char* tc_net_ir_text(const tc_net* net);
TC_API const char* tc_net_memory_table(const tc_net* net, int csv);
TC_API tc_status tc_net_memory_summary(const tc_net* net, tc_mem_summary* out);
TC_API const char* tc_net_verify(const tc_net* net);
/* Fig. 2 text of one train statement. */
TC_API const char* tc_net_stmt_text(const tc_net* net, int index);

#ifdef __cplusplus
}
#endif

#endif /* TC_PLAN_H */
