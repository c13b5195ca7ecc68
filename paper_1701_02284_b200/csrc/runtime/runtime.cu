// sm_100a executor of the memory-scheduled plan (tc_runtime.h).
//
// Replaces the reference runtime's per-statement exec + MemoryPool
// with:
//   * a static device arena: every storage (alias chain from inline_inplace)
//     and every companion buffer (max-pool argmax indices, BN statistics) gets
//     an offset from lifetime-interval packing over the statement order, so
//     the step performs no allocation (the paper's cudaMalloc/cudaFree churn,
//     PAPER.md:323, 512-513, disappears);
//   * a persistent parameter slab: fp32 master weights / velocities /
//     gradients in device layouts plus bf16 GEMM-operand shadows refreshed by
//     the fused momentum update;
//   * peephole fusion of in-place BiasAdd / ReLU into the producing GEMM
//     epilogue (adjacent statements exposed by CSE + in-place inlining);
//   * optional NCCL gradient all-reduce (one process per GPU) before each
//     Update, and CUDA-graph capture of the whole step.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <memory>
#include <string>
#include <unordered_map>
#include <thread>
#include <condition_variable>
#include <mutex>
#include <vector>

#include "kernels/common.cuh"
#include "kernels/ops.cuh"
#include "tc_philox.h"
#include "tc_runtime.h"

namespace tcb {
namespace {

enum DType { DT_BF16 = 0, DT_F32 = 1, DT_U8 = 2 };

inline int ceil8(long long v) { return static_cast<int>((v + 7) / 8 * 8); }
inline size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

struct VarL {
    int id = -1;
    int rank = 0;
    int64_t d[4] = {1, 1, 1, 1};
    int dtype = DT_BF16;
    bool nhwc = false;  // device layout NHWC (4-D, or 2-D gradient of a flattened 4-D tensor)
    int N = 1, H = 1, W = 1, C = 1, cs = 8;  // 2-D: H = W = 1, C = F, cs = row stride
    int storage = -1;
    int def = -1;
    size_t bytes() const {
        const size_t el = static_cast<size_t>(N) * H * W * cs;
        return el * (dtype == DT_F32 ? 4 : dtype == DT_U8 ? 1 : 2);
    }
    long long elems() const { return static_cast<long long>(N) * H * W * cs; }
    Act4 act() const { return Act4{N, H, W, C, cs}; }
};

struct ParamL {
    int rank = 0;
    int64_t d[4] = {1, 1, 1, 1};
    enum Kind { VEC, CONV, FC } kind = VEC;
    // conv: [K][R][S][cs]; fc: [out][in_dev]; vec: [K]
    int K = 1, C = 1, R = 1, S = 1, cs = 8, ks = 8;
    bool fc_from4d = false;
    int fH = 1, fW = 1, fC = 1, fcs = 8;  // flattened 4-D input of an FC layer
    // conv filter row stride: Kw = ceil8(R*S*cs) (== R*S*cs unless cs = 4, the
    // channel-stride-4 first-layer input whose taps are gathered 8 bytes at a time)
    int Kw = 0;
    int in_dev = 0;
    int update_stmt = -1;  // the param's Update statement
    // space-to-depth first-layer conv: taps regrouped into an Rp x Rp stride-1 conv over
    // s2d*s2d*cs channels; device layout [K][Rp][Rp][s2d][s2d][cs] (taps outside R x S are 0)
    int s2d = 0, Rp = 0;
    long long n = 0;  // device elements
    float* p = nullptr;
    float* v = nullptr;
    float* g = nullptr;
    bf16* shadow = nullptr;
    bf16* rskc = nullptr;
    bool crsk = false;  // rskc holds [cs][R][S][ks] (K-major bwd-data operand) instead of [R][S][ks][cs]
};

struct Item {  // arena allocation
    size_t bytes = 0;
    int first = 0, last = 0;
    size_t off = 0;
};

}  // namespace
}  // namespace tcb

using namespace tcb;

// Fork-join pool of host threads for the fp32 -> bf16 rounding of staged host batches.
struct HostPool {
    // The batch is cut into `nchunks` chunks; every worker converts its share of chunk 0, then of
    // chunk 1, ..., counting each finished share in done[chunk], so the caller can start a chunk's
    // host -> device copy while the workers round the next one.
    static constexpr int kMaxChunks = 64;
    std::vector<std::thread> th;
    std::mutex m;
    std::condition_variable cv, done_cv;
    const float* src = nullptr;
    uint16_t* dst = nullptr;
    size_t n = 0, chunk = 0;
    int nchunks = 1;
    std::atomic<int> done[kMaxChunks];
    int gen = 0, pending = 0;
    bool stop = false;
    explicit HostPool(int workers) {
        for (auto& d : done) d.store(0);
        for (int w = 0; w < workers; ++w)
            th.emplace_back([this, w, workers] {
                int seen = 0;
                for (;;) {
                    std::unique_lock<std::mutex> lk(m);
                    cv.wait(lk, [&] { return stop || gen != seen; });
                    if (stop) return;
                    seen = gen;
                    const float* s0 = src;
                    uint16_t* d0 = dst;
                    const size_t total = n, ck = chunk;
                    const int nc = nchunks;
                    lk.unlock();
                    for (int c = 0; c < nc; ++c) {
                        const size_t ca = std::min(total, ck * c), cn = std::min(total, ca + ck) - ca;
                        const size_t share = (cn / workers + 63) / 64 * 64;
                        const size_t a = std::min(cn, share * w), b = std::min(cn, a + share);
                        round_bf16(s0 + ca + a, d0 + ca + a, b - a);
                        done[c].fetch_add(1, std::memory_order_release);
                    }
                    lk.lock();
                    if (--pending == 0) done_cv.notify_all();
                }
            });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(m);
            stop = true;
        }
        cv.notify_all();
        for (auto& t : th) t.join();
    }
    // round-to-nearest-even, as __float2bfloat16_rn for every finite value (NaN / Inf keep their
    // top half); written so the compiler vectorises it
    __attribute__((optimize("O3"))) static void round_bf16(const float* __restrict__ s, uint16_t* __restrict__ d, size_t n) {
        const uint32_t* u = reinterpret_cast<const uint32_t*>(s);
        for (size_t i = 0; i < n; ++i) {
            const uint32_t x = u[i];
            const uint32_t r = ((x & 0x7f800000u) == 0x7f800000u) ? x : x + 0x7fffu + ((x >> 16) & 1u);
            d[i] = static_cast<uint16_t>(r >> 16);
        }
    }
    // Round s[0, count) into d; on_chunk(begin, len) runs on the calling thread as soon as a chunk
    // is complete (in chunk order).  Returns the first non-OK status of on_chunk.
    template <typename F>
    tc_status run(const float* s, uint16_t* d, size_t count, int chunks, F&& on_chunk) {
        chunks = std::max(1, std::min(kMaxChunks, chunks));
        const size_t ck = ((count + chunks - 1) / chunks + 63) / 64 * 64;
        const int nc = static_cast<int>(std::max<size_t>(1, (count + ck - 1) / ck));
        const int workers = static_cast<int>(th.size());
        {
            std::lock_guard<std::mutex> lk(m);
            src = s;
            dst = d;
            n = count;
            chunk = ck;
            nchunks = nc;
            for (int c = 0; c < nc; ++c) done[c].store(0, std::memory_order_relaxed);
            pending = workers;
            ++gen;
        }
        cv.notify_all();
        tc_status st = TC_OK;
        for (int c = 0; c < nc; ++c) {
            for (int spin = 0; done[c].load(std::memory_order_acquire) < workers; ++spin)
                if (spin > 64) std::this_thread::yield();
            const size_t a = std::min(count, ck * c);
            if (st == TC_OK) st = on_chunk(a, std::min(count, a + ck) - a);
        }
        std::unique_lock<std::mutex> lk(m);
        done_cv.wait(lk, [&] { return pending == 0; });
        return st;
    }
};

struct tc_ctx {
    const tc_plan* plan = nullptr;
    tc_ctx_desc desc{};
    int device = 0;
    cudaStream_t st = nullptr;
    ncclComm_t comm = nullptr;

    std::unordered_map<int, VarL> vars;
    std::vector<ParamL> params;
    std::unordered_map<int, int> storage_item;      // storage id -> item
    std::unordered_map<int, int> pool_idx_item;     // pool output var -> item (1-byte window-local argmax)
    std::unordered_map<int, int> bn_stats_item;     // BN input var -> item (2*C fp32)
    std::unordered_map<int, float> mask_rate;       // dropout mask var -> rate
    // BatchNorm backward: the BETA / DATA / GAMMA statements of one BN share the
    // reductions (sum dy, sum dy*xhat), computed once at the group's first statement
    struct BnGroup {
        int x_var = -1, up_var = -1, first = -1, gamma = -1;
        float* sums = nullptr;  // 5*C persistent floats: sum dy, sum dy*xhat, data-gradient k1..k3
    };
    std::vector<BnGroup> bn_groups;
    std::unordered_map<int, int> stmt_bn_group;     // BN_BWD_* stmt -> group
    float* bn_sums = nullptr;
    std::vector<Item> items;
    std::vector<uint8_t> fused;                     // stmt folded into its producer
    std::vector<uint8_t> fuse_bias, fuse_relu;      // producer flags
    std::vector<int> fuse_bias_param;
    std::vector<int> fuse_mask_var;                 // data-gradient producer: ReLU output var folded in (-1)
    std::vector<int> dropout_apply;                 // forward dropout product: its DropoutMask statement, folded in (-1)
    std::vector<int> fuse_add_res, fuse_add_out;    // BN forward: folded residual add (other operand, output var)
    std::vector<char> sgd_fused;                    // per param: momentum update fused into its FC filter gradient
    // bias gradient folded into the halo filter-gradient kernel of the same conv (bf16 mode):
    // per filter-gradient stmt the bias param it also produces; per bias stmt the producer (-1)
    std::vector<int> wgrad_bias_param, bias_fold_by;
    bool fuse_sgd_active = false;                   // set by run_body for update steps
    std::vector<char> pool_flag_nonpos;             // max-pool forward: flag windows with max <= 0 in the index
    std::vector<char> pool_mask_in_idx;             // max-pool backward: its folded ReLU mask is in the index
    // Softmax log-loss head: Softmax, Log(S.copy), 1/(S.copy), Y * c, product and
    // the softmax backward of one head as one row-wise kernel at the chain's first statement
    struct XentHead {
        int pos = -1;                    // statement that launches the fused kernel
        int z = -1, L = -1, Y = -1, dz = -1;
        bool write_y = false;            // the head also produces Cuda(Indicator(Y)) (fused LOAD_Y)
        float scale = 1.f;
    };
    std::vector<XentHead> xent;
    std::vector<int> stmt_xent;                     // stmt -> head launched there, or -1
    std::vector<std::pair<int, int>> early_start;   // (storage, stmt): written earlier than its Let

    uint8_t* arena = nullptr;
    size_t arena_bytes = 0, arena_keep_bytes = 0;
    uint8_t* slab = nullptr;
    size_t slab_bytes = 0;
    uint8_t* ws = nullptr;
    size_t ws_bytes = 0;
    float* partials = nullptr;
    int max_partials = 0;
    void* d_input = nullptr;  // staged input batch (bf16, or fp32 in TC_PREC_F32)
    int32_t* d_labels = nullptr;
    // Input pipeline: host batches are copied (NCHW fp32 + labels) into one of two
    // device staging slots on copy_st, overlapping the running step; the next step
    // converts the pending slot into the staged input layout on the main stream.
    float* d_stage[2] = {nullptr, nullptr};
    // bf16 host staging (TCB_HOST_BF16=1, bf16 mode): the host batch is rounded to bf16 by a pool
    // of host threads into pinned memory (chunk by chunk, each chunk's copy overlapping the next
    // chunk's rounding), so half the bytes cross the host link; the device staging kernel then
    // reads bf16 (bit-identical staged values).  Off by default: on a 16-core host the rounding is
    // host-memory bound (1.3 ms per AlexNet b128 batch) and costs more than the fp32 copy it halves
    // (1.4 ms, hidden under the 1.56 ms step): e2e 68k vs 77k images/s.
    uint16_t* h_stage16[2] = {nullptr, nullptr};
    bool host_bf16 = false;
    struct HostPool* pool = nullptr;
    int32_t* d_label_stage[2] = {nullptr, nullptr};
    cudaStream_t copy_st = nullptr;
    cudaEvent_t h2d_done[2] = {nullptr, nullptr}, conv_done[2] = {nullptr, nullptr};
    int stage_pending = -1, stage_next = 0;
    float* d_loss = nullptr;
    uint32_t* d_iter = nullptr;
    uint32_t* h_iter = nullptr;  // pinned
    float* h_loss = nullptr;     // pinned: two loss slots 16 floats apart (the last two steps)
    cudaEvent_t loss_ev[2] = {nullptr, nullptr};  // the slot's D2H has landed
    int loss_slot = 0, loss_count = 0;            // slot of the most recent loss; losses enqueued
    int input_cs = 8;
    StageLayout in_layout{};  // staged input image layout (space-to-depth when in_layout.s2d > 0)
    bool f32 = false;         // TC_PREC_F32: fp32 activations, 6-term bf16 split contractions
    uint8_t* split_buf = nullptr;  // split operand copies of the current contraction (f32 mode)
    size_t split_bytes = 0;
    size_t input_bytes = 0;

    // gradient buckets (backward production order); all-reduce + fused momentum
    // update run on comm_st, overlapped with the rest of the backward
    struct Bucket {
        int last_stmt = -1;      // Update statement that completes the bucket
        size_t off = 0;          // float offset into grads
        long long n = 0;         // floats (all-reduce count, includes alignment gaps)
        std::vector<int> params;
        cudaEvent_t ready = nullptr;
    };
    std::vector<Bucket> buckets;
    std::vector<std::vector<int>> stmt_flush;  // stmt -> buckets flushed after it (bucket order)
    float* grads = nullptr;        // contiguous gradient region inside the slab
    long long grads_n = 0;
    cudaStream_t comm_st = nullptr;
    cudaEvent_t join_ev = nullptr;
    bool overlap = true;

    // global-L2 gradient clipping (plan->clip > 0): every update waits for the
    // whole gradient; the clip factor is a device scalar read by the update kernel
    double* clip_partials = nullptr;
    float* d_clip = nullptr;  // [0] scale, [1] norm
    int last_update_stmt = -1;

    cudaGraph_t graph[2] = {nullptr, nullptr};
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    int runs[2] = {0, 0};
    int launches_per_step = -1;
    std::vector<int> prof_launches;  // kernels each statement launched in the last tc_profile_step
    std::vector<float> prof_update_ms;  // bucket all-reduce + momentum update completed after statement i
    // test body: the train-body Lets the main logits depend on, test-mode dropout
    std::vector<uint8_t> in_test;
    bool test_mode = false;
    unsigned* d_hits = nullptr;
    unsigned* h_hits = nullptr;  // pinned
    int64_t device_used = 0;
};

namespace {

// ------------------------------------------------------------------ analysis
tc_status analyze_layouts(tc_ctx* c) {
    const tc_plan* p = c->plan;
    for (int i = 0; i < p->nvars; ++i) {
        VarL v;
        v.id = p->vars[i].id;
        v.rank = p->vars[i].rank;
        for (int j = 0; j < v.rank; ++j) v.d[j] = p->vars[i].dims[j];
        c->vars[v.id] = v;
    }
    // params
    c->params.resize(p->nparams);
    for (int i = 0; i < p->nparams; ++i) {
        ParamL& q = c->params[i];
        const tc_param_desc& pd = p->params[i];
        q.rank = pd.rank;
        for (int j = 0; j < pd.rank; ++j) q.d[j] = pd.dims[j];
        if (pd.rank == 4) {
            q.kind = ParamL::CONV;
            q.K = static_cast<int>(pd.dims[0]);
            q.C = static_cast<int>(pd.dims[1]);
            q.R = static_cast<int>(pd.dims[2]);
            q.S = static_cast<int>(pd.dims[3]);
            q.cs = ceil8(q.C);
            q.ks = ceil8(q.K);
            q.n = static_cast<long long>(q.K) * q.R * q.S * q.cs;
        } else if (pd.rank == 2) {
            q.kind = ParamL::FC;
            q.K = static_cast<int>(pd.dims[0]);
            q.C = static_cast<int>(pd.dims[1]);
        } else {
            q.kind = ParamL::VEC;
            q.K = static_cast<int>(pd.dims[0]);
            q.n = q.K;
        }
    }
    // dtypes and layouts, in statement order
    std::unordered_map<int, int> fc_input_of_param;  // FC weight param -> forward input var
    for (int i = 0; i < p->nstmts; ++i) {
        const tc_stmt& s = p->stmts[i];
        if (s.kind == TC_STMT_LET) {
            VarL& v = c->vars.at(s.var);
            v.storage = s.storage;
            v.def = i;
        }
        if (s.op == TC_OP_MATMUL_FWD && s.in[1].kind == TC_REF_PARAM) fc_input_of_param[s.in[1].index] = s.in[0].index;
        if (s.op == TC_OP_DROPOUT_MASK) c->mask_rate[s.var] = static_cast<float>(s.rate);
    }
    for (int i = 0; i < p->nstmts; ++i) {
        const tc_stmt& s = p->stmts[i];
        if (s.kind != TC_STMT_LET) continue;
        VarL& v = c->vars.at(s.var);
        int dt = DT_BF16;
        switch (s.op) {
            case TC_OP_LOAD_Y:
            case TC_OP_SOFTMAX_FWD:
            case TC_OP_LOG:
            case TC_OP_RECIP: dt = DT_F32; break;
            case TC_OP_DROPOUT_MASK: dt = DT_U8; break;
            case TC_OP_SCALE:
            case TC_OP_MUL:
            case TC_OP_ADD:
                for (int k = 0; k < s.nin; ++k)
                    if (s.in[k].kind == TC_REF_VAR && c->vars.at(s.in[k].index).dtype == DT_F32) dt = DT_F32;
                break;
            default: break;
        }
        const bool head = dt == DT_F32;  // loss-head tensors: fp32 [N][F] in both precisions
        if (c->f32 && dt == DT_BF16) dt = DT_F32;
        v.dtype = dt;
        if (v.rank == 4) {
            v.nhwc = true;
            v.N = static_cast<int>(v.d[0]);
            v.C = static_cast<int>(v.d[1]);
            v.H = static_cast<int>(v.d[2]);
            v.W = static_cast<int>(v.d[3]);
            // the input image of <= 4 channels is staged with channel stride 4 (8-byte taps)
            v.cs = (s.op == TC_OP_LOAD_X && v.C <= 4 && !c->f32) ? 4 : ceil8(v.C);
        } else if (v.rank == 2) {
            v.N = static_cast<int>(v.d[0]);
            v.C = static_cast<int>(v.d[1]);
            v.cs = head ? v.C : ceil8(v.C);
            if (s.op == TC_OP_MATMUL_BWD_DATA && s.in[1].kind == TC_REF_PARAM) {
                // gradient of a flattened 4-D activation keeps that activation's NHWC layout
                auto it = fc_input_of_param.find(s.in[1].index);
                if (it != fc_input_of_param.end()) {
                    const VarL& a = c->vars.at(it->second);
                    if (a.nhwc) {
                        v.nhwc = true;
                        v.N = a.N;
                        v.H = a.H;
                        v.W = a.W;
                        v.C = a.C;
                        v.cs = a.cs;
                    }
                }
            }
        } else {
            return fail(TC_SHAPE_FAULT, "runtime: unsupported var rank " + std::to_string(v.rank));
        }
    }
    // conv filters follow their input's channel stride (cs = 4 for a <= 4-channel input image)
    for (int i = 0; i < p->nstmts; ++i) {
        const tc_stmt& s = p->stmts[i];
        if (s.kind != TC_STMT_LET || s.op != TC_OP_CONV_FWD || s.in[0].kind != TC_REF_VAR) continue;
        ParamL& q = c->params[s.in[1].index];
        q.cs = c->vars.at(s.in[0].index).cs;
    }
    // Space-to-depth for a strided first-layer conv on the cs = 4 input (AlexNet 11x11/4):
    // staging the image as [N][Hs][Ws][s*s*cs] turns it into a stride-1 Rp x Rp conv over
    // s*s*cs channels, which takes the TMA im2col operand path instead of 8-byte gathers:
    // 64 channels (SW128 boxes) for stride 4.
    {
        int xv = -1;
        for (int i = 0; i < p->nstmts; ++i)
            if (p->stmts[i].kind == TC_STMT_LET && p->stmts[i].op == TC_OP_LOAD_X) xv = p->stmts[i].var;
        int fwd = -1, uses = 0, other = 0;
        for (int i = 0; xv >= 0 && i < p->nstmts; ++i) {
            const tc_stmt& s = p->stmts[i];
            for (int k = 0; k < s.nin; ++k) {
                if (s.in[k].kind != TC_REF_VAR || s.in[k].index != xv) continue;
                if (s.op == TC_OP_CONV_FWD && k == 0) {
                    fwd = i;
                    ++uses;
                } else if (s.op != TC_OP_CONV_BWD_FILTER) {
                    ++other;
                }
            }
        }
        const char* e = std::getenv("TCB_S2D");
        const bool allowed = !(e && e[0] == '0') && !c->f32;
        if (allowed && xv >= 0 && uses == 1 && other == 0) {
            const tc_stmt& s = p->stmts[fwd];
            VarL& x = c->vars.at(xv);
            const VarL& y = c->vars.at(s.var);
            ParamL& q = c->params[s.in[1].index];
            const int st = s.stride;
            // (a stride-2 variant staging the image with channel stride 8 -> 32-channel SW64 boxes
            // measured slower for ResNet-50 / GoogLeNet conv1: wgrad 0.43 -> 0.56 ms)
            const int cs = (st * st * 4) % 64 == 0 ? 4 : 0;
            bool ok = x.cs == 4 && cs > 0 && st >= 2 && st <= 8 && q.R == q.S;
            for (int i = 0; ok && i < p->nstmts; ++i)
                if (p->stmts[i].op == TC_OP_CONV_BWD_DATA && p->stmts[i].in[1].kind == TC_REF_PARAM &&
                    p->stmts[i].in[1].index == s.in[1].index)
                    ok = false;
            if (ok) {
                x.cs = cs;
                q.cs = cs;
                q.s2d = st;
                q.Rp = (q.R + st - 1) / st;
                c->in_layout.s2d = st;
                c->in_layout.pad = s.pad;
                c->in_layout.Hs = y.H + q.Rp - 1;
                c->in_layout.Ws = y.W + q.Rp - 1;
            }
        }
    }
    for (ParamL& q : c->params) {
        if (q.kind != ParamL::CONV) continue;
        q.Kw = q.s2d ? q.Rp * q.Rp * q.s2d * q.s2d * q.cs : ceil8(static_cast<long long>(q.R) * q.S * q.cs);
        q.n = static_cast<long long>(q.K) * q.Kw;
    }
    // FC weight device layout follows its forward input
    for (int i = 0; i < p->nparams; ++i) {
        ParamL& q = c->params[i];
        if (q.kind != ParamL::FC) continue;
        auto it = fc_input_of_param.find(i);
        if (it != fc_input_of_param.end() && c->vars.at(it->second).nhwc) {
            const VarL& a = c->vars.at(it->second);
            q.fc_from4d = true;
            q.fH = a.H;
            q.fW = a.W;
            q.fC = a.C;
            q.fcs = a.cs;
            q.in_dev = a.H * a.W * a.cs;
        } else {
            q.in_dev = ceil8(q.C);
        }
        q.n = static_cast<long long>(q.K) * q.in_dev;
    }
    return TC_OK;
}

// Peephole fusion: GEMM producer followed by in-place BiasAdd / ReLU on its storage.
// TCB_POOL_IDX_FLAG=0 keeps the ReLU output read in the pooling backward (A/B switch).
// Fusion switches are read per context (plan_fusion), so tests can A/B them in one process.
static bool env_on(const char* name) {
    const char* e = std::getenv(name);
    return !(e && e[0] == '0');
}
static bool pool_idx_flag_enabled() { return env_on("TCB_POOL_IDX_FLAG"); }

// Softmax log-loss head fold (shared arena only: the parity mode materialises every var).  Per
// SOFTMAX_BWD(G, S): S = SOFTMAX_FWD(z), G = MUL(A, R), R = RECIP(S), A = SCALE(Y), Y = LOAD_Y, and
// L = LOG(S) (read by the Print).  The fused kernel runs at the chain's first statement and writes
// L, dz (and Y when LOAD_Y comes later); those storages start there (early_start).  It repeats the
// separate kernels' arithmetic operation for operation, so the fold is bit-identical.
void plan_xent_fusion(tc_ctx* c) {
    const tc_plan* p = c->plan;
    c->stmt_xent.assign(p->nstmts, -1);
    if (c->desc.keep || !env_on("TCB_XENT_FOLD")) return;
    std::unordered_map<int, int> def;     // var -> defining stmt
    std::unordered_map<int, int> readers;  // var -> number of reading statements
    for (int i = 0; i < p->nstmts; ++i) {
        const tc_stmt& s = p->stmts[i];
        if (s.kind == TC_STMT_LET) def[s.var] = i;
        if (s.kind == TC_STMT_DEALLOC) continue;
        for (int k = 0; k < s.nin; ++k)
            if (s.in[k].kind == TC_REF_VAR) readers[s.in[k].index]++;
    }
    auto op_of = [&](int var) { auto it = def.find(var); return it == def.end() ? -1 : p->stmts[it->second].op; };
    struct Cand {
        tc_ctx::XentHead h;
        std::vector<int> chain;
        int ly;
    };
    std::vector<Cand> cands;
    for (int b = 0; b < p->nstmts; ++b) {
        const tc_stmt& sb = p->stmts[b];
        if (sb.kind != TC_STMT_LET || sb.op != TC_OP_SOFTMAX_BWD || sb.nin != 2 || c->fused[b]) continue;
        const int G = sb.in[0].index, S = sb.in[1].index;
        if (op_of(S) != TC_OP_SOFTMAX_FWD || op_of(G) != TC_OP_MUL) continue;
        const tc_stmt& sm = p->stmts[def[G]];
        int A = sm.in[0].index, R = sm.in[1].index;
        if (op_of(A) == TC_OP_RECIP) std::swap(A, R);
        if (op_of(R) != TC_OP_RECIP || op_of(A) != TC_OP_SCALE) continue;
        const tc_stmt& sr = p->stmts[def[R]];
        const tc_stmt& sa = p->stmts[def[A]];
        if (sr.in[0].index != S) continue;
        const int Y = sa.in[0].index;
        if (op_of(Y) != TC_OP_LOAD_Y) continue;
        int lg = -1;
        for (int i = 0; i < p->nstmts; ++i)
            if (p->stmts[i].kind == TC_STMT_LET && p->stmts[i].op == TC_OP_LOG && p->stmts[i].in[0].index == S) lg = i;
        if (lg < 0) continue;
        // the intermediates feed only this chain
        if (readers[S] != 3 || readers[R] != 1 || readers[A] != 1 || readers[G] != 1) continue;
        const int f = def[S];
        const VarL& z = c->vars.at(p->stmts[f].in[0].index);
        const VarL& d = c->vars.at(sb.var);
        const VarL& Sv = c->vars.at(S);
        if (z.rank != 2 || d.rank != 2 || d.cs != z.cs || Sv.dtype != DT_F32 || Sv.cs != Sv.C) continue;
        Cand cd;
        cd.chain = {f, lg, def[R], def[A], def[G], b};
        cd.h.pos = *std::min_element(cd.chain.begin(), cd.chain.end());
        cd.h.z = p->stmts[f].in[0].index;
        cd.h.L = p->stmts[lg].var;
        cd.h.dz = sb.var;
        cd.h.Y = Y;
        cd.h.scale = static_cast<float>(sa.scale);
        cd.ly = def[Y];
        cands.push_back(cd);
    }
    // heads in launch order; the first one writes Y (and absorbs LOAD_Y) when LOAD_Y comes later
    std::sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) { return a.h.pos < b.h.pos; });
    std::unordered_map<int, int> y_written;
    for (Cand& cd : cands) {
        tc_ctx::XentHead& h = cd.h;
        if (cd.ly > h.pos && !y_written.count(h.Y)) {
            h.write_y = true;
            c->fused[cd.ly] = 1;
            c->early_start.emplace_back(c->vars.at(h.Y).storage, h.pos);
        }
        y_written[h.Y] = 1;
        for (int i : cd.chain) c->fused[i] = 1;
        c->early_start.emplace_back(c->vars.at(h.L).storage, h.pos);
        c->early_start.emplace_back(c->vars.at(h.dz).storage, h.pos);
        c->stmt_xent[h.pos] = static_cast<int>(c->xent.size());
        c->xent.push_back(h);
    }
}

void plan_fusion(tc_ctx* c) {
    const tc_plan* p = c->plan;
    c->fused.assign(p->nstmts, 0);
    c->fuse_bias.assign(p->nstmts, 0);
    c->fuse_relu.assign(p->nstmts, 0);
    c->fuse_bias_param.assign(p->nstmts, -1);
    c->fuse_mask_var.assign(p->nstmts, -1);
    c->dropout_apply.assign(p->nstmts, -1);
    c->pool_flag_nonpos.assign(p->nstmts, 0);
    c->fuse_add_res.assign(p->nstmts, -1);
    c->fuse_add_out.assign(p->nstmts, -1);
    c->pool_mask_in_idx.assign(p->nstmts, 0);
    auto next_let = [&](int i) {
        for (int j = i + 1; j < p->nstmts; ++j) {
            if (p->stmts[j].kind == TC_STMT_DEALLOC) continue;
            return p->stmts[j].kind == TC_STMT_LET ? j : -1;
        }
        return -1;
    };
    // In-place ReLU backward folded into the statement that produces its upstream gradient:
    // data-gradient GEMMs (bf16 mode: the epilogue multiplies by [relu output > 0] before the
    // store), pooling backward and LRN backward (both precisions)
    for (int i = 0; i < p->nstmts; ++i) {
        const tc_stmt& s = p->stmts[i];
        if (s.kind != TC_STMT_LET) continue;
        const bool gemm_fold = env_on("TCB_GEMM_RELU_FOLD");
        const bool gemm = s.op == TC_OP_CONV_BWD_DATA || s.op == TC_OP_MATMUL_BWD_DATA;
        // dropout backward product (one operand the byte mask) followed by the ReLU backward
        const bool drop_mul = s.op == TC_OP_MUL && s.nin == 2 && s.in[0].kind == TC_REF_VAR && s.in[1].kind == TC_REF_VAR &&
                              (c->vars.at(s.in[0].index).dtype == DT_U8 || c->vars.at(s.in[1].index).dtype == DT_U8);
        if (drop_mul && !env_on("TCB_DROPOUT_FOLD")) continue;
        // adjoint sum of an activation gradient (vector add kernel) followed by the ReLU backward
        const bool act_add = s.op == TC_OP_ADD && s.nin == 2 && c->vars.at(s.var).cs % 8 == 0 &&
                             c->vars.at(s.var).dtype == (c->f32 ? DT_F32 : DT_BF16) && env_on("TCB_ADD_RELU_FOLD");
        // concat backward slice copy (8-channel aligned) followed by the branch's ReLU backward
        const bool cat_bwd = s.op == TC_OP_CONCAT_BWD && s.offset % 8 == 0 && s.extent % 8 == 0 &&
                             c->vars.at(s.var).cs % 8 == 0 && s.in[0].kind == TC_REF_VAR &&
                             c->vars.at(s.in[0].index).cs % 8 == 0 && env_on("TCB_ADD_RELU_FOLD");
        if (!(gemm && !c->f32) && s.op != TC_OP_POOL_BWD && s.op != TC_OP_LRN_BWD && !drop_mul && !act_add && !cat_bwd)
            continue;
        // the next Let, skipping Update / Print statements that do not read this output (the
        // filter-gradient Update sits between a data gradient and its ReLU backward)
        int j = -1;
        for (int k = i + 1; k < p->nstmts; ++k) {
            const tc_stmt& t = p->stmts[k];
            if (t.kind == TC_STMT_DEALLOC) continue;
            if (t.kind == TC_STMT_LET) {
                j = k;
                break;
            }
            bool reads = false;
            for (int q = 0; q < t.nin; ++q) reads |= t.in[q].kind == TC_REF_VAR && t.in[q].index == s.var;
            if (reads) break;
        }
        if (j < 0) continue;
        const tc_stmt& r = p->stmts[j];
        if (r.op != TC_OP_RELU_BWD || !r.inplace || r.in[0].kind != TC_REF_VAR || r.in[0].index != s.var ||
            r.in[1].kind != TC_REF_VAR)
            continue;
        const VarL& y = c->vars.at(s.var);
        const VarL& m = c->vars.at(r.in[1].index);
        if (m.dtype != y.dtype || m.cs != y.cs || m.elems() != y.elems()) continue;
        if (s.op == TC_OP_LRN_BWD && r.in[1].index != s.in[2].index) continue;  // mask must be the LRN input
        // (FC data-gradient GEMMs run unsplit whether or not the mask is folded in, so the fold
        // changes nothing but the launch count: bit-identical)
        if (gemm && !gemm_fold) continue;
        c->fuse_mask_var[i] = r.in[1].index;
        c->fused[j] = 1;
        if (s.op == TC_OP_POOL_BWD && s.max_pool && s.k * s.k <= 127 && pool_idx_flag_enabled()) {
            // max pooling over the ReLU output: the mask at the argmax travels in the index byte
            const int f = c->vars.at(s.in[1].index).def;
            if (f >= 0 && p->stmts[f].op == TC_OP_POOL_FWD && p->stmts[f].in[0].kind == TC_REF_VAR &&
                p->stmts[f].in[0].index == r.in[1].index) {
                c->pool_flag_nonpos[f] = 1;
                c->pool_mask_in_idx[i] = 1;
            }
        }
    }
    for (int i = 0; i < p->nstmts; ++i) {
        const tc_stmt& s = p->stmts[i];
        if (s.kind != TC_STMT_LET || (s.op != TC_OP_CONV_FWD && s.op != TC_OP_MATMUL_FWD && s.op != TC_OP_BN_FWD &&
                                      s.op != TC_OP_ADD))
            continue;
        int j = next_let(i);
        if (s.op == TC_OP_MATMUL_FWD && j >= 0 && p->stmts[j].op == TC_OP_BIAS_ADD && p->stmts[j].inplace &&
            p->stmts[j].in[0].kind == TC_REF_VAR && p->stmts[j].in[0].index == s.var &&
            p->stmts[j].in[1].kind == TC_REF_PARAM) {
            c->fuse_bias[i] = 1;
            c->fuse_bias_param[i] = p->stmts[j].in[1].index;
            c->fused[j] = 1;
            const int prev = p->stmts[j].var;
            j = next_let(j);
            if (j >= 0 && p->stmts[j].op == TC_OP_RELU_FWD && p->stmts[j].inplace && p->stmts[j].in[0].index == prev) {
                c->fuse_relu[i] = 1;
                c->fused[j] = 1;
            }
            continue;
        }
        if ((s.op == TC_OP_CONV_FWD || s.op == TC_OP_BN_FWD || s.op == TC_OP_ADD) && j >= 0 &&
            p->stmts[j].op == TC_OP_RELU_FWD &&
            p->stmts[j].inplace &&
            p->stmts[j].in[0].kind == TC_REF_VAR && p->stmts[j].in[0].index == s.var) {
            c->fuse_relu[i] = 1;
            c->fused[j] = 1;
        }
    }
    // BatchNorm followed by the residual add that is its only reader (ResNet's y = relu(BN(x) + r)):
    // the BN apply pass reads r and writes the add's output (and its folded ReLU), saving the
    // write + re-read of the BN output.  Not in keep mode, where every var is materialised.
    const bool bn_add = env_on("TCB_BN_ADD_FOLD");
    for (int i = 0; bn_add && !c->desc.keep && i < p->nstmts; ++i) {
        const tc_stmt& s = p->stmts[i];
        if (s.kind != TC_STMT_LET || s.op != TC_OP_BN_FWD || c->fused[i] || c->fuse_relu[i]) continue;
        const int j = next_let(i);
        if (j < 0 || c->fused[j]) continue;
        const tc_stmt& a = p->stmts[j];
        if (a.op != TC_OP_ADD || a.nin != 2 || a.in[0].kind != TC_REF_VAR || a.in[1].kind != TC_REF_VAR) continue;
        const int k = a.in[0].index == s.var ? 1 : a.in[1].index == s.var ? 0 : -1;
        if (k < 0 || a.in[k].index == s.var) continue;
        int readers = 0;
        for (int q = 0; q < p->nstmts; ++q)
            for (int r = 0; p->stmts[q].kind != TC_STMT_DEALLOC && r < p->stmts[q].nin; ++r)
                readers += p->stmts[q].in[r].kind == TC_REF_VAR && p->stmts[q].in[r].index == s.var;
        if (readers != 1) continue;
        const VarL& y = c->vars.at(s.var);
        const VarL& r = c->vars.at(a.in[k].index);
        const VarL& o = c->vars.at(a.var);
        if (r.dtype != y.dtype || o.dtype != y.dtype || r.cs != y.cs || o.cs != y.cs || r.elems() != y.elems() ||
            o.elems() != y.elems())
            continue;
        c->fuse_add_res[i] = a.in[k].index;
        c->fuse_add_out[i] = a.var;
        c->fuse_relu[i] = c->fuse_relu[j];
        c->fused[j] = 1;
    }
    // DropoutMask folded into the forward product that consumes it: the product statement writes
    // the mask (kept for the backward) and x * mask * scale in one pass (TCB_DROPOUT_FOLD=0: off)
    for (int i = 0; env_on("TCB_DROPOUT_FOLD") && i < p->nstmts; ++i) {
        const tc_stmt& d = p->stmts[i];
        if (d.kind != TC_STMT_LET || d.op != TC_OP_DROPOUT_MASK || d.in[0].kind != TC_REF_VAR || c->fused[i]) continue;
        const int j = next_let(i);
        if (j < 0 || c->fused[j]) continue;
        const tc_stmt& m = p->stmts[j];
        if (m.op != TC_OP_MUL || m.nin != 2 || m.in[0].kind != TC_REF_VAR || m.in[1].kind != TC_REF_VAR) continue;
        const int xi = m.in[0].index == d.var ? 1 : m.in[1].index == d.var ? 0 : -1;
        if (xi < 0 || m.in[xi].index != d.in[0].index) continue;
        const VarL& x = c->vars.at(d.in[0].index);
        const VarL& y = c->vars.at(m.var);
        if (x.cs % 8 || y.cs != x.cs || y.dtype != x.dtype || c->vars.at(d.var).cs != x.cs) continue;
        c->dropout_apply[j] = i;
        c->fused[i] = 1;
    }
    plan_xent_fusion(c);
}

// Lifetime-interval packing of storages and companions into one arena.
void pack_items(std::vector<Item>& items, bool keep, size_t* total, size_t* keep_total) {
    std::vector<int> order(items.size());
    for (size_t i = 0; i < items.size(); ++i) order[i] = static_cast<int>(i);
    std::sort(order.begin(), order.end(), [&](int a, int b) {
        if (items[a].bytes != items[b].bytes) return items[a].bytes > items[b].bytes;
        return items[a].first < items[b].first;
    });
    *keep_total = 0;
    for (const Item& it : items) *keep_total += align256(it.bytes);
    std::vector<int> placed;
    size_t top = 0;
    for (int idx : order) {
        Item& it = items[idx];
        const size_t sz = align256(it.bytes);
        if (keep) {
            it.off = top;
            top += sz;
            continue;
        }
        // collect conflicting intervals sorted by offset, then first fit
        std::vector<std::pair<size_t, size_t>> busy;
        for (int o : placed) {
            const Item& q = items[o];
            if (q.last < it.first || it.last < q.first) continue;
            busy.emplace_back(q.off, q.off + align256(q.bytes));
        }
        std::sort(busy.begin(), busy.end());
        size_t off = 0;
        for (auto& [b0, b1] : busy) {
            if (off + sz <= b0) break;
            off = std::max(off, b1);
        }
        it.off = off;
        top = std::max(top, off + sz);
        placed.push_back(idx);
    }
    *total = top;
}

tc_status plan_arena(tc_ctx* c) {
    const tc_plan* p = c->plan;
    const int n = p->nstmts;
    // storage lifetimes
    std::unordered_map<int, Item> st;
    auto touch = [&](int storage, int i) {
        auto& it = st[storage];
        it.last = std::max(it.last, i);
    };
    for (int i = 0; i < n; ++i) {
        const tc_stmt& s = p->stmts[i];
        if (s.kind == TC_STMT_LET) {
            const VarL& v = c->vars.at(s.var);
            if (s.op == TC_OP_LOAD_X) continue;  // lives in the persistent input buffer
            auto f = st.find(s.storage);
            if (f == st.end()) {
                Item it;
                it.first = i;
                it.last = i;
                it.bytes = v.bytes();
                st[s.storage] = it;
            } else {
                f->second.bytes = std::max(f->second.bytes, v.bytes());
                f->second.last = std::max(f->second.last, i);
            }
        }
        if (s.kind == TC_STMT_LET || s.kind == TC_STMT_UPDATE || s.kind == TC_STMT_PRINT)
            for (int k = 0; k < s.nin; ++k)
                if (s.in[k].kind == TC_REF_VAR) {
                    const VarL& v = c->vars.at(s.in[k].index);
                    if (st.count(v.storage)) touch(v.storage, i);
                }
        if (s.kind == TC_STMT_DEALLOC && st.count(s.storage)) touch(s.storage, i);
    }
    for (const auto& [sid, pos] : c->early_start) {  // storages a fused kernel writes before their Let
        auto f = st.find(sid);
        if (f != st.end()) f->second.first = std::min(f->second.first, pos);
    }
    for (auto& [sid, it] : st) {
        c->storage_item[sid] = static_cast<int>(c->items.size());
        c->items.push_back(it);
    }
    // companions
    for (int i = 0; i < n; ++i) {
        const tc_stmt& s = p->stmts[i];
        if (s.kind != TC_STMT_LET) continue;
        if (s.op == TC_OP_POOL_FWD && s.max_pool) {
            Item it;
            it.first = i;
            it.last = i;
            it.bytes = static_cast<size_t>(c->vars.at(s.var).elems());
            for (int j = i + 1; j < n; ++j)
                if (p->stmts[j].op == TC_OP_POOL_BWD && p->stmts[j].in[1].kind == TC_REF_VAR &&
                    p->stmts[j].in[1].index == s.var)
                    it.last = j;
            c->pool_idx_item[s.var] = static_cast<int>(c->items.size());
            c->items.push_back(it);
        }
        if (s.op == TC_OP_BN_FWD) {
            const int xv = s.in[0].index;
            Item it;
            it.first = i;
            it.last = i;
            it.bytes = static_cast<size_t>(c->vars.at(xv).C) * 2 * 4;
            for (int j = i + 1; j < n; ++j) {
                const tc_stmt& b = p->stmts[j];
                if ((b.op == TC_OP_BN_BWD_DATA || b.op == TC_OP_BN_BWD_GAMMA) && b.in[1].kind == TC_REF_VAR &&
                    b.in[1].index == xv)
                    it.last = j;
                if (b.op == TC_OP_BN_BWD_BETA && b.in[0].kind == TC_REF_VAR) it.last = std::max(it.last, it.last);
            }
            c->bn_stats_item[xv] = static_cast<int>(c->items.size());
            c->items.push_back(it);
        }
    }
    pack_items(c->items, c->desc.keep != 0, &c->arena_bytes, &c->arena_keep_bytes);
    return TC_OK;
}

// ------------------------------------------------------------------ host layout permutations
// Device column of tap (r, s), channel c of a space-to-depth filter.
long long s2d_col(const ParamL& q, int r, int sx, int c) {
    const int st = q.s2d;
    return ((static_cast<long long>(r / st) * q.Rp + sx / st) * st * st + (r % st) * st + sx % st) * q.cs + c;
}

void ref_to_dev(const ParamL& q, const float* ref, std::vector<float>& dev) {
    dev.assign(q.n, 0.f);
    if (q.kind == ParamL::CONV && q.s2d) {
        for (int k = 0; k < q.K; ++k)
            for (int c = 0; c < q.C; ++c)
                for (int r = 0; r < q.R; ++r)
                    for (int sx = 0; sx < q.S; ++sx)
                        dev[static_cast<long long>(k) * q.Kw + s2d_col(q, r, sx, c)] =
                            ref[((static_cast<long long>(k) * q.C + c) * q.R + r) * q.S + sx];
    } else if (q.kind == ParamL::CONV) {  // [K][Kw], Kw >= R*S*cs, (r, s, c) order
        for (int k = 0; k < q.K; ++k)
            for (int c = 0; c < q.C; ++c)
                for (int r = 0; r < q.R; ++r)
                    for (int s = 0; s < q.S; ++s)
                        dev[static_cast<long long>(k) * q.Kw + (static_cast<long long>(r) * q.S + s) * q.cs + c] =
                            ref[((static_cast<long long>(k) * q.C + c) * q.R + r) * q.S + s];
    } else if (q.kind == ParamL::FC) {
        for (int o = 0; o < q.K; ++o) {
            if (q.fc_from4d) {
                for (int c = 0; c < q.fC; ++c)
                    for (int h = 0; h < q.fH; ++h)
                        for (int w = 0; w < q.fW; ++w)
                            dev[static_cast<long long>(o) * q.in_dev + (static_cast<long long>(h) * q.fW + w) * q.fcs + c] =
                                ref[static_cast<long long>(o) * q.C + (static_cast<long long>(c) * q.fH + h) * q.fW + w];
            } else {
                for (int j = 0; j < q.C; ++j) dev[static_cast<long long>(o) * q.in_dev + j] = ref[static_cast<long long>(o) * q.C + j];
            }
        }
    } else {
        for (int k = 0; k < q.K; ++k) dev[k] = ref[k];
    }
}

void dev_to_ref(const ParamL& q, const float* dev, float* ref) {
    if (q.kind == ParamL::CONV && q.s2d) {
        for (int k = 0; k < q.K; ++k)
            for (int c = 0; c < q.C; ++c)
                for (int r = 0; r < q.R; ++r)
                    for (int sx = 0; sx < q.S; ++sx)
                        ref[((static_cast<long long>(k) * q.C + c) * q.R + r) * q.S + sx] =
                            dev[static_cast<long long>(k) * q.Kw + s2d_col(q, r, sx, c)];
    } else if (q.kind == ParamL::CONV) {
        for (int k = 0; k < q.K; ++k)
            for (int c = 0; c < q.C; ++c)
                for (int r = 0; r < q.R; ++r)
                    for (int s = 0; s < q.S; ++s)
                        ref[((static_cast<long long>(k) * q.C + c) * q.R + r) * q.S + s] =
                            dev[static_cast<long long>(k) * q.Kw + (static_cast<long long>(r) * q.S + s) * q.cs + c];
    } else if (q.kind == ParamL::FC) {
        for (int o = 0; o < q.K; ++o) {
            if (q.fc_from4d) {
                for (int c = 0; c < q.fC; ++c)
                    for (int h = 0; h < q.fH; ++h)
                        for (int w = 0; w < q.fW; ++w)
                            ref[static_cast<long long>(o) * q.C + (static_cast<long long>(c) * q.fH + h) * q.fW + w] =
                                dev[static_cast<long long>(o) * q.in_dev + (static_cast<long long>(h) * q.fW + w) * q.fcs + c];
            } else {
                for (int j = 0; j < q.C; ++j) ref[static_cast<long long>(o) * q.C + j] = dev[static_cast<long long>(o) * q.in_dev + j];
            }
        }
    } else {
        for (int k = 0; k < q.K; ++k) ref[k] = dev[k];
    }
}

uint16_t f2bf(float f) {  // round to nearest even
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return static_cast<uint16_t>(u >> 16);
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

float bf2f(uint16_t b) {
    const uint32_t u = static_cast<uint32_t>(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

tc_status upload_dev_param(tc_ctx* c, int i, const std::vector<float>& dev) {
    ParamL& q = c->params[i];
    TCB_CUDA_CHECK(cudaMemcpyAsync(q.p, dev.data(), q.n * 4, cudaMemcpyHostToDevice, c->st));
    if (q.shadow) {
        std::vector<uint16_t> sh(q.n);
        for (long long j = 0; j < q.n; ++j) sh[j] = f2bf(dev[j]);
        TCB_CUDA_CHECK(cudaMemcpyAsync(q.shadow, sh.data(), q.n * 2, cudaMemcpyHostToDevice, c->st));
        if (q.rskc) {
            const int RS = q.R * q.S;
            std::vector<uint16_t> r(static_cast<size_t>(RS) * q.ks * q.cs, 0);
            for (int k = 0; k < q.K; ++k)
                for (int rs = 0; rs < RS; ++rs)
                    for (int cc = 0; cc < q.cs; ++cc)
                        r[q.crsk ? (static_cast<size_t>(cc) * RS + rs) * q.ks + k : (static_cast<size_t>(rs) * q.ks + k) * q.cs + cc] =
                            sh[(static_cast<size_t>(k) * RS + rs) * q.cs + cc];
            TCB_CUDA_CHECK(cudaMemcpyAsync(q.rskc, r.data(), r.size() * 2, cudaMemcpyHostToDevice, c->st));
        }
        TCB_CUDA_CHECK(cudaStreamSynchronize(c->st));  // host staging vectors go out of scope
    } else {
        TCB_CUDA_CHECK(cudaStreamSynchronize(c->st));
    }
    return TC_OK;
}

// ------------------------------------------------------------------ execution helpers
struct Ptrs {
    tc_ctx* c;
    void* var(int id) const {
        const VarL& v = c->vars.at(id);
        if (c->plan && v.def >= 0 && c->plan->stmts[v.def].op == TC_OP_LOAD_X) return c->d_input;
        auto it = c->storage_item.find(v.storage);
        return c->arena + c->items[it->second].off;
    }
    template <class T>
    T* as(const tc_ref& r) const {
        if (r.kind == TC_REF_PARAM) return reinterpret_cast<T*>(c->params[r.index].p);
        return reinterpret_cast<T*>(var(r.index));
    }
    const VarL& L(const tc_ref& r) const { return c->vars.at(r.index); }
};

tc_conv_desc conv_desc(const VarL& x, const ParamL& w, const VarL& y, const tc_stmt& s) {
    tc_conv_desc d;
    if (w.s2d) {  // stride-1 Rp x Rp conv over the space-to-depth staged input
        d.N = x.N;
        d.C = w.s2d * w.s2d * w.cs;
        d.H = y.H + w.Rp - 1;
        d.W = y.W + w.Rp - 1;
        d.K = w.K;
        d.R = d.S = w.Rp;
        d.stride = 1;
        d.pad = 0;
        d.Ho = y.H;
        d.Wo = y.W;
        d.cs = d.C;
        d.ks = y.cs;
        d.wld = w.Kw;
        return d;
    }
    d.N = x.N;
    d.C = x.C;
    d.H = x.H;
    d.W = x.W;
    d.K = w.K;
    d.R = w.R;
    d.S = w.S;
    d.stride = s.stride;
    d.pad = s.pad;
    d.Ho = y.H;
    d.Wo = y.W;
    d.cs = x.cs;
    d.ks = y.cs;
    d.wld = w.Kw;
    return d;
}

tc_status run_gemm_args(tc_ctx* c, tc_gemm_args& a) {
    a.workspace = c->ws;
    a.workspace_bytes = c->ws_bytes;
    return tc_gemm_bf16(&a, c->st);
}

// ---- fp32 precision mode: every contraction as one bf16 contraction over kSplitN bf16
// operand copies (hi / mid / lo parts pairing to the fp32 product down to 2^-24), laid side
// by side along channels / columns or stacked along images / rows (ops.cuh launch_split).
// Same tcgen05 kernels, fp32 outputs.
inline size_t al256(size_t v) { return (v + 255) & ~size_t(255); }

tc_conv_desc split_desc(const tc_conv_desc& d0, int which) {
    tc_conv_desc d = d0;
    if (which == 0) {  // fprop: input channels x3
        d.cs = d.C = kSplitN * d0.cs;
        d.wld = d0.R * d0.S * d.cs;
    } else if (which == 1) {  // bwd-data: output-gradient channels x3
        d.ks = kSplitN * d0.ks;
    } else {  // bwd-filter: images x3
        d.N = kSplitN * d0.N;
    }
    return d;
}

// bytes of the split operand copies of a contraction (A' then B', 256-aligned)
size_t split_need(const tc_conv_desc& d0, int which, const ParamL& w) {
    const size_t pin = static_cast<size_t>(d0.N) * d0.H * d0.W, pout = static_cast<size_t>(d0.N) * d0.Ho * d0.Wo;
    const size_t rs = static_cast<size_t>(d0.R) * d0.S;
    if (which == 0) return al256(pin * kSplitN * d0.cs * 2) + al256(static_cast<size_t>(w.K) * rs * kSplitN * d0.cs * 2);
    if (which == 1) return al256(pout * kSplitN * d0.ks * 2) + al256(rs * kSplitN * d0.ks * d0.cs * 2);
    return al256(kSplitN * pout * d0.ks * 2) + al256(kSplitN * pin * d0.cs * 2);
}

// which: 0 fprop (act = x; aux = bias), 1 bwd-data (act = dy), 2 bwd-filter (act = dy; aux = x)
tc_status split_conv(tc_ctx* c, int which, const tc_conv_desc& d0, const ParamL& w, const float* act, const float* aux,
                     int relu, float* out) {
    bf16* A = reinterpret_cast<bf16*>(c->split_buf);
    const size_t pin = static_cast<size_t>(d0.N) * d0.H * d0.W, pout = static_cast<size_t>(d0.N) * d0.Ho * d0.Wo;
    const int RS = d0.R * d0.S;
    const tc_conv_desc d = split_desc(d0, which);
    tc_status r;
    if (which == 0) {  // act = x [pin][cs]; weights p [K][RS][cs]
        bf16* B = A + al256(pin * kSplitN * d0.cs * 2) / 2;
        r = launch_split(act, pin, d0.cs, A, pin, d0.cs, SPLIT_COLS, SPLIT_A, c->st);
        if (r == TC_OK) r = launch_split(w.p, static_cast<long long>(w.K) * RS, d0.cs, B, static_cast<long long>(w.K) * RS,
                                          d0.cs, SPLIT_COLS, SPLIT_B, c->st);
        if (r == TC_OK) r = conv_fwd_ex(&d, A, B, aux, relu, out, 1, c->ws, c->ws_bytes, c->st);
    } else if (which == 1) {  // act = dy [pout][ks]
        bf16* B = A + al256(pout * kSplitN * d0.ks * 2) / 2;
        r = launch_split(act, pout, d0.ks, A, pout, d0.ks, SPLIT_COLS, SPLIT_A, c->st);
        if (r == TC_OK) r = launch_split_rskc(w.p, w.Kw, w.K, RS, d0.cs, d0.ks, B, SPLIT_B, c->st);
        if (r == TC_OK) r = conv_bwd_data_ex(&d, A, B, out, 1, c->ws, c->ws_bytes, c->st);
    } else {  // act = dy [pout][ks], aux = x [pin][cs]
        bf16* B = A + al256(kSplitN * pout * d0.ks * 2) / 2;
        r = launch_split(act, pout, d0.ks, A, pout, d0.ks, SPLIT_ROWS, SPLIT_A, c->st);
        if (r == TC_OK) r = launch_split(aux, pin, d0.cs, B, pin, d0.cs, SPLIT_ROWS, SPLIT_B, c->st);
        if (r == TC_OK) r = tc_conv2d_bwd_filter(&d, A, B, out, c->ws, c->ws_bytes, c->st);
    }
    return r;
}

// FC forms: 0 fwd  Y[M][N] = A[M][K] W[N][K]^T;  1 bwd-data  dX = dY[M][Kd] W[Kd][N] (W rows Kr <= Kd);
//           2 bwd-W  dW[Nout][N] = dY^T (rows = batch)
size_t split_fc_need(int form, int M, int N, int K) {
    if (form == 0) return al256(static_cast<size_t>(M) * kSplitN * K * 2) + al256(static_cast<size_t>(N) * kSplitN * K * 2);
    if (form == 1) return al256(static_cast<size_t>(M) * kSplitN * K * 2) + al256(static_cast<size_t>(kSplitN) * K * N * 2);
    return al256(static_cast<size_t>(kSplitN) * K * M * 2) + al256(static_cast<size_t>(kSplitN) * K * N * 2);
}

// (sum dy, sum dy*xhat) of the BN group of BN_BWD_* statement i; reduced at the group's first statement.
template <typename T>
tc_status bn_group_sums(tc_ctx* c, int i, const float** sums) {
    auto it = c->stmt_bn_group.find(i);
    if (it == c->stmt_bn_group.end()) return fail(TC_INTERNAL, "runtime: BN backward statement without a group");
    const tc_ctx::BnGroup& gr = c->bn_groups[it->second];
    if (gr.first == i) {
        Ptrs P{c};
        const VarL& x = c->vars.at(gr.x_var);
        const float* stats = reinterpret_cast<float*>(c->arena + c->items[c->bn_stats_item.at(x.id)].off);
        tc_status r = launch_bn_bwd_reduce(reinterpret_cast<const T*>(P.var(gr.up_var)),
                                           reinterpret_cast<const T*>(P.var(x.id)), c->params[gr.gamma].p, stats, gr.sums,
                                           static_cast<long long>(x.N) * x.H * x.W, x.C, x.cs, c->partials,
                                           c->max_partials, c->st);
        if (r != TC_OK) return r;
    }
    *sums = gr.sums;
    return TC_OK;
}

// Gradient op of an Update (or a parameter-shaped Let) into `g` (device param layout).
SgdTensor sgd_tensor(tc_ctx* c, int pidx);

template <typename T>
tc_status compute_param_grad(tc_ctx* c, int idx, int pidx, float* g) {
    const tc_stmt& s = c->plan->stmts[idx];
    Ptrs P{c};
    const ParamL& q = c->params[pidx];
    cudaStream_t st = c->st;
    switch (s.op) {
        case TC_OP_CONV_BWD_FILTER: {
            const VarL& dy = P.L(s.in[0]);
            const VarL& x = P.L(s.in[1]);
            tc_conv_desc d = conv_desc(x, q, dy, s);
            if constexpr (std::is_same_v<T, float>)
                return split_conv(c, 2, d, q, static_cast<const float*>(P.var(dy.id)), static_cast<const float*>(P.var(x.id)),
                                  0, g);
            const int bp = c->wgrad_bias_param[idx];
            tc_status r = conv_bwd_filter_ex(&d, P.var(dy.id), P.var(x.id), g, bp >= 0 ? c->params[bp].g : nullptr,
                                             c->ws, c->ws_bytes, st);
            if (r != TC_OK || !q.s2d) return r;
            return launch_s2d_mask_grad(g, q.K, q.Kw, q.Rp, q.s2d, q.cs, q.R, q.S, st);
        }
        case TC_OP_BN_BWD_BETA:
        case TC_OP_BN_BWD_GAMMA: {
            const float* sums = nullptr;
            tc_status r = bn_group_sums<T>(c, idx, &sums);
            if (r != TC_OK) return r;
            TCB_CUDA_CHECK(cudaMemcpyAsync(g, sums + (s.op == TC_OP_BN_BWD_GAMMA ? q.K : 0), q.K * sizeof(float),
                                           cudaMemcpyDeviceToDevice, st));
            return TC_OK;
        }
        case TC_OP_CONV_BWD_BIAS:
        case TC_OP_BIAS_GRAD: {
            const VarL& up = P.L(s.in[0]);
            return launch_colsum(reinterpret_cast<const T*>(P.var(up.id)), static_cast<long long>(up.N) * up.H * up.W,
                                 q.K, up.cs, g, c->partials, c->max_partials, st);
        }
        case TC_OP_MATMUL_BWD_W: {
            const VarL& up = P.L(s.in[0]);
            const VarL& a = P.L(s.in[1]);
            tc_gemm_args ga{};
            if constexpr (std::is_same_v<T, float>) {  // K = batch: copies stacked along the rows
                bf16* As = reinterpret_cast<bf16*>(c->split_buf);
                bf16* Bs = As + al256(static_cast<size_t>(kSplitN) * up.N * up.cs * 2) / 2;
                tc_status r = launch_split(static_cast<const float*>(P.var(up.id)), up.N, up.cs, As, up.N, up.cs,
                                            SPLIT_ROWS, SPLIT_A, st);
                if (r == TC_OK)
                    r = launch_split(static_cast<const float*>(P.var(a.id)), up.N, q.in_dev, Bs, up.N, q.in_dev, SPLIT_ROWS,
                                      SPLIT_B, st);
                if (r != TC_OK) return r;
                ga.M = q.K;
                ga.N = q.in_dev;
                ga.K = kSplitN * up.N;
                ga.a_layout = TC_LAYOUT_MN;
                ga.A = As;
                ga.lda = up.cs;
                ga.b_layout = TC_LAYOUT_MN;
                ga.B = Bs;
                ga.ldb = q.in_dev;
                ga.D = g;
                ga.ldd = q.in_dev;
                ga.d_dtype = TC_DTYPE_F32;
                ga.alpha = 1.f;
                return run_gemm_args(c, ga);
            }
            ga.M = q.K;
            ga.N = q.in_dev;
            ga.K = up.N;
            ga.a_layout = TC_LAYOUT_MN;
            ga.A = P.var(up.id);
            ga.lda = up.cs;
            ga.b_layout = TC_LAYOUT_MN;
            ga.B = P.var(a.id);
            ga.ldb = q.in_dev;
            ga.D = g;
            ga.ldd = q.in_dev;
            ga.d_dtype = TC_DTYPE_F32;
            ga.alpha = 1.f;
            const int bp = c->wgrad_bias_param[idx];  // folded FC bias gradient (column sums of dy)
            if (c->fuse_sgd_active && c->sgd_fused[pidx]) {  // update fused into the epilogue
                const SgdTensor t = sgd_tensor(c, pidx);
                ga.workspace = c->ws;
                ga.workspace_bytes = c->ws_bytes;
                return gemm_args_ex(&ga, &t, c->st, bp >= 0 ? c->params[bp].g : nullptr);
            }
            if (bp >= 0) {
                ga.workspace = c->ws;
                ga.workspace_bytes = c->ws_bytes;
                return gemm_args_ex(&ga, nullptr, c->st, c->params[bp].g);
            }
            return run_gemm_args(c, ga);
        }
        default: break;
    }
    return fail(TC_INTERNAL, "runtime: unsupported parameter-gradient op " + std::to_string(s.op));
}

template <typename T>
tc_status exec_let(tc_ctx* c, int i) {
    const tc_stmt& s = c->plan->stmts[i];
    Ptrs P{c};
    cudaStream_t st = c->st;
    const VarL& out = c->vars.at(s.var);
    void* y = P.var(s.var);
    if (c->test_mode && s.op == TC_OP_DROPOUT_MASK) return TC_OK;  // test-mode dropout = identity
    if (c->test_mode && s.op == TC_OP_MUL) {
        const VarL& a = P.L(s.in[0]);
        const VarL& b = P.L(s.in[1]);
        if (a.dtype == DT_U8 || b.dtype == DT_U8) {
            const VarL& x = b.dtype == DT_U8 ? a : b;
            TCB_CUDA_CHECK(cudaMemcpyAsync(y, P.var(x.id), out.bytes(), cudaMemcpyDeviceToDevice, st));
            return TC_OK;
        }
    }
    switch (s.op) {
        case TC_OP_LOAD_X: return TC_OK;  // the staged input buffer is the var's storage
        case TC_OP_LOAD_Y: return launch_onehot(c->d_labels, reinterpret_cast<float*>(y), out.N, out.C, st);
        case TC_OP_CONV_FWD: {
            const VarL& x = P.L(s.in[0]);
            const ParamL& w = c->params[s.in[1].index];
            const float* bias = s.nin > 2 ? c->params[s.in[2].index].p : nullptr;
            tc_conv_desc d = conv_desc(x, w, out, s);
            if constexpr (std::is_same_v<T, float>)
                return split_conv(c, 0, d, w, static_cast<const float*>(P.var(x.id)), bias, c->fuse_relu[i],
                                  static_cast<float*>(y));
            return tc_conv2d_fwd(&d, P.var(x.id), w.shadow, bias, c->fuse_relu[i], y, c->ws, c->ws_bytes, st);
        }
        case TC_OP_CONV_BWD_DATA: {
            const VarL& dy = P.L(s.in[0]);
            const ParamL& w = c->params[s.in[1].index];
            tc_conv_desc d = conv_desc(out, w, dy, s);
            if constexpr (std::is_same_v<T, float>)
                return split_conv(c, 1, d, w, static_cast<const float*>(P.var(dy.id)), nullptr, 0, static_cast<float*>(y));
            return conv_bwd_data_ex(&d, P.var(dy.id), w.rskc, y, 0, c->ws, c->ws_bytes, st,
                                    c->fuse_mask_var[i] >= 0 ? P.var(c->fuse_mask_var[i]) : nullptr, w.crsk ? 1 : 0);
        }
        case TC_OP_POOL_FWD: {
            const VarL& x = P.L(s.in[0]);
            uint8_t* idx = s.max_pool ? reinterpret_cast<uint8_t*>(c->arena + c->items[c->pool_idx_item.at(s.var)].off) : nullptr;
            return launch_pool_fwd(reinterpret_cast<const T*>(P.var(x.id)), x.act(), reinterpret_cast<T*>(y),
                                   out.act(), idx, s.k, s.stride, s.pad, s.max_pool, c->pool_flag_nonpos[i], st);
        }
        case TC_OP_POOL_BWD: {
            const VarL& up = P.L(s.in[0]);
            const VarL& fy = P.L(s.in[1]);
            const uint8_t* idx = s.max_pool ? reinterpret_cast<uint8_t*>(c->arena + c->items[c->pool_idx_item.at(fy.id)].off)
                                            : nullptr;
            Act4 ya = fy.act();
            return launch_pool_bwd(reinterpret_cast<const T*>(P.var(up.id)), ya, idx, reinterpret_cast<T*>(y),
                                   out.act(), s.k, s.stride, s.pad, s.max_pool,
                                   c->fuse_mask_var[i] >= 0 && !c->pool_mask_in_idx[i]
                                       ? reinterpret_cast<const T*>(P.var(c->fuse_mask_var[i]))
                                                            : static_cast<const T*>(nullptr),
                                   st);
        }
        case TC_OP_RELU_FWD:
            return launch_relu_fwd(reinterpret_cast<const T*>(P.var(s.in[0].index)), reinterpret_cast<T*>(y),
                                   out.elems(), st);
        case TC_OP_RELU_BWD:
            return launch_relu_bwd(reinterpret_cast<const T*>(P.var(s.in[0].index)),
                                   reinterpret_cast<const T*>(P.var(s.in[1].index)), reinterpret_cast<T*>(y),
                                   out.elems(), st);
        case TC_OP_SOFTMAX_FWD: {
            const VarL& x = P.L(s.in[0]);
            return launch_softmax_fwd(reinterpret_cast<const T*>(P.var(x.id)), x.cs, reinterpret_cast<float*>(y), out.N,
                                      out.C, st);
        }
        case TC_OP_SOFTMAX_BWD:
            return launch_softmax_bwd(reinterpret_cast<const float*>(P.var(s.in[0].index)),
                                      reinterpret_cast<const float*>(P.var(s.in[1].index)), reinterpret_cast<T*>(y),
                                      out.cs, out.N, out.C, st);
        case TC_OP_LRN_FWD:
            return launch_lrn_fwd(reinterpret_cast<const T*>(P.var(s.in[0].index)), reinterpret_cast<T*>(y), out.act(),
                                  s.lrn_size, static_cast<float>(s.alpha), static_cast<float>(s.beta),
                                  static_cast<float>(s.lrn_k), st);
        case TC_OP_LRN_BWD:
            return launch_lrn_bwd(reinterpret_cast<const T*>(P.var(s.in[0].index)),
                                  reinterpret_cast<const T*>(P.var(s.in[2].index)),
                                  reinterpret_cast<const T*>(P.var(s.in[1].index)), reinterpret_cast<T*>(y),
                                  out.act(), s.lrn_size, static_cast<float>(s.alpha), static_cast<float>(s.beta),
                                  static_cast<float>(s.lrn_k), c->fuse_mask_var[i] >= 0 ? 1 : 0, st);
        case TC_OP_DROPOUT_MASK:
            return launch_dropout_mask(reinterpret_cast<uint8_t*>(y), out.N, out.H, out.W, out.C, out.cs,
                                       static_cast<float>(s.rate), c->desc.seed, static_cast<uint32_t>(s.var), c->d_iter,
                                       st);
        case TC_OP_MUL: {
            const VarL& a = P.L(s.in[0]);
            const VarL& b = P.L(s.in[1]);
            if (out.dtype == DT_F32 && a.dtype != DT_U8 && b.dtype != DT_U8)  // loss-head product
                return launch_f32_ew(F32_MUL, reinterpret_cast<const float*>(P.var(a.id)),
                                     reinterpret_cast<const float*>(P.var(b.id)), 1.f, reinterpret_cast<float*>(y),
                                     out.elems(), st);
            const VarL& m = b.dtype == DT_U8 ? b : a;
            const VarL& x = b.dtype == DT_U8 ? a : b;
            if (m.dtype != DT_U8) return fail(TC_INTERNAL, "runtime: activation x activation MUL is not in the op set");
            const float rate = c->mask_rate.at(m.id);
            if (const int di = c->dropout_apply[i]; di >= 0)  // the folded DropoutMask statement
                return launch_dropout_apply(reinterpret_cast<const T*>(P.var(x.id)), reinterpret_cast<uint8_t*>(P.var(m.id)),
                                            reinterpret_cast<T*>(y), m.N, m.H, m.W, m.C, m.cs, rate, c->desc.seed,
                                            static_cast<uint32_t>(c->plan->stmts[di].var), c->d_iter, st);
            return launch_mask_mul(reinterpret_cast<const T*>(P.var(x.id)), reinterpret_cast<const uint8_t*>(P.var(m.id)),
                                   1.f / (1.f - rate), reinterpret_cast<T*>(y), out.elems(), st,
                                   c->fuse_mask_var[i] >= 0 ? reinterpret_cast<const T*>(P.var(c->fuse_mask_var[i])) : nullptr);
        }
        case TC_OP_ADD:
            // loss-head sums (fp32, unpadded rows) take the scalar kernel; activations the vector one
            if (out.dtype == DT_F32 && (!std::is_same_v<T, float> || out.cs % 8))
                return launch_f32_ew(F32_ADD, reinterpret_cast<const float*>(P.var(s.in[0].index)),
                                     reinterpret_cast<const float*>(P.var(s.in[1].index)), 1.f, reinterpret_cast<float*>(y),
                                     out.elems(), st);
            return launch_add(reinterpret_cast<const T*>(P.var(s.in[0].index)),
                                   reinterpret_cast<const T*>(P.var(s.in[1].index)), reinterpret_cast<T*>(y),
                                   out.elems(), c->fuse_relu[i], st,
                                   c->fuse_mask_var[i] >= 0 ? reinterpret_cast<const T*>(P.var(c->fuse_mask_var[i])) : nullptr);
        case TC_OP_SCALE:
        case TC_OP_LOG:
        case TC_OP_RECIP: {
            if (out.dtype != DT_F32) return fail(TC_INTERNAL, "runtime: Log/Recip/Scale expected on fp32 loss-head tensors");
            const int op = s.op == TC_OP_LOG ? F32_LOG : s.op == TC_OP_RECIP ? F32_RECIP : F32_SCALE;
            return launch_f32_ew(op, reinterpret_cast<const float*>(P.var(s.in[0].index)), nullptr,
                                 static_cast<float>(s.scale), reinterpret_cast<float*>(y), out.elems(), st);
        }
        case TC_OP_MATMUL_FWD: {
            const VarL& a = P.L(s.in[0]);
            const ParamL& w = c->params[s.in[1].index];
            tc_gemm_args ga{};
            if constexpr (std::is_same_v<T, float>) {  // copies side by side along K
                bf16* As = reinterpret_cast<bf16*>(c->split_buf);
                bf16* Bs = As + al256(static_cast<size_t>(a.N) * kSplitN * w.in_dev * 2) / 2;
                tc_status r = launch_split(static_cast<const float*>(P.var(a.id)), a.N, w.in_dev, As, a.N, w.in_dev,
                                            SPLIT_COLS, SPLIT_A, st);
                if (r == TC_OK)
                    r = launch_split(w.p, out.C, w.in_dev, Bs, out.C, w.in_dev, SPLIT_COLS, SPLIT_B, st);
                if (r != TC_OK) return r;
                ga.M = a.N;
                ga.N = out.cs;
                ga.K = kSplitN * w.in_dev;
                ga.a_layout = TC_LAYOUT_K;
                ga.A = As;
                ga.lda = kSplitN * w.in_dev;
                ga.b_layout = TC_LAYOUT_K;
                ga.B = Bs;
                ga.ldb = kSplitN * w.in_dev;
                ga.D = y;
                ga.ldd = out.cs;
                ga.d_dtype = TC_DTYPE_F32;
                ga.bias = c->fuse_bias[i] ? c->params[c->fuse_bias_param[i]].p : nullptr;
                ga.bias_n = out.C;
                ga.b_rows = out.C;
                ga.relu = c->fuse_relu[i];
                ga.alpha = 1.f;
                return run_gemm_args(c, ga);
            }
            ga.M = a.N;
            ga.N = out.cs;  // padded columns come out as zeros (zero weight rows, masked bias)
            ga.K = w.in_dev;
            ga.a_layout = TC_LAYOUT_K;
            ga.A = P.var(a.id);
            ga.lda = w.in_dev;
            ga.b_layout = TC_LAYOUT_K;
            ga.B = w.shadow;
            ga.ldb = w.in_dev;
            ga.D = y;
            ga.ldd = out.cs;
            ga.d_dtype = TC_DTYPE_BF16;
            ga.bias = c->fuse_bias[i] ? c->params[c->fuse_bias_param[i]].p : nullptr;
            ga.bias_n = out.C;  // the bias param has exactly out.C entries; padded columns get 0
            ga.b_rows = out.C;  // the weight has out.C rows: never read past it
            ga.relu = c->fuse_relu[i];
            ga.alpha = 1.f;
            return run_gemm_args(c, ga);
        }
        case TC_OP_MATMUL_BWD_DATA: {
            const VarL& up = P.L(s.in[0]);
            const ParamL& w = c->params[s.in[1].index];
            tc_gemm_args ga{};
            if constexpr (std::is_same_v<T, float>) {  // K = up.cs: A copies side by side, W copies stacked
                bf16* As = reinterpret_cast<bf16*>(c->split_buf);
                bf16* Bs = As + al256(static_cast<size_t>(up.N) * kSplitN * up.cs * 2) / 2;
                tc_status r = launch_split(static_cast<const float*>(P.var(up.id)), up.N, up.cs, As, up.N, up.cs,
                                            SPLIT_COLS, SPLIT_A, st);
                if (r == TC_OK)
                    r = launch_split(w.p, w.K, w.in_dev, Bs, up.cs, w.in_dev, SPLIT_ROWS, SPLIT_B, st);
                if (r != TC_OK) return r;
                ga.M = up.N;
                ga.N = w.in_dev;
                ga.K = kSplitN * up.cs;
                ga.a_layout = TC_LAYOUT_K;
                ga.A = As;
                ga.lda = kSplitN * up.cs;
                ga.b_layout = TC_LAYOUT_MN;
                ga.B = Bs;
                ga.ldb = w.in_dev;
                ga.D = y;
                ga.ldd = w.in_dev;
                ga.d_dtype = TC_DTYPE_F32;
                ga.alpha = 1.f;
                return run_gemm_args(c, ga);
            }
            ga.M = up.N;
            ga.N = w.in_dev;
            ga.K = w.K;
            ga.a_layout = TC_LAYOUT_K;
            ga.A = P.var(up.id);
            ga.lda = up.cs;
            ga.b_layout = TC_LAYOUT_MN;
            ga.B = w.shadow;
            ga.ldb = w.in_dev;
            ga.D = y;
            ga.ldd = w.in_dev;
            ga.d_dtype = TC_DTYPE_BF16;
            ga.alpha = 1.f;
            if (c->fuse_mask_var[i] >= 0) {  // the following ReLU backward, folded into the epilogue
                ga.relu_mask = P.var(c->fuse_mask_var[i]);
                ga.mask_ld = w.in_dev;
            }
            // unsplit: the mask is applied by the tile epilogue, not by a split-K reduce (unfolded,
            // the same contraction runs: identical summation order either way), and without a mask
            // the N = in-features side already fills the grid (AlexNet fc6 bwd-data, 128 x 9216 x
            // 4096: 15.1 us unsplit vs 23.5 us with the cost model's split-K + reduce, in-graph)
            ga.splits = 1;
            return run_gemm_args(c, ga);
        }
        case TC_OP_BIAS_ADD: {
            const VarL& x = P.L(s.in[0]);
            return launch_bias_add(reinterpret_cast<const T*>(P.var(x.id)), c->params[s.in[1].index].p,
                                   reinterpret_cast<T*>(y), static_cast<long long>(x.N) * x.H * x.W, x.C, x.cs, 0, st);
        }
        case TC_OP_CONCAT: {
            if (out.cs != out.C) {
                tc_status r = launch_zero(y, out.bytes(), st);
                if (r != TC_OK) return r;
            }
            int off = 0;
            for (int k = 0; k < s.nin; ++k) {
                const VarL& part = P.L(s.in[k]);
                tc_status r = launch_channel_copy(reinterpret_cast<const T*>(P.var(part.id)), part.cs,
                                                  reinterpret_cast<T*>(y), out.cs, off, part.C,
                                                  static_cast<long long>(out.N) * out.H * out.W, st);
                if (r != TC_OK) return r;
                off += part.C;
            }
            return TC_OK;
        }
        case TC_OP_CONCAT_BWD: {
            const VarL& up = P.L(s.in[0]);
            if (out.cs != out.C) {
                tc_status r = launch_zero(y, out.bytes(), st);
                if (r != TC_OK) return r;
            }
            return launch_channel_copy(reinterpret_cast<const T*>(P.var(up.id)) + s.offset, up.cs,
                                       reinterpret_cast<T*>(y), out.cs, 0, static_cast<int>(s.extent),
                                       static_cast<long long>(out.N) * out.H * out.W, st,
                                       c->fuse_mask_var[i] >= 0 ? reinterpret_cast<const T*>(P.var(c->fuse_mask_var[i])) : nullptr);
        }
        case TC_OP_BN_FWD: {
            const VarL& x = P.L(s.in[0]);
            float* stats = reinterpret_cast<float*>(c->arena + c->items[c->bn_stats_item.at(x.id)].off);
            const bool add = c->fuse_add_res[i] >= 0;  // folded residual add (its output var is written)
            return launch_bn_fwd(reinterpret_cast<const T*>(P.var(x.id)), c->params[s.in[1].index].p,
                                 c->params[s.in[2].index].p,
                                 reinterpret_cast<T*>(add ? P.var(c->fuse_add_out[i]) : y), stats,
                                 static_cast<long long>(x.N) * x.H * x.W, x.C, x.cs, static_cast<float>(s.eps),
                                 c->fuse_relu[i],
                                 add ? reinterpret_cast<const T*>(P.var(c->fuse_add_res[i])) : static_cast<const T*>(nullptr),
                                 c->partials, c->max_partials, st);
        }
        case TC_OP_BN_BWD_DATA: {
            const VarL& up = P.L(s.in[0]);
            const VarL& x = P.L(s.in[1]);
            const float* sums = nullptr;  // sums[2C..5C): k1..k3 from the group's reduction
            tc_status r = bn_group_sums<T>(c, i, &sums);
            if (r != TC_OK) return r;
            return launch_bn_bwd_apply(reinterpret_cast<const T*>(P.var(up.id)),
                                       reinterpret_cast<const T*>(P.var(x.id)), sums + 2 * x.C, reinterpret_cast<T*>(y),
                                       static_cast<long long>(x.N) * x.H * x.W, x.C, x.cs, st);
        }
        default: break;
    }
    return fail(TC_INTERNAL, "runtime: unsupported Let op " + std::to_string(s.op));
}

tc_status exec_stmt(tc_ctx* c, int i) {
    const tc_stmt& s = c->plan->stmts[i];
    if (s.kind == TC_STMT_DEALLOC) return TC_OK;  // static arena: lifetimes were resolved at plan load
    if (!c->stmt_xent.empty() && c->stmt_xent[i] >= 0) {
        const tc_ctx::XentHead& h = c->xent[c->stmt_xent[i]];
        Ptrs P{c};
        const VarL& z = c->vars.at(h.z);
        const VarL& L = c->vars.at(h.L);
        float* y = h.write_y ? static_cast<float*>(P.var(h.Y)) : nullptr;
        return c->f32 ? launch_softmax_xent(static_cast<const float*>(P.var(h.z)), z.cs, c->d_labels, h.scale,
                                            static_cast<float*>(P.var(h.L)), y, static_cast<float*>(P.var(h.dz)), z.N, L.C,
                                            c->st)
                      : launch_softmax_xent(static_cast<const bf16*>(P.var(h.z)), z.cs, c->d_labels, h.scale,
                                            static_cast<float*>(P.var(h.L)), y, static_cast<bf16*>(P.var(h.dz)), z.N, L.C,
                                            c->st);
    }
    if (s.kind == TC_STMT_LET) return c->fused[i] ? TC_OK : c->f32 ? exec_let<float>(c, i) : exec_let<bf16>(c, i);
    if (s.kind == TC_STMT_PRINT) {
        Ptrs P{c};
        const float* a[4];
        const float* b[4];
        long long n[4];
        double coef[4];
        for (int t = 0; t < s.nterms; ++t) {
            a[t] = reinterpret_cast<const float*>(P.var(s.in[2 * t].index));
            b[t] = reinterpret_cast<const float*>(P.var(s.in[2 * t + 1].index));
            n[t] = c->vars.at(s.in[2 * t].index).elems();
            coef[t] = s.coef[t];
        }
        return launch_loss(a, b, n, coef, s.nterms, c->d_loss, c->st);
    }
    // Update: the gradient only; all-reduce + momentum SGD run per bucket (flush_bucket)
    if (c->bias_fold_by[i] >= 0) return TC_OK;  // produced by its conv's filter-gradient kernel
    ParamL& q = c->params[s.param];
    return c->f32 ? compute_param_grad<float>(c, i, s.param, q.g) : compute_param_grad<bf16>(c, i, s.param, q.g);
}

SgdTensor sgd_tensor(tc_ctx* c, int pidx) {
    const ParamL& q = c->params[pidx];
    const tc_stmt& s = c->plan->stmts[q.update_stmt];
    SgdTensor t{};
    t.p = q.p;
    t.v = q.v;
    t.g = q.g;
    t.n = q.n;
    t.shadow = q.shadow;
    t.shadow_rskc = q.crsk ? nullptr : q.rskc;  // K-major copies: refresh_crsk after the update
    t.rskc_kmajor = 0;
    t.K = q.K;
    t.RS = q.R * q.S;
    t.cs = q.cs;
    t.ks = q.ks;
    t.lr_alpha = static_cast<float>(s.lr_alpha);
    t.momentum = static_cast<float>(s.momentum);
    t.decay = static_cast<float>(s.decay);
    return t;
}

// Gradient all-reduce (world > 1) and the fused multi-tensor momentum update of one
// bucket.  With overlap, both run on comm_st after the bucket's last gradient: every
// read of these parameters by the backward precedes their Update statements in the
// plan (PAPER.md:292-293 ordering), hence precedes the event.
// K-major bwd-data filter copies ([cs][R][S][ks]) of the updated conv filters, transposed from
// the fresh bf16 shadow in one coalesced pass each (the update kernel itself writes only the
// [K][R][S][cs] shadow for these).
tc_status refresh_crsk(tc_ctx* c, const std::vector<int>& params, cudaStream_t s2) {
    for (int pidx : params) {
        const ParamL& q = c->params[pidx];
        if (!q.crsk || !q.rskc || !q.shadow || q.s2d || c->f32) continue;
        tc_status r = launch_krsc_to_crsk(q.shadow, q.K, q.R * q.S, q.cs, q.Kw, q.rskc, q.ks, s2);
        if (r != TC_OK) return r;
    }
    return TC_OK;
}

tc_status flush_bucket(tc_ctx* c, int b, int update, bool overlap) {
    tc_ctx::Bucket& bk = c->buckets[b];
    cudaStream_t s2 = c->st;
    if (overlap) {
        TCB_CUDA_CHECK(cudaEventRecord(bk.ready, c->st));
        TCB_CUDA_CHECK(cudaStreamWaitEvent(c->comm_st, bk.ready, 0));
        s2 = c->comm_st;
    }
    if (c->comm && ncclAllReduce(c->grads + bk.off, c->grads + bk.off, bk.n, ncclFloat, ncclSum, c->comm, s2) != ncclSuccess)
        return fail(TC_NCCL_ERROR, "ncclAllReduce failed");
    if (!update || c->plan->clip > 0) return TC_OK;  // clipped updates wait for the whole gradient (clip_update)
    std::vector<SgdTensor> ts;
    for (int pidx : bk.params)
        if (!(c->fuse_sgd_active && c->sgd_fused[pidx])) ts.push_back(sgd_tensor(c, pidx));
    tc_status r = launch_sgd(ts.data(), static_cast<int>(ts.size()), nullptr, s2);
    return r != TC_OK ? r : refresh_crsk(c, bk.params, s2);
}

// Clipped momentum update of every parameter (plan->clip > 0): the global norm of
// g + decay p over the whole (all-reduced) gradient, then one multi-tensor update.
tc_status clip_update(tc_ctx* c, cudaStream_t s2) {
    std::vector<SgdTensor> ts;
    for (size_t i = 0; i < c->params.size(); ++i) ts.push_back(sgd_tensor(c, static_cast<int>(i)));
    tc_status r = launch_clip_scale(ts.data(), static_cast<int>(ts.size()), static_cast<float>(c->plan->clip),
                                    c->clip_partials, c->d_clip, s2);
    if (r != TC_OK) return r;
    for (SgdTensor& t : ts) t.gscale = c->d_clip;
    r = launch_sgd(ts.data(), static_cast<int>(ts.size()), nullptr, s2);
    if (r != TC_OK) return r;
    std::vector<int> all(c->params.size());
    for (size_t i = 0; i < all.size(); ++i) all[i] = static_cast<int>(i);
    return refresh_crsk(c, all, s2);
}

// Data parallel: every rank's Print holds its share of the global-batch loss (|N| = G*B);
// the sum over ranks is the loss of the global batch.
tc_status allreduce_loss(tc_ctx* c) {
    if (c->comm && ncclAllReduce(c->d_loss, c->d_loss, 1, ncclFloat, ncclSum, c->comm, c->st) != ncclSuccess)
        return fail(TC_NCCL_ERROR, "ncclAllReduce (loss) failed");
    return TC_OK;
}

// D2H of the step's loss into the next of two pinned slots, enqueued after the (possibly graph-
// replayed) step on the main stream: tc_loss reads the newest, tc_loss_prev the one before it
// without waiting for the newest step.
static tc_status enqueue_loss_read(tc_ctx* c) {
    const int k = c->loss_count ? c->loss_slot ^ 1 : 0;
    TCB_CUDA_CHECK(cudaMemcpyAsync(c->h_loss + 16 * k, c->d_loss, sizeof(float), cudaMemcpyDeviceToHost, c->st));
    TCB_CUDA_CHECK(cudaEventRecord(c->loss_ev[k], c->st));
    c->loss_slot = k;
    ++c->loss_count;
    return TC_OK;
}

// Bias gradient of a conv (CONV_BWD_BIAS over the same dy) computed by its halo filter-gradient
// kernel (conv_bwd_filter_ex): the kernel's epilogue warps sum the staged dy tiles while the MMA
// runs, and the split-K reduce adds the per-split partials -- no separate two-pass column sum
// over dy.  The gradient-bucket flush that ran after the bias statement moves to the producer
// when the bias statement comes first.  TCB_WGRAD_BIAS_FOLD=0 disables.
void plan_bias_fold(tc_ctx* c) {
    const tc_plan* p = c->plan;
    c->wgrad_bias_param.assign(p->nstmts, -1);
    c->bias_fold_by.assign(p->nstmts, -1);
    if (c->f32) return;
    Ptrs P{c};
    for (int i = 0; i < p->nstmts; ++i) {
        const tc_stmt& b = p->stmts[i];
        const bool conv_bias = b.op == TC_OP_CONV_BWD_BIAS, fc_bias = b.op == TC_OP_BIAS_GRAD;
        if (b.kind != TC_STMT_UPDATE || !(conv_bias || fc_bias) || b.in[0].kind != TC_REF_VAR) continue;
        for (int j = 0; j < p->nstmts; ++j) {
            const tc_stmt& f = p->stmts[j];
            if (f.kind != TC_STMT_UPDATE || f.op != (conv_bias ? TC_OP_CONV_BWD_FILTER : TC_OP_MATMUL_BWD_W) ||
                f.in[0].kind != TC_REF_VAR || f.in[0].index != b.in[0].index || c->wgrad_bias_param[j] >= 0)
                continue;
            const ParamL& w = c->params[f.param];
            if (c->params[b.param].K != w.K) continue;
            if (conv_bias) {
                const tc_conv_desc d = conv_desc(P.L(f.in[1]), w, P.L(f.in[0]), f);
                if (!wgrad_bias_foldable(&d)) continue;
            } else {
                // the FC filter gradient's GEMM view (compute_param_grad): M = out features,
                // N = in features, K = batch, A = dy MN-major
                const VarL& up = P.L(f.in[0]);
                tc_gemm_args ga{};
                ga.M = w.K;
                ga.N = w.in_dev;
                ga.K = up.N;
                ga.a_layout = TC_LAYOUT_MN;
                ga.b_layout = TC_LAYOUT_MN;
                ga.d_dtype = TC_DTYPE_F32;
                if (up.cs < w.K || !gemm_bias_foldable(&ga)) continue;
            }
            if (i < j) {  // bucket flushes at statements i .. j-1 move to just before j's own, in order
                std::vector<int> moved;
                for (int k = i; k < j; ++k) {
                    moved.insert(moved.end(), c->stmt_flush[k].begin(), c->stmt_flush[k].end());
                    c->stmt_flush[k].clear();
                }
                c->stmt_flush[j].insert(c->stmt_flush[j].begin(), moved.begin(), moved.end());
                for (int bki : moved) c->buckets[bki].last_stmt = j;
            }
            c->wgrad_bias_param[j] = b.param;
            c->bias_fold_by[i] = j;
            break;
        }
    }
}

// Per-statement form of one parameter's all-reduce + momentum update (tc_exec_stmt).
static tc_status exec_stmt_update(tc_ctx* c, int index, int param) {
    ParamL& q = c->params[param];
    if (c->comm && ncclAllReduce(q.g, q.g, q.n, ncclFloat, ncclSum, c->comm, c->st) != ncclSuccess)
        return fail(TC_NCCL_ERROR, "ncclAllReduce failed");
    if (c->plan->clip > 0)  // the clipped update needs the whole gradient: applied at the last Update
        return index == c->last_update_stmt ? clip_update(c, c->st) : TC_OK;
    SgdTensor t = sgd_tensor(c, param);
    tc_status r = launch_sgd(&t, 1, nullptr, c->st);
    return r != TC_OK ? r : refresh_crsk(c, {param}, c->st);
}

tc_status run_body(tc_ctx* c, int update, bool overlap, bool set_iter) {
    tc_status r = set_iter ? launch_set_iter(c->d_iter, c->h_iter[0], c->h_iter[1], c->st) : TC_OK;
    if (r != TC_OK) return r;
    struct ActiveScope {  // the fused FC updates apply to update steps of the whole-step path only
        tc_ctx* c;
        ActiveScope(tc_ctx* cc, bool on) : c(cc) { c->fuse_sgd_active = on; }
        ~ActiveScope() { c->fuse_sgd_active = false; }
    } active(c, update != 0);
    for (int i = 0; i < c->plan->nstmts; ++i) {
        r = exec_stmt(c, i);
        if (r != TC_OK) return r;
        for (int bki : c->stmt_flush[i]) {
            r = flush_bucket(c, bki, update, overlap);
            if (r != TC_OK) return r;
        }
    }
    if (update && c->plan->clip > 0) {
        r = clip_update(c, overlap ? c->comm_st : c->st);
        if (r != TC_OK) return r;
    }
    if (overlap) {
        TCB_CUDA_CHECK(cudaEventRecord(c->join_ev, c->comm_st));
        TCB_CUDA_CHECK(cudaStreamWaitEvent(c->st, c->join_ev, 0));
    }
    return allreduce_loss(c);  // the loss read-back is enqueued by tc_step, outside any capture
}

// Largest split-K workspace over the plan's contractions (and, in TC_PREC_F32, the largest
// split-operand buffer, returned through *split).
size_t workspace_need(tc_ctx* c, size_t* split) {
    size_t need = 0, sp = 0;
    const tc_plan* p = c->plan;
    Ptrs P{c};
    auto conv = [&](tc_conv_desc d, int which, const ParamL& w) {
        if (c->f32) {
            sp = std::max(sp, split_need(d, which, w));
            d = split_desc(d, which);
        }
        need = std::max(need, tc_conv2d_workspace_bytes(&d, which));
    };
    for (int i = 0; i < p->nstmts; ++i) {
        const tc_stmt& s = p->stmts[i];
        if (s.kind != TC_STMT_LET && s.kind != TC_STMT_UPDATE) continue;
        switch (s.op) {
            case TC_OP_CONV_FWD: {
                const ParamL& w = c->params[s.in[1].index];
                conv(conv_desc(P.L(s.in[0]), w, c->vars.at(s.var), s), 0, w);
                break;
            }
            case TC_OP_CONV_BWD_DATA: {
                const ParamL& w = c->params[s.in[1].index];
                conv(conv_desc(c->vars.at(s.var), w, P.L(s.in[0]), s), 1, w);
                break;
            }
            case TC_OP_CONV_BWD_FILTER: {
                const ParamL& w = c->params[s.param];
                conv(conv_desc(P.L(s.in[1]), w, P.L(s.in[0]), s), 2, w);
                break;
            }
            case TC_OP_MATMUL_FWD:
            case TC_OP_MATMUL_BWD_DATA:
            case TC_OP_MATMUL_BWD_W: {
                tc_gemm_args ga{};
                ga.d_dtype = c->f32 ? TC_DTYPE_F32 : TC_DTYPE_BF16;
                if (s.op == TC_OP_MATMUL_FWD) {
                    const ParamL& w = c->params[s.in[1].index];
                    ga.M = P.L(s.in[0]).N;
                    ga.N = c->vars.at(s.var).cs;
                    ga.K = c->f32 ? kSplitN * w.in_dev : w.in_dev;
                    if (c->f32) sp = std::max(sp, split_fc_need(0, ga.M, ga.N, w.in_dev));
                } else if (s.op == TC_OP_MATMUL_BWD_DATA) {
                    const ParamL& w = c->params[s.in[1].index];
                    const VarL& up = P.L(s.in[0]);
                    ga.M = up.N;
                    ga.N = w.in_dev;
                    ga.K = c->f32 ? kSplitN * up.cs : w.K;
                    if (c->f32) sp = std::max(sp, split_fc_need(1, ga.M, ga.N, up.cs));
                } else {
                    const ParamL& w = c->params[s.param];
                    const VarL& up = P.L(s.in[0]);
                    ga.M = w.K;
                    ga.N = w.in_dev;
                    ga.K = c->f32 ? kSplitN * up.N : up.N;
                    ga.d_dtype = TC_DTYPE_F32;
                    if (c->f32) sp = std::max(sp, split_fc_need(2, up.cs, ga.N, up.N));
                }
                need = std::max(need, tc_gemm_workspace_bytes(&ga));
                break;
            }
            default: break;
        }
    }
    if (split) *split = sp;
    return need;
}

}  // namespace

// ================================================================== C ABI
extern "C" {

tc_status tc_nccl_unique_id(void* out128) {
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return fail(TC_NCCL_ERROR, "ncclGetUniqueId failed");
    std::memcpy(out128, &id, sizeof id);
    return TC_OK;
}

tc_status tc_ctx_create(const tc_plan* plan, const tc_ctx_desc* desc, tc_ctx** out) {
    if (!plan || !desc || !out) return fail(TC_INVALID_ARG, "tc_ctx_create: null argument");
    *out = nullptr;
    auto c = std::make_unique<tc_ctx>();
    c->plan = plan;
    c->desc = *desc;
    if (c->desc.seed == 0) c->desc.seed = 42;
    TCB_CUDA_CHECK(cudaSetDevice(desc->device));
    TCB_CUDA_CHECK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    c->f32 = desc->precision == TC_PREC_F32;
    tc_status r = analyze_layouts(c.get());
    if (r != TC_OK) return r;
    plan_fusion(c.get());
    r = plan_arena(c.get());
    if (r != TC_OK) return r;
    // gradient buckets: parameters in Update-statement order (backward production order)
    std::vector<int> order;
    for (int i = 0; i < plan->nstmts; ++i) {
        const tc_stmt& s = plan->stmts[i];
        if (s.kind != TC_STMT_UPDATE) continue;
        ParamL& q = c->params.at(s.param);
        if (q.update_stmt >= 0) return fail(TC_INTERNAL, "runtime: parameter with two Update statements");
        q.update_stmt = i;
        order.push_back(s.param);
    }
    for (size_t i = 0; i < c->params.size(); ++i)
        if (c->params[i].update_stmt < 0) return fail(TC_INTERNAL, "runtime: parameter without an Update statement");
    if (!(plan->clip >= 0.0)) return fail(TC_INVALID_ARG, "solver clip must be >= 0 (0 = no clipping)");
    for (int i = 0; i < plan->nstmts; ++i)
        if (plan->stmts[i].kind == TC_STMT_UPDATE) c->last_update_stmt = i;
    // FC filter gradients whose momentum update runs in the GEMM epilogue (world size 1, no
    // gradient clipping, not the keep / fp32 parity modes): the gradient never reaches HBM and
    // the separate update pass skips them.  Opt-in (TCB_SGD_FUSE=1): bit-identical to the
    // separate update (tests/test_step_gpu.py), but the epilogue's per-row fp32 p / v traffic is
    // uncoalesced (one row per lane) and measured AlexNet 74.8k -> 60.4k images/s; a TMA-staged
    // p / v tile would be needed to make it pay.
    {
        const char* e = std::getenv("TCB_SGD_FUSE");
        const bool on = e && e[0] == '1' && c->desc.world <= 1 && !c->desc.keep && !c->f32 && plan->clip == 0.0;
        c->sgd_fused.assign(c->params.size(), 0);
        for (size_t i = 0; on && i < c->params.size(); ++i) {
            const ParamL& q = c->params[i];
            if (q.kind == ParamL::FC && q.update_stmt >= 0 && plan->stmts[q.update_stmt].op == TC_OP_MATMUL_BWD_W &&
                q.in_dev % 4 == 0)
                c->sgd_fused[i] = 1;
        }
    }
    const char* bmb = std::getenv("TCB_BUCKET_MB");
    const long long bucket_cap = static_cast<long long>((bmb ? std::atof(bmb) : 32.0) * (1 << 20) / 4);
    c->stmt_flush.assign(plan->nstmts, {});
    long long goff = 0;
    for (size_t j = 0; j < order.size(); ++j) {
        ParamL& q = c->params[order[j]];
        if (c->buckets.empty() || c->buckets.back().last_stmt >= 0) {
            c->buckets.emplace_back();
            c->buckets.back().off = static_cast<size_t>(goff);
        }
        tc_ctx::Bucket& bk = c->buckets.back();
        bk.params.push_back(order[j]);
        goff += (q.n + 63) / 64 * 64;  // 256-byte aligned gradient tensors
        bk.n = goff - static_cast<long long>(bk.off);
        if (bk.n >= bucket_cap || j + 1 == order.size() || bk.params.size() >= 32) {
            bk.last_stmt = q.update_stmt;
            c->stmt_flush[q.update_stmt].push_back(static_cast<int>(c->buckets.size()) - 1);
        }
    }
    c->grads_n = goff;
    plan_bias_fold(c.get());
    // parameter slab: [gradients (contiguous, bucket order)] then per parameter p, v, bf16 shadows
    size_t slab = static_cast<size_t>(goff) * 4;
    auto reserve = [&](size_t bytes) {
        const size_t off = slab;
        slab += align256(bytes);
        return off;
    };
    std::vector<size_t> offs;
    for (ParamL& q : c->params) {
        offs.push_back(reserve(q.n * 4));  // p
        offs.push_back(reserve(q.n * 4));  // v
        offs.push_back(q.kind != ParamL::VEC ? reserve(q.n * 2) : SIZE_MAX);
        offs.push_back(q.kind == ParamL::CONV && q.cs % 8 == 0 ? reserve(static_cast<size_t>(q.R) * q.S * q.ks * q.cs * 2)
                                                           : SIZE_MAX);
    }
    c->slab_bytes = slab;
    TCB_CUDA_CHECK(cudaMalloc(&c->slab, std::max<size_t>(slab, 256)));
    TCB_CUDA_CHECK(cudaMemsetAsync(c->slab, 0, std::max<size_t>(slab, 256), c->st));
    c->grads = reinterpret_cast<float*>(c->slab);
    {
        long long o = 0;
        for (int pi : order) {
            c->params[pi].g = c->grads + o;
            o += (c->params[pi].n + 63) / 64 * 64;
        }
    }
    for (size_t i = 0; i < c->params.size(); ++i) {
        ParamL& q = c->params[i];
        q.p = reinterpret_cast<float*>(c->slab + offs[4 * i]);
        q.v = reinterpret_cast<float*>(c->slab + offs[4 * i + 1]);
        if (offs[4 * i + 2] != SIZE_MAX) q.shadow = reinterpret_cast<bf16*>(c->slab + offs[4 * i + 2]);
        if (offs[4 * i + 3] != SIZE_MAX) {
            q.rskc = reinterpret_cast<bf16*>(c->slab + offs[4 * i + 3]);
            // bwd-data filter operand K-major ([cs][R][S][ks]; TCB_DGRAD_KMAJOR=0: [R][S][ks][cs]):
            // the MMA issues exactly Cin columns (N = 96: 96 instead of 128) and the halo kernel
            // loads only those filter rows; refreshed by a transpose of the shadow after the update
            static const bool kmajor = [] {
                const char* e = std::getenv("TCB_DGRAD_KMAJOR");
                return !(e && e[0] == '0');
            }();
            q.crsk = kmajor;
        }
    }
    {
        const char* ov = std::getenv("TCB_OVERLAP");
        c->overlap = !(ov && ov[0] == '0');
    }
    TCB_CUDA_CHECK(cudaStreamCreateWithFlags(&c->comm_st, cudaStreamNonBlocking));
    TCB_CUDA_CHECK(cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming));
    for (auto& bk : c->buckets) TCB_CUDA_CHECK(cudaEventCreateWithFlags(&bk.ready, cudaEventDisableTiming));
    // arena
    TCB_CUDA_CHECK(cudaMalloc(&c->arena, std::max<size_t>(c->arena_bytes, 256)));
    TCB_CUDA_CHECK(cudaMemsetAsync(c->arena, 0, std::max<size_t>(c->arena_bytes, 256), c->st));
    // input staging: NHWC bf16 batch + labels + NCHW fp32 staging for host batches
    c->input_cs = plan->input_dims[1] <= 4 && !c->f32 ? 4 : ceil8(plan->input_dims[1]);
    for (int i = 0; i < plan->nstmts; ++i)  // = the LOAD_X var layout (cs 8 for a stride-2 space-to-depth)
        if (plan->stmts[i].kind == TC_STMT_LET && plan->stmts[i].op == TC_OP_LOAD_X)
            c->input_cs = c->vars.at(plan->stmts[i].var).cs;
    c->in_layout.N = static_cast<int>(plan->input_dims[0]);
    c->in_layout.C = static_cast<int>(plan->input_dims[1]);
    c->in_layout.H = static_cast<int>(plan->input_dims[2]);
    c->in_layout.W = static_cast<int>(plan->input_dims[3]);
    c->in_layout.cs = c->input_cs;
    const size_t in_el = static_cast<size_t>(c->in_layout.elems());
    const size_t in_es = c->f32 ? 4 : 2;
    const size_t stage_el = static_cast<size_t>(plan->input_dims[0]) * plan->input_dims[1] * plan->input_dims[2] * plan->input_dims[3];
    c->input_bytes = in_el * in_es + 2 * stage_el * 4;
    TCB_CUDA_CHECK(cudaMalloc(&c->d_input, in_el * in_es));
    TCB_CUDA_CHECK(cudaMemsetAsync(c->d_input, 0, in_el * in_es, c->st));
    for (int k = 0; k < 2; ++k) {
        TCB_CUDA_CHECK(cudaMalloc(&c->d_stage[k], stage_el * 4));
        TCB_CUDA_CHECK(cudaMalloc(&c->d_label_stage[k], plan->input_dims[0] * sizeof(int32_t)));
        TCB_CUDA_CHECK(cudaEventCreateWithFlags(&c->h2d_done[k], cudaEventDisableTiming));
        TCB_CUDA_CHECK(cudaEventCreateWithFlags(&c->conv_done[k], cudaEventDisableTiming));
        TCB_CUDA_CHECK(cudaEventRecord(c->conv_done[k], c->st));
    }
    TCB_CUDA_CHECK(cudaStreamCreateWithFlags(&c->copy_st, cudaStreamNonBlocking));
    {
        const char* e = std::getenv("TCB_HOST_BF16");
        c->host_bf16 = !c->f32 && e && e[0] == '1';
        if (c->host_bf16) {
            for (int k = 0; k < 2; ++k) TCB_CUDA_CHECK(cudaMallocHost(&c->h_stage16[k], stage_el * 2));
            const unsigned hw = std::thread::hardware_concurrency();
            const char* te = std::getenv("TCB_HOST_THREADS");
            const int want = te ? std::atoi(te) : static_cast<int>(std::min(16u, hw ? hw : 4u));
            c->pool = new HostPool(std::max(1, want));
        }
    }
    TCB_CUDA_CHECK(cudaMalloc(&c->d_labels, plan->input_dims[0] * sizeof(int32_t)));
    TCB_CUDA_CHECK(cudaMemsetAsync(c->d_labels, 0, plan->input_dims[0] * sizeof(int32_t), c->st));
    TCB_CUDA_CHECK(cudaMalloc(&c->d_loss, 4096));  // loss, fp64 block partials, ticket (launch_loss)
    TCB_CUDA_CHECK(cudaMemsetAsync(c->d_loss, 0, 4096, c->st));
    TCB_CUDA_CHECK(cudaMalloc(&c->d_iter, 256));
    TCB_CUDA_CHECK(cudaMallocHost(&c->h_iter, 256));
    TCB_CUDA_CHECK(cudaMallocHost(&c->h_loss, 256));
    c->h_iter[0] = c->h_iter[1] = 0;
    for (int k = 0; k < 2; ++k) {
        c->h_loss[16 * k] = 0.f;
        TCB_CUDA_CHECK(cudaEventCreateWithFlags(&c->loss_ev[k], cudaEventDisableTiming));
    }
    // workspace + reduction partials
    c->ws_bytes = workspace_need(c.get(), &c->split_bytes);
    if (c->split_bytes) TCB_CUDA_CHECK(cudaMalloc(&c->split_buf, c->split_bytes));
    int maxc = 8;
    for (auto& [id, v] : c->vars) maxc = std::max(maxc, v.cs);
    for (const ParamL& q : c->params) maxc = std::max(maxc, q.K);
    c->max_partials = static_cast<int>(colsum_partials_floats(maxc));
    TCB_CUDA_CHECK(cudaMalloc(&c->ws, std::max<size_t>(c->ws_bytes, 256)));
    if (const char* e = std::getenv("TCB_POISON"); e && e[0] == '1') {  // debug: NaN-fill scratch, arena, gradients
        TCB_CUDA_CHECK(cudaMemset(c->ws, 0xFF, std::max<size_t>(c->ws_bytes, 256)));
        TCB_CUDA_CHECK(cudaMemset(c->arena, 0xFF, std::max<size_t>(c->arena_bytes, 256)));
        TCB_CUDA_CHECK(cudaMemset(c->grads, 0xFF, static_cast<size_t>(c->grads_n) * 4));
    }
    TCB_CUDA_CHECK(cudaMalloc(&c->partials, (static_cast<size_t>(c->max_partials) + 3 * maxc + 64) * sizeof(float)));
    // BN backward groups
    {
        std::unordered_map<int, int> beta_x, gamma_of_x, group_of_x;
        for (int i = 0; i < plan->nstmts; ++i) {
            const tc_stmt& s = plan->stmts[i];
            if (s.kind == TC_STMT_LET && s.op == TC_OP_BN_FWD) {
                beta_x[s.in[2].index] = s.in[0].index;
                gamma_of_x[s.in[0].index] = s.in[1].index;
            }
        }
        size_t total = 0;
        std::vector<size_t> offs;
        for (int i = 0; i < plan->nstmts; ++i) {
            const tc_stmt& s = plan->stmts[i];
            if (s.op != TC_OP_BN_BWD_BETA && s.op != TC_OP_BN_BWD_DATA && s.op != TC_OP_BN_BWD_GAMMA) continue;
            if (s.kind != TC_STMT_LET && s.kind != TC_STMT_UPDATE) continue;
            int xv = -1;
            if (s.op == TC_OP_BN_BWD_BETA) {
                auto f = beta_x.find(s.kind == TC_STMT_UPDATE ? s.param : s.in[1].index);
                if (f == beta_x.end()) return fail(TC_INTERNAL, "runtime: BN beta gradient without its BatchNorm");
                xv = f->second;
            } else {
                xv = s.in[1].index;
            }
            auto g = group_of_x.find(xv);
            if (g == group_of_x.end()) {
                tc_ctx::BnGroup gr;
                gr.x_var = xv;
                gr.up_var = s.in[0].index;
                gr.first = i;
                gr.gamma = gamma_of_x.at(xv);
                group_of_x[xv] = static_cast<int>(c->bn_groups.size());
                c->bn_groups.push_back(gr);
                offs.push_back(total);
                total += 5 * static_cast<size_t>(c->vars.at(xv).C) + 64;
                g = group_of_x.find(xv);
            } else if (c->bn_groups[g->second].up_var != s.in[0].index) {
                return fail(TC_INTERNAL, "runtime: BN backward statements disagree on the upstream gradient");
            }
            c->stmt_bn_group[i] = g->second;
        }
        if (total) {
            TCB_CUDA_CHECK(cudaMalloc(&c->bn_sums, total * sizeof(float)));
            for (size_t k = 0; k < c->bn_groups.size(); ++k) c->bn_groups[k].sums = c->bn_sums + offs[k];
        }
    }
    if (plan->clip > 0) {
        TCB_CUDA_CHECK(cudaMalloc(&c->clip_partials, clip_partials_doubles(static_cast<int>(c->params.size())) * sizeof(double)));
        TCB_CUDA_CHECK(cudaMalloc(&c->d_clip, 256));
    }
    // NCCL: world > 1, or a 1-rank communicator when an id is supplied (exercises the
    // all-reduce path, captured in the step's graph, on a single GPU)
    if (desc->world > 1 || (desc->world == 1 && desc->nccl_id)) {
        if (!desc->nccl_id) return fail(TC_INVALID_ARG, "world > 1 needs an NCCL unique id");
        ncclUniqueId id;
        std::memcpy(&id, desc->nccl_id, sizeof id);
        if (ncclCommInitRank(&c->comm, desc->world, id, desc->rank) != ncclSuccess)
            return fail(TC_NCCL_ERROR, "ncclCommInitRank failed");
    }
    TCB_CUDA_CHECK(cudaStreamSynchronize(c->st));
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) c->device_used = static_cast<int64_t>(tot - fr);
    *out = c.release();
    return TC_OK;
}

void tc_ctx_destroy(tc_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->desc.device);
    if (c->st) cudaStreamSynchronize(c->st);
    for (int k = 0; k < 2; ++k) {
        if (c->gexec[k]) cudaGraphExecDestroy(c->gexec[k]);
        if (c->graph[k]) cudaGraphDestroy(c->graph[k]);
    }
    if (c->comm_st) cudaStreamSynchronize(c->comm_st);
    if (c->comm) ncclCommDestroy(c->comm);
    for (auto& bk : c->buckets)
        if (bk.ready) cudaEventDestroy(bk.ready);
    if (c->join_ev) cudaEventDestroy(c->join_ev);
    if (c->comm_st) cudaStreamDestroy(c->comm_st);
    cudaFree(c->arena);
    cudaFree(c->slab);
    cudaFree(c->ws);
    cudaFree(c->split_buf);
    cudaFree(c->partials);
    cudaFree(c->bn_sums);
    cudaFree(c->clip_partials);
    cudaFree(c->d_hits);
    if (c->h_hits) cudaFreeHost(c->h_hits);
    cudaFree(c->d_clip);
    cudaFree(c->d_input);
    if (c->copy_st) cudaStreamSynchronize(c->copy_st);
    delete c->pool;
    for (int k = 0; k < 2; ++k) {
        if (c->h_stage16[k]) cudaFreeHost(c->h_stage16[k]);
        cudaFree(c->d_stage[k]);
        cudaFree(c->d_label_stage[k]);
        if (c->h2d_done[k]) cudaEventDestroy(c->h2d_done[k]);
        if (c->conv_done[k]) cudaEventDestroy(c->conv_done[k]);
    }
    if (c->copy_st) cudaStreamDestroy(c->copy_st);
    cudaFree(c->d_labels);
    cudaFree(c->d_loss);
    cudaFree(c->d_iter);
    cudaFreeHost(c->h_iter);
    cudaFreeHost(c->h_loss);
    for (int k = 0; k < 2; ++k)
        if (c->loss_ev[k]) cudaEventDestroy(c->loss_ev[k]);
    if (c->st) cudaStreamDestroy(c->st);
    delete c;
}

void* tc_ctx_stream(tc_ctx* c) { return c ? c->st : nullptr; }

tc_status tc_param_upload(tc_ctx* c, int i, const float* host) {
    if (!c || !host || i < 0 || i >= static_cast<int>(c->params.size())) return fail(TC_INVALID_ARG, "tc_param_upload");
    std::vector<float> dev;
    ref_to_dev(c->params[i], host, dev);
    return upload_dev_param(c, i, dev);
}

tc_status tc_velocity_upload(tc_ctx* c, int i, const float* host) {
    if (!c || !host || i < 0 || i >= static_cast<int>(c->params.size())) return fail(TC_INVALID_ARG, "tc_velocity_upload");
    std::vector<float> dev;
    ref_to_dev(c->params[i], host, dev);
    TCB_CUDA_CHECK(cudaMemcpyAsync(c->params[i].v, dev.data(), c->params[i].n * 4, cudaMemcpyHostToDevice, c->st));
    TCB_CUDA_CHECK(cudaStreamSynchronize(c->st));
    return TC_OK;
}

const tc_plan* tc_ctx_plan(tc_ctx* c) { return c ? c->plan : nullptr; }

static tc_status download_slab(tc_ctx* c, int i, const float* dptr, float* host) {
    const ParamL& q = c->params[i];
    std::vector<float> dev(q.n);
    TCB_CUDA_CHECK(cudaMemcpyAsync(dev.data(), dptr, q.n * 4, cudaMemcpyDeviceToHost, c->st));
    TCB_CUDA_CHECK(cudaStreamSynchronize(c->st));
    dev_to_ref(q, dev.data(), host);
    return TC_OK;
}

tc_status tc_param_download(tc_ctx* c, int i, float* host) {
    if (!c || !host || i < 0 || i >= static_cast<int>(c->params.size())) return fail(TC_INVALID_ARG, "tc_param_download");
    return download_slab(c, i, c->params[i].p, host);
}
tc_status tc_velocity_download(tc_ctx* c, int i, float* host) {
    if (!c || !host || i < 0 || i >= static_cast<int>(c->params.size())) return fail(TC_INVALID_ARG, "tc_velocity_download");
    return download_slab(c, i, c->params[i].v, host);
}
tc_status tc_grad_download(tc_ctx* c, int i, float* host) {
    if (!c || !host || i < 0 || i >= static_cast<int>(c->params.size())) return fail(TC_INVALID_ARG, "tc_grad_download");
    return download_slab(c, i, c->params[i].g, host);
}

tc_status tc_init_params(tc_ctx* c) {
    if (!c) return fail(TC_INVALID_ARG, "tc_init_params");
    const tc_plan* p = c->plan;
    for (int i = 0; i < p->nparams; ++i) {
        const tc_param_desc& pd = p->params[i];
        long long n = 1;
        for (int j = 0; j < pd.rank; ++j) n *= pd.dims[j];
        std::vector<float> ref(n);
        if (pd.init_kind == TC_INIT_CONSTANT) {
            std::fill(ref.begin(), ref.end(), static_cast<float>(pd.init_value));
        } else if (pd.init_kind == TC_INIT_XAVIER) {
            const double a = std::sqrt(6.0 / static_cast<double>(pd.fan_in + pd.fan_out));
            for (long long j = 0; j < n; ++j)
                ref[j] = static_cast<float>((2.0 * tcp_param_uniform(c->desc.seed, i, static_cast<uint32_t>(j)) - 1.0) * a);
        } else {
            for (long long j = 0; j < n; ++j) {
                const double u1 = tcp_param_uniform(c->desc.seed, i, static_cast<uint32_t>(2 * j));
                const double u2 = tcp_param_uniform(c->desc.seed, i, static_cast<uint32_t>(2 * j + 1));
                ref[j] = static_cast<float>(pd.sigma * std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2));
            }
        }
        tc_status r = tc_param_upload(c, i, ref.data());
        if (r != TC_OK) return r;
        TCB_CUDA_CHECK(cudaMemsetAsync(c->params[i].v, 0, c->params[i].n * 4, c->st));
    }
    TCB_CUDA_CHECK(cudaStreamSynchronize(c->st));
    return TC_OK;
}

tc_status tc_stage_batch(tc_ctx* c, const float* x, const int32_t* labels) {
    if (!c || !x || !labels) return fail(TC_INVALID_ARG, "tc_stage_batch: null argument");
    const tc_plan* p = c->plan;
    const size_t el = static_cast<size_t>(p->input_dims[0]) * p->input_dims[1] * p->input_dims[2] * p->input_dims[3];
    // the slot's previous batch must have been converted by its step before it is overwritten
    const int k = c->stage_next;
    TCB_CUDA_CHECK(cudaStreamWaitEvent(c->copy_st, c->conv_done[k], 0));
    if (c->host_bf16) {
        // the slot's previous host->device copy has finished reading the pinned buffer
        TCB_CUDA_CHECK(cudaEventSynchronize(c->h2d_done[k]));
        // each rounded chunk is copied while the pool rounds the next (TCB_STAGE_CHUNKS, default 8)
        static const int chunks = [] {
            const char* e = std::getenv("TCB_STAGE_CHUNKS");
            return e ? std::max(1, std::atoi(e)) : 8;
        }();
        uint16_t* h = c->h_stage16[k];
        uint16_t* dv = reinterpret_cast<uint16_t*>(c->d_stage[k]);
        tc_status r = c->pool->run(x, h, el, chunks, [&](size_t a, size_t len) -> tc_status {
            TCB_CUDA_CHECK(cudaMemcpyAsync(dv + a, h + a, len * 2, cudaMemcpyHostToDevice, c->copy_st));
            return TC_OK;
        });
        if (r != TC_OK) return r;
    } else {
        TCB_CUDA_CHECK(cudaMemcpyAsync(c->d_stage[k], x, el * 4, cudaMemcpyHostToDevice, c->copy_st));
    }
    TCB_CUDA_CHECK(cudaMemcpyAsync(c->d_label_stage[k], labels, p->input_dims[0] * 4, cudaMemcpyHostToDevice, c->copy_st));
    TCB_CUDA_CHECK(cudaEventRecord(c->h2d_done[k], c->copy_st));
    c->stage_pending = k;
    c->stage_next = k ^ 1;
    return TC_OK;
}

int64_t tc_stage_bytes(const tc_ctx* c) {
    if (!c) return 0;
    const tc_plan* p = c->plan;
    const int64_t el = p->input_dims[0] * p->input_dims[1] * p->input_dims[2] * p->input_dims[3];
    return el * (c->host_bf16 ? 2 : 4) + p->input_dims[0] * 4;
}

// Convert a pending host batch (if any) into the staged input layout on the main stream.
static tc_status consume_staged(tc_ctx* c) {
    const int k = c->stage_pending;
    if (k < 0) return TC_OK;
    c->stage_pending = -1;
    TCB_CUDA_CHECK(cudaStreamWaitEvent(c->st, c->h2d_done[k], 0));
    TCB_CUDA_CHECK(cudaMemcpyAsync(c->d_labels, c->d_label_stage[k], c->plan->input_dims[0] * sizeof(int32_t),
                                   cudaMemcpyDeviceToDevice, c->st));
    tc_status r = c->f32 ? launch_nchw_to_nhwc(static_cast<const float*>(c->d_stage[k]), static_cast<float*>(c->d_input),
                                               c->in_layout, c->st)
                  : c->host_bf16 ? launch_nchw_to_nhwc(reinterpret_cast<const bf16*>(c->d_stage[k]),
                                                       static_cast<bf16*>(c->d_input), c->in_layout, c->st)
                                 : launch_nchw_to_nhwc(static_cast<const float*>(c->d_stage[k]),
                                                       static_cast<bf16*>(c->d_input), c->in_layout, c->st);
    if (r != TC_OK) return r;
    TCB_CUDA_CHECK(cudaEventRecord(c->conv_done[k], c->st));
    return TC_OK;
}

tc_status tc_stage_synthetic(tc_ctx* c, int iter, int n0) {
    if (!c) return fail(TC_INVALID_ARG, "tc_stage_synthetic");
    tc_status r0 = consume_staged(c);  // keep slot bookkeeping consistent; the synthetic batch wins
    if (r0 != TC_OK) return r0;
    const tc_plan* p = c->plan;
    if (c->f32)
        return launch_synth_batch(static_cast<float*>(c->d_input), c->d_labels, c->in_layout, static_cast<int>(p->classes),
                                  c->desc.seed, static_cast<uint32_t>(iter), static_cast<uint32_t>(n0), c->st);
    return launch_synth_batch(static_cast<bf16*>(c->d_input), c->d_labels, c->in_layout, static_cast<int>(p->classes),
                              c->desc.seed, static_cast<uint32_t>(iter), static_cast<uint32_t>(n0), c->st);
}

tc_status tc_step(tc_ctx* c, int iter, int n0, int update) {
    if (!c) return fail(TC_INVALID_ARG, "tc_step");
    TCB_CUDA_CHECK(cudaSetDevice(c->desc.device));
    {
        tc_status r0 = consume_staged(c);
        if (r0 != TC_OK) return r0;
    }
    const int k = update ? 1 : 0;
    // The iteration / first-sample counters that the dropout kernels read live in
    // device memory; a one-thread kernel sets them ahead of the (captured) step, so
    // the host never waits for the previous step.
    if (c->gexec[k]) {
        tc_status r = launch_set_iter(c->d_iter, static_cast<uint32_t>(iter), static_cast<uint32_t>(n0), c->st);
        if (r != TC_OK) return r;
        TCB_CUDA_CHECK(cudaGraphLaunch(c->gexec[k], c->st));
        count_launch(static_cast<unsigned>(std::max(0, c->launches_per_step - 1)));
        return enqueue_loss_read(c);
    }
    c->h_iter[0] = static_cast<uint32_t>(iter);
    c->h_iter[1] = static_cast<uint32_t>(n0);
    const char* ng = std::getenv("TCB_NCCL_GRAPH");
    const bool capture = c->desc.use_graph && c->runs[k] >= 1 && (!c->comm || !(ng && ng[0] == '0'));
    const unsigned long long before = g_launches.load();
    if (capture) {
        tc_status r = launch_set_iter(c->d_iter, c->h_iter[0], c->h_iter[1], c->st);
        if (r != TC_OK) return r;
        TCB_CUDA_CHECK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
    }
    tc_status r = run_body(c, update, c->overlap, /*set_iter=*/!capture);
    if (capture) {
        cudaGraph_t g = nullptr;
        cudaError_t e = cudaStreamEndCapture(c->st, &g);
        if (r != TC_OK) return r;
        if (e != cudaSuccess) return fail(TC_CUDA_ERROR, std::string("graph capture: ") + cudaGetErrorString(e));
        c->graph[k] = g;
        TCB_CUDA_CHECK(cudaGraphInstantiate(&c->gexec[k], g, 0));
        TCB_CUDA_CHECK(cudaGraphLaunch(c->gexec[k], c->st));
    }
    if (r != TC_OK) return r;
    if (c->launches_per_step < 0) c->launches_per_step = static_cast<int>(g_launches.load() - before);
    c->runs[k]++;
    return enqueue_loss_read(c);
}

tc_status tc_exec_stmt(tc_ctx* c, int index, int iter, int n0) {
    if (!c || index < 0 || index >= c->plan->nstmts) return fail(TC_INVALID_ARG, "tc_exec_stmt");
    tc_status r = consume_staged(c);
    if (r != TC_OK) return r;
    r = launch_set_iter(c->d_iter, static_cast<uint32_t>(iter), static_cast<uint32_t>(n0), c->st);
    if (r != TC_OK) return r;
    r = exec_stmt(c, index);
    if (r != TC_OK) return r;
    const tc_stmt& s = c->plan->stmts[index];
    if (s.kind == TC_STMT_PRINT) {
        r = allreduce_loss(c);
        if (r != TC_OK) return r;
        return enqueue_loss_read(c);
    }
    if (s.kind != TC_STMT_UPDATE) return TC_OK;
    // a folded bias gradient computed by a later statement is updated there
    if (c->bias_fold_by[index] > index) return TC_OK;
    r = exec_stmt_update(c, index, s.param);
    const int bp = c->wgrad_bias_param[index];
    if (r == TC_OK && bp >= 0 && c->params[bp].update_stmt < index && c->plan->clip <= 0)  // (clip: one pass did all)
        r = exec_stmt_update(c, index, bp);
    return r;
}

tc_status tc_test(tc_ctx* c, int iter, int n0, double* precision) {
    if (!c || !precision) return fail(TC_INVALID_ARG, "tc_test: null argument");
    const tc_plan* p = c->plan;
    if (p->ntest <= 0 || c->vars.find(p->logits_var) == c->vars.end()) return fail(TC_INVALID_ARG, "tc_test: plan has no test body");
    TCB_CUDA_CHECK(cudaSetDevice(c->desc.device));
    tc_status r = consume_staged(c);
    if (r != TC_OK) return r;
    if (c->in_test.empty()) {
        std::unordered_map<int, int> want;
        for (int i = 0; i < p->ntest; ++i) want[p->test_stmts[i].var] = 1;
        c->in_test.assign(p->nstmts, 0);
        for (int i = 0; i < p->nstmts; ++i)
            c->in_test[i] = p->stmts[i].kind == TC_STMT_LET && want.count(p->stmts[i].var) ? 1 : 0;
        TCB_CUDA_CHECK(cudaMalloc(&c->d_hits, 256));
        TCB_CUDA_CHECK(cudaMallocHost(&c->h_hits, 256));
    }
    r = launch_set_iter(c->d_iter, static_cast<uint32_t>(iter), static_cast<uint32_t>(n0), c->st);
    if (r != TC_OK) return r;
    c->test_mode = true;
    for (int i = 0; i < p->nstmts && r == TC_OK; ++i)
        if (c->in_test[i]) r = exec_stmt(c, i);
    c->test_mode = false;
    if (r != TC_OK) return r;
    Ptrs P{c};
    const VarL& lg = c->vars.at(p->logits_var);
    r = lg.dtype == DT_F32 ? launch_argmax_hits(static_cast<const float*>(P.var(lg.id)), lg.cs, lg.N, lg.C, c->d_labels,
                                                c->d_hits, c->st)
                           : launch_argmax_hits(static_cast<const bf16*>(P.var(lg.id)), lg.cs, lg.N, lg.C, c->d_labels,
                                                c->d_hits, c->st);
    if (r != TC_OK) return r;
    TCB_CUDA_CHECK(cudaMemcpyAsync(c->h_hits, c->d_hits, sizeof(unsigned), cudaMemcpyDeviceToHost, c->st));
    TCB_CUDA_CHECK(cudaStreamSynchronize(c->st));
    *precision = static_cast<double>(c->h_hits[0]) / static_cast<double>(lg.N);
    return TC_OK;
}

tc_status tc_loss(tc_ctx* c, double* loss) {
    if (!c || !loss) return fail(TC_INVALID_ARG, "tc_loss");
    TCB_CUDA_CHECK(cudaStreamSynchronize(c->st));
    *loss = c->h_loss[16 * c->loss_slot];
    return TC_OK;
}

tc_status tc_loss_prev(tc_ctx* c, double* loss) {
    if (!c || !loss) return fail(TC_INVALID_ARG, "tc_loss_prev");
    if (c->loss_count < 2) return fail(TC_INVALID_ARG, "tc_loss_prev: fewer than two steps enqueued");
    const int k = c->loss_slot ^ 1;
    TCB_CUDA_CHECK(cudaEventSynchronize(c->loss_ev[k]));  // that step only, not the one running now
    *loss = c->h_loss[16 * k];
    return TC_OK;
}

tc_status tc_sync(tc_ctx* c) {
    if (!c) return fail(TC_INVALID_ARG, "tc_sync");
    TCB_CUDA_CHECK(cudaStreamSynchronize(c->copy_st));
    TCB_CUDA_CHECK(cudaStreamSynchronize(c->st));
    return TC_OK;
}

tc_status tc_var_download(tc_ctx* c, int var, float* host, int64_t max_elems) {
    if (!c || !host) return fail(TC_INVALID_ARG, "tc_var_download");
    auto it = c->vars.find(var);
    if (it == c->vars.end() || it->second.def < 0) return fail(TC_INVALID_ARG, "tc_var_download: unknown var");
    const VarL& v = it->second;
    Ptrs P{c};
    const bool s2d_input = c->in_layout.s2d && c->plan->stmts[v.def].op == TC_OP_LOAD_X;
    std::vector<uint8_t> raw(s2d_input ? static_cast<size_t>(c->in_layout.elems()) * 2 : v.bytes());
    TCB_CUDA_CHECK(cudaStreamSynchronize(c->st));
    TCB_CUDA_CHECK(cudaMemcpy(raw.data(), P.var(var), raw.size(), cudaMemcpyDeviceToHost));
    auto at = [&](long long e) -> float {
        if (v.dtype == DT_F32) return reinterpret_cast<const float*>(raw.data())[e];
        if (v.dtype == DT_U8) return raw[e] ? 1.f / (1.f - c->mask_rate.at(var)) : 0.f;
        return bf2f(reinterpret_cast<const uint16_t*>(raw.data())[e]);
    };
    long long count = 1;
    for (int j = 0; j < v.rank; ++j) count *= v.d[j];
    if (count > max_elems) return fail(TC_INVALID_ARG, "tc_var_download: buffer too small");
    if (s2d_input) {  // space-to-depth staged image -> NCHW (pixels past the last window are not staged: 0)
        const StageLayout& L = c->in_layout;
        for (int n = 0; n < v.N; ++n)
            for (int ch = 0; ch < v.C; ++ch)
                for (int h = 0; h < v.H; ++h)
                    for (int w = 0; w < v.W; ++w) {
                        const int hp = h + L.pad, wp = w + L.pad;
                        const int P = hp / L.s2d, Q = wp / L.s2d;
                        float val = 0.f;
                        if (P < L.Hs && Q < L.Ws)
                            val = at((((static_cast<long long>(n) * L.Hs + P) * L.Ws + Q) * L.s2d * L.s2d +
                                      (hp % L.s2d) * L.s2d + wp % L.s2d) * L.cs + ch);
                        host[((static_cast<long long>(n) * v.C + ch) * v.H + h) * v.W + w] = val;
                    }
    } else if (v.nhwc) {  // reference NCHW order (also for the 2-D view of a flattened tensor)
        for (int n = 0; n < v.N; ++n)
            for (int ch = 0; ch < v.C; ++ch)
                for (int h = 0; h < v.H; ++h)
                    for (int w = 0; w < v.W; ++w)
                        host[((static_cast<long long>(n) * v.C + ch) * v.H + h) * v.W + w] =
                            at(((static_cast<long long>(n) * v.H + h) * v.W + w) * v.cs + ch);
    } else {
        for (int n = 0; n < v.N; ++n)
            for (int f = 0; f < v.C; ++f) host[static_cast<long long>(n) * v.C + f] = at(static_cast<long long>(n) * v.cs + f);
    }
    return TC_OK;
}

tc_status tc_pool_indices_download(tc_ctx* c, int var, int32_t* host, int64_t max_elems) {
    if (!c || !host) return fail(TC_INVALID_ARG, "tc_pool_indices_download");
    auto it = c->pool_idx_item.find(var);
    if (it == c->pool_idx_item.end()) return fail(TC_INVALID_ARG, "not a max-pool output var");
    const VarL& v = c->vars.at(var);
    const tc_stmt& s = c->plan->stmts[v.def];
    const VarL& x = c->vars.at(s.in[0].index);
    std::vector<uint8_t> raw(v.elems());
    TCB_CUDA_CHECK(cudaStreamSynchronize(c->st));
    TCB_CUDA_CHECK(cudaMemcpy(raw.data(), c->arena + c->items[it->second].off, raw.size(), cudaMemcpyDeviceToHost));
    const long long count = static_cast<long long>(v.N) * v.C * v.H * v.W;
    if (count > max_elems) return fail(TC_INVALID_ARG, "buffer too small");
    // window-local argmax (r*k + s) -> flat NCHW index of the input
    for (int n = 0; n < v.N; ++n)
        for (int ch = 0; ch < v.C; ++ch)
            for (int h = 0; h < v.H; ++h)
                for (int w = 0; w < v.W; ++w) {
                    int loc = raw[((static_cast<long long>(n) * v.H + h) * v.W + w) * v.cs + ch];
                    int32_t flat = -1;
                    if (loc != 255) {
                        if (c->pool_flag_nonpos[v.def]) loc &= 0x7F;  // drop the folded-ReLU flag
                        const int ih = h * s.stride - s.pad + loc / s.k, iw = w * s.stride - s.pad + loc % s.k;
                        flat = static_cast<int32_t>(((static_cast<long long>(n) * x.C + ch) * x.H + ih) * x.W + iw);
                    }
                    host[((static_cast<long long>(n) * v.C + ch) * v.H + h) * v.W + w] = flat;
                }
    return TC_OK;
}

tc_status tc_memory(tc_ctx* c, tc_rt_memory* out) {
    if (!c || !out) return fail(TC_INVALID_ARG, "tc_memory");
    out->arena_bytes = static_cast<int64_t>(c->arena_bytes);
    out->arena_keep_bytes = static_cast<int64_t>(c->arena_keep_bytes);
    out->param_bytes = static_cast<int64_t>(c->slab_bytes);
    out->workspace_bytes = static_cast<int64_t>(c->ws_bytes);
    out->input_bytes = static_cast<int64_t>(c->input_bytes);
    out->device_used_bytes = c->device_used;
    return TC_OK;
}

int tc_launches_per_step(tc_ctx* c) { return c ? c->launches_per_step : -1; }

int tc_profile_launches(tc_ctx* c, int* out, int max) {
    if (!c || !out) return -1;
    const int n = std::min<int>(max, static_cast<int>(c->prof_launches.size()));
    for (int i = 0; i < n; ++i) out[i] = c->prof_launches[i];
    return n;
}

tc_status tc_profile_step(tc_ctx* c, int iter, int n0, int update, float* stmt_ms, int max) {
    if (!c || !stmt_ms || max < c->plan->nstmts) return fail(TC_INVALID_ARG, "tc_profile_step");
    tc_status r = consume_staged(c);
    if (r != TC_OK) return r;
    r = launch_set_iter(c->d_iter, static_cast<uint32_t>(iter), static_cast<uint32_t>(n0), c->st);
    if (r != TC_OK) return r;
    const int n = c->plan->nstmts;
    // ev[i] .. evx[i]: the statement's own kernels; evx[i] .. ev[i + 1]: the bucket all-reduce +
    // momentum update it completes (serial form, main stream), reported separately
    std::vector<cudaEvent_t> ev(n + 1), evx(n);
    for (auto& e : ev) TCB_CUDA_CHECK(cudaEventCreate(&e));
    for (auto& e : evx) TCB_CUDA_CHECK(cudaEventCreate(&e));
    TCB_CUDA_CHECK(cudaEventRecord(ev[0], c->st));
    c->prof_launches.assign(n, 0);
    c->prof_update_ms.assign(n, 0.f);
    for (int i = 0; i < n && r == TC_OK; ++i) {
        const unsigned long long l0 = g_launches.load();
        r = exec_stmt(c, i);
        c->prof_launches[i] = static_cast<int>(g_launches.load() - l0);
        cudaEventRecord(evx[i], c->st);
        for (size_t b = 0; r == TC_OK && b < c->stmt_flush[i].size(); ++b) r = flush_bucket(c, c->stmt_flush[i][b], update, false);
        if (r == TC_OK && update && i == c->last_update_stmt && c->plan->clip > 0) r = clip_update(c, c->st);
        cudaEventRecord(ev[i + 1], c->st);
    }
    cudaStreamSynchronize(c->st);
    for (int i = 0; i < n; ++i) {
        float ms = 0.f, mu = 0.f;
        cudaEventElapsedTime(&ms, ev[i], evx[i]);
        cudaEventElapsedTime(&mu, evx[i], ev[i + 1]);
        stmt_ms[i] = ms;
        c->prof_update_ms[i] = mu;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    for (auto& e : evx) cudaEventDestroy(e);
    return r;
}

int tc_profile_updates(tc_ctx* c, float* out, int max) {
    if (!c || !out) return -1;
    const int n = std::min<int>(max, static_cast<int>(c->prof_update_ms.size()));
    for (int i = 0; i < n; ++i) out[i] = c->prof_update_ms[i];
    return n;
}

}  // extern "C"
