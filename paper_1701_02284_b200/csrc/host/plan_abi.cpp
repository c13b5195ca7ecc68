// C ABI of the plan producers (tc_plan.h): compile a configured network and
// expose its IrProgram as flat tc_stmt records.  This is the only place the
// host compiler's C++ types meet the C boundary; exceptions stop here.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

#include "host/compiler.hpp"
#include "host/netspec.hpp"
#include "status.hpp"
#include "tc_plan.h"

using namespace tensorc;

struct tc_net {
    NetworkDef net;
    IrProgram prog;
    MemoryReport report;
    std::vector<tc_param_desc> params;
    std::vector<tc_stmt> stmts, test;
    std::vector<tc_var_desc> vars;
    tc_plan plan{};
    std::string ir_text, table_text, table_csv, verify_text;
    uint64_t spec_seed = 42;                       // netspec data source synthetic(seed)
    int64_t spec_iters = 0, spec_test_iters = 0;   // netspec solver iters / test_iters
    std::string codegen_text;
};

namespace {

struct Flattener {
    const IrProgram& p;
    std::unordered_map<const ParamSpec*, int> pindex;

    explicit Flattener(const IrProgram& prog) : p(prog) {
        for (std::size_t i = 0; i < p.params.size(); ++i) pindex[p.params[i].get()] = static_cast<int>(i);
    }

    tc_ref ref(const TPtr& t) {
        TPtr b = base_of(t);
        if (b->kind == TKind::Param) return tc_ref{TC_REF_PARAM, pindex.at(b->param.get())};
        return tc_ref{TC_REF_VAR, b->id};
    }

    void hyper(tc_stmt& s, const Hyper& h) {
        s.k = h.k;
        s.stride = h.stride;
        s.pad = h.pad;
        s.max_pool = h.max_pool;
        s.has_bias = h.has_bias;
        s.lrn_size = h.lrn_size;
        s.alpha = h.alpha;
        s.beta = h.beta;
        s.lrn_k = h.lrn_k;
        s.rate = h.rate;
        s.scale = h.scale;
        s.eps = h.eps;
        s.offset = h.offset;
        s.extent = h.extent;
    }

    void add(tc_stmt& s, const TPtr& t) { s.in[s.nin++] = ref(t); }

    // op code + operand list of the expression computing a Let / Update.
    void rhs(tc_stmt& s, const TPtr& n) {
        hyper(s, n->hyper);
        s.slot = n->slot;
        if (n->kind == TKind::Load) {
            s.op = n->hyper.indicator ? TC_OP_LOAD_Y : TC_OP_LOAD_X;
            return;
        }
        if (n->kind == TKind::Concat) {
            s.op = TC_OP_CONCAT;
            for (const TPtr& o : n->operands) add(s, o);
            return;
        }
        if (n->kind == TKind::GradPrim) {
            add(s, n->upstream);
            for (const TPtr& o : n->saved) add(s, o);
            switch (n->prim) {
                case PrimOp::Convolv:
                    s.op = n->slot == 0 ? TC_OP_CONV_BWD_DATA : n->slot == 1 ? TC_OP_CONV_BWD_FILTER : TC_OP_CONV_BWD_BIAS;
                    return;
                case PrimOp::Pooling: s.op = TC_OP_POOL_BWD; return;
                case PrimOp::ReLU: s.op = TC_OP_RELU_BWD; return;
                case PrimOp::Softmax: s.op = TC_OP_SOFTMAX_BWD; return;
                case PrimOp::LRN: s.op = TC_OP_LRN_BWD; return;
                case PrimOp::MatMul: s.op = n->slot == 0 ? TC_OP_MATMUL_BWD_DATA : TC_OP_MATMUL_BWD_W; return;
                case PrimOp::BiasAdd: s.op = TC_OP_BIAS_GRAD; return;
                case PrimOp::Eltwise: s.op = TC_OP_MUL; return;  // d(a*b)/da = up * b
                case PrimOp::Concat: s.op = TC_OP_CONCAT_BWD; return;
                case PrimOp::BatchNorm:
                    s.op = n->slot == 0 ? TC_OP_BN_BWD_DATA : n->slot == 1 ? TC_OP_BN_BWD_GAMMA : TC_OP_BN_BWD_BETA;
                    return;
                default: break;
            }
            fail(ErrKind::Internal, std::string("flatten: no runtime op for d_") + prim_name(n->prim));
        }
        if (n->kind != TKind::Prim) fail(ErrKind::Internal, "flatten: unexpected node kind for " + n->display_name());
        for (const TPtr& o : n->operands) add(s, o);
        switch (n->prim) {
            case PrimOp::Convolv: s.op = TC_OP_CONV_FWD; return;
            case PrimOp::Pooling: s.op = TC_OP_POOL_FWD; return;
            case PrimOp::ReLU: s.op = TC_OP_RELU_FWD; return;
            case PrimOp::Softmax: s.op = TC_OP_SOFTMAX_FWD; return;
            case PrimOp::LRN: s.op = TC_OP_LRN_FWD; return;
            case PrimOp::DropoutMask: s.op = TC_OP_DROPOUT_MASK; return;
            case PrimOp::MatMul: s.op = TC_OP_MATMUL_FWD; return;
            case PrimOp::BiasAdd: s.op = TC_OP_BIAS_ADD; return;
            case PrimOp::Eltwise: s.op = n->hyper.eltwise == ELT_MUL ? TC_OP_MUL : TC_OP_ADD; return;
            case PrimOp::Log: s.op = TC_OP_LOG; return;
            case PrimOp::Recip: s.op = TC_OP_RECIP; return;
            case PrimOp::Scale: s.op = TC_OP_SCALE; return;
            case PrimOp::BatchNorm: s.op = TC_OP_BN_FWD; return;
            default: break;
        }
        fail(ErrKind::Internal, std::string("flatten: no runtime op for ") + prim_name(n->prim));
    }

    // loss = sum coef * dot(Y, logS)
    void loss_terms(tc_stmt& s, const SPtr& e, double coef) {
        switch (e->kind) {
            case SKind::Const:
            case SKind::NamedConst: return;
            case SKind::Add: loss_terms(s, e->args[0], coef); loss_terms(s, e->args[1], coef); return;
            case SKind::Neg: loss_terms(s, e->args[0], -coef); return;
            case SKind::Mul:
                if (e->args[1]->kind == SKind::Const || e->args[1]->kind == SKind::NamedConst)
                    return loss_terms(s, e->args[0], coef * e->args[1]->value);
                return loss_terms(s, e->args[1], coef * e->args[0]->value);
            case SKind::Div: return loss_terms(s, e->args[0], coef / e->args[1]->value);
            case SKind::Dot:
                if (s.nterms >= 4) fail(ErrKind::Internal, "flatten: more than 4 loss terms");
                s.coef[s.nterms++] = coef;
                add(s, e->tensor);
                add(s, e->tensor2);
                return;
            default: fail(ErrKind::Internal, "flatten: unsupported loss form");
        }
    }

    tc_stmt stmt(const IrStmt& ir) {
        tc_stmt s;
        std::memset(&s, 0, sizeof s);
        s.var = ir.var;
        s.storage = ir.storage;
        s.bytes = ir.bytes;
        s.param = -1;
        switch (ir.kind) {
            case StmtKind::Let:
                s.kind = TC_STMT_LET;
                s.inplace = ir.inplace;
                rhs(s, ir.node);
                s.rank = ir.shape.rank();
                for (int i = 0; i < s.rank && i < 4; ++i) s.dims[i] = ir.shape.dims[i];
                break;
            case StmtKind::Dealloc: s.kind = TC_STMT_DEALLOC; break;
            case StmtKind::Update:
                s.kind = TC_STMT_UPDATE;
                rhs(s, ir.node);
                s.param = pindex.at(ir.param.get());
                s.lr_alpha = ir.lr_alpha;
                s.momentum = ir.momentum;
                s.decay = ir.decay;
                break;
            case StmtKind::Print:
                s.kind = TC_STMT_PRINT;
                s.op = TC_OP_PRINT_LOSS;
                loss_terms(s, ir.loss, 1.0);
                break;
        }
        return s;
    }
};

void fill_param(tc_param_desc& d, const ParamSpec& ps, const Shape& s) {
    std::memset(&d, 0, sizeof d);
    std::strncpy(d.name, ps.name.c_str(), sizeof d.name - 1);
    d.rank = s.rank();
    for (int i = 0; i < s.rank() && i < 4; ++i) d.dims[i] = s.dims[i];
    d.init_kind = ps.init == InitKind::Xavier ? TC_INIT_XAVIER : ps.init == InitKind::Constant ? TC_INIT_CONSTANT
                                                                                               : TC_INIT_GAUSSIAN;
    d.init_value = ps.init_value;
    d.sigma = ps.sigma;
    d.lr_mult = ps.lr_mult;
    d.decay_mult = ps.decay_mult;
    // Xavier fans: conv (Cout, Cin, k, k) -> Cin*k^2, Cout*k^2; full (out, in) -> in, out.
    if (s.rank() == 4) {
        d.fan_in = s.dims[1] * s.dims[2] * s.dims[3];
        d.fan_out = s.dims[0] * s.dims[2] * s.dims[3];
    } else if (s.rank() == 2) {
        d.fan_in = s.dims[1];
        d.fan_out = s.dims[0];
    } else {
        d.fan_in = d.fan_out = s.count();
    }
}



void apply_opts(CompileOptions& co, const tc_compile_opts* opts) {
    co.solver.lr = opts->lr;
    co.solver.momentum = opts->momentum;
    co.solver.decay = opts->decay;
    co.solver.clip = opts->clip;
    co.mode = opts->mode == TC_MODE_REUSE ? MemMode::Reuse : MemMode::Dealloc;
    co.workspace_cap_mb = opts->workspace_cap_mb;
    co.greedy_schedule = opts->greedy_schedule != 0;
    co.cse = opts->no_cse == 0;
}

// Gradient derivation + IR pipeline + memplan of an elaborated network, flattened to tc_plan.
void compile_into(tc_net* h, const CompileOptions& co) {
    if (!(co.solver.clip >= 0.0)) fail(ErrKind::SyntaxError, "solver clip must be >= 0 (0 disables, SPEC.md:36)");
    h->prog = compile_network(h->net, co);
    h->report = analyze(h->prog);
    Flattener fl(h->prog);
    for (std::size_t i = 0; i < h->prog.params.size(); ++i) {
        tc_param_desc d;
        fill_param(d, *h->prog.params[i], h->prog.param_shapes[i]);
        h->params.push_back(d);
    }
    for (const IrStmt& s : h->prog.train) h->stmts.push_back(fl.stmt(s));
    for (const IrStmt& s : h->prog.test) h->test.push_back(fl.stmt(s));
    int max_var = 0;
    for (const auto& [id, shp] : h->prog.var_shapes) {
        tc_var_desc v;
        std::memset(&v, 0, sizeof v);
        v.id = id;
        v.rank = shp.rank();
        for (int i = 0; i < v.rank && i < 4; ++i) v.dims[i] = shp.dims[i];
        h->vars.push_back(v);
        max_var = std::max(max_var, id + 1);
    }
    std::sort(h->vars.begin(), h->vars.end(), [](const tc_var_desc& a, const tc_var_desc& b) { return a.id < b.id; });
    h->ir_text = dump_ir(h->prog);
    h->table_text = format_report(h->report, false);
    h->table_csv = format_report(h->report, true);
    h->verify_text = verify(h->prog);
    tc_plan& p = h->plan;
    p.name = h->net.name.c_str();
    p.batch = h->prog.batch;
    p.classes = h->prog.classes;
    for (int i = 0; i < 4; ++i) p.input_dims[i] = h->prog.input_shape.dims[i];
    p.nparams = static_cast<int>(h->params.size());
    p.params = h->params.data();
    p.nstmts = static_cast<int>(h->stmts.size());
    p.stmts = h->stmts.data();
    p.ntest = static_cast<int>(h->test.size());
    p.test_stmts = h->test.data();
    p.logits_var = h->prog.logits_var;
    p.nvars = static_cast<int>(h->vars.size());
    p.vars = h->vars.data();
    p.max_var = max_var;
    p.lr = co.solver.lr;
    p.momentum = co.solver.momentum;
    p.decay = co.solver.decay;
    p.clip = co.solver.clip;
    p.mode = co.mode == MemMode::Reuse ? TC_MODE_REUSE : TC_MODE_DEALLOC;
}

template <class Fn>
tc_status guarded(Fn&& fn) {
    try {
        fn();
        return TC_OK;
    } catch (const CompileError& e) {
        return tcb::fail(TC_COMPILE_ERROR, std::string(err_kind_name(e.kind)) + " at " + e.loc.to_string() + ": " + e.what());
    } catch (const std::exception& e) {
        return tcb::fail(TC_INTERNAL, e.what());
    }
}

}  // namespace

extern "C" {

tc_status tc_net_compile(const char* name, int64_t batch, const tc_compile_opts* opts, tc_net** out) {
    if (!name || !out || batch <= 0) return tcb::fail(TC_INVALID_ARG, "tc_net_compile: bad arguments");
    *out = nullptr;
    return guarded([&] {
        auto h = std::make_unique<tc_net>();
        if (opts && opts->global_batch > 0) h->net.loss_card = opts->global_batch;
        build_by_name(h->net, name, batch);
        CompileOptions co;
        if (opts) apply_opts(co, opts);
        co.solver.name = name;
        compile_into(h.get(), co);
        *out = h.release();
    });
}

tc_status tc_net_compile_spec(const char* text, int64_t batch, const tc_compile_opts* opts, tc_net** out) {
    if (!text || !out || batch < 0) return tcb::fail(TC_INVALID_ARG, "tc_net_compile_spec: bad arguments");
    *out = nullptr;
    return guarded([&] {
        auto h = std::make_unique<tc_net>();
        if (opts && opts->global_batch > 0) h->net.loss_card = opts->global_batch;
        SpecSolver sv;
        build_from_spec(h->net, text, batch, &sv);
        CompileOptions co;
        co.solver.lr = sv.lr;
        co.solver.momentum = sv.momentum;
        co.solver.decay = sv.decay;
        co.solver.clip = sv.clip;
        if (opts) apply_opts(co, opts);  // explicit options override the spec's solver section
        co.solver.name = h->net.name;
        h->spec_seed = sv.seed;
        h->spec_iters = sv.iters;
        h->spec_test_iters = sv.test_iters;
        compile_into(h.get(), co);
        *out = h.release();
    });
}

tc_status tc_net_spec_info(const tc_net* net, uint64_t* seed, int64_t* iters, int64_t* test_iters) {
    if (!net) return tcb::fail(TC_INVALID_ARG, "tc_net_spec_info: null net");
    if (seed) *seed = net->spec_seed;
    if (iters) *iters = net->spec_iters;
    if (test_iters) *test_iters = net->spec_test_iters;
    return TC_OK;
}

// Serialized plan (raw little-endian POD records, guarded by a header of record sizes): lets a
// consumer that does not link this library (the CPU oracle's reference arm in bench.py) execute the
// exact plan the runtime executes.
tc_status tc_plan_save(const tc_plan* p, const char* path) {
    if (!p || !path) return tcb::fail(TC_INVALID_ARG, "tc_plan_save: null argument");
    FILE* f = std::fopen(path, "wb");
    if (!f) return tcb::fail(TC_IO_ERROR, std::string("tc_plan_save: cannot open ") + path);
    bool ok = true;
    auto put = [&](const void* d, std::size_t n) { ok = ok && std::fwrite(d, 1, n, f) == n; };
    const uint32_t hdr[6] = {0x4c504354u /* "TCPL" */, 1u, static_cast<uint32_t>(sizeof(tc_stmt)),
                             static_cast<uint32_t>(sizeof(tc_param_desc)), static_cast<uint32_t>(sizeof(tc_var_desc)),
                             static_cast<uint32_t>(TC_MAX_IN)};
    put(hdr, sizeof hdr);
    char name[64] = {0};
    std::strncpy(name, p->name ? p->name : "", sizeof name - 1);
    put(name, sizeof name);
    const int64_t head[6] = {p->batch, p->classes, p->input_dims[0], p->input_dims[1], p->input_dims[2], p->input_dims[3]};
    put(head, sizeof head);
    const int32_t counts[7] = {p->nparams, p->nstmts, p->ntest, p->logits_var, p->nvars, p->max_var, p->mode};
    put(counts, sizeof counts);
    const double solver[4] = {p->lr, p->momentum, p->decay, p->clip};
    put(solver, sizeof solver);
    put(p->params, sizeof(tc_param_desc) * p->nparams);
    put(p->stmts, sizeof(tc_stmt) * p->nstmts);
    put(p->test_stmts, sizeof(tc_stmt) * p->ntest);
    put(p->vars, sizeof(tc_var_desc) * p->nvars);
    ok = (std::fclose(f) == 0) && ok;
    return ok ? TC_OK : tcb::fail(TC_IO_ERROR, std::string("tc_plan_save: write failed: ") + path);
}

// ---------------------------------------------------------------- codegen
}  // extern "C"

namespace {

std::string fmt_d(double v) {
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}

std::string c_str_lit(const std::string& t) {
    std::string o = "\"";
    for (char ch : t) {
        if (ch == '"' || ch == '\\') o += '\\';
        o += ch;
    }
    return o + "\"";
}

// Designated initializer of a tc_stmt: non-default fields only, in declaration order.
std::string stmt_init(const tc_stmt& s) {
    std::string o = "{";
    auto fi = [&](const char* n, long long v) {
        if (v) o += std::string(".") + n + " = " + std::to_string(v) + ", ";
    };
    auto fd = [&](const char* n, double v) {
        if (v != 0.0) o += std::string(".") + n + " = " + fmt_d(v) + ", ";
    };
    fi("kind", s.kind);
    fi("op", s.op);
    fi("var", s.var);
    fi("storage", s.storage);
    fi("inplace", s.inplace);
    fi("param", s.param);
    fi("nin", s.nin);
    if (s.nin) {
        o += ".in = {";
        for (int i = 0; i < s.nin; ++i) o += "{" + std::to_string(s.in[i].kind) + ", " + std::to_string(s.in[i].index) + "}, ";
        o += "}, ";
    }
    fi("rank", s.rank);
    if (s.rank) {
        o += ".dims = {";
        for (int i = 0; i < 4; ++i) o += std::to_string(s.dims[i]) + (i < 3 ? ", " : "");
        o += "}, ";
    }
    fi("bytes", s.bytes);
    fi("k", s.k);
    fi("stride", s.stride);
    fi("pad", s.pad);
    fi("max_pool", s.max_pool);
    fi("has_bias", s.has_bias);
    fi("lrn_size", s.lrn_size);
    fi("slot", s.slot);
    fd("alpha", s.alpha);
    fd("beta", s.beta);
    fd("lrn_k", s.lrn_k);
    fd("rate", s.rate);
    fd("scale", s.scale);
    fd("eps", s.eps);
    fi("offset", s.offset);
    fi("extent", s.extent);
    fd("lr_alpha", s.lr_alpha);
    fd("momentum", s.momentum);
    fd("decay", s.decay);
    fi("nterms", s.nterms);
    if (s.nterms) {
        o += ".coef = {";
        for (int i = 0; i < 4; ++i) o += fmt_d(s.coef[i]) + (i < 3 ? ", " : "");
        o += "}, ";
    }
    if (o.size() > 1) o.resize(o.size() - 2);
    return o + "}";
}

std::string emit_program(const tc_net* h, int mode, long long iters, long long test_iters) {
    const tc_plan& p = h->plan;
    const std::string& nm = h->net.name;
    std::string o;
    o += "// " + nm + ".gen.cpp -- generated by tc_net_codegen from the IrProgram of network '" + nm + "' (batch " +
         std::to_string(p.batch) + ").\n";
    o += "// A standalone training program: one compilation unit that depends only on the runtime library\n"
         "// (libtcb200, tc_runtime.h), not on the compiler.  One runtime call per IR statement, with the\n"
         "// statement in Fig. 2 syntax as the comment above it (PAPER.md section 5, SPEC.md:422-451).\n"
         "//   build: g++ -std=c++20 -O2 -I<repo>/include " + nm + ".gen.cpp -L<repo>/paper_1701_02284_b200/_lib -ltcb200\n"
         "//   run:   ./a.out [iters] [snapshot_dir]     (TENSORC_SEED overrides the seed, default 42)\n";
    o += "#include <cstdio>\n#include <cstdlib>\n\n#include \"tc_runtime.h\"\n\n";
    o += std::string("static const int kMode = ") + (mode == TC_MODE_REUSE ? "TC_MODE_REUSE" : "TC_MODE_DEALLOC") +
         ";  // memory mode: TC_MODE_REUSE | TC_MODE_DEALLOC (edit this line)\n";
    o += "static const long long kTrainIters = " + std::to_string(iters) + ", kTestIters = " + std::to_string(test_iters) + ";\n\n";
    o += "static const tc_param_desc kParams[] = {\n";
    for (const tc_param_desc& d : h->params) {
        o += "    {" + c_str_lit(d.name) + ", " + std::to_string(d.rank) + ", {";
        for (int i = 0; i < 4; ++i) o += std::to_string(d.dims[i]) + (i < 3 ? ", " : "");
        o += "}, " + std::to_string(d.init_kind) + ", " + fmt_d(d.init_value) + ", " + fmt_d(d.sigma) + ", " +
             fmt_d(d.lr_mult) + ", " + fmt_d(d.decay_mult) + ", " + std::to_string(d.fan_in) + ", " +
             std::to_string(d.fan_out) + "},\n";
    }
    o += "};\n\n// train-loop body\nstatic const tc_stmt kTrain[] = {\n";
    for (std::size_t i = 0; i < h->stmts.size(); ++i) o += "    " + stmt_init(h->stmts[i]) + ",  // [" + std::to_string(i) + "]\n";
    o += "};\n\n// test body: the forward statements the main logits depend on\nstatic const tc_stmt kTest[] = {\n";
    for (const tc_stmt& s : h->test) o += "    " + stmt_init(s) + ",\n";
    if (h->test.empty()) o += "    {},\n";
    o += "};\n\nstatic const tc_var_desc kVars[] = {\n";
    for (const tc_var_desc& v : h->vars)
        o += "    {" + std::to_string(v.id) + ", " + std::to_string(v.rank) + ", {" + std::to_string(v.dims[0]) + ", " +
             std::to_string(v.dims[1]) + ", " + std::to_string(v.dims[2]) + ", " + std::to_string(v.dims[3]) + "}},\n";
    o += "};\n\n";
    o += "static void check(tc_status s, const char* what) {\n"
         "    if (s != TC_OK) {\n"
         "        std::fprintf(stderr, \"%s: status %d: %s\\n\", what, static_cast<int>(s), tc_last_error());\n"
         "        std::exit(s == TC_IO_ERROR || s == TC_FORMAT_ERROR ? 2 : 1);\n"
         "    }\n"
         "}\n\n";
    o += "// One training iteration: one runtime call per IR statement.\n"
         "static void train(tc_ctx* ctx, int it) {\n";
    for (std::size_t i = 0; i < h->prog.train.size(); ++i) {
        std::string t = h->prog.train[i].text;
        for (char& ch : t)
            if (ch == '\n') ch = ' ';
        o += "    // " + t + "\n    check(tc_exec_stmt(ctx, " + std::to_string(i) + ", it, 0), \"statement " +
             std::to_string(i) + "\");\n";
    }
    o += "}\n\n";
    o += "int main(int argc, char** argv) {\n"
         "    const long long iters = argc > 1 ? std::atoll(argv[1]) : kTrainIters;\n"
         "    const char* snapshot = argc > 2 ? argv[2] : nullptr;\n"
         "    tc_plan plan{};\n"
         "    plan.name = " + c_str_lit(nm) + ";\n"
         "    plan.batch = " + std::to_string(p.batch) + ";\n"
         "    plan.classes = " + std::to_string(p.classes) + ";\n";
    for (int i = 0; i < 4; ++i) o += "    plan.input_dims[" + std::to_string(i) + "] = " + std::to_string(p.input_dims[i]) + ";\n";
    o += "    plan.nparams = " + std::to_string(p.nparams) + ";\n"
         "    plan.params = kParams;\n"
         "    plan.nstmts = " + std::to_string(p.nstmts) + ";\n"
         "    plan.stmts = kTrain;\n"
         "    plan.ntest = " + std::to_string(p.ntest) + ";\n"
         "    plan.test_stmts = kTest;\n"
         "    plan.logits_var = " + std::to_string(p.logits_var) + ";\n"
         "    plan.nvars = " + std::to_string(p.nvars) + ";\n"
         "    plan.vars = kVars;\n"
         "    plan.max_var = " + std::to_string(p.max_var) + ";\n"
         "    plan.lr = " + fmt_d(p.lr) + ";\n"
         "    plan.momentum = " + fmt_d(p.momentum) + ";\n"
         "    plan.decay = " + fmt_d(p.decay) + ";\n"
         "    plan.clip = " + fmt_d(p.clip) + ";\n"
         "    plan.mode = kMode;\n"
         "    tc_ctx_desc desc{};\n"
         "    desc.world = 1;\n"
         "    const char* seed = std::getenv(\"TENSORC_SEED\");\n"
         "    desc.seed = seed ? std::strtoull(seed, nullptr, 10) : 42;\n"
         "    tc_ctx* ctx = nullptr;\n"
         "    check(tc_ctx_create(&plan, &desc, &ctx), \"tc_ctx_create\");\n"
         "    check(tc_init_params(ctx), \"init\");\n"
         "    if (snapshot) {  // resume from the snapshot directory's parameters (missing files keep their init)\n"
         "        int loaded = 0, missing = 0;\n"
         "        check(tc_snapshot_load(ctx, snapshot, &loaded, &missing), \"snapshot load\");\n"
         "        std::fprintf(stderr, \"snapshot %s: %d loaded, %d missing\\n\", snapshot, loaded, missing);\n"
         "    }\n"
         "    for (long long it = 0; it < iters; ++it) {\n"
         "        check(tc_stage_synthetic(ctx, static_cast<int>(it), 0), \"data\");\n"
         "        train(ctx, static_cast<int>(it));\n"
         "        double loss = 0.0;\n"
         "        check(tc_loss(ctx, &loss), \"loss\");\n"
         "        std::printf(\"%lld,%.9g\\n\", it, loss);\n"
         "    }\n"
         "    if (snapshot) check(tc_snapshot_save(ctx, snapshot), \"snapshot save\");\n";
    if (!h->test.empty())
        o += "    double prec = 0.0;\n"
             "    for (long long t = 0; t < kTestIters; ++t) {  // test procedure: argmax-match precision\n"
             "        double pr = 0.0;\n"
             "        check(tc_stage_synthetic(ctx, static_cast<int>(iters + t), 0), \"data\");\n"
             "        check(tc_test(ctx, static_cast<int>(iters + t), 0, &pr), \"test\");\n"
             "        prec += pr;\n"
             "    }\n"
             "    std::printf(\"precision %.6f\\n\", kTestIters ? prec / kTestIters : 0.0);\n";
    o += "    tc_ctx_destroy(ctx);\n"
         "    return 0;\n"
         "}\n";
    return o;
}

}  // namespace

extern "C" {

const char* tc_net_codegen(tc_net* net, int mode, int64_t iters, int64_t test_iters) {
    if (!net) return "";
    try {
        const long long it = iters > 0 ? iters : (net->spec_iters > 0 ? net->spec_iters : 1000);
        const long long ti = test_iters >= 0 ? test_iters : (net->spec_test_iters > 0 ? net->spec_test_iters : 10);
        net->codegen_text = emit_program(net, mode, it, ti);
    } catch (const std::exception& e) {
        tcb::fail(TC_INTERNAL, e.what());
        return "";
    }
    return net->codegen_text.c_str();
}

void tc_net_destroy(tc_net* net) { delete net; }
const tc_plan* tc_net_plan(const tc_net* net) { return net ? &net->plan : nullptr; }
const char* tc_net_ir_text(const tc_net* net) { return net ? net->ir_text.c_str() : ""; }
const char* tc_net_memory_table(const tc_net* net, int csv) {
    return net ? (csv ? net->table_csv.c_str() : net->table_text.c_str()) : "";
}
const char* tc_net_verify(const tc_net* net) { return net ? net->verify_text.c_str() : "null net"; }
const char* tc_net_stmt_text(const tc_net* net, int index) {
    if (!net || index < 0 || index >= static_cast<int>(net->prog.train.size())) return "";
    return net->prog.train[index].text.c_str();
}
tc_status tc_net_memory_summary(const tc_net* net, tc_mem_summary* out) {
    if (!net || !out) return tcb::fail(TC_INVALID_ARG, "tc_net_memory_summary: null argument");
    const MemoryReport& r = net->report;
    out->peak_dealloc_bytes = r.peak_dealloc_bytes;
    out->peak_reuse_bytes = r.peak_reuse_bytes;
    out->param_bytes = r.param_bytes;
    out->workspace_bytes = r.workspace_bytes;
    out->peak_dealloc_mb = r.peak_dealloc_mb();
    out->peak_reuse_mb = r.peak_reuse_mb();
    out->param_mb = static_cast<float>(r.param_bytes) / 1e6f;
    out->workspace_mb = static_cast<float>(r.workspace_bytes) / 1e6f;
    return TC_OK;
}

}  // extern "C"
