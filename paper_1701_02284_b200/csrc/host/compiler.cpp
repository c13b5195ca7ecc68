// Compilation pipeline: vectorize -> shapes -> gradients -> IR -> memory plan.
// See compiler.hpp for the stage list and the SPEC.md sections each follows.
#include "host/compiler.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <set>
#include <iomanip>
#include <sstream>
#include <unordered_set>

namespace tensorc {

const Shape& ShapeTable::of(const TPtr& e) const {
    auto it = t.find(e.get());
    if (it == t.end()) fail(ErrKind::Internal, "no shape for " + e->display_name());
    return it->second;
}
const Shape& ShapeTable::of(const ParamSpec* ps) const {
    auto it = p.find(ps);
    if (it == p.end()) fail(ErrKind::Internal, "no shape for parameter " + ps->name);
    return it->second;
}

// ================================================================ vectorize
namespace {

bool is_ivar(const SPtr& s, int id) { return s && s->kind == SKind::IndexVar && s->ivar == id; }

// IndexAbs[i,j] Sum_k a(i,k) * w(j,k)  ->  (a, w)
bool match_contraction(const TensorExpr& t, TPtr* a, TPtr* w) {
    if (t.kind != TKind::IndexAbs || t.binders.size() != 2 || !t.body || t.body->kind != SKind::Sum) return false;
    const int k = t.body->ivar;
    const SPtr& m = t.body->args[0];
    if (m->kind != SKind::Mul) return false;
    const SPtr& ea = m->args[0];
    const SPtr& ew = m->args[1];
    if (ea->kind != SKind::Elem || ew->kind != SKind::Elem || ea->args.size() != 2 || ew->args.size() != 2) return false;
    if (!is_ivar(ea->args[0], t.binders[0]) || !is_ivar(ea->args[1], k)) return false;
    if (!is_ivar(ew->args[0], t.binders[1]) || !is_ivar(ew->args[1], k)) return false;
    *a = ea->tensor;
    *w = ew->tensor;
    return true;
}

class Vectorizer {
public:
    explicit Vectorizer(bool cse) : cse_(cse) {}
    int merged() const { return merged_; }
    TPtr run(const TPtr& t) {
        if (!t) return t;
        auto hit = memo_.find(t);
        if (hit != memo_.end()) return hit->second;
        auto c = std::make_shared<TensorExpr>(*t);
        for (auto& op : c->operands) op = run(op);
        for (auto& sv : c->saved) sv = run(sv);
        c->upstream = run(c->upstream);
        if (c->body) c->body = run_s(c->body);
        TPtr a, w;
        TPtr out = c;
        if (match_contraction(*c, &a, &w)) {
            Hyper h;
            h.transpose_b = true;
            h.out = c->hyper.out;
            out = t_prim(PrimOp::MatMul, h, {a, w}, 2, c->id);
        } else if (c->kind == TKind::AddT && c->operands[1]->kind == TKind::RowBcast) {
            out = t_prim(PrimOp::BiasAdd, Hyper{}, {c->operands[0], c->operands[1]->operands[0]}, c->rank, c->id);
        }
        if (cse_) out = canonical(out);
        memo_.emplace(t, out);
        return out;
    }
    SPtr run_s(const SPtr& s) {
        if (!s) return s;
        auto hit = smemo_.find(s);
        if (hit != smemo_.end()) return hit->second;
        auto c = std::make_shared<ScalarExpr>(*s);
        for (auto& x : c->args) x = run_s(x);
        c->tensor = run(c->tensor);
        c->tensor2 = run(c->tensor2);
        c->range_of = run(c->range_of);
        SPtr out = c;
        smemo_.emplace(s, out);
        return out;
    }

private:
    // cse: operands are already canonical, so syntactic identity is identity of (kind, operator,
    // hyper-parameters, operand nodes); leaves are keyed by what they denote.
    TPtr canonical(const TPtr& t) {
        std::ostringstream k;
        k << std::setprecision(17);
        switch (t->kind) {
            case TKind::Param: k << "P" << t->param.get(); break;
            case TKind::Input: k << "I" << t->name; break;
            case TKind::Prim:
                if (t->prim == PrimOp::DropoutMask) return t;  // randomized: never merged
                k << "F" << static_cast<int>(t->prim) << ":" << t->rank;
                break;
            case TKind::AddT: k << "A" << t->rank; break;
            case TKind::Concat: k << "C" << t->rank; break;
            case TKind::Flatten: k << "L" << t->flat_axis; break;
            case TKind::Reshape: k << "R" << t->reshape_to.to_string(); break;
            default: return t;  // Copy (each backs its own in-place op), Var, Load, index expressions, grads
        }
        const Hyper& h = t->hyper;
        k << "|" << h.k << "," << h.stride << "," << h.pad << "," << h.max_pool << "," << h.rank << "," << h.rate << ","
          << h.lrn_size << "," << h.alpha << "," << h.beta << "," << h.transpose_a << "," << h.transpose_b << ","
          << h.scale << "," << h.classes << "," << h.indicator << "," << h.has_bias << "," << h.eps << "," << h.lrn_k << ","
          << h.offset << "," << h.extent << "," << h.eltwise << "," << h.out << "|";
        for (const TPtr& o : t->operands) k << o.get() << ";";
        auto [it, fresh] = canon_.emplace(k.str(), t);
        if (!fresh) ++merged_;
        return it->second;
    }
    bool cse_ = false;
    int merged_ = 0;
    std::unordered_map<std::string, TPtr> canon_;
    std::unordered_map<TPtr, TPtr> memo_;
    std::unordered_map<SPtr, SPtr> smemo_;
};

}  // namespace

int vectorize(NetworkDef& net, bool cse) {
    Vectorizer v(cse);
    net.loss = v.run_s(net.loss);
    net.logits_main = v.run(net.logits_main);
    net.x_load = v.run(net.x_load);
    net.y_load = v.run(net.y_load);
    return v.merged();
}

// ================================================================ shapes
namespace {

std::int64_t out_extent(std::int64_t in, int k, int s, int p, const std::string& site) {
    const std::int64_t num = in + 2LL * p - k;
    if (num < 0) fail(ErrKind::NonPositiveExtent, site + ": window larger than padded input");
    const std::int64_t o = num / s + 1;
    if (o < 1) fail(ErrKind::NonPositiveExtent, site + ": non-positive output extent");
    return o;
}

void bind_param(ShapeTable& st, const TPtr& p, const Shape& s) {
    auto it = st.p.find(p->param.get());
    if (it == st.p.end()) {
        st.p.emplace(p->param.get(), s);
        st.t[p.get()] = s;
    } else if (it->second != s) {
        fail(ErrKind::ShapeMismatch, "parameter " + p->param->name + ": expected " + it->second.to_string() +
                                         ", found " + s.to_string());
    } else {
        st.t[p.get()] = s;
    }
}

void need_rank(const Shape& s, int r, const std::string& site) {
    if (s.rank() != r)
        fail(ErrKind::ShapeMismatch, site + ": expected rank " + std::to_string(r) + ", found " + s.to_string());
}

}  // namespace

void infer_shapes(const NetworkDef& net, ShapeTable& st) {
    auto visit = [&](const TPtr& t) {
        if (st.t.count(t.get())) return;
        const std::string site = t->display_name();
        auto sh = [&](int i) -> const Shape& { return st.of(t->operands[i]); };
        Shape out;
        switch (t->kind) {
            case TKind::Param: return;  // bound at first constraining use
            case TKind::Var: fail(ErrKind::UnboundName, "free variable " + site + " after normalisation");
            case TKind::Input:
                out = t->name == "Y" ? Shape{net.batch} : net.input_shape;
                break;
            case TKind::Load:
                out = t->hyper.indicator ? Shape{sh(0).dims[0], t->hyper.classes} : sh(0);
                break;
            case TKind::Flatten: {
                const Shape& s = sh(0);
                std::vector<std::int64_t> d(s.dims.begin(), s.dims.begin() + t->flat_axis);
                std::int64_t rest = 1;
                for (int i = t->flat_axis; i < s.rank(); ++i) rest *= s.dims[i];
                d.push_back(rest);
                out = Shape(d);
                break;
            }
            case TKind::Reshape: out = t->reshape_to; break;
            case TKind::Copy: out = sh(0); break;
            case TKind::Concat: {
                out = sh(0);
                need_rank(out, 4, site);
                for (std::size_t i = 1; i < t->operands.size(); ++i) {
                    const Shape& s = sh(static_cast<int>(i));
                    need_rank(s, 4, site);
                    if (s.dims[0] != out.dims[0] || s.dims[2] != out.dims[2] || s.dims[3] != out.dims[3])
                        fail(ErrKind::ShapeMismatch, site + ": concat operands disagree outside the channel axis (" +
                                                         out.to_string() + " vs " + s.to_string() + ")");
                    out.dims[1] += s.dims[1];
                }
                break;
            }
            case TKind::Prim: {
                const Hyper& h = t->hyper;
                switch (t->prim) {
                    case PrimOp::Convolv: {
                        const Shape& x = sh(0);
                        need_rank(x, 4, site);
                        bind_param(st, t->operands[1], Shape{h.out, x.dims[1], h.k, h.k});
                        if (h.has_bias) bind_param(st, t->operands[2], Shape{h.out});
                        out = Shape{x.dims[0], h.out, out_extent(x.dims[2], h.k, h.stride, h.pad, site),
                                    out_extent(x.dims[3], h.k, h.stride, h.pad, site)};
                        break;
                    }
                    case PrimOp::Pooling: {
                        const Shape& x = sh(0);
                        need_rank(x, 4, site);
                        out = Shape{x.dims[0], x.dims[1], out_extent(x.dims[2], h.k, h.stride, h.pad, site),
                                    out_extent(x.dims[3], h.k, h.stride, h.pad, site)};
                        break;
                    }
                    case PrimOp::MatMul: {
                        const Shape& a = sh(0);
                        need_rank(a, 2, site);
                        bind_param(st, t->operands[1], Shape{h.out, a.dims[1]});
                        out = Shape{a.dims[0], h.out};
                        break;
                    }
                    case PrimOp::BiasAdd: {
                        out = sh(0);
                        bind_param(st, t->operands[1], Shape{out.dims[1]});
                        break;
                    }
                    case PrimOp::BatchNorm: {
                        out = sh(0);
                        need_rank(out, 4, site);
                        bind_param(st, t->operands[1], Shape{out.dims[1]});
                        bind_param(st, t->operands[2], Shape{out.dims[1]});
                        break;
                    }
                    case PrimOp::Eltwise: {
                        out = sh(0);
                        if (sh(1) != out)
                            fail(ErrKind::ShapeMismatch, site + ": elementwise operands " + out.to_string() + " vs " +
                                                             sh(1).to_string());
                        break;
                    }
                    case PrimOp::Softmax: out = sh(0); need_rank(out, 2, site); break;
                    case PrimOp::ReLU:
                        out = sh(0);
                        if (h.rank && out.rank() != h.rank)
                            fail(ErrKind::ShapeMismatch, site + ": relu(" + std::to_string(h.rank) + ") applied to " +
                                                             out.to_string());
                        break;
                    default: out = sh(0); break;
                }
                break;
            }
            case TKind::IndexAbs: {
                TPtr a, w;
                if (!match_contraction(*t, &a, &w)) fail(ErrKind::Internal, site + ": unsupported index pattern");
                const Shape& as = st.of(a);
                if (as.rank() != 2)
                    fail(ErrKind::ShapeMismatch, site + ": full layer applied to rank-" + std::to_string(as.rank()) +
                                                     " tensor " + as.to_string() + " (missing flatten?)");
                bind_param(st, w, Shape{t->hyper.out, as.dims[1]});
                out = Shape{as.dims[0], t->hyper.out};
                break;
            }
            case TKind::RowBcast: return;
            case TKind::AddT: {
                out = sh(0);
                if (t->operands[1]->kind == TKind::RowBcast) bind_param(st, t->operands[1]->operands[0], Shape{out.dims[1]});
                break;
            }
            case TKind::GradPrim:
            case TKind::Apply: fail(ErrKind::Internal, site + ": unexpected node in forward shape inference");
        }
        st.t[t.get()] = out;
    };
    // Parameters get their shape from their consumer, so visit consumers with
    // a post-order that binds params lazily.
    postorder_scalar(net.loss, visit);
    if (net.logits_main) postorder(net.logits_main, visit);
    // Scalar Dot operands must agree.
    std::function<void(const SPtr&)> chk = [&](const SPtr& s) {
        if (!s) return;
        for (const auto& a : s->args) chk(a);
        if (s->kind == SKind::Dot && st.of(s->tensor) != st.of(s->tensor2))
            fail(ErrKind::ShapeMismatch, "dot operands " + st.of(s->tensor).to_string() + " vs " +
                                             st.of(s->tensor2).to_string());
    };
    chk(net.loss);
}

// ================================================================ gradients
namespace {

class GradBuilder {
public:
    GradBuilder(NetworkDef& net, ShapeTable& st, GradInfo& gi) : net_(net), st_(st), gi_(gi) {}

    void run() {
        std::vector<TPtr> topo;
        postorder_scalar(net_.loss, [&](const TPtr& t) { topo.push_back(t); });
        for (const TPtr& t : topo) req_[t.get()] = compute_req(t);
        seed(net_.loss, 1.0);
        for (auto it = topo.rbegin(); it != topo.rend(); ++it) {
            const TPtr& n = *it;
            auto a = adj_.find(n.get());
            if (a == adj_.end() || !req_[n.get()]) continue;
            TPtr g = accumulate(n, a->second);
            if (n->kind == TKind::Param) {
                gi_.param_grads.emplace_back(n->param, g);
                continue;
            }
            backward(n, g);
        }
        // seed dependence
        for (const TPtr& c : gi_.created) {
            bool dep = seeds_.count(c.get()) != 0;
            for (const TPtr& d : c->deps()) {
                TPtr b = base_of(d);
                auto f = gi_.seed_dep.find(b.get());
                if (f != gi_.seed_dep.end() && f->second) dep = true;
            }
            gi_.seed_dep[c.get()] = dep;
        }
    }

private:
    bool compute_req(const TPtr& t) {
        switch (t->kind) {
            case TKind::Param: return true;
            case TKind::Input:
            case TKind::Load: return false;
            case TKind::Prim:
                if (t->prim == PrimOp::DropoutMask) return false;
                break;
            default: break;
        }
        for (const TPtr& d : t->deps())
            if (req_[d.get()]) return true;
        return false;
    }
    bool req(const TPtr& t) const {
        auto it = req_.find(t.get());
        return it != req_.end() && it->second;
    }

    TPtr reg(TPtr node, const Shape& s) {
        st_.t[node.get()] = s;
        gi_.created.push_back(node);
        return node;
    }
    void contrib(const TPtr& to, const TPtr& g) {
        if (req(to)) adj_[to.get()].push_back(g);
    }
    std::string wrt(const TPtr& t) const {
        TPtr b = base_of(t);
        return b->display_name();
    }

    TPtr accumulate(const TPtr& n, const std::vector<TPtr>& gs) {
        TPtr g = gs[0];
        for (std::size_t i = 1; i < gs.size(); ++i) {
            Hyper h;
            h.eltwise = ELT_ADD;
            g = reg(t_prim(PrimOp::Eltwise, h, {g, gs[i]}, n->rank, net_.ctx.fresh_id()), st_.of(n));
        }
        return g;
    }

    // Adjoint seeds from the scalar loss (SPEC.md:188-195 diff_scalar).
    void seed(const SPtr& s, double coef) {
        switch (s->kind) {
            case SKind::Const:
            case SKind::NamedConst: return;
            case SKind::Add: seed(s->args[0], coef); seed(s->args[1], coef); return;
            case SKind::Neg: seed(s->args[0], -coef); return;
            case SKind::Mul: {
                const SPtr& a = s->args[0];
                const SPtr& b = s->args[1];
                if (is_const(b)) return seed(a, coef * b->value);
                if (is_const(a)) return seed(b, coef * a->value);
                fail(ErrKind::NotDifferentiable, "product of two non-constant scalars in the loss");
            }
            case SKind::Div:
                if (!is_const(s->args[1])) fail(ErrKind::NotDifferentiable, "division by a non-constant scalar");
                return seed(s->args[0], coef / s->args[1]->value);
            case SKind::Dot: {
                auto one = [&](const TPtr& wrt_t, const TPtr& other) {
                    if (!req(wrt_t)) return;
                    Hyper h;
                    h.scale = coef;
                    TPtr g = reg(t_prim(PrimOp::Scale, h, {other}, other->rank, net_.ctx.fresh_id()), st_.of(other));
                    seeds_.insert(g.get());
                    contrib(wrt_t, g);
                };
                one(s->tensor2, s->tensor);
                one(s->tensor, s->tensor2);
                return;
            }
            default: fail(ErrKind::NotDifferentiable, "unsupported scalar form in the loss: " + to_string(s));
        }
    }
    static bool is_const(const SPtr& s) { return s->kind == SKind::Const || s->kind == SKind::NamedConst; }

    TPtr gp(const TPtr& n, int slot, std::vector<TPtr> saved, const TPtr& up, const TPtr& wrt_t) {
        const Shape& s = st_.of(wrt_t);
        TPtr g = t_grad_prim(n->prim, n->hyper, slot, std::move(saved), up, s.rank(), wrt(wrt_t), net_.ctx.fresh_id());
        return reg(g, s);
    }

    void backward(const TPtr& n, const TPtr& g) {
        const auto& op = n->operands;
        switch (n->kind) {
            case TKind::Flatten:
            case TKind::Reshape: {
                TPtr r = t_reshape(g, st_.of(op[0]));
                st_.t[r.get()] = st_.of(op[0]);
                contrib(op[0], r);
                return;
            }
            case TKind::Copy: contrib(op[0], g); return;
            case TKind::Concat: {
                std::int64_t off = 0;
                for (std::size_t i = 0; i < op.size(); ++i) {
                    const std::int64_t c = st_.of(op[i]).dims[1];
                    if (req(op[i])) {
                        // Concat backward = channel slice [off, off + c) of the upstream
                        Hyper h;
                        h.offset = off;
                        h.extent = c;
                        TPtr s = t_grad_prim(PrimOp::Concat, h, static_cast<int>(i), {}, g, 4, wrt(op[i]),
                                             net_.ctx.fresh_id());
                        contrib(op[i], reg(s, st_.of(op[i])));
                    }
                    off += c;
                }
                return;
            }
            case TKind::Prim: break;
            default: fail(ErrKind::NotDifferentiable, "no gradient rule for node " + n->display_name());
        }
        switch (n->prim) {
            case PrimOp::Convolv:
                // Creation order bias, data, filter: the data gradient reads W before
                // W's in-place update.
                if (n->hyper.has_bias && req(op[2])) contrib(op[2], gp(n, 2, {}, g, op[2]));
                if (req(op[0])) contrib(op[0], gp(n, 0, {op[1]}, g, op[0]));
                if (req(op[1])) contrib(op[1], gp(n, 1, {op[0]}, g, op[1]));
                return;
            case PrimOp::Pooling: contrib(op[0], gp(n, 0, {n, op[0]}, g, op[0])); return;
            // ReLU saves its output: Fig. 2 runs ReLU in place (X15 = ReLU()(X14), 0 bytes),
            // so the input no longer exists; [y > 0] == [x > 0].
            case PrimOp::ReLU: contrib(op[0], gp(n, 0, {n}, g, op[0])); return;
            case PrimOp::Softmax: contrib(op[0], gp(n, 0, {n}, g, op[0])); return;
            case PrimOp::LRN: contrib(op[0], gp(n, 0, {n, op[0]}, g, op[0])); return;
            case PrimOp::MatMul:
                if (req(op[0])) contrib(op[0], gp(n, 0, {op[1]}, g, op[0]));
                if (req(op[1])) contrib(op[1], gp(n, 1, {op[0]}, g, op[1]));
                return;
            case PrimOp::BiasAdd:
                if (req(op[1])) contrib(op[1], gp(n, 1, {}, g, op[1]));
                contrib(op[0], g);
                return;
            case PrimOp::BatchNorm:
                if (req(op[2])) contrib(op[2], gp(n, 2, {}, g, op[2]));
                if (req(op[0])) contrib(op[0], gp(n, 0, {op[0], op[1]}, g, op[0]));
                if (req(op[1])) contrib(op[1], gp(n, 1, {op[0]}, g, op[1]));
                return;
            case PrimOp::Eltwise:
                if (n->hyper.eltwise == ELT_ADD) {
                    contrib(op[0], g);
                    contrib(op[1], g);
                } else {
                    if (req(op[0])) contrib(op[0], gp(n, 0, {op[1]}, g, op[0]));
                    if (req(op[1])) contrib(op[1], gp(n, 1, {op[0]}, g, op[1]));
                }
                return;
            case PrimOp::Log: {
                // d log(x) = dx / x : the adjoint is g * (1/x)  (Fig. 2 "X52 = 1/(X19.copy)")
                TPtr r = reg(t_prim(PrimOp::Recip, Hyper{}, {op[0]}, n->rank, net_.ctx.fresh_id()), st_.of(op[0]));
                Hyper h;
                h.eltwise = ELT_MUL;
                contrib(op[0], reg(t_prim(PrimOp::Eltwise, h, {g, r}, n->rank, net_.ctx.fresh_id()), st_.of(op[0])));
                return;
            }
            case PrimOp::Scale: {
                Hyper h;
                h.scale = n->hyper.scale;
                contrib(op[0], reg(t_prim(PrimOp::Scale, h, {g}, n->rank, net_.ctx.fresh_id()), st_.of(op[0])));
                return;
            }
            default: fail(ErrKind::NotDifferentiable, std::string("no gradient rule for ") + prim_name(n->prim));
        }
    }

    NetworkDef& net_;
    ShapeTable& st_;
    GradInfo& gi_;
    std::unordered_map<const TensorExpr*, bool> req_;
    std::unordered_map<const TensorExpr*, std::vector<TPtr>> adj_;
    std::unordered_set<const TensorExpr*> seeds_;
};

}  // namespace

TPtr base_of(const TPtr& t) {
    TPtr b = t;
    while (b && (b->kind == TKind::Flatten || b->kind == TKind::Reshape || b->kind == TKind::Copy)) b = b->operands[0];
    return b;
}

GradInfo derive_gradients(NetworkDef& net, ShapeTable& st) {
    GradInfo gi;
    GradBuilder(net, st, gi).run();
    return gi;
}

// ================================================================ IR
namespace {

bool is_storage_node(const TPtr& t) {
    return t && t->kind != TKind::Param && t->kind != TKind::Input && !is_view(*t) && t->kind != TKind::Copy &&
           t->kind != TKind::RowBcast;
}

// Dependencies of a node in print order: GradPrim -> upstream, saved...; others -> operands.
std::vector<TPtr> ordered_deps(const TPtr& t) {
    if (t->kind == TKind::GradPrim) {
        std::vector<TPtr> d{t->upstream};
        d.insert(d.end(), t->saved.begin(), t->saved.end());
        return d;
    }
    return t->operands;
}

void loss_reads(const SPtr& s, std::vector<TPtr>& out) {
    if (!s) return;
    for (const auto& a : s->args) loss_reads(a, out);
    if (s->kind == SKind::Dot) {
        out.push_back(s->tensor);
        out.push_back(s->tensor2);
    }
}

bool inplace_capable(const TPtr& t) {
    if (t->kind == TKind::GradPrim) return t->prim == PrimOp::ReLU;
    if (t->kind != TKind::Prim) return false;
    switch (t->prim) {
        case PrimOp::Log:
        case PrimOp::Recip:
        case PrimOp::BiasAdd:
        case PrimOp::ReLU:
        case PrimOp::Scale: return true;
        case PrimOp::Eltwise: return t->hyper.eltwise == ELT_ADD;  // adjoint accumulation (Accum)
        default: return false;
    }
}

// Operand an in-place op overwrites.
TPtr inplace_target(const TPtr& t) { return t->kind == TKind::GradPrim ? t->upstream : t->operands[0]; }

}  // namespace

std::vector<int> stmt_reads(const IrStmt& s) {
    std::vector<int> out;
    auto add = [&](const TPtr& t) {
        TPtr b = base_of(t);
        if (is_storage_node(b)) out.push_back(b->id);
    };
    switch (s.kind) {
        case StmtKind::Let:
        case StmtKind::Update:
            for (const TPtr& d : ordered_deps(s.node)) add(d);
            break;
        case StmtKind::Print: {
            std::vector<TPtr> r;
            loss_reads(s.loss, r);
            for (const TPtr& t : r) add(t);
            break;
        }
        case StmtKind::Dealloc: break;
    }
    return out;
}

IrProgram compile_network(NetworkDef& net, const CompileOptions& opt) {
    vectorize(net, opt.cse);
    ShapeTable st;
    infer_shapes(net, st);
    GradInfo gi = derive_gradients(net, st);

    IrProgram p;
    p.name = net.name;
    p.batch = net.batch;
    p.classes = net.classes;
    p.input_shape = net.input_shape;
    p.solver = opt.solver;
    p.mode = opt.mode;
    p.workspace_cap_mb = opt.workspace_cap_mb;
    p.params = net.params;
    for (const auto& pp : p.params) p.param_shapes.push_back(st.of(pp.get()));

    // ---- to_ssa: forward Lets by post-order from the loss heads' softmax outputs,
    // then the labels, then the Log nodes (Fig. 2 order X7..X19, X20, X21).
    std::vector<TPtr> dots;
    loss_reads(net.loss, dots);
    std::vector<TPtr> roots;
    for (std::size_t i = 0; i + 1 < dots.size(); i += 2) roots.push_back(dots[i + 1]->operands[0]);
    roots.push_back(net.y_load);
    for (std::size_t i = 0; i + 1 < dots.size(); i += 2) roots.push_back(dots[i + 1]);
    std::vector<TPtr> order;
    std::unordered_set<const TensorExpr*> seen;
    std::function<void(const TPtr&)> dfs = [&](const TPtr& t) {
        if (!t || seen.count(t.get())) return;
        seen.insert(t.get());
        for (const TPtr& d : t->deps()) dfs(d);
        if (is_storage_node(t)) order.push_back(t);
    };
    for (const TPtr& r : roots) dfs(r);

    // ---- form_updates: param gradients are the Update right-hand sides.
    std::unordered_map<const TensorExpr*, ParamPtr> grad_root;
    for (auto& [pp, g] : gi.param_grads) grad_root[g.get()] = pp;

    std::vector<IrStmt> phaseF, phaseB;
    auto make_let = [&](const TPtr& t) {
        IrStmt s;
        s.kind = StmtKind::Let;
        s.node = t;
        s.var = t->id;
        s.shape = st.of(t);
        return s;
    };
    for (const TPtr& t : order) phaseF.push_back(make_let(t));
    for (const TPtr& t : gi.created) {
        if (!is_storage_node(t)) continue;
        auto gr = grad_root.find(t.get());
        if (gr != grad_root.end() && t->kind == TKind::GradPrim) {
            const ParamPtr& pp = gr->second;
            IrStmt u;
            u.kind = StmtKind::Update;
            u.node = t;
            u.param = pp;
            u.lr_alpha = -opt.solver.lr * pp->lr_mult;
            u.momentum = opt.solver.momentum;
            u.decay = opt.solver.decay * pp->decay_mult;
            phaseB.push_back(u);
            continue;
        }
        IrStmt s = make_let(t);
        if (gi.seed_dep[t.get()]) phaseB.push_back(s);
        else phaseF.push_back(s);
        if (gr != grad_root.end()) {  // summed parameter gradient: Update reads the sum
            IrStmt u;
            u.kind = StmtKind::Update;
            u.node = t;
            u.param = gr->second;
            u.lr_alpha = -opt.solver.lr * gr->second->lr_mult;
            u.momentum = opt.solver.momentum;
            u.decay = opt.solver.decay * gr->second->decay_mult;
            phaseB.push_back(u);
        }
    }
    std::vector<IrStmt> body = phaseF;
    {
        IrStmt pr;
        pr.kind = StmtKind::Print;
        pr.loss = net.loss;
        body.push_back(pr);
    }
    body.insert(body.end(), phaseB.begin(), phaseB.end());

    // ---- schedule.  Default: generation order, which is a
    // valid topological order and reproduces Fig. 2.  Optional greedy list
    // scheduler: among ready statements prefer the one that frees the most
    // bytes, then the smallest allocation, then generation order.
    if (opt.greedy_schedule) {
        const std::size_t n = body.size();
        std::unordered_map<int, std::size_t> def;
        for (std::size_t i = 0; i < n; ++i)
            if (body[i].kind == StmtKind::Let) def[body[i].var] = i;
        std::vector<std::vector<std::size_t>> preds(n);
        std::unordered_map<const ParamSpec*, std::vector<std::size_t>> param_readers;
        std::unordered_map<int, int> remaining_reads;
        for (std::size_t i = 0; i < n; ++i) {
            for (int v : stmt_reads(body[i])) {
                preds[i].push_back(def.at(v));
                remaining_reads[v]++;
            }
            const TPtr& nd = body[i].node;
            if (nd)
                for (const TPtr& d : nd->deps())
                    if (d->kind == TKind::Param && body[i].kind == StmtKind::Let) param_readers[d->param.get()].push_back(i);
        }
        for (std::size_t i = 0; i < n; ++i) {
            if (body[i].kind == StmtKind::Update)
                for (std::size_t r : param_readers[body[i].param.get()]) preds[i].push_back(r);
            if (body[i].kind == StmtKind::Print)  // the loss is printed before the backward pass starts
                for (std::size_t j = 0; j < i; ++j) preds[i].push_back(j);
        }
        std::vector<int> indeg(n, 0);
        std::vector<std::vector<std::size_t>> succ(n);
        for (std::size_t i = 0; i < n; ++i) {
            std::sort(preds[i].begin(), preds[i].end());
            preds[i].erase(std::unique(preds[i].begin(), preds[i].end()), preds[i].end());
            indeg[i] = static_cast<int>(preds[i].size());
            for (std::size_t q : preds[i]) succ[q].push_back(i);
        }
        std::vector<IrStmt> out;
        std::vector<bool> done(n, false);
        for (std::size_t step = 0; step < n; ++step) {
            std::size_t best = n;
            std::int64_t best_free = -1, best_alloc = 0;
            for (std::size_t i = 0; i < n; ++i) {
                if (done[i] || indeg[i] != 0) continue;
                std::int64_t freed = 0;
                for (int v : stmt_reads(body[i]))
                    if (remaining_reads[v] == 1) freed += body[def.at(v)].shape.bytes();
                const std::int64_t alloc = body[i].kind == StmtKind::Let ? body[i].shape.bytes() : 0;
                if (best == n || freed > best_free || (freed == best_free && alloc < best_alloc)) {
                    best = i;
                    best_free = freed;
                    best_alloc = alloc;
                }
            }
            if (best == n) fail(ErrKind::CycleDetected, "schedule: dependency cycle");
            done[best] = true;
            for (int v : stmt_reads(body[best])) remaining_reads[v]--;
            for (std::size_t q : succ[best]) indeg[q]--;
            out.push_back(body[best]);
        }
        body = std::move(out);
    }

    // ---- inline_inplace and storage assignment.
    std::unordered_map<int, int> storage_of;             // var -> storage
    std::unordered_map<int, std::int64_t> storage_bytes;
    std::unordered_map<int, std::size_t> last_read;      // var -> last statement index reading it
    for (std::size_t i = 0; i < body.size(); ++i)
        for (int v : stmt_reads(body[i])) last_read[v] = i;
    std::unordered_map<int, std::vector<int>> storage_vars;
    auto storage_last_use = [&](int stg) {
        std::size_t last = 0;
        for (int v : storage_vars[stg]) {
            auto it = last_read.find(v);
            if (it != last_read.end()) last = std::max(last, it->second);
        }
        return last;
    };
    for (std::size_t i = 0; i < body.size(); ++i) {
        IrStmt& s = body[i];
        if (s.kind != StmtKind::Let) continue;
        s.storage = s.var;
        s.bytes = s.shape.bytes();
        if (inplace_capable(s.node)) {
            TPtr tgt = base_of(inplace_target(s.node));
            if (is_storage_node(tgt) && storage_of.count(tgt->id)) {
                const int stg = storage_of[tgt->id];
                if (storage_last_use(stg) <= i && storage_bytes[stg] == s.shape.bytes()) {
                    s.inplace = true;
                    s.storage = stg;
                    s.bytes = 0;
                } else {
                    s.copy_operand = true;
                }
            }
        }
        storage_of[s.var] = s.storage;
        storage_vars[s.storage].push_back(s.var);
        if (!s.inplace) storage_bytes[s.storage] = s.shape.bytes();
    }

    // ---- insert_dealloc: free each storage right after its last use.
    std::vector<IrStmt> final_body;
    std::unordered_set<int> freed;
    for (std::size_t i = 0; i < body.size(); ++i) {
        final_body.push_back(body[i]);
        std::vector<int> cands = stmt_reads(body[i]);
        if (body[i].kind == StmtKind::Let) cands.push_back(body[i].var);
        for (int v : cands) {
            const int stg = storage_of.at(v);
            if (freed.count(stg)) continue;
            // last use of the storage (reads of any alias) and of its last alias definition
            std::size_t last = storage_last_use(stg);
            for (std::size_t j = 0; j < body.size(); ++j)
                if (body[j].kind == StmtKind::Let && storage_of[body[j].var] == stg) last = std::max(last, j);
            if (last != i) continue;
            freed.insert(stg);
            IrStmt d;
            d.kind = StmtKind::Dealloc;
            // name the most recent alias of the storage that this statement touched
            int shown = v;
            for (int a : storage_vars[stg])
                if (std::find(cands.begin(), cands.end(), a) != cands.end()) shown = a;
            d.var = shown;
            d.storage = stg;
            d.bytes = storage_bytes[stg];
            final_body.push_back(d);
        }
    }
    p.train = std::move(final_body);

    // ---- printable text (Fig. 2 surface syntax)
    for (IrStmt& s : p.train) {
        switch (s.kind) {
            case StmtKind::Let: {
                std::string rhs = to_string(s.node);
                if (s.copy_operand) {
                    TPtr tgt = base_of(inplace_target(s.node));
                    const std::string nm = tgt->display_name();
                    if (s.node->kind == TKind::Prim && s.node->prim == PrimOp::Log) rhs = "Log " + nm + ".copy";
                    else if (s.node->kind == TKind::Prim && s.node->prim == PrimOp::Recip) rhs = "1/(" + nm + ".copy)";
                    else {
                        const std::size_t pos = rhs.find(nm);
                        if (pos != std::string::npos) rhs.replace(pos, nm.size(), nm + ".copy");
                    }
                }
                s.text = "val X" + std::to_string(s.var) + " = " + rhs;
                break;
            }
            case StmtKind::Dealloc: s.text = "Dealloc(X" + std::to_string(s.var) + ")"; break;
            case StmtKind::Update: s.text = s.param->name + " <~~ " + to_string(s.node); break;
            case StmtKind::Print: s.text = "Print(" + to_string(s.loss) + ")"; break;
        }
    }
    for (const auto& [node, shp] : st.t)
        if (node->id >= 0) p.var_shapes[node->id] = shp;

    // ---- test body: forward Lets needed by the main logits (test-mode dropout = identity).
    {
        std::unordered_set<const TensorExpr*> need;
        postorder(net.logits_main, [&](const TPtr& t) { need.insert(t.get()); });
        for (const IrStmt& s : p.train)
            if (s.kind == StmtKind::Let && need.count(s.node.get())) p.test.push_back(s);
        p.logits_var = net.logits_main->id;
    }
    return p;
}

// ================================================================ memplan
namespace {
double mb(std::int64_t bytes) { return static_cast<double>(static_cast<float>(bytes) / 1e6f); }
}  // namespace

MemoryReport analyze(const IrProgram& p) {
    MemoryReport r;
    std::int64_t dealloc_total = 0, reuse_total = 0;
    std::multiset<std::int64_t> free_blocks;  // reuse-mode pool: blocks keyed by size
    for (const IrStmt& s : p.train) {
        MemoryRow row;
        row.stmt = s.text;
        std::int64_t delta = 0;
        switch (s.kind) {
            case StmtKind::Let:
                row.dims = s.shape.to_string();
                delta = s.bytes;
                if (delta > 0) {
                    // The paper's runtime-efficient pool hands back a released block
                    // of the same size; otherwise it allocates afresh (Fig. 2: X20
                    // reuses X18's 0.02 MB block, X72's 5.76 MB is fresh).
                    auto it = free_blocks.find(delta);
                    if (it != free_blocks.end()) free_blocks.erase(it);
                    else reuse_total += delta;
                }
                dealloc_total += delta;
                break;
            case StmtKind::Dealloc:
                delta = -s.bytes;
                dealloc_total -= s.bytes;
                free_blocks.insert(s.bytes);
                break;
            default: break;
        }
        r.peak_dealloc_bytes = std::max(r.peak_dealloc_bytes, dealloc_total);
        r.peak_reuse_bytes = std::max(r.peak_reuse_bytes, reuse_total);
        row.delta_mb = delta >= 0 ? mb(delta) : -mb(-delta);
        row.total_dealloc_mb = mb(dealloc_total);
        row.total_reuse_mb = mb(reuse_total);
        r.rows.push_back(row);
    }
    // static_memory
    for (const Shape& s : p.param_shapes) r.param_bytes += 2 * s.bytes();  // weights + velocities
    std::int64_t ws = 0;
    for (const IrStmt& s : p.train) {
        if (s.kind != StmtKind::Let || s.node->kind != TKind::Prim || s.node->prim != PrimOp::Convolv) continue;
        const TPtr& x = s.node->operands[0];
        const Shape& xs = p.var_shapes.at(base_of(x)->id);
        const std::int64_t k = s.node->hyper.k;
        ws = std::max(ws, 4 * xs.dims[0] * xs.dims[1] * k * k * s.shape.dims[2] * s.shape.dims[3]);
    }
    if (p.workspace_cap_mb >= 0) ws = std::min<std::int64_t>(ws, static_cast<std::int64_t>(p.workspace_cap_mb * 1e6));
    r.workspace_bytes = ws;
    return r;
}

std::string format_report(const MemoryReport& r, bool csv) {
    std::ostringstream os;
    char buf[512];
    if (csv) {
        os << "ir_expression,dimensions,current_mb,total_mb,wo_dealloc_mb\n";
        for (const auto& row : r.rows) {
            std::snprintf(buf, sizeof buf, "\"%s\",%s,%.6f,%.6f,%.6f\n", row.stmt.c_str(), row.dims.c_str(),
                          row.delta_mb, row.total_dealloc_mb, row.total_reuse_mb);
            os << buf;
        }
        return os.str();
    }
    std::snprintf(buf, sizeof buf, "%-46s %-14s %12s %12s %12s\n", "IR expression", "Dimensions", "Current mem", "Total",
                  "w/o dealloc");
    os << buf << std::string(100, '-') << "\n";
    for (const auto& row : r.rows) {
        std::snprintf(buf, sizeof buf, "%-46s %-14s %12.6f %12.6f %12.6f\n", row.stmt.c_str(), row.dims.c_str(),
                      row.delta_mb, row.total_dealloc_mb, row.total_reuse_mb);
        os << buf;
    }
    std::snprintf(buf, sizeof buf, "peak (dealloc) %.6f MB, peak (reuse) %.6f MB, params+velocities %.6f MB, workspace %.6f MB\n",
                  r.peak_dealloc_mb(), r.peak_reuse_mb(), static_cast<float>(r.param_bytes) / 1e6f,
                  static_cast<float>(r.workspace_bytes) / 1e6f);
    os << buf;
    return os.str();
}

std::string dump_ir(const IrProgram& p) {
    std::ostringstream os;
    for (const IrStmt& s : p.train) {
        os << s.text;
        if (s.kind == StmtKind::Let) os << "    # " << s.shape.to_string() << (s.inplace ? " (in place)" : "");
        os << "\n";
    }
    return os.str();
}

std::string verify(const IrProgram& p) {
    std::unordered_set<int> defined, dead;
    std::unordered_map<int, int> storage;
    std::unordered_map<int, std::size_t> last_use;
    for (std::size_t i = 0; i < p.train.size(); ++i)
        for (int v : stmt_reads(p.train[i])) last_use[v] = i;
    for (std::size_t i = 0; i < p.train.size(); ++i) {
        const IrStmt& s = p.train[i];
        for (int v : stmt_reads(s)) {
            if (!defined.count(v)) return "use before definition of X" + std::to_string(v) + " at: " + s.text;
            if (dead.count(storage[v])) return "use after dealloc of X" + std::to_string(v) + " at: " + s.text;
        }
        if (s.kind == StmtKind::Let) {
            if (!defined.insert(s.var).second) return "SSA violation: X" + std::to_string(s.var) + " assigned twice";
            storage[s.var] = s.storage;
        }
        if (s.kind == StmtKind::Dealloc) {
            if (dead.count(s.storage)) return "double dealloc of storage " + std::to_string(s.storage);
            dead.insert(s.storage);
            // must be immediately after the last use of every alias
            for (const auto& [v, stg] : storage) {
                if (stg != s.storage) continue;
                auto it = last_use.find(v);
                if (it != last_use.end() && it->second > i) return "dealloc before last use of X" + std::to_string(v);
            }
        }
    }
    return "";
}

}  // namespace tensorc
