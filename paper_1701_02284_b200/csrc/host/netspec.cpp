// Text network description parser + elaborator.  See netspec.hpp.
#include "host/netspec.hpp"

#include <cctype>
#include <map>
#include <memory>
#include <set>
#include <vector>

namespace tensorc {
namespace {

// ----------------------------------------------------------------- lexer
enum class Tok { Ident, Number, Punct, End };

struct Token {
    Tok kind = Tok::End;
    std::string text;
    double num = 0.0;
    SrcLoc loc;
};

std::vector<Token> lex(const std::string& src) {
    std::vector<Token> out;
    int line = 1, col = 1;
    std::size_t i = 0;
    auto adv = [&](std::size_t n) {
        for (std::size_t k = 0; k < n; ++k, ++i) {
            if (src[i] == '\n') {
                ++line;
                col = 1;
            } else {
                ++col;
            }
        }
    };
    while (i < src.size()) {
        const char c = src[i];
        if (c == '#') {
            while (i < src.size() && src[i] != '\n') adv(1);
            continue;
        }
        if (std::isspace(static_cast<unsigned char>(c)) || c == ';') {
            adv(1);
            continue;
        }
        Token t;
        t.loc = SrcLoc{line, col};
        const bool digit = std::isdigit(static_cast<unsigned char>(c)) != 0;
        const bool neg = c == '-' && i + 1 < src.size() && (std::isdigit(static_cast<unsigned char>(src[i + 1])) || src[i + 1] == '.');
        if (digit || neg || (c == '.' && i + 1 < src.size() && std::isdigit(static_cast<unsigned char>(src[i + 1])))) {
            std::size_t used = 0;
            t.num = std::stod(src.substr(i), &used);
            t.kind = Tok::Number;
            t.text = src.substr(i, used);
            adv(used);
        } else if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
            std::size_t j = i;
            while (j < src.size() && (std::isalnum(static_cast<unsigned char>(src[j])) || src[j] == '_')) ++j;
            t.kind = Tok::Ident;
            t.text = src.substr(i, j - i);
            adv(j - i);
        } else if (std::string("(){}=,.+*").find(c) != std::string::npos) {
            t.kind = Tok::Punct;
            t.text = std::string(1, c);
            adv(1);
        } else {
            fail(ErrKind::SyntaxError, t.loc, std::string("unexpected character '") + c + "'");
        }
        out.push_back(t);
    }
    Token e;
    e.loc = SrcLoc{line, col};
    out.push_back(e);
    return out;
}

// ----------------------------------------------------------------- AST
struct Value;
struct Arg {
    std::string key;  // "" = positional
    std::shared_ptr<Value> v;
};
struct Value {  // number | ident | call(args) | tuple
    enum Kind { Num, Id, Call, Tuple } kind = Num;
    double num = 0.0;
    std::string id;
    std::vector<Arg> args;
    SrcLoc loc;
};
struct Term {
    std::string id;
    bool call = false;
    std::vector<Arg> args;
    SrcLoc loc;
};
struct Decl {
    std::string name;
    SrcLoc loc;
    std::vector<Term> chain;                          // compose
    std::vector<std::pair<double, Term>> loss_terms;  // lossexpr: weight * logloss(ident)
    std::shared_ptr<Value> value;                     // data / solver keys
};
struct Section {
    std::string kind, name;
    SrcLoc loc;
    std::vector<Decl> decls;
};

class Parser {
public:
    explicit Parser(std::vector<Token> t) : t_(std::move(t)) {}

    std::vector<Section> file() {
        std::vector<Section> out;
        while (peek().kind != Tok::End) out.push_back(section());
        if (out.empty()) fail(ErrKind::SyntaxError, peek().loc, "expected a section (net | solver | data)");
        return out;
    }

private:
    const Token& peek(int k = 0) const { return t_[std::min(pos_ + k, t_.size() - 1)]; }
    bool is(const char* p, int k = 0) const { return peek(k).kind == Tok::Punct && peek(k).text == p; }
    Token take() { return t_[std::min(pos_++, t_.size() - 1)]; }
    Token expect_ident(const char* what) {
        if (peek().kind != Tok::Ident) fail(ErrKind::SyntaxError, peek().loc, std::string("expected ") + what);
        return take();
    }
    void expect(const char* p) {
        if (!is(p)) fail(ErrKind::SyntaxError, peek().loc, std::string("expected '") + p + "'");
        take();
    }

    Section section() {
        Section s;
        Token k = expect_ident("a section (net | solver | data)");
        if (k.text != "net" && k.text != "solver" && k.text != "data")
            fail(ErrKind::SyntaxError, k.loc, "expected a section (net | solver | data), got '" + k.text + "'");
        s.kind = k.text;
        s.loc = k.loc;
        if (peek().kind == Tok::Ident) s.name = take().text;
        expect("{");
        while (!is("}")) {
            if (peek().kind == Tok::End) fail(ErrKind::SyntaxError, peek().loc, "expected '}'");
            s.decls.push_back(decl(s.kind == "net"));
        }
        take();
        return s;
    }

    Decl decl(bool net) {
        Decl d;
        Token n = expect_ident("a declaration name");
        d.name = n.text;
        d.loc = n.loc;
        expect("=");
        if (!net) {
            d.value = value();
            return d;
        }
        const bool loss = (peek().kind == Tok::Ident && peek().text == "logloss") ||
                          (peek().kind == Tok::Number && is("*", 1));
        if (loss) {
            do {
                double w = 1.0;
                if (peek().kind == Tok::Number) {
                    w = take().num;
                    expect("*");
                }
                Token l = expect_ident("logloss");
                if (l.text != "logloss") fail(ErrKind::SyntaxError, l.loc, "expected logloss(...)");
                expect("(");
                Term t;
                t.loc = peek().loc;
                t.id = expect_ident("a network name").text;
                expect(")");
                d.loss_terms.emplace_back(w, t);
            } while (is("+") && (take(), true));
            return d;
        }
        d.chain.push_back(term());
        while (is(".")) {
            take();
            d.chain.push_back(term());
        }
        if (d.chain.empty()) fail(ErrKind::SyntaxError, peek().loc, "expected composition");
        return d;
    }

    Term term() {
        Term t;
        t.loc = peek().loc;
        t.id = expect_ident("a layer or network name").text;
        if (is("(")) {
            t.call = true;
            t.args = args();
        }
        return t;
    }

    std::vector<Arg> args() {
        std::vector<Arg> out;
        expect("(");
        if (is(")")) {
            take();
            return out;
        }
        for (;;) {
            Arg a;
            if (peek().kind == Tok::Ident && is("=", 1)) {
                a.key = take().text;
                take();
            }
            a.v = value();
            out.push_back(std::move(a));
            if (is(",")) {
                take();
                continue;
            }
            expect(")");
            return out;
        }
    }

    std::shared_ptr<Value> value() {
        auto v = std::make_shared<Value>();
        v->loc = peek().loc;
        if (peek().kind == Tok::Number) {
            v->kind = Value::Num;
            v->num = take().num;
        } else if (peek().kind == Tok::Ident) {
            v->id = take().text;
            v->kind = Value::Id;
            if (is("(")) {
                v->kind = Value::Call;
                v->args = args();
            }
        } else if (is("(")) {
            v->kind = Value::Tuple;
            v->args = args();
        } else {
            fail(ErrKind::SyntaxError, v->loc, "expected a value");
        }
        return v;
    }

    std::vector<Token> t_;
    std::size_t pos_ = 0;
};

// ----------------------------------------------------------------- elaboration
const std::set<std::string> kLayerKinds = {"conv", "maxpool", "avgpool", "relu", "full", "flatten", "softmax",
                                           "dropout", "lrn", "concat", "batchnorm", "residual"};

class Elaborator {
public:
    Elaborator(NetworkDef& net, std::int64_t classes) : net_(net), L_(net), classes_(classes) {}

    void declare(const Decl& d) {
        if (funs_.count(d.name) || losses_.count(d.name)) fail(ErrKind::DuplicateName, d.loc, "'" + d.name + "' declared twice");
        if (!d.loss_terms.empty()) {
            losses_[d.name] = d;
            loss_order_.push_back(d.name);
            return;
        }
        if (d.chain.size() == 1) {
            const Term& t = d.chain[0];
            if (t.call || (kLayerKinds.count(t.id) && !funs_.count(t.id))) {
                funs_[d.name] = layer(t, d.name);
            } else {
                funs_[d.name] = lookup(t);  // alias
                if (chains_.count(t.id)) chains_[d.name] = chains_[t.id];
            }
            return;
        }
        // composition t1 . t2 . ... . tn, left associative; when the first-applied term is
        // itself a composition, its application is shared (applied once per input, see apply())
        std::vector<FunPtr> fs;
        for (std::size_t i = 0; i < d.chain.size(); ++i)
            fs.push_back(d.chain[i].call || (kLayerKinds.count(d.chain[i].id) && !funs_.count(d.chain[i].id))
                             ? layer(d.chain[i], d.name + "_" + std::to_string(i))
                             : lookup(d.chain[i]));
        const Term& last = d.chain.back();
        Chain ch;
        if (!last.call && chains_.count(last.id)) {
            ch.inner = last.id;
            fs.pop_back();
        }
        FunPtr f = fs[0];
        for (std::size_t i = 1; i < fs.size(); ++i) f = L_.compose(f, fs[i]);
        ch.head = f;
        chains_[d.name] = ch;
        funs_[d.name] = ch.inner.empty() ? f : nullptr;
    }

    // logits of a network name applied to the loaded input (shared prefixes applied once)
    TPtr apply(const std::string& name, const SrcLoc& loc) {
        auto hit = applied_.find(name);
        if (hit != applied_.end()) return hit->second;
        TPtr out;
        auto ch = chains_.find(name);
        if (ch != chains_.end() && !ch->second.inner.empty()) {
            TPtr in = apply(ch->second.inner, loc);
            out = normalize(net_.ctx, t_apply(ch->second.head, in));
        } else {
            auto f = funs_.find(name);
            if (f == funs_.end() || !f->second) fail(ErrKind::UnboundName, loc, "unknown network '" + name + "'");
            out = normalize(net_.ctx, t_apply(f->second, net_.x_load));
        }
        applied_[name] = out;
        return out;
    }

    void finish() {
        if (loss_order_.empty()) fail(ErrKind::SyntaxError, SrcLoc{}, "the net section needs a loss = logloss(...) declaration");
        if (loss_order_.size() > 1)
            fail(ErrKind::DuplicateName, losses_[loss_order_[1]].loc, "exactly one loss expression is allowed");
        const Decl& d = losses_[loss_order_[0]];
        net_.x_load = t_load(t_input("X", 4), net_.ctx.fresh_id());
        std::vector<TPtr> soft;
        FunPtr softmax = L_.softmax();
        for (const auto& [w, t] : d.loss_terms) {
            TPtr logits = apply(t.id, t.loc);
            if (!net_.logits_main) net_.logits_main = logits;
            soft.push_back(normalize(net_.ctx, t_apply(softmax, logits)));
        }
        net_.y_load = t_load_indicator(t_input("Y", 1), net_.classes, net_.ctx.fresh_id());
        SPtr loss;
        for (std::size_t i = 0; i < soft.size(); ++i) {
            const double w = d.loss_terms[i].first;
            SPtr l = L_.log_loss(soft[i], w, w == 1.0 ? "" : "loss" + std::to_string(i));
            loss = loss ? s_add(loss, l) : l;
        }
        net_.loss = loss;
        net_.params = free_params_scalar(net_.loss);
    }

private:
    struct Chain {
        FunPtr head;
        std::string inner;  // first-applied composition whose application is shared
    };

    FunPtr lookup(const Term& t) {
        auto f = funs_.find(t.id);
        if (f == funs_.end()) fail(ErrKind::UnboundName, t.loc, "unknown name '" + t.id + "'");
        if (!f->second) fail(ErrKind::ArityError, t.loc, "'" + t.id + "' is a network with a shared prefix; use it first-applied");
        return f->second;
    }

    // positional / keyword argument access
    struct Args {
        const std::vector<Arg>& a;
        const SrcLoc& loc;
        const std::string& kind;
        std::int64_t classes;
        std::set<std::string> used;
        const Value* get(const std::string& key, std::size_t pos) {
            for (const Arg& x : a)
                if (x.key == key) {
                    used.insert(key);
                    return x.v.get();
                }
            std::size_t k = 0;
            for (const Arg& x : a) {
                if (!x.key.empty()) continue;
                if (k++ == pos) return x.v.get();
            }
            return nullptr;
        }
        double num(const std::string& key, std::size_t pos, double dflt, bool required = false) {
            const Value* v = get(key, pos);
            if (!v) {
                if (required) fail(ErrKind::ArityError, loc, kind + ": missing argument '" + key + "'");
                return dflt;
            }
            if (v->kind == Value::Id && v->id == "K") return static_cast<double>(classes);
            if (v->kind != Value::Num) fail(ErrKind::SyntaxError, v->loc, kind + ": '" + key + "' must be a number");
            return v->num;
        }
        std::size_t positional() const {
            std::size_t n = 0;
            for (const Arg& x : a) n += x.key.empty();
            return n;
        }
    };

    static ParamInit init_of(const Value* v, ParamInit dflt) {
        if (!v) return dflt;
        if (v->kind == Value::Id && v->id == "xavier") return ParamInit::xavier();
        auto arg = [&](std::size_t i, double d) {
            if (i >= v->args.size()) return d;
            const Value& a = *v->args[i].v;
            if (a.kind != Value::Num) fail(ErrKind::SyntaxError, a.loc, "initialiser arguments must be numbers");
            return a.num;
        };
        if (v->kind == Value::Call && (v->id == "const" || v->id == "constant"))
            return ParamInit::constant(arg(0, 0.0), arg(1, 1.0), arg(2, 1.0));
        if (v->kind == Value::Call && v->id == "gaussian") {
            ParamInit p;
            p.kind = InitKind::Gaussian;
            p.sigma = arg(0, 0.01);
            p.lr_mult = arg(1, 1.0);
            p.decay_mult = arg(2, 1.0);
            return p;
        }
        fail(ErrKind::SyntaxError, v->loc, "unknown initialiser (xavier | const(v, lrm, dcm) | gaussian(sigma, lrm, dcm))");
    }

    FunPtr branch(const Value* v, const std::string& pname) {
        if (!v) return nullptr;
        if (v->kind == Value::Id) {
            Term t;
            t.id = v->id;
            t.loc = v->loc;
            return kLayerKinds.count(v->id) && !funs_.count(v->id) ? layer(t, pname) : lookup(t);
        }
        if (v->kind == Value::Call) {
            Term t;
            t.id = v->id;
            t.call = true;
            t.args = v->args;
            t.loc = v->loc;
            return layer(t, pname);
        }
        fail(ErrKind::SyntaxError, v->loc, "expected a layer or network");
    }

    FunPtr layer(const Term& t, const std::string& name) {
        if (!kLayerKinds.count(t.id)) fail(ErrKind::UnknownLayerKind, t.loc, "unknown layer kind '" + t.id + "'");
        Args A{t.args, t.loc, t.id, classes_, {}};
        const std::string& k = t.id;
        if (k == "conv") {
            const int kk = static_cast<int>(A.num("k", 0, 0, true));
            const auto out = static_cast<std::int64_t>(A.num("out", 1, 0, true));
            const int stride = static_cast<int>(A.num("stride", 2, 1));
            const int pad = static_cast<int>(A.num("pad", 3, 0));
            const ParamInit w = init_of(A.get("w", 99), ParamInit::xavier());
            const ParamInit b = init_of(A.get("b", 99), ParamInit::constant(0.0));
            const bool bias = A.num("bias", 99, 1) != 0;
            return L_.convolv(name, kk, out, stride, pad, w, b, bias);
        }
        if (k == "maxpool" || k == "avgpool") {
            const int kk = static_cast<int>(A.num("k", 0, 0, true));
            const int stride = static_cast<int>(A.num("stride", 1, kk));
            const int pad = static_cast<int>(A.num("pad", 2, 0));
            return k == "maxpool" ? L_.max_pool(kk, stride, pad) : L_.avg_pool(kk, stride, pad);
        }
        if (k == "relu") return L_.relu(static_cast<int>(A.num("rank", 0, 4)));
        if (k == "softmax") return L_.softmax();
        if (k == "full") {
            const auto out = static_cast<std::int64_t>(A.num("out", 0, 0, true));
            return L_.full(name, out, init_of(A.get("w", 1), ParamInit::xavier()), init_of(A.get("b", 2), ParamInit::constant(0.0)));
        }
        if (k == "flatten") return L_.flatten(static_cast<int>(A.num("rank", 0, 4)), static_cast<int>(A.num("axis", 1, 1)));
        if (k == "dropout") return L_.dropout(A.num("rate", 0, 0.5, true), static_cast<int>(A.num("rank", 1, 2)));
        if (k == "lrn")
            return L_.lrn(static_cast<int>(A.num("size", 0, 5)), A.num("alpha", 1, 1e-4), A.num("beta", 2, 0.75));
        if (k == "batchnorm") return L_.batchnorm(name);
        if (k == "concat") {
            if (t.args.size() < 2) fail(ErrKind::ArityError, t.loc, "concat needs at least two branches");
            std::vector<FunPtr> bs;
            for (std::size_t i = 0; i < t.args.size(); ++i) bs.push_back(branch(t.args[i].v.get(), name + "_" + std::to_string(i)));
            return L_.concat(bs);
        }
        if (k == "residual") {
            if (t.args.empty() || t.args.size() > 2) fail(ErrKind::ArityError, t.loc, "residual(branch[, shortcut])");
            return L_.residual(branch(t.args[0].v.get(), name + "_b"),
                               t.args.size() > 1 ? branch(t.args[1].v.get(), name + "_s") : nullptr);
        }
        fail(ErrKind::UnknownLayerKind, t.loc, "unknown layer kind '" + k + "'");
    }

    NetworkDef& net_;
    LayerFactory L_;
    std::int64_t classes_;
    std::map<std::string, FunPtr> funs_;
    std::map<std::string, Chain> chains_;
    std::map<std::string, Decl> losses_;
    std::vector<std::string> loss_order_;
    std::map<std::string, TPtr> applied_;
};

double num_value(const Decl& d) {
    if (d.value->kind != Value::Num) fail(ErrKind::SyntaxError, d.value->loc, "'" + d.name + "' must be a number");
    return d.value->num;
}

}  // namespace

void build_from_spec(NetworkDef& net, const std::string& text, std::int64_t batch, SpecSolver* solver) {
    std::vector<Section> secs = Parser(lex(text)).file();
    SpecSolver sv;
    std::int64_t C = 0, H = 0, W = 0, K = 0, N = 0;
    const Section* netsec = nullptr;
    for (const Section& s : secs) {
        if (s.kind == "net") {
            if (netsec) fail(ErrKind::DuplicateName, s.loc, "more than one net section");
            netsec = &s;
            continue;
        }
        std::set<std::string> seen;
        for (const Decl& d : s.decls) {
            if (!seen.insert(d.name).second) fail(ErrKind::DuplicateName, d.loc, "'" + d.name + "' declared twice");
            if (s.kind == "solver") {
                const double v = num_value(d);
                if (d.name == "lr") sv.lr = v;
                else if (d.name == "momentum") sv.momentum = v;
                else if (d.name == "decay") sv.decay = v;
                else if (d.name == "clip") sv.clip = v;
                else if (d.name == "iters") sv.iters = static_cast<std::int64_t>(v);
                else if (d.name == "test_iters") sv.test_iters = static_cast<std::int64_t>(v);
                else if (d.name == "snapshot_every") sv.snapshot_every = static_cast<std::int64_t>(v);
                else fail(ErrKind::SyntaxError, d.loc, "unknown solver key '" + d.name + "'");
            } else {  // data
                if (d.name == "batch") N = static_cast<std::int64_t>(num_value(d));
                else if (d.name == "classes") K = static_cast<std::int64_t>(num_value(d));
                else if (d.name == "shape") {
                    const Value& v = *d.value;
                    if (v.kind != Value::Tuple || v.args.size() != 3) fail(ErrKind::SyntaxError, v.loc, "shape = (C, H, W)");
                    std::int64_t* dst[3] = {&C, &H, &W};
                    for (int i = 0; i < 3; ++i) {
                        if (v.args[i].v->kind != Value::Num) fail(ErrKind::SyntaxError, v.args[i].v->loc, "shape entries are numbers");
                        *dst[i] = static_cast<std::int64_t>(v.args[i].v->num);
                    }
                } else if (d.name == "source") {
                    const Value& v = *d.value;
                    if (v.kind == Value::Call && v.id == "synthetic") {
                        if (!v.args.empty() && v.args[0].v->kind == Value::Num) sv.seed = static_cast<std::uint64_t>(v.args[0].v->num);
                    } else {
                        fail(ErrKind::SyntaxError, v.loc, "data source: only synthetic(seed) is available (IDX ingestion is out of scope)");
                    }
                } else {
                    fail(ErrKind::SyntaxError, d.loc, "unknown data key '" + d.name + "'");
                }
            }
        }
    }
    if (!netsec) fail(ErrKind::SyntaxError, SrcLoc{}, "missing net section");
    if (batch > 0) N = batch;
    if (N < 1) fail(ErrKind::NonPositiveExtent, SrcLoc{}, "data batch must be >= 1");
    if (K < 2) fail(ErrKind::NonPositiveExtent, SrcLoc{}, "data classes must be >= 2");
    if (C < 1 || H < 1 || W < 1) fail(ErrKind::NonPositiveExtent, SrcLoc{}, "data shape = (C, H, W) with positive extents");
    if (!(sv.lr > 0) || sv.momentum < 0 || sv.momentum >= 1 || sv.decay < 0 || sv.clip < 0)
        fail(ErrKind::SyntaxError, SrcLoc{}, "solver: lr > 0, 0 <= momentum < 1, decay >= 0, clip >= 0 (SPEC.md:36)");
    net.name = netsec->name.empty() ? "net" : netsec->name;
    net.batch = N;
    net.input_shape = Shape{N, C, H, W};
    net.classes = K;
    Elaborator el(net, K);
    for (const Decl& d : netsec->decls) el.declare(d);
    el.finish();
    if (solver) *solver = sv;
}

}  // namespace tensorc
