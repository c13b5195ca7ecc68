// Layer templates and the configured networks.  See nets.hpp.
#include "host/nets.hpp"

#include <cmath>

namespace tensorc {

namespace {
int index_var_counter = 1000;  // index-variable ids live in their own namespace
}

ParamPtr LayerFactory::param(const std::string& name, const ParamInit& init, int rank) {
    auto p = std::make_shared<ParamSpec>();
    p->name = name;
    p->init = init.kind;
    p->init_value = init.value;
    p->sigma = init.sigma;
    p->lr_mult = init.lr_mult;
    p->decay_mult = init.decay_mult;
    p->rank = rank;
    return p;
}

FunPtr LayerFactory::convolv(const std::string& name, int k, std::int64_t out, int stride, int pad, ParamInit w,
                             ParamInit b, bool has_bias) {
    TPtr v = t_var(-1, 4);
    Hyper h;
    h.k = k;
    h.stride = stride;
    h.pad = pad;
    h.out = out;
    h.has_bias = has_bias;
    std::vector<TPtr> ops{v, t_param(param(name + "_W", w, 4), 4)};
    if (has_bias) ops.push_back(t_param(param(name + "_B", b, 1), 1));
    return fun_of(v, t_prim(PrimOp::Convolv, h, ops, 4, -1), name);
}

FunPtr LayerFactory::max_pool(int k, int stride, int pad) {
    TPtr v = t_var(-1, 4);
    Hyper h;
    h.k = k;
    h.stride = stride < 0 ? k : stride;
    h.pad = pad;
    h.max_pool = true;
    return fun_of(v, t_prim(PrimOp::Pooling, h, {v}, 4, -1), "max_pool");
}

FunPtr LayerFactory::avg_pool(int k, int stride, int pad) {
    TPtr v = t_var(-1, 4);
    Hyper h;
    h.k = k;
    h.stride = stride < 0 ? k : stride;
    h.pad = pad;
    h.max_pool = false;
    return fun_of(v, t_prim(PrimOp::Pooling, h, {v}, 4, -1), "avg_pool");
}

FunPtr LayerFactory::relu(int rank) {
    TPtr v = t_var(-1, rank);
    Hyper h;
    h.rank = rank;
    return fun_of(v, t_prim(PrimOp::ReLU, h, {v}, rank, -1), "relu");
}

FunPtr LayerFactory::softmax() {
    TPtr v = t_var(-1, 2);
    Hyper h;
    h.rank = 2;
    return fun_of(v, t_prim(PrimOp::Softmax, h, {v}, 2, -1), "softmax");
}

FunPtr LayerFactory::lrn(int size, double alpha, double beta) {
    TPtr v = t_var(-1, 4);
    Hyper h;
    h.lrn_size = size;
    h.alpha = alpha;
    h.beta = beta;
    return fun_of(v, t_prim(PrimOp::LRN, h, {v}, 4, -1), "lrn");
}

FunPtr LayerFactory::dropout(double rate, int rank) {
    // y = x * M with M an explicit IR value: inverted-dropout
    // mask holding 0 or 1/(1-rate), drawn from a counter RNG.
    TPtr v = t_var(-1, rank);
    Hyper hm;
    hm.rate = rate;
    TPtr mask = t_prim(PrimOp::DropoutMask, hm, {v}, rank, -1);
    Hyper hy;
    hy.eltwise = ELT_MUL;
    return fun_of(v, t_prim(PrimOp::Eltwise, hy, {v, mask}, rank, -1), "dropout");
}

FunPtr LayerFactory::flatten(int rank, int axis) {
    TPtr v = t_var(-1, rank);
    return fun_of(v, t_flatten(v, axis), "flatten");
}

FunPtr LayerFactory::full(const std::string& name, std::int64_t out, ParamInit w, ParamInit b) {
    // Fig. 2 form: X12 = (X11[1><3])(i | @) * (fc1_W)(j | @); X14 = (X12 + (i) => fc1_B)
    // i.e. IndexAbs[i,j] Sum_k v(i,k) * W(j,k), then a row-broadcast bias add.
    // vectorize() turns these into MatMul / BiasAdd.
    TPtr v = t_var(-1, 2);
    TPtr W = t_param(param(name + "_W", w, 2), 2);
    TPtr B = t_param(param(name + "_B", b, 1), 1);
    const int i = index_var_counter++, j = index_var_counter++, k = index_var_counter++;
    SPtr body = s_sum(k, W, 1, s_mul(s_elem(v, {s_ivar(i), s_ivar(k)}), s_elem(W, {s_ivar(j), s_ivar(k)})));
    auto mm = std::make_shared<TensorExpr>(*t_index_abs({i, j}, body, 2, -1));
    mm->hyper.out = out;
    TPtr rb = t_row_bcast(i, B, -1);
    return fun_of(v, t_add(mm, rb, -1), name);
}

FunPtr LayerFactory::batchnorm(const std::string& name) {
    TPtr v = t_var(-1, 4);
    Hyper h;
    h.eps = 1e-5;
    TPtr g = t_param(param(name + "_G", ParamInit::constant(1.0, 1.0, 0.0), 1), 1);
    TPtr b = t_param(param(name + "_Bt", ParamInit::constant(0.0, 1.0, 0.0), 1), 1);
    return fun_of(v, t_prim(PrimOp::BatchNorm, h, {v, g, b}, 4, -1), name);
}

FunPtr LayerFactory::concat(const std::vector<FunPtr>& branches) {
    TPtr v = t_var(-1, 4);
    std::vector<TPtr> parts;
    for (const auto& b : branches) parts.push_back(t_apply(b, v));
    return fun_of(v, t_concat(parts, -1), "concat");
}

FunPtr LayerFactory::residual(const FunPtr& branch, const FunPtr& shortcut) {
    TPtr v = t_var(-1, 4);
    TPtr a = t_apply(branch, v);
    TPtr s = shortcut ? t_apply(shortcut, v) : v;
    Hyper h;
    h.eltwise = ELT_ADD;
    TPtr sum = t_prim(PrimOp::Eltwise, h, {a, s}, 4, -1);
    Hyper hr;
    hr.rank = 4;
    return fun_of(v, t_prim(PrimOp::ReLU, hr, {sum}, 4, -1), "residual");
}

FunPtr LayerFactory::seq(const std::vector<FunPtr>& fs) {
    const int rank = fs.empty() ? 4 : fs.front()->bound->rank;
    TPtr v = t_var(-1, rank);
    TPtr cur = v;
    for (const auto& f : fs) cur = t_apply(f, cur);
    return fun_of(v, cur, "seq");
}

SPtr LayerFactory::log_loss(const TPtr& softmax_out, double weight, const std::string& weight_name) {
    // (0 - (Y . Log S)) / |N|; Log gets the next SSA number.
    TPtr logs = t_prim(PrimOp::Log, Hyper{}, {softmax_out}, 2, net_.ctx.fresh_id());
    SPtr l = s_div(s_add(s_const(0.0), s_neg(s_dot(net_.y_load, logs))),
                   s_card(net_.loss_card > 0 ? net_.loss_card : net_.batch));
    if (!weight_name.empty()) l = s_mul(l, s_named(weight, weight_name));
    return l;
}

// ================================================================= networks
namespace {

void init_net(NetworkDef& net, const std::string& name, std::int64_t batch, Shape in, std::int64_t classes) {
    net.name = name;
    net.batch = batch;
    net.input_shape = std::move(in);
    net.classes = classes;
}

TPtr apply_norm(NetworkDef& net, const FunPtr& f, const TPtr& x) { return normalize(net.ctx, t_apply(f, x)); }

void finish(NetworkDef& net) { net.params = free_params_scalar(net.loss); }

}  // namespace

// Fig. 1.  Seven compositions draw X0..X6, Cuda(X) is X7,
// normalisation numbers the network X8..X19 and the loss head X20, X21.
void build_lenet(NetworkDef& net, std::int64_t batch) {
    init_net(net, "lenet", batch, Shape{batch, 1, 28, 28}, 10);
    LayerFactory L(net);
    FunPtr cv1 = L.convolv("cv1", 5, 20);
    FunPtr cv2 = L.convolv("cv2", 5, 50);
    FunPtr mp = L.max_pool(2);
    FunPtr flat = L.flatten(4, 1);
    FunPtr f = L.full("fc1", 500);
    FunPtr f2 = L.full("fc2", net.classes);
    FunPtr relu = L.relu(2);
    FunPtr softmax = L.softmax();
    // f2 o relu o f o flat o mp o cv2 o mp o cv1, left associative
    FunPtr network = L.compose(L.compose(L.compose(L.compose(L.compose(L.compose(L.compose(f2, relu), f), flat), mp), cv2), mp), cv1);
    net.x_load = t_load(t_input("X", 4), net.ctx.fresh_id());
    TPtr logits = apply_norm(net, network, net.x_load);
    TPtr s = apply_norm(net, softmax, logits);
    net.logits_main = logits;
    net.y_load = t_load_indicator(t_input("Y", 1), net.classes, net.ctx.fresh_id());
    net.loss = L.log_loss(s, 1.0, "");
    finish(net);
}

// AlexNet per PAPER.md:168-175 with Caffe bvlc_alexnet hyper-parameters, no
// conv groups, floor pooling at 224 input.
void build_alexnet(NetworkDef& net, std::int64_t batch) {
    init_net(net, "alexnet", batch, Shape{batch, 3, 224, 224}, 1000);
    LayerFactory L(net);
    auto b01 = ParamInit::constant(0.1);
    FunPtr cv1 = L.convolv("cv1", 11, 96, 4, 0);
    FunPtr cv2 = L.convolv("cv2", 5, 256, 1, 2, ParamInit::xavier(), b01);
    FunPtr cv3 = L.convolv("cv3", 3, 384, 1, 1);
    FunPtr cv4 = L.convolv("cv4", 3, 384, 1, 1, ParamInit::xavier(), b01);
    FunPtr cv5 = L.convolv("cv5", 3, 256, 1, 1, ParamInit::xavier(), b01);
    FunPtr full6 = L.full("fc6", 4096, ParamInit::xavier(), b01);
    FunPtr full7 = L.full("fc7", 4096, ParamInit::xavier(), b01);
    FunPtr full8 = L.full("fc8", net.classes);
    FunPtr relu = L.relu(4), relu2 = L.relu(2);
    FunPtr pool = L.max_pool(3, 2);
    FunPtr lrn = L.lrn(5, 1e-4, 0.75);
    FunPtr drop = L.dropout(0.5, 2);
    FunPtr flat = L.flatten(4, 1);
    FunPtr network = L.seq({cv1, relu, lrn, pool, cv2, relu, lrn, pool, cv3, relu, cv4, relu, cv5, relu, pool, flat,
                            full6, relu2, drop, full7, relu2, drop, full8});
    net.x_load = t_load(t_input("X", 4), net.ctx.fresh_id());
    TPtr logits = apply_norm(net, network, net.x_load);
    TPtr s = apply_norm(net, L.softmax(), logits);
    net.logits_main = logits;
    net.y_load = t_load_indicator(t_input("Y", 1), net.classes, net.ctx.fresh_id());
    net.loss = L.log_loss(s, 1.0, "");
    finish(net);
}

void build_vgg16(NetworkDef& net, std::int64_t batch) {
    init_net(net, "vgg16", batch, Shape{batch, 3, 224, 224}, 1000);
    LayerFactory L(net);
    FunPtr relu = L.relu(4), relu2 = L.relu(2), pool = L.max_pool(2, 2);
    std::vector<FunPtr> layers;
    const int cfg[5][2] = {{64, 2}, {128, 2}, {256, 3}, {512, 3}, {512, 3}};
    for (int s = 0; s < 5; ++s) {
        for (int i = 0; i < cfg[s][1]; ++i) {
            layers.push_back(L.convolv("conv" + std::to_string(s + 1) + "_" + std::to_string(i + 1), 3, cfg[s][0], 1, 1));
            layers.push_back(relu);
        }
        layers.push_back(pool);
    }
    FunPtr drop = L.dropout(0.5, 2);
    layers.push_back(L.flatten(4, 1));
    layers.push_back(L.full("fc6", 4096));
    layers.push_back(relu2);
    layers.push_back(drop);
    layers.push_back(L.full("fc7", 4096));
    layers.push_back(relu2);
    layers.push_back(drop);
    layers.push_back(L.full("fc8", net.classes));
    net.x_load = t_load(t_input("X", 4), net.ctx.fresh_id());
    TPtr logits = apply_norm(net, L.seq(layers), net.x_load);
    TPtr s = apply_norm(net, L.softmax(), logits);
    net.logits_main = logits;
    net.y_load = t_load_indicator(t_input("Y", 1), net.classes, net.ctx.fresh_id());
    net.loss = L.log_loss(s, 1.0, "");
    finish(net);
}

namespace {
struct InceptionCfg {
    const char* tag;
    int c1, r3, c3, r5, c5, pp;
};
const InceptionCfg kInception[9] = {
    {"3a", 64, 96, 128, 16, 32, 32},    {"3b", 128, 128, 192, 32, 96, 64},  {"4a", 192, 96, 208, 16, 48, 64},
    {"4b", 160, 112, 224, 24, 64, 64},  {"4c", 128, 128, 256, 24, 64, 64},  {"4d", 112, 144, 288, 32, 64, 64},
    {"4e", 256, 160, 320, 32, 128, 128}, {"5a", 256, 160, 320, 32, 128, 128}, {"5b", 384, 192, 384, 48, 128, 128},
};

// PAPER.md:192-213 inception(n): four branches concatenated; biases const 0.2
// with lr/decay multipliers (2, 0) ("b02 = Param.const(0.2f, 2, 0)").
FunPtr inception(LayerFactory& L, int n, const InceptionCfg& c, const FunPtr& relu) {
    auto b02 = ParamInit::constant(0.2, 2.0, 0.0);
    auto w = ParamInit::xavier();
    const std::string p = "cv" + std::to_string(n);
    FunPtr icv1 = L.convolv(p + "1", 1, c.c1, 1, 0, w, b02);
    FunPtr icv2 = L.convolv(p + "2", 1, c.r3, 1, 0, w, b02);
    FunPtr icv3 = L.convolv(p + "3", 3, c.c3, 1, 1, w, b02);
    FunPtr icv4 = L.convolv(p + "4", 1, c.r5, 1, 0, w, b02);
    FunPtr icv5 = L.convolv(p + "5", 5, c.c5, 1, 2, w, b02);
    FunPtr icv6 = L.convolv(p + "6", 1, c.pp, 1, 0, w, b02);
    FunPtr ipool = L.max_pool(3, 1, 1);
    return L.concat({L.seq({icv1, relu}), L.seq({icv2, relu, icv3, relu}), L.seq({icv4, relu, icv5, relu}),
                     L.seq({ipool, icv6, relu})});
}
}  // namespace

// GoogLeNet per PAPER.md:215-240 (three loss heads, aux weight 0.3) with the
// Caffe bvlc_googlenet channel table; stride-2 max-pools use pad 1 so floor
// pooling reproduces Caffe's ceil shapes 112->56->28->14->7.
void build_googlenet(NetworkDef& net, std::int64_t batch) {
    init_net(net, "googlenet", batch, Shape{batch, 3, 224, 224}, 1000);
    LayerFactory L(net);
    auto b02 = ParamInit::constant(0.2, 2.0, 0.0);
    auto b0 = ParamInit::constant(0.0, 2.0, 0.0);
    auto w = ParamInit::xavier();
    FunPtr relu = L.relu(4), relu2 = L.relu(2);
    FunPtr pool = L.max_pool(3, 2, 1);
    FunPtr lrn = L.lrn(5, 1e-4, 0.75);
    FunPtr cv1 = L.convolv("cv1", 7, 64, 2, 3, w, b02);
    FunPtr cv2 = L.convolv("cv2", 1, 64, 1, 0, w, b02);
    FunPtr cv3 = L.convolv("cv3", 3, 192, 1, 1, w, b02);
    std::vector<FunPtr> inc;
    for (int i = 0; i < 9; ++i) inc.push_back(inception(L, i + 1, kInception[i], relu));
    FunPtr network1 = L.seq({cv1, relu, pool, lrn, cv2, relu, cv3, relu, lrn, pool, inc[0], inc[1], pool, inc[2]});
    FunPtr network2 = L.seq({inc[3], inc[4], inc[5]});
    FunPtr network3 = L.seq({inc[6], pool, inc[7], inc[8], L.avg_pool(7, 1), L.dropout(0.4, 4), L.flatten(4, 1),
                             L.full("fc7", net.classes, w, b0)});
    auto branch = [&](int n) {
        FunPtr bpool = L.avg_pool(5, 3);
        FunPtr cv = L.convolv("b" + std::to_string(n) + "cv", 1, 128, 1, 0, w, b02);
        FunPtr f1 = L.full("b" + std::to_string(n) + "fc1", 1024, w, b02);
        FunPtr f2 = L.full("b" + std::to_string(n) + "fc2", net.classes, w, b0);
        return L.seq({bpool, cv, relu, L.flatten(4, 1), f1, relu2, L.dropout(0.7, 2), f2});
    };
    FunPtr softmax = L.softmax();
    net.x_load = t_load(t_input("X", 4), net.ctx.fresh_id());
    TPtr h1 = apply_norm(net, network1, net.x_load);
    TPtr h2 = apply_norm(net, network2, h1);
    TPtr logits = apply_norm(net, network3, h2);
    TPtr s_main = apply_norm(net, softmax, logits);
    TPtr s_b2 = apply_norm(net, softmax, apply_norm(net, branch(2), h2));
    TPtr s_b1 = apply_norm(net, softmax, apply_norm(net, branch(1), h1));
    net.logits_main = logits;
    net.y_load = t_load_indicator(t_input("Y", 1), net.classes, net.ctx.fresh_id());
    SPtr l_main = L.log_loss(s_main, 1.0, "");
    SPtr l2 = L.log_loss(s_b2, 0.3, "loss2");
    SPtr l1 = L.log_loss(s_b1, 0.3, "loss1");
    net.loss = s_add(s_add(l_main, l2), l1);
    finish(net);
}

// ResNet-50 (He et al. Caffe prototxt): bias-free convs followed
// by BatchNorm (channel affine), stride on the first 1x1 of each stage,
// projection shortcuts on the first block of every stage.
void build_resnet50(NetworkDef& net, std::int64_t batch) {
    init_net(net, "resnet50", batch, Shape{batch, 3, 224, 224}, 1000);
    LayerFactory L(net);
    auto w = ParamInit::xavier();
    auto nob = ParamInit::constant(0.0);
    FunPtr relu = L.relu(4);
    auto conv_bn = [&](const std::string& name, int k, int out, int stride, int pad, bool with_relu) {
        std::vector<FunPtr> fs{L.convolv(name, k, out, stride, pad, w, nob, false), L.batchnorm("bn_" + name)};
        if (with_relu) fs.push_back(relu);
        return L.seq(fs);
    };
    std::vector<FunPtr> layers{conv_bn("conv1", 7, 64, 2, 3, true), L.max_pool(3, 2, 1)};
    const int blocks[4] = {3, 4, 6, 3};
    const int width[4] = {64, 128, 256, 512};
    for (int s = 0; s < 4; ++s) {
        for (int b = 0; b < blocks[s]; ++b) {
            const std::string tag = "res" + std::to_string(s + 2) + static_cast<char>('a' + b);
            const int stride = (b == 0 && s > 0) ? 2 : 1;
            FunPtr br = L.seq({conv_bn(tag + "_branch2a", 1, width[s], stride, 0, true),
                               conv_bn(tag + "_branch2b", 3, width[s], 1, 1, true),
                               conv_bn(tag + "_branch2c", 1, width[s] * 4, 1, 0, false)});
            FunPtr sc = b == 0 ? conv_bn(tag + "_branch1", 1, width[s] * 4, stride, 0, false) : nullptr;
            layers.push_back(L.residual(br, sc));
        }
    }
    layers.push_back(L.avg_pool(7, 1));
    layers.push_back(L.flatten(4, 1));
    layers.push_back(L.full("fc1000", net.classes));
    net.x_load = t_load(t_input("X", 4), net.ctx.fresh_id());
    TPtr logits = apply_norm(net, L.seq(layers), net.x_load);
    TPtr s = apply_norm(net, L.softmax(), logits);
    net.logits_main = logits;
    net.y_load = t_load_indicator(t_input("Y", 1), net.classes, net.ctx.fresh_id());
    net.loss = L.log_loss(s, 1.0, "");
    finish(net);
}

// One inception block ("one inception-block network") on a small
// image, followed by a classifier: exercises Concat and adjoint accumulation.
void build_inception_block(NetworkDef& net, std::int64_t batch) {
    init_net(net, "inception", batch, Shape{batch, 3, 16, 16}, 10);
    LayerFactory L(net);
    FunPtr relu = L.relu(4);
    InceptionCfg c{"t", 8, 8, 16, 4, 8, 8};
    FunPtr network = L.seq({L.convolv("stem", 3, 16, 1, 1), relu, inception(L, 1, c, relu), L.max_pool(2),
                            L.flatten(4, 1), L.full("fc", net.classes)});
    net.x_load = t_load(t_input("X", 4), net.ctx.fresh_id());
    TPtr logits = apply_norm(net, network, net.x_load);
    TPtr s = apply_norm(net, L.softmax(), logits);
    net.logits_main = logits;
    net.y_load = t_load_indicator(t_input("Y", 1), net.classes, net.ctx.fresh_id());
    net.loss = L.log_loss(s, 1.0, "");
    finish(net);
}

// A small net with a duplicated sub-expression for the cse pass: the same
// full layer applied twice to the same hidden activations, the two logits summed.  With cse the
// second MatMul / BiasAdd pair is the first one (one Let each); without, two identical Lets.
void build_csedemo(NetworkDef& net, std::int64_t batch) {
    init_net(net, "csedemo", batch, Shape{batch, 1, 8, 8}, 10);
    LayerFactory L(net);
    FunPtr body = L.seq({L.flatten(4, 1), L.full("fc1", 32), L.relu(2)});
    FunPtr head = L.full("fc2", net.classes);
    net.x_load = t_load(t_input("X", 4), net.ctx.fresh_id());
    TPtr h = apply_norm(net, body, net.x_load);
    TPtr a = apply_norm(net, head, h);
    TPtr b = apply_norm(net, head, h);
    Hyper add;
    add.eltwise = ELT_ADD;
    TPtr logits = t_prim(PrimOp::Eltwise, add, {a, b}, 2, net.ctx.fresh_id());
    TPtr s = apply_norm(net, L.softmax(), logits);
    net.logits_main = logits;
    net.y_load = t_load_indicator(t_input("Y", 1), net.classes, net.ctx.fresh_id());
    net.loss = L.log_loss(s, 1.0, "");
    finish(net);
}

void build_by_name(NetworkDef& net, const std::string& name, std::int64_t batch) {
    if (name == "csedemo") return build_csedemo(net, batch);
    if (name == "lenet") return build_lenet(net, batch);
    if (name == "alexnet") return build_alexnet(net, batch);
    if (name == "vgg16") return build_vgg16(net, batch);
    if (name == "googlenet") return build_googlenet(net, batch);
    if (name == "resnet50") return build_resnet50(net, batch);
    if (name == "inception") return build_inception_block(net, batch);
    fail(ErrKind::UnboundName, "unknown network '" + name + "'");
}

}  // namespace tensorc
