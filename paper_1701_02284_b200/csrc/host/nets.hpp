// Network definition layer: the layer vocabulary of the paper's listings
// (CudaLayer.convolv / max_pool / relu / softmax / lrn / concat, Layer.full /
// flatten / log_loss) as TensorFun templates over the
// expression core, plus the five configured networks.
//
// This is the `elaborate` step of SPEC.md:52-61 done through the C++ API (the
// text netspec parser is out of scope).  Layer bodies are
// templates (node ids < 0); ids are assigned when an application is
// normalised, so LeNet reproduces the X7..X21 numbering of Fig. 2
// (PAPER.md:272-287).
#pragma once

#include <map>
#include <string>

#include "host/expr.hpp"

namespace tensorc {

struct ParamInit {
    InitKind kind = InitKind::Xavier;
    double value = 0.0;
    double lr_mult = 1.0;
    double decay_mult = 1.0;
    double sigma = 0.0;  // Gaussian
    static ParamInit xavier() { return {}; }
    static ParamInit constant(double v, double lrm = 1.0, double dcm = 1.0) {
        return {InitKind::Constant, v, lrm, dcm};
    }
};

// Everything downstream stages need about a network instance.
struct NetworkDef {
    std::string name;
    std::int64_t batch = 0;
    std::int64_t loss_card = 0;  // |N| of the log-loss; data parallel: global batch (0 = batch)
    Shape input_shape;       // (N, C, H, W)
    std::int64_t classes = 0;
    ExprContext ctx;
    TPtr x_load;             // Cuda(X)
    TPtr y_load;             // Cuda(Indicator(Y, K))
    SPtr loss;               // scalar training loss
    TPtr logits_main;        // pre-softmax output of the main branch (test body)
    std::vector<ParamPtr> params;             // free_params(loss), first-use order
};

class LayerFactory {
public:
    explicit LayerFactory(NetworkDef& net) : net_(net) {}

    FunPtr convolv(const std::string& name, int k, std::int64_t out, int stride = 1, int pad = 0,
                   ParamInit w = ParamInit::xavier(), ParamInit b = ParamInit::constant(0.0), bool has_bias = true);
    FunPtr max_pool(int k, int stride = -1, int pad = 0);
    FunPtr avg_pool(int k, int stride = -1, int pad = 0);
    FunPtr relu(int rank);
    FunPtr softmax();
    FunPtr lrn(int size, double alpha, double beta);
    FunPtr dropout(double rate, int rank);
    FunPtr flatten(int rank, int axis);
    FunPtr full(const std::string& name, std::int64_t out, ParamInit w = ParamInit::xavier(),
                ParamInit b = ParamInit::constant(0.0));
    FunPtr batchnorm(const std::string& name);                 // ResNet extension
    FunPtr concat(const std::vector<FunPtr>& branches);        // CudaLayer.concat
    FunPtr residual(const FunPtr& branch, const FunPtr& shortcut);  // y = relu(branch(x) + shortcut(x))
    FunPtr seq(const std::vector<FunPtr>& fs);  // f_n o ... o f_1 without fresh compose ids
    FunPtr compose(const FunPtr& f, const FunPtr& g) { return tensorc::compose(net_.ctx, f, g); }

    // Softmax log-loss head: (0 - (Y . Log S)) / |N|.
    SPtr log_loss(const TPtr& softmax_out, double weight, const std::string& weight_name);

private:
    ParamPtr param(const std::string& name, const ParamInit& init, int rank);
    NetworkDef& net_;
};

// Parameter shapes are fixed later by shape inference from their first
// constraining use.  All builders fill `net` completely.
void build_lenet(NetworkDef& net, std::int64_t batch);
void build_alexnet(NetworkDef& net, std::int64_t batch);
void build_vgg16(NetworkDef& net, std::int64_t batch);
void build_googlenet(NetworkDef& net, std::int64_t batch);
void build_resnet50(NetworkDef& net, std::int64_t batch);
// Small networks for tests: a 2-conv inception block and an MLP.
void build_inception_block(NetworkDef& net, std::int64_t batch);
void build_by_name(NetworkDef& net, const std::string& name, std::int64_t batch);

}  // namespace tensorc
