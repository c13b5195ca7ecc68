// Text network description (the reference's netspec-frontend):
// parse a `.net` file and elaborate it through the layer vocabulary of nets.hpp
// into a NetworkDef, so user networks reach the compiler and the sm_100a runtime
// without C++ code (C ABI: tc_net_compile_spec, tc_plan.h).
//
// Grammar (`#` line comments, whitespace-insensitive):
//   file    := section+
//   section := ("net" | "solver" | "data") ident? "{" decl* "}"
//   decl    := ident "=" (compose | lossexpr | value)
//   compose := term ("." term)*          left-associative, like the paper's `o`
//   term    := ident | ident "(" args ")"
//   args    := arg ("," arg)* ; arg := [ident "="] (number | ident | call)
//   lossexpr:= lterm ("+" lterm)* ; lterm := [number "*"] "logloss" "(" ident ")"
// Layer kinds: conv(k, out[, stride=1][, pad=0][, w=xavier][, b=const(v[, lrm, dcm])][, bias=1]),
//   maxpool(k[, stride=k][, pad=0]), avgpool(...), relu(rank), full(out[, w, b]),
//   flatten(rank, axis), softmax, dropout(rate[, rank=2]), lrn(size, alpha, beta),
//   concat(branch, ...), and the ResNet extensions batchnorm, residual(branch[, shortcut]).
//   Initialisers: xavier | const(v[, lr_mult, decay_mult]) | gaussian(sigma[, lr_mult, decay_mult]).
//   The identifier K in a layer argument is the data section's class count.
// data keys: source = synthetic(seed), batch, shape = (C, H, W), classes.
// solver keys: lr, momentum, decay, clip, iters, test_iters, snapshot_every.
//
// Errors are CompileError (diag.hpp) with the line / column of the offending
// token: SyntaxError, DuplicateName, UnknownLayerKind, UnboundName, ArityError.
#pragma once

#include <cstdint>
#include <string>

#include "host/nets.hpp"

namespace tensorc {

struct SpecSolver {
    double lr = 0.01, momentum = 0.9, decay = 0.0005, clip = 0.0;  // Fig. 1 defaults
    std::int64_t iters = 1000, test_iters = 10, snapshot_every = 0;
    std::uint64_t seed = 42;  // data source synthetic(seed)
};

// Parse + elaborate.  batch > 0 overrides the data section's batch.
void build_from_spec(NetworkDef& net, const std::string& text, std::int64_t batch, SpecSolver* solver);

}  // namespace tensorc
