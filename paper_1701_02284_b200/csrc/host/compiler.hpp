// Compilation pipeline from a NetworkDef to the memory-scheduled execution plan.
//
//   vectorize  ->  infer_shapes
//   -> grad / prim_backward
//   -> to_ssa, cse, form_updates, schedule, inline_inplace, insert_dealloc
//   -> analyze / static_memory
//
// The resulting IrProgram is what crosses the boundary to
// the runtime: it is flattened into tc_plan.h structs for the sm_100a executor
// and for the CPU oracle alike.
#pragma once

#include <map>
#include <string>
#include <unordered_map>
#include <vector>

#include "host/nets.hpp"

namespace tensorc {

struct SolverConfig {
    std::string name = "net";
    int train_iters = 1000;
    int test_iters = 10;
    double lr = 0.01;
    double momentum = 0.9;
    double decay = 0.0005;
    double clip = 0.0;
};

enum class MemMode { Reuse, Dealloc };

struct ShapeTable {
    std::unordered_map<const TensorExpr*, Shape> t;
    std::unordered_map<const ParamSpec*, Shape> p;
    const Shape& of(const TPtr& e) const;
    const Shape& of(const ParamSpec* ps) const;
    bool has(const TPtr& e) const { return t.count(e.get()) != 0; }
};

// Rewrites FC index patterns into MatMul / BiasAdd (in place on net).
// Contraction / bias-add recognition; with cse, syntactically identical pure nodes (same kind,
// operator, hyper-parameters and operands) are built once (Copy and the
// randomized dropout mask are never merged).  Returns the number of nodes merged.
int vectorize(NetworkDef& net, bool cse = false);
void infer_shapes(const NetworkDef& net, ShapeTable& st);

struct GradInfo {
    std::vector<TPtr> created;                               // backward nodes in creation order
    std::vector<std::pair<ParamPtr, TPtr>> param_grads;      // in creation order
    std::unordered_map<const TensorExpr*, bool> seed_dep;    // depends on the loss adjoint
};
GradInfo derive_gradients(NetworkDef& net, ShapeTable& st);

enum class StmtKind { Let, Dealloc, Update, Print };

struct IrStmt {
    StmtKind kind = StmtKind::Let;
    TPtr node;          // Let: defining expression; Update: gradient expression (GradPrim)
    ParamPtr param;     // Update target
    SPtr loss;          // Print
    int var = -1;       // Let / Dealloc
    Shape shape;        // Let result shape (reference NCHW)
    std::int64_t bytes = 0;      // bytes this statement allocates (0 for in-place)
    int storage = -1;   // Let: storage id (alias root); Dealloc: storage freed
    bool inplace = false;        // Let writes into its first operand's storage
    bool copy_operand = false;   // an always-in-place op on a live operand: "X.copy"
    // Update: v = momentum * v - lr*lr_mult * (g + decay*decay_mult * p); p += v
    double lr_alpha = 0.0, momentum = 0.0, decay = 0.0;
    std::string text;   // Fig. 2 surface syntax
};

struct IrProgram {
    std::string name;
    std::int64_t batch = 0;
    std::int64_t classes = 0;
    Shape input_shape;
    SolverConfig solver;
    MemMode mode = MemMode::Dealloc;
    double workspace_cap_mb = -1.0;   // < 0: unlimited
    std::vector<ParamPtr> params;
    std::vector<Shape> param_shapes;
    std::vector<IrStmt> train;        // train-loop body
    std::vector<IrStmt> test;         // test body: forward to the main logits
    int logits_var = -1;
    std::unordered_map<int, Shape> var_shapes;
};

struct CompileOptions {
    SolverConfig solver;
    MemMode mode = MemMode::Dealloc;
    double workspace_cap_mb = -1.0;
    bool greedy_schedule = false;   // SPEC.md:331 greedy release-most-bytes list scheduler
    bool cse = true;                // SPEC.md:313-319 common sub-expression elimination
};

IrProgram compile_network(NetworkDef& net, const CompileOptions& opt);

// ---------------------------------------------------------------- memplan
struct MemoryRow {
    std::string stmt;
    std::string dims;
    double delta_mb = 0;
    double total_dealloc_mb = 0;
    double total_reuse_mb = 0;
};

struct MemoryReport {
    std::vector<MemoryRow> rows;
    std::int64_t peak_dealloc_bytes = 0;
    std::int64_t peak_reuse_bytes = 0;
    std::int64_t param_bytes = 0;       // weights + biases + velocities (fp32)
    std::int64_t workspace_bytes = 0;   // shared im2col workspace (min(cap, max conv))
    double peak_dealloc_mb() const { return static_cast<float>(peak_dealloc_bytes) / 1e6f; }
    double peak_reuse_mb() const { return static_cast<float>(peak_reuse_bytes) / 1e6f; }
};

MemoryReport analyze(const IrProgram& p);
std::string format_report(const MemoryReport& r, bool csv);
std::string dump_ir(const IrProgram& p);
// Verifier: SSA, def-before-use, dealloc after last use,
// no use after dealloc.  Returns "" when valid, else the first violation.
std::string verify(const IrProgram& p);

// Variables read by a statement (vars only, views resolved to their base).
std::vector<int> stmt_reads(const IrStmt& s);
// Storage-owning base of a view / copy chain.
TPtr base_of(const TPtr& t);

}  // namespace tensorc
