// planner.hpp -- fused operations, pass plans and their kernel lowering.
#pragma once

#include <cstdint>
#include <cstdio>
#include <vector>

#include "common.hpp"
#include "kernels.hpp"

namespace qcs {

using u64 = std::uint64_t;

// One state operation in circuit order, in a form the tile kernel can run.
struct FOp {
    int kind = TOP_GATE;          // TileOpKind
    bool diagonal = false;        // commutes with every other diagonal operation
    u64 touch = 0;                // basis bits the operation reads (its support)
    // TOP_GATE (controls peeled off) / TOP_WHT (K = 1)
    int K = 0;
    int tpos[3] = {0, 0, 0};      // target basis bits, most significant first
    u64 ctrl_mask = 0, ctrl_val = 0;
    int nrows = 0;
    std::uint8_t row_member[8] = {};
    std::uint8_t nnz[8] = {};
    std::uint8_t col_member[8][8] = {};
    double2 val[8][8] = {};
    // TOP_DIAG
    int dk = 0;
    int dpos[3] = {0, 0, 0};
    double2 dval[8] = {};
    std::uint8_t dskip[8] = {};
    // TOP_SIGN
    std::vector<u64> flips;
    bool flip_rest = false;
    // TOP_SCALE
    double scale = 1.0;
    // the placement it came from (gate / diag ops): single-op passes use the gate kernel
    GateOp src;
};

bool make_fop(const GateOp& op, FOp& f);  // false: identity, nothing to do
FOp make_sign(int n, std::vector<u64> flips, bool flip_rest);
FOp make_scale(double s);
FOp make_wht(int bit);

struct PlannedPass {
    u64 tile = 0;               // tile bit set
    std::vector<int> ops;       // indices into the op list, execution order
};
struct Plan {
    std::vector<PlannedPass> passes;
};
Plan plan_ops(int n, const std::vector<FOp>& ops, int max_bits);
void merge_single_qubit(int n, std::vector<FOp>& ops);
void split_phases(std::vector<FOp>& ops);

struct Lowered {
    std::vector<PassParams> passes;
    std::vector<TileOp> big;                 // shared-memory gates, sign steps, 3-bit diagonals
    std::vector<u64> flips;
    std::vector<u64> tables;                 // per pass: run offsets (PassParams::hi_off), tile lists
    std::vector<std::vector<int>> pass_ops;  // FOp indices per pass
    std::vector<u64> single_flip_off, single_flip_cnt;  // sign step of a single-op pass
    std::vector<u64> reached;  // per pass: the bits operations before it may have changed (support)
};
void lower_plan(int n, const std::vector<FOp>& ops, const Plan& plan, Lowered& out);
// compile (in parallel, NVRTC) the specialised kernels of the plan's passes that will use one (jit.cpp)
void jit_prepare(int n, const std::vector<PassParams>& passes, const std::vector<std::vector<int>>& pass_ops);
// one line per round and operation (planner debugging, QCS_PLAN_DUMP)
void dump_pass(std::FILE* f, const PassParams& p, std::size_t nsrc);

}  // namespace qcs
