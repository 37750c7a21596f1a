// Lowers planner passes (planner.hpp) into the device micro-programs that
// k_tile_pass executes (internal.hpp: MicroOpDev, PermDev, PointDev ...).
#pragma once

#include <string>
#include <vector>

#include "../internal.hpp"
#include "planner.hpp"

namespace sdb {

struct HostPlanArrays {
    std::vector<PassDev> passes;
    std::vector<MicroOpDev> ops;
    std::vector<PermDev> perms;
    std::vector<PointDev> points;
    std::vector<SegDev> segs;
    std::vector<uint32_t> lo_pairs;
    std::vector<uint64_t> oo_pairs;
    std::vector<uint64_t> qt_words;
    std::vector<CfgThreadDev> cfg_tb;
    std::vector<uint64_t> term_hmask;
    std::vector<uint32_t> term_lmask;
    std::vector<double> term_coeffs;
    std::vector<int> pass_class;   // 0 = transform pass, 1 = diagonal-only pass
    std::vector<int> transposes;   // shared-memory transposes per pass (CFG with a write side)
    // Specialised kernels stage tile loads through TMA (jit.cpp): -1 default
    // (on unless SDB_TMA=0), 0 off, 1 on. Set per plan by the caller.
    int tma = -1;
    int ring = -1;  // specialised kernels run the ring pipeline: -1 default (R = 5 programs), 0 off, 1 on
};

// table_threshold: POINT stages with more terms use the per-tile WHT table.
// rbits: register coordinates per thread config (3 or 4).
HostPlanArrays lower_plan(const StepPlan& sp, int n_local, int table_threshold, int rbits);

std::string describe_program(const HostPlanArrays& a);

// Checks the register-config bookkeeping of every pass (throws on a mismatch).
void verify_lowering(const HostPlanArrays& a);

}  // namespace sdb
