// Clifford synthesis that simultaneously diagonalises a commuting group.
//
// Drop-in for reference proj/include/simdiag/diagonalize.hpp:1-63 (steps
// (i)-(iv) and the two drivers). Implementation:
// paper_2206_11664_b200/csrc/host/synthesis.cpp.
#pragma once

#include <cstdint>
#include <span>
#include <utility>
#include <vector>

#include "simdiag/clifford_circuit.hpp"
#include "simdiag/hamiltonian.hpp"
#include "simdiag/tableau.hpp"

namespace simdiag {

enum class ColumnKind { diag_only, flip_only, general };

std::vector<ColumnKind> classify_columns(const CommutingGroup& group);

/// (i) H trials over active qubits, high -> low, kept on strict rank gain.
std::vector<int> maximize_x_rank(BinaryTableau& tab, std::uint64_t active);

struct XSweep {
    std::vector<std::pair<int, int>> cnots;
    std::vector<std::pair<std::size_t, int>> pivots;  // (row, column)
};

/// (ii) Clear X entries right of each pivot with CNOTs.
XSweep clear_upper_x(BinaryTableau& tab, std::uint64_t active);

struct PhaseGates {
    std::vector<std::pair<int, int>> czs;
    std::vector<int> s_layer;
};

/// (iii) Clear the pivot rows' Z entries with CZ (off-pivot) and S (pivot).
PhaseGates clear_z_block(BinaryTableau& tab, std::uint64_t active,
                         std::span<const std::pair<std::size_t, int>> pivots);

/// (iv) H on every qubit whose X column is non-zero.
std::vector<int> x_to_z(BinaryTableau& tab);

CliffordCircuit find_clifford(const CommutingGroup& group);
DiagonalGroup diagonalize_group(const CommutingGroup& group);

}  // namespace simdiag
