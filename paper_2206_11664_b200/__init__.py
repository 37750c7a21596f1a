"""simdiag-b200: B200-native Trotter hot path of arXiv 2206.11664.

Grouping and Clifford synthesis run in from-scratch host C++ (bit-exact with
the reference); the state-vector work runs as hand-written sm_100a CUDA tile
passes behind the C ABI in include/simdiag_c.h. This package is the Python
mirror of the reference's C++ API over that ABI.
"""
from .simdiag import (  # noqa: F401
    K_DROP_TOLERANCE,
    K_MAX_QUBITS,
    CliffordCircuit,
    CommutingGroup,
    DiagonalGroup,
    EvolutionPlan,
    Hamiltonian,
    LocalShards,
    PauliString,
    StateVector,
    TrotterPlan,
    WeightedTerm,
    comm_unique_id,
    commutes,
    diagonalize_group,
    evolve_baseline,
    evolve_grouped,
    exact_evolve,
    gen_syk,
    gen_tfim,
    exchange_routes,
    expectation,
    fidelity,
    greedy_partition,
    norm,
    partition_and_diagonalize,
    plan_preview,
)
from . import models  # noqa: F401

__all__ = [
    "CliffordCircuit", "CommutingGroup", "DiagonalGroup", "EvolutionPlan", "Hamiltonian",
    "PauliString", "StateVector", "TrotterPlan", "WeightedTerm", "commutes", "diagonalize_group",
    "evolve_grouped", "fidelity", "greedy_partition", "norm", "partition_and_diagonalize", "models",
    "LocalShards", "comm_unique_id", "plan_preview", "evolve_baseline", "expectation", "exact_evolve", "gen_tfim", "gen_syk",
]
