// Per-subdomain sparse factorisation used by the BDDC setup.
//
// Replaces the reference's equilibrate -> AMD -> threshold-LU pipeline
// (reference src/sparse_lu.cpp:80-195,239-243, src/amd.cpp:32-148) for the two
// systems the apply needs:
//   * the interior block A_II (reference preconditioner.cpp:64), factored as a
//     supernodal Cholesky L L^T in a nested-dissection order, and
//   * the constrained saddle system [[A_i, C_i^T], [C_i, 0]] (preconditioner.cpp:48),
//     which is reduced EXACTLY to the interface: with A_i ordered interior-first,
//     eliminating the interior leaves the dense Schur complement
//         S = A_GG - A_GI A_II^{-1} A_IG
//     (obtained for free as the root update of the multifrontal factorisation), and
//     the saddle inverse restricted to the interface is a small dense matrix.
#pragma once

#include <cstdint>
#include <vector>

#include "csr.hpp"

namespace bddc_b200 {

struct Supernode {
    index_t col_begin = 0;   // permuted interior positions [col_begin, col_end)
    index_t col_end = 0;
    index_t parent = -1;     // supernode id, -1 for roots of the interior forest
    index_t height = 0;      // 0 for leaves; parent height > child height
    std::vector<index_t> rows;  // R_s, ascending: interior positions, then n_I + gamma
    index_t n_interior_rows = 0;
    std::vector<double> L;   // n_s x n_s lower triangle of the diagonal block (row-major)
    std::vector<double> Linv;  // its inverse (row-major, lower)
    std::vector<double> B;   // |rows| x n_s (row-major): L[rows, cols]
    index_t size() const { return col_end - col_begin; }
};

struct InteriorFactor {
    index_t n_interior = 0;
    index_t n_iface = 0;
    std::vector<index_t> perm;   // perm[p] = local interior index at permuted position p
    std::vector<index_t> iperm;  // inverse
    std::vector<Supernode> snodes;  // postorder (children before parents)
    std::vector<double> schur;   // n_iface x n_iface, row-major, symmetric
    std::int64_t factor_values() const;  // sum of |L| (diag lower + interior-row B) entries
};

struct FactorOptions {
    index_t leaf_size = 16;       // regions at or below this size become dense leaves
    index_t max_supernode = 128;  // separators are split into chains above this width
};

// A_local: n_local x n_local Neumann matrix, interior dofs first (n_interior of them).
// coords: optional (x, y) integer coordinates per local dof (2*n_local), enabling
// geometric nested dissection; nullptr selects graph (BFS level-set) bisection.
// Throws std::runtime_error when A_II is not positive definite.
InteriorFactor factor_subdomain(const CsrMatrix& A_local, index_t n_interior,
                                const index_t* coords, const FactorOptions& opt = {});

// The pattern-only part of factor_subdomain: ordering, supernodes, row structures and heights
// (numeric members L / Linv / B and schur left empty). Identical for every subdomain with the
// same local pattern, split and relative coordinates, whatever the values.
InteriorFactor symbolic_factor(const CsrMatrix& A_local, index_t n_interior, const index_t* coords,
                               const FactorOptions& opt = {});

// In-place multi-RHS solve A_II X = B; X is n_interior x nrhs row-major, indexed by
// the original local interior order. Host-side setup helper (coarse basis).
void factor_solve(const InteriorFactor& F, double* X, index_t nrhs);

}  // namespace bddc_b200
