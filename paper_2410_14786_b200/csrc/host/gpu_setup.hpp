// GPU setup, host part (reference setup_subdomain / assemble_coarse,
// src/preconditioner.cpp:34-98, and lu_factor, src/sparse_lu.cpp:80-195).
//
// The setup is split by what depends on the VALUES of a subdomain and what only on its
// PATTERN. Subdomains with the same local sparsity pattern, interior split, constraint
// matrix and relative coordinates form a "setup class" (C2: 9 classes for 64 subdomains; a
// heterogeneous problem like C5 keeps its classes, only the values differ). Per class, the
// host does the pattern-only work ONCE:
//   * the nested-dissection ordering and supernodal symbolic factorisation (factor.hpp),
//   * the multifrontal plan the device factorisation follows: front sizes and offsets, the
//     scatter of the local matrix into each front, the extend-add maps of every child into
//     its parent, the supernodes grouped by tree height, the A_GG scatter into the Schur
//     complement,
//   * the three interior-solve programs as TEMPLATES (solve_program.hpp ValueLayout): every
//     tile value is a reference into the subdomain's value array D = [L_ss^-1 | BL_s].
// Everything numeric runs on the device for every subdomain (device/setup.cu): the batched
// multifrontal Cholesky, the Schur complements, L_ss^-1 and BL_s, the program fill, the
// saddle reduction to K_i / Phi_G / Lambda_i, Phi_I by interior solves, A_ci and A_c^-1.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "factor.hpp"
#include "problem.hpp"
#include "solve_program.hpp"

namespace bddc_b200 {

struct SetupClass {
    std::vector<index_t> members;  // subdomains of the class, ascending
    index_t rep = -1;              // the member whose pattern / constraints / coordinates define the class
    index_t n_local = 0, n_interior = 0, n_iface = 0, n_primal = 0, nnz = 0;
    InteriorFactor sym;  // symbolic factor (numeric members empty)

    // ---- multifrontal plan; fronts are column-major f x f (lower triangle used), per subdomain
    // at front_off[s] of a front_total-double scratch block
    std::vector<std::int32_t> sn_nc, sn_m, sn_mi;  // columns, rows (|R_s|), interior rows of R_s
    std::vector<std::int64_t> front_off;
    std::int64_t front_total = 0;
    std::int32_t max_front = 0;
    std::vector<std::int32_t> level_ptr, level_sn;  // supernodes by height, heights ascending
    std::vector<std::int32_t> asc_ptr, asc_pos, asc_csr;  // per supernode: front position <- local CSR value
    std::vector<std::int32_t> ch_ptr, ch_id;              // per supernode: its children
    std::vector<std::int32_t> em_ptr, em_pos;             // per supernode: its rows -> front position in the parent
    // ---- interface Schur complement S (n_iface^2, row-major): A_GG scatter + root updates
    std::vector<std::int32_t> sgg_pos, sgg_csr;
    std::vector<std::int32_t> roots;
    std::vector<std::int32_t> root_gamma_ptr, root_gamma;  // per root: interface index of each row
    // ---- constraints (pattern and values shared by the class), C_G on the interface columns
    std::vector<std::int32_t> c_ptr, c_col;  // n_primal rows, interface column index
    std::vector<double> c_val;
    // ---- templates: 0 = full solve (stage hook), 1 = harmonic (pruned forward), 2 = head (pruned
    // backward); their gmap holds local dof indices, couple_src local CSR value indices
    ValueLayout layout;
    SolvePools prog[3];
    std::int64_t factor_values = 0;
};

// Exact pattern key of subdomain i's setup (values of A excluded).
std::string setup_pattern_key(const CsrMatrix& A, index_t n_interior, const CsrMatrix& C,
                              const std::vector<index_t>& rel_coords);

// Groups the subdomains into classes and builds every class's symbolic factor, multifrontal
// plan and program templates (host threads over classes). coords: global (x, y) per dof or null.
std::vector<SetupClass> plan_gpu_setup(const std::vector<CsrMatrix>& locals, const Decomposition& d,
                                       const ConstraintSet& cs, const index_t* coords, const FactorOptions& fopt,
                                       int parts, int unit_bytes, bool harmonic, int workers);

}  // namespace bddc_b200
