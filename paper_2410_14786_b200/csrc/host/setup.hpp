// BDDC setup on the host (not timed in the apply; reported as setup_seconds).
//
// Produces, per subdomain, everything the device apply consumes:
//   * the supernodal Cholesky of A_II (interior solves; reference preconditioner.cpp:64),
//   * K_i   = interface block of the constrained saddle inverse,
//   * Phi_i = coarse basis, Lambda_i, A_ci = Phi_i^T A_i Phi_i (reference
//             preconditioner.cpp:34-66 / SubdomainData, preconditioner.hpp:27-35),
// and the coarse problem A_c (assemble_coarse, preconditioner.cpp:68-98) with its
// dense inverse for the replicated coarse GEMV.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "factor.hpp"
#include "problem.hpp"

namespace bddc_b200 {

struct SubdomainSetup {
    InteriorFactor factor;
    index_t n_local = 0, n_interior = 0, n_iface = 0, n_primal = 0;
    std::vector<double> K;       // n_iface x n_iface row-major
    std::vector<double> phi;     // n_local x n_primal row-major (reference layout)
    std::vector<double> lambda;  // n_primal x n_primal
    std::vector<double> aci;     // n_primal x n_primal
    std::int64_t dedup_of = -1;  // index of an identical earlier subdomain, if any
};

struct BddcSetup {
    std::vector<SubdomainSetup> subs;
    CsrMatrix coarse_matrix;              // A_c
    std::vector<double> coarse_inverse;   // dense n_c x n_c, row-major
    double seconds = 0.0;
    index_t unique_subdomains = 0;
};

// coords: optional global (ix, iy) per dof (2*global_dofs); enables geometric ND.
// Throws std::runtime_error("bddc setup: subdomain i: ...") like the reference ctor
// (preconditioner.cpp:119-121).
// assemble = false skips the coarse problem (multi-GPU: assembled after gathering every
// rank's A_ci, see assemble_coarse).
// dense_inverse = false skips A_c^-1 (coarse CG mode); a non-SPD A_c leaves it empty.
BddcSetup bddc_setup(const std::vector<CsrMatrix>& locals, const Decomposition& d,
                     const ConstraintSet& cs, const index_t* coords, index_t workers,
                     const FactorOptions& fopt = {}, bool assemble = true, bool dense_inverse = true);

// A_c = sum_i R_ci^T A_ci R_ci in ascending i (reference assemble_coarse,
// preconditioner.cpp:68-98) and its dense inverse, into out.coarse_matrix / coarse_inverse.
void assemble_coarse(BddcSetup& out, const std::vector<const std::vector<double>*>& aci,
                     const std::vector<std::vector<index_t>>& primal_maps, index_t n_coarse,
                     bool dense_inverse = true);

// Dense helpers (row-major).
// In-place inverse via LU with partial pivoting; throws "singular" on a zero pivot.
void dense_inverse(std::vector<double>& a, index_t n, const char* what);
// SPD inverse via Cholesky; throws on a non-positive pivot.
void spd_inverse(std::vector<double>& a, index_t n, const char* what);

}  // namespace bddc_b200
