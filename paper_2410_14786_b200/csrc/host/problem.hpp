// Problem layer: structured Q1 Poisson grid, kx x ky subdomain decomposition,
// dof classes, partition-of-unity weights and primal constraints.
//
// Integer maps are bit-exact with the reference (tests/test_host_problem.py):
//   classify_dofs        reference src/decomposition.cpp:30-59 (entity numbering
//                        generalised to kx x ky; reduces to the reference when kx == ky)
//   build_decomposition  src/decomposition.cpp:73-110
//   build_weights        src/decomposition.cpp:61-71
//   build_constraints    src/decomposition.cpp:112-159
//   assemble_poisson     src/decomposition.cpp:161-203
//   global_from_locals   src/decomposition.cpp:205-222
//   q1_element_matrix    src/grid.cpp:19-39
//   study_rhs            src/study.cpp:69-75
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "csr.hpp"

namespace bddc_b200 {

enum class DofKind : std::uint8_t { interior = 0, edge = 1, corner = 2 };

struct DofClass {
    DofKind kind = DofKind::interior;
    index_t entity = -1;
};

struct Decomposition {
    index_t k = 0;   // subdomains per side when square (reference field), else 0
    index_t kx = 0;
    index_t ky = 0;
    index_t n_subdomains = 0;
    index_t global_dofs = 0;
    std::vector<std::vector<index_t>> subdomain_dofs;  // interior first, ascending
    std::vector<index_t> interior_counts;
    std::vector<DofClass> classes;
    std::vector<index_t> multiplicity;
    std::vector<std::vector<double>> weights;
};

struct ConstraintSet {
    std::vector<CsrMatrix> constraint_matrices;
    std::vector<std::vector<index_t>> primal_maps;
    index_t n_coarse = 0;
};

struct PoissonProblem {
    index_t cells_x = 0, cells_y = 0;
    Decomposition decomposition;
    CsrMatrix global_matrix;
    std::vector<CsrMatrix> local_matrices;
    // (ix, iy) vertex coordinates of every global dof; used only to pick a
    // geometric nested-dissection ordering during setup.
    std::vector<index_t> coords;
};

// 4x4 Q1 element stiffness, node order SW, SE, NE, NW (2x2 Gauss).
void q1_element_matrix(double K[4][4]);

std::vector<DofClass> classify_dofs(index_t cells_x, index_t cells_y, index_t kx, index_t ky);
std::vector<std::vector<double>> build_weights(const Decomposition& d);
Decomposition build_decomposition(index_t cells_x, index_t cells_y, index_t kx, index_t ky);
ConstraintSet build_constraints(const Decomposition& d);
CsrMatrix global_from_locals(const Decomposition& d, const std::vector<CsrMatrix>& locals);

// kappa (optional): per-element coefficient, row-major over cells_x x cells_y cells.
PoissonProblem assemble_poisson(index_t cells_x, index_t cells_y, index_t kx, index_t ky,
                                const double* kappa = nullptr);

// Deterministic heterogeneous coefficient for config C5:
// kappa_e = 10^(contrast_decades * u_e), u_e = (splitmix64(seed ^ e) >> 11) * 2^-53.
std::vector<double> log_uniform_kappa(index_t cells_x, index_t cells_y, double contrast_decades,
                                      std::uint64_t seed);

// Seeded standard-normal rhs: libstdc++ mt19937_64 + normal_distribution.
std::vector<double> study_rhs(index_t n, std::uint64_t seed);

// Reference bundle format (reference src/bundle.cpp:59-111): manifest, Matrix Market
// local matrices (%.17g), maps, classes, rhs. Lets the reference oracle ingest
// rectangular / heterogeneous problems produced here.
std::string export_bundle(const Decomposition& d, const std::vector<CsrMatrix>& locals,
                          const std::vector<double>& rhs, const std::string& directory);

// Matrix Market "coordinate real general|symmetric" (reference src/matrix_market.cpp:23-71):
// 1-based entries, symmetric files mirrored, duplicates summed in file order (from_triplets).
CsrMatrix read_matrix_market_file(const std::string& path);

// Bundle ingestion (reference src/bundle.cpp:113-290): manifest keys, rhs / classes / maps /
// Matrix Market locals, multiplicity validation with the reference's messages, stable
// interior-first reorder of every map (and its matrix), weights 1/multiplicity, constraints and
// the global matrix rebuilt from the locals.
struct IngestedProblem {
    Decomposition decomposition;
    std::vector<CsrMatrix> local_matrices;
    ConstraintSet constraints;
    CsrMatrix global_matrix;
    std::vector<double> rhs;
};
IngestedProblem ingest_bundle(const std::string& manifest_path);

}  // namespace bddc_b200
