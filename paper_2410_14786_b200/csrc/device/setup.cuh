// GPU setup kernels (reference setup_subdomain / assemble_coarse,
// src/preconditioner.cpp:34-98, lu_factor src/sparse_lu.cpp:80-195). The host plans a class
// of identically patterned subdomains once (host/gpu_setup.hpp); these kernels do the numeric
// work of every member at once:
//   mf_front      batched multifrontal Cholesky of A_II, one launch per height of the
//                 elimination tree, one CTA per (front, member), 32-column panels in shared memory
//   schur         S_i = A_GG + extend-add of the roots' updates
//   linv_bl       L_ss^-1 and BL_s = L_{R_s,s} L_ss^-1 into the member's value array D
//   fill          program streams = template words / D values (solve_program.hpp srcmap codes)
//   saddle        Gauss-Jordan inverse (partial pivoting) of [[S, C^T], [C, 0]] -> K_i, Phi_G,
//                 Lambda_i and A_ci = Phi^T A Phi = Phi_G^T S_i Phi_G
//   phi_*         Phi_I columns from interior solves
//   gj_step       dense SPD inverse of A_c (Gauss-Jordan, one launch pair per pivot, all SMs)
#pragma once

#include "common.cuh"

namespace bddc_b200 {

struct MfPlanDev {  // device copy of a SetupClass plan (pointers into one upload)
    const std::int32_t* sn_nc;
    const std::int32_t* sn_m;
    const std::int32_t* sn_mi;
    const std::int64_t* front_off;
    const std::int32_t* level_sn;
    const std::int32_t* asc_ptr;
    const std::int32_t* asc_pos;
    const std::int32_t* asc_csr;
    const std::int32_t* ch_ptr;
    const std::int32_t* ch_id;
    const std::int32_t* em_ptr;
    const std::int32_t* em_pos;
    const std::int32_t* sgg_pos;
    const std::int32_t* sgg_csr;
    const std::int32_t* roots;
    const std::int32_t* root_gamma_ptr;
    const std::int32_t* root_gamma;
    const std::int32_t* c_ptr;
    const std::int32_t* c_col;
    const double* c_val;
    const std::int64_t* linv_off;
    const std::int64_t* bl_off;
    const std::int32_t* a_ptr;  // local CSR pattern (n_local + 1)
    const std::int32_t* a_col;
    std::int64_t front_total, d_total;
    int nnz, n_local, n_interior, n_iface, n_primal, n_roots, n_sn, sgg_n;
};

struct MfBatch {  // one batch of members of a class
    const double* aval;  // member-major local CSR values (nnz each)
    double* fronts;      // member-major fronts (front_total each)
    double* S;           // member-major Schur complements (n_iface^2 each)
    double* D;           // member-major value arrays (d_total each)
    double* M;           // member-major saddle matrices / inverses ((n_iface + n_primal)^2 each)
    int* piv;            // member-major pivot rows (n_iface + n_primal each)
    int* status;         // [0] first failing member + 1 (multifrontal), [1] its pivot; [2], [3] saddle
    int n;               // members in the batch
    int first;           // index of the batch's first member within the class (status reports)
};

// Multifrontal factorisation of the supernodes level_sn[lb, le) for every member.
void launch_mf_level(const MfPlanDev& P, const MfBatch& B, int lb, int le, int max_f, cudaStream_t s);
void launch_schur(const MfPlanDev& P, const MfBatch& B, int max_root_f, cudaStream_t s);
void launch_linv_bl(const MfPlanDev& P, const MfBatch& B, int max_nc, cudaStream_t s);

struct FillJob {
    std::int64_t dst;    // word offset in the destination stream
    std::int64_t tmpl;   // word offset of the template stream / srcmap
    std::int64_t words;
    std::int64_t d_off;  // offset of the member's value array in the batch's D
};
void launch_fill(double* dst, const double* tmpl, const std::int32_t* srcmap, const double* D, const FillJob* jobs,
                 int n_jobs, cudaStream_t s);

// Saddle inverse per member; then K_i, Phi_G (and the interface rows of Phi), Lambda_i and A_ci
// out to the image offsets of each member.
struct SaddleOut {
    const std::int64_t* off;  // per member: {kmat, phig, phi, lambda, aci} offsets into the buffers below
    double* kmat;
    double* phig;
    double* phi;
    double* lambda;
    double* aci;  // A_ci = Phi^T A Phi, evaluated as Phi_G^T (S_i Phi_G) (A Phi vanishes on the interior rows)
};
void launch_saddle(const MfPlanDev& P, const MfBatch& B, const SaddleOut& O, cudaStream_t s);

// Phi_I columns: hbuf slots of every subdomain <- Phi_G[:, j] (0 past n_primal), then (after an
// interior solve with the coupling rhs) Phi[l, j] <- x[local_dofs[l]] for the interior rows.
void launch_phi_to_hbuf(const SubdomainDesc* subs, int n_sub, const double* phig, double* hbuf, int j,
                        cudaStream_t s);
void launch_phi_from_solution(const SubdomainDesc* subs, int n_sub, const std::int32_t* local_dofs, const double* x,
                              double* phi, int j, cudaStream_t s);

// In-place inverse of the dense SPD n x n matrix A (row-major) by Gauss-Jordan without
// pivoting; status[0] = 1 + the first non-positive pivot, 0 if A is SPD to working precision.
void dense_spd_inverse(double* A, int n, double* scratch, int* status, cudaStream_t s);

}  // namespace bddc_b200
