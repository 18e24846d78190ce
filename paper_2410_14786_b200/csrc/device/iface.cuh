#pragma once

#include "common.cuh"

namespace bddc_b200 {

struct IfaceParams {
    const SubdomainDesc* subs;
    int n_subdomains;
    int max_iface;
    int max_primal;
    // interface dofs
    const std::int32_t* iface_dof;
    const double* iface_w;
    const std::int32_t* iface_gid;
    const std::int32_t* gi_row_ptr;
    const std::int32_t* gi_row_col;
    const double* gi_row_val;
    // dense blocks
    const double* kmat;
    const double* phig;
    const std::int32_t* primal;
    // coarse
    int n_coarse;
    const std::int32_t* c_own_ptr;
    const std::int32_t* c_own_ref;
    const double* coarse_inv;
    // scratch
    double* gbuf;   // w * r'_G per (subdomain, gamma)
    double* hbuf;   // w * (Phi_G x_c + K g) per (subdomain, gamma)
    double* cbuf;   // Phi_G^T g per (subdomain, primal)
    double* xc;     // coarse solution
};

// K3: g_i = W_i (r_G - A_GI u0_I) restricted to subdomain i, c_i = Phi_Gi^T g_i.
void launch_iface_restrict(const IfaceParams& P, const double* r, const double* u0, cudaStream_t s);
// K4: x_c = A_c^{-1} r_c with r_c = sum_i R_ci^T c_i (ascending i).
void launch_coarse_direct(const IfaceParams& P, cudaStream_t s);
// K5: h_i = W_i (Phi_Gi x_c[map_i] + K_i g_i); rows split over blocks_per_sub CTAs.
void launch_iface_local(const IfaceParams& P, int blocks_per_sub, cudaStream_t s);

}  // namespace bddc_b200
