#pragma once

#include "fused_comm.cuh"

namespace bddc_b200 {

struct IfaceParams {
    const double* skip;  // pipelined PCG: skip when scal[2] / scal[3] is set (null: never)
    // multi-GPU fused LL exchanges (null on one GPU): restrict reads the u0 halo (vector index
    // >= ll_u_base) from its LL buffer and publishes the c_i; the K_i kernel reads the other
    // ranks' c_i (outside [c_own_lo, c_own_hi)) from theirs and publishes the shared h_i
    const ll_word* ll_u;
    const std::uint64_t* seq_u;
    int ll_u_base;
    const ll_word* ll_c;
    const std::uint64_t* seq_c;
    int c_own_lo, c_own_hi;
    Publish pub_c, pub_h;
    const SubdomainDesc* subs;
    int n_subdomains;
    int max_iface;
    int max_primal;
    // interface dofs
    const std::int32_t* iface_dof;
    const double* iface_w;
    const std::int32_t* iface_gid;
    const std::int32_t* gi_row_ptr;
    const std::int32_t* slot_rows;  // per local interface slot: its global A_GI row range {begin, end}
    const std::int32_t* gi_row_col;
    const double* gi_row_val;
    // dense blocks. kpacked: K_i stored as its upper triangle of 32 x 32 tiles (iface.cu,
    // pack_sym_k), applied by one CTA per subdomain; kpart: per tile two 32-vectors of partial
    // sums (kmat offset / 16)
    const double* kmat;
    int kpacked;
    int kcluster;  // packed: CTAs per subdomain (a thread-block cluster); 1 for the cooperative grid
    double* kpart;
    const double* phig;
    const std::int32_t* primal;
    // coarse
    int n_coarse;
    const std::int32_t* c_own_ptr;
    const std::int32_t* c_own_ref;
    // per coarse dof: its owners' cbuf slots (ascending subdomain, -1 padded) as an int4; x <= -2:
    // more than four owners (the owner list); null: owner lists only
    const std::int32_t* c_own4;
    const double* coarse_inv;
    // scratch
    double* gbuf;   // w * r'_G per (subdomain, gamma)
    double* hbuf;   // w * (Phi_G x_c + K g) per (subdomain, gamma)
    double* cbuf;   // Phi_G^T g per (subdomain, primal)
    double* xc;     // coarse solution
    // fused coarse solve (K_i kernel, cooperative launch): r_c formed once per GPU, each CTA
    // its share, exchanged through rc_g and a grid barrier on the monotonic coarse_ctr
    double* rc_g;
    unsigned long long* coarse_ctr;
};

struct StageParams {
    const SubdomainDesc* subs;
    int n_subdomains;
    int n_vector;
    int max_primal;
    const std::int32_t* local_dofs;
    const double* phi;
    const double* iface_w;     // per local interface slot
    const std::int32_t* iface_dof;
    const std::int32_t* gi_dof;
    int n_gi;
    const std::int32_t* gi_own_ptr;
    const std::int32_t* gi_own_ref;
    const std::int32_t* dof_own_ptr;
    const std::int32_t* dof_own_ref;
    const std::int32_t* lrow_ptr;
    const std::int32_t* lrow_col;
    const double* lrow_val;
    const std::int32_t* primal;
    const double* weights_local;  // per local slot
    double* lbuf;                 // per local slot
    double* gbuf;
    double* cbuf;
    const double* xc;
};

// Reference-faithful coarse CG on A_c (src/preconditioner.cpp:149-157 + pcg.cpp:40-109,
// no preconditioner). status: [0]=iterations, [1]=relative residual, [2]=converged.
struct CoarseCgParams {
    int n;
    const std::int32_t* ptr;
    const std::int32_t* col;
    const double* val;
    const std::int32_t* c_own_ptr;
    const std::int32_t* c_own_ref;
    const double* cbuf;
    double* xc;
    double* status;
    double rtol, atol;
    int max_it;
};
void launch_coarse_cg(const CoarseCgParams& P, cudaStream_t s);

// Stage hooks (not on the hot path): general-r coarse/local corrections.
void launch_stage_phi_restrict(const StageParams& P, const double* r, cudaStream_t s);
void launch_stage_phi_prolong(const StageParams& P, cudaStream_t s);
void launch_stage_gather_local(const StageParams& P, double* out, cudaStream_t s);
void launch_stage_local_g(const StageParams& P, const double* r, const double* y, cudaStream_t s);
void launch_stage_iface_gather(const StageParams& P, const double* h, double* out, cudaStream_t s);

// K3: g_i = W_i (r_G - A_GI u0_I) restricted to subdomain i, c_i = Phi_Gi^T g_i.
void launch_iface_restrict(const IfaceParams& P, const double* r, const double* u0, cudaStream_t s);
// K4: x_c = A_c^{-1} r_c with r_c = sum_i R_ci^T c_i (ascending i).
void launch_coarse_direct(const IfaceParams& P, cudaStream_t s);
// K5: h_i = W_i (Phi_Gi x_c[map_i] + K_i g_i); rows split over blocks_per_sub CTAs.
// with_coarse = false: h_i = K_i g_i (unweighted; local_correction stage)
// coarse: 0 = h_i = K_i g_i; 1 = W_i(Phi x_c[map] + K g) with x_c from the coarse kernel;
// 2 = the same with the rows of x_c = A_c^{-1} r_c formed in the kernel (dense direct mode)
void launch_iface_local(const IfaceParams& P, int blocks_per_sub, cudaStream_t s, int coarse);
// Whether the fused-coarse K_i grid (n_subdomains * blocks_per_sub CTAs) can be co-resident on
// `device` (cooperative launch, one r_c per GPU); otherwise every CTA forms r_c itself.
bool iface_local_cooperative_fits(const IfaceParams& P, int blocks_per_sub, int device);
// Packed K_i kernel: the first h row of CTA c of a subdomain's cluster of C (whole 32-row blocks)
__host__ __device__ inline int sym_rows_begin(int ng, int C, int c) {
    const int nt = (ng + 31) / 32;
    const int r = (c * nt / C) * 32;
    return r < ng ? r : ng;
}
// Doubles of subdomain K_i (n_iface = ng) in the packed symmetric layout: the tiles (a, b),
// a <= b, of the zero-padded ceil(ng / 32)^2 tiling, 1024 row-major values each.
std::int64_t sym_k_values(int ng);
// Packs every subdomain's row-major K_i (full_off) into the tiled upper triangle (sym_off).
void launch_pack_sym_k(const double* full, const std::int64_t* full_off, double* packed, const std::int64_t* sym_off,
                       const std::int32_t* ng, int n_subdomains, cudaStream_t s);

}  // namespace bddc_b200
