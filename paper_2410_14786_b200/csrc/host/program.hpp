// Compiles the host setup (supernodal factors, K_i, Phi_i, coarse inverse) into the
// flat device image the sm_100a kernels consume (layout: device_format.hpp).
// With a RankPlan (multi-GPU, host/distribute.hpp) the image describes one rank: interface
// sums also read the remote slots filled by the interface exchange, and the coarse
// residual is summed from the gathered c_i of every subdomain, both in ascending global
// subdomain order.
#pragma once

#include <cstdint>
#include <vector>

#include "../device_format.hpp"
#include "setup.hpp"
#include "solve_program.hpp"

namespace bddc_b200 {

struct RankPlan;
struct SetupClass;

struct DeviceImage {
    std::vector<SubdomainDesc> subs;
    SolvePools solve;  // interior-solve parts
    SolvePools harm;   // harmonic-extension parts (pruned forward sweep; empty when disabled)
    SolvePools head;   // the apply's first solve: full forward, pruned backward (with harm)
    int parts = 1;     // CTAs per subdomain in the interior solve
    std::vector<std::int32_t> iface_dof;     // per (subdomain, gamma): vector index
    std::vector<double> iface_w;             // weight
    std::vector<std::int32_t> iface_gid;     // global interface id
    std::vector<std::int32_t> iface_writer;  // 1 if this subdomain is the lowest owner
    std::vector<double> kmat, phig, phi;
    std::vector<std::int32_t> primal;
    std::vector<std::int32_t> local_dofs;
    std::vector<std::int32_t> lrow_ptr, lrow_col;  // local A_GI rows (stage hooks)
    std::vector<double> lrow_val;
    // interface dofs of the vector (one entry per distinct interface dof)
    std::vector<std::int32_t> gi_dof;
    std::vector<std::int32_t> gi_row_ptr, gi_row_col;
    std::vector<double> gi_row_val;
    std::vector<std::int32_t> gi_own_ptr, gi_own_ref;  // -> hbuf slots, ascending subdomain
    // every vector dof: owners as local-dof slots (ascending subdomain) for stage gathers
    std::vector<std::int32_t> dof_own_ptr, dof_own_ref;
    // coarse owners: per coarse dof, cbuf slots ascending subdomain
    std::vector<std::int32_t> c_own_ptr, c_own_ref;
    std::vector<double> coarse_inv;
    std::int64_t hbuf_total = 0, cbuf_total = 0, local_total = 0;
    std::int32_t max_interior = 0, max_iface = 0, max_primal = 0, n_coarse = 0;
    std::int32_t n_vector = 0;
    std::int64_t factor_values = 0;
    // GPU setup (classes given): K_i, Phi and the program values are produced on the device;
    // the host vectors kmat / phig / phi stay empty, these are their lengths
    bool device_values = false;
    std::int64_t kmat_total = 0, phig_total = 0, phi_total = 0, lambda_total = 0;
    std::vector<std::int64_t> lambda_off;  // per subdomain (device Lambda_i, n_primal^2)
    std::vector<std::int32_t> sub_class;   // class of each subdomain
    struct Fill {
        std::int64_t dst;  // word offset in the pool's device stream
        std::int64_t words;
        std::int32_t cls, prog;
        index_t sub;
    };
    std::vector<Fill> fills[3];  // per pool: 0 solve, 1 harm, 2 head
};

DeviceImage build_device_image(const Decomposition& d, const ConstraintSet& cs,
                               const std::vector<CsrMatrix>& locals, const CsrMatrix& global,
                               const BddcSetup& setup, int parts, int unit_bytes = 4096,
                               const RankPlan* plan = nullptr, bool harmonic = false,
                               const std::vector<SetupClass>* classes = nullptr);

}  // namespace bddc_b200
