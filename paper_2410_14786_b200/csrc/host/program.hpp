// Compiles the host setup (supernodal factors, K_i, Phi_i, coarse inverse) into the
// flat device image the sm_100a kernels consume (layout: device_format.hpp).
#pragma once

#include <cstdint>
#include <vector>

#include "../device_format.hpp"
#include "setup.hpp"

namespace bddc_b200 {

struct DeviceImage {
    std::vector<SubdomainDesc> subs;
    std::vector<double> stream;
    std::vector<TileTask> tasks;
    std::vector<std::int32_t> phases;
    std::vector<std::int32_t> idx;
    std::vector<std::int32_t> gmap;
    std::vector<std::int32_t> couple_ptr;
    std::vector<std::int32_t> couple_gamma;
    std::vector<double> couple_val;
    std::vector<std::int32_t> iface_dof;     // per (subdomain, gamma): vector index
    std::vector<double> iface_w;             // weight
    std::vector<std::int32_t> iface_gid;     // global interface id
    std::vector<std::int32_t> iface_writer;  // 1 if this subdomain is the lowest owner
    std::vector<double> kmat, phig, phi;
    std::vector<std::int32_t> primal;
    std::vector<std::int32_t> local_dofs;
    // interface dofs of the vector (one entry per distinct interface dof)
    std::vector<std::int32_t> gi_dof;
    std::vector<std::int32_t> gi_row_ptr, gi_row_col;
    std::vector<double> gi_row_val;
    std::vector<std::int32_t> gi_own_ptr, gi_own_ref;  // -> hbuf slots, ascending subdomain
    // coarse owners: per coarse dof, cbuf slots ascending subdomain
    std::vector<std::int32_t> c_own_ptr, c_own_ref;
    std::vector<double> coarse_inv;
    std::int64_t hbuf_total = 0, cbuf_total = 0;
    std::int32_t max_interior = 0, max_iface = 0, max_primal = 0, n_coarse = 0;
    std::int32_t n_vector = 0;
    // accounting (bytes of FP64 values actually streamed per interior-solve pass pair)
    std::int64_t fwd_values = 0, bwd_values = 0, factor_values = 0;
    std::int64_t fwd_tasks_total = 0, bwd_tasks_total = 0;
};

// vec_index: per subdomain local dof -> device vector index (global dof on 1 GPU).
// global matrix rows (CSR over the device vector) provide the interface residual rows.
DeviceImage build_device_image(const Decomposition& d, const ConstraintSet& cs,
                               const std::vector<CsrMatrix>& locals, const CsrMatrix& global,
                               const BddcSetup& setup);

}  // namespace bddc_b200
