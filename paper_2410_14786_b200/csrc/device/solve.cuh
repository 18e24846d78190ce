#pragma once

#include "common.cuh"

namespace bddc_b200 {

struct SolveParams {
    const SubdomainDesc* subs;
    int first_subdomain;
    const double* stream;
    const TileTask* tasks;
    const std::int32_t* phases;
    const std::int32_t* idx;
    const std::int32_t* gmap;
    // MODE 1 (second interior solve of the apply): coupling + interface gather
    const std::int32_t* couple_ptr;
    const std::int32_t* couple_gamma;
    const double* couple_val;
    const std::int32_t* iface_gid;
    const std::int32_t* iface_dof;
    const std::int32_t* iface_writer;
    const std::int32_t* gi_own_ptr;
    const std::int32_t* gi_own_ref;
    const double* hbuf;
    // vectors
    const double* in;
    double* out;
};

std::size_t interior_solve_smem(int max_interior, int max_iface);
void launch_interior_solve(const SolveParams& P, int mode, int n_subdomains, std::size_t smem,
                           cudaStream_t stream);

}  // namespace bddc_b200
