#pragma once

#include "fused_comm.cuh"

#include "common.cuh"

namespace bddc_b200 {

// static shared memory of the solve kernel (reductions, fused-exchange bookkeeping), kept out
// of the dynamic carve-up
constexpr int kSolveStaticSmemReserve = 1024;

struct SolveParams {
    const double* skip;  // pipelined PCG: skip when scal[2] / scal[3] is set (null: never)
    const PartDesc* parts;
    const SubdomainDesc* subs;
    const double* stream;
    const std::int32_t* units;   // {offset16, bytes} pairs
    const std::int32_t* phases;
    const std::int32_t* gmap;
    // MODE 1 (second interior solve of the apply): coupling + interface gather
    const std::int32_t* couple_ptr;
    const std::int32_t* couple_gamma;
    const double* couple_val;
    const std::int32_t* iface_gid;
    const std::int32_t* iface_dof;
    const std::int32_t* iface_writer;  // per local interface slot: the dof it writes (its writer), else -1
    const std::int32_t* gi_own_ptr;
    // per local interface slot: the hbuf slots of its owners (ascending subdomain, -1 padded) as
    // an int4; x <= -2: more than four owners, the owner list of global interface dof -2 - x
    const std::int32_t* iface_own4;
    const std::int32_t* gi_own_ref;
    const double* hbuf;
    const double* in;
    double* out;
    const double* u0;  // MODE 3: the first interior solve's result (z_I = u0 - harmonic extension)
    // Split apply (head program + harmonic program): MODE 0 stores its forward result y0 =
    // L^-1 r_I (part-local order, at part.gmap) into y_out before the (pruned) backward sweep;
    // MODE 3 with y_in forms y0 - L^-1 A_IG z_G before its backward sweep, whose result is z_I
    // itself (one full backward sweep per apply instead of two). Null: off.
    double* y_out;
    const double* y_in;
    // MODE 3, fused PCG dot product: per CTA, sum of dot_r[i] * z[i] over the z entries it writes
    // with i < n_dot, into dot_part[blockIdx.x] (null: off)
    const double* dot_r;
    double* dot_part;
    int n_dot;
    int unit_bytes;  // set by the launcher
    int slot_shift;  // log2(ring slots per warp)
    int max_loc;
    int max_top;
    int max_iface;
    long long* stats;  // diagnostics (BDDC_SOLVE_STATS): per CTA, per warp {total, mbarrier wait,
                       // CTA-barrier wait, units} cycles of the launch; null = off
    // multi-GPU fused LL exchanges (null on one GPU): MODE 0 publishes the halo of u0; MODE 3
    // reads the peers' h_i (hbuf slots >= ll_h_base) from its LL buffer and publishes the halo
    // of z with r.z
    Publish pub;
    const ll_word* ll_h;
    const std::uint64_t* seq_h;
    int ll_h_base;
};

struct SolveLaunch {
    int n_parts = 0;      // CTAs
    int cluster = 1;      // parts per subdomain (1 or 2)
    std::size_t smem = 0;
    int unit_bytes = 0;
    int slot_shift = 1;
};

std::size_t interior_solve_smem(int max_loc, int max_top, int max_iface, int unit_bytes, int slots_per_warp);
int max_solve_smem(int device);
// mode 0: out[I] = A_II^{-1} in[I]
// mode 1: z_G = sum of h over owners (written to out), out[I] = A_II^{-1}(in_I - A_IG z_G)
// mode 2: out[I] = A_II^{-1}(in_I - A_IG h_own)   (local saddle solve, stage hook)
// mode 3: z_G as mode 1, out[I] = u0_I - A_II^{-1} A_IG z_G  (harmonic-extension program)
void launch_interior_solve(SolveParams P, const SolveLaunch& L, int mode, cudaStream_t stream);

}  // namespace bddc_b200
