// Multi-GPU partition of a decomposed problem: one rank per B200.
//
// The reference is single-process (src/parallel.hpp:19-45 is its only parallelism; every
// cross-subdomain sum is a serial loop in ascending subdomain order, e.g.
// src/preconditioner.cpp:141-147,168-169,189-190). Here each rank owns a rectangular block
// of subdomains and works on a rank-local vector index space
//
//     [ owned dofs | other dofs of my subdomains | halo ]
//       0 .. n_owned  .. n_rows                   .. n_local
//
// * owned: the rank of the lowest-index subdomain containing the dof owns it; PCG dot
//   products sum over owned entries only (then a gather of per-rank partials, summed in
//   rank order on every rank, so every rank takes identical decisions);
// * rows [0, n_rows): every dof of the rank's subdomains; the rank computes them
//   redundantly and bit-identically to its neighbours (same global CSR rows in the same
//   column order, same owner-ordered interface sums);
// * halo: the one-layer A-graph neighbours of the rank's dofs that live only on other
//   ranks; refreshed by a halo exchange (grouped by owner rank, ascending global dof).
//
// Cross-rank sums keep the reference's order: an interface dof's z = sum of the h_i of
// every subdomain containing it in ascending global subdomain index (remote h_i arrive
// by the interface exchange into "remote slots"), and r_c sums the c_i of ALL subdomains
// in ascending order from a gathered buffer; the distributed apply is therefore
// bit-identical to the single-GPU one.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "../context.hpp"

namespace bddc_b200 {

// Rectangular blocks of the kx x ky subdomain layout (factor world = px * py as square as
// possible, px | kx, py | ky); contiguous id ranges when the problem is not a grid.
std::vector<int> block_partition(const Decomposition& d, int world);

struct RankPlan {
    int rank = 0;
    int world = 1;
    std::vector<int> sub_rank;               // rank of every global subdomain
    std::vector<index_t> subdomains;         // this rank's global subdomain ids, ascending
    std::vector<index_t> local_to_global;    // rank-local vector index -> global dof
    index_t n_owned = 0;
    index_t n_rows = 0;
    index_t n_local = 0;

    // halo exchange of a vector (u0 and p): per peer, ncclSend of the packed entries
    // halo_send_idx[send_off[q] .. send_off[q+1]) and ncclRecv into [n_rows + recv_off[q], ...)
    std::vector<int> halo_peers;
    std::vector<index_t> halo_send_off, halo_send_idx, halo_recv_off;

    // interface exchange of h_i values: local hbuf slots packed per peer; received values
    // land in remote slots [recv_off[q], recv_off[q+1]) after the local slots
    std::vector<int> iface_peers;
    std::vector<index_t> iface_send_off, iface_send_slot, iface_recv_off;
    index_t n_local_slots = 0;   // sum of n_iface over the rank's subdomains
    index_t n_remote_slots = 0;
    // per local row: remote contributions (global subdomain id, remote slot index)
    std::vector<std::vector<std::pair<index_t, index_t>>> remote_owners;

    // gathered coarse contributions: rank q's c_i occupy [q * cbuf_pad, (q+1) * cbuf_pad)
    index_t cbuf_pad = 0;
    std::vector<index_t> cbuf_offset;        // per global subdomain
    std::vector<std::vector<index_t>> primal_all;  // every global subdomain's primal map

    ProblemData local;                       // rank-local problem (vector space above)
};

// sub_rank: optional subdomain -> rank assignment (nullptr: block_partition).
RankPlan make_rank_plan(const ProblemData& global, int rank, int world, const int* sub_rank = nullptr);

}  // namespace bddc_b200
