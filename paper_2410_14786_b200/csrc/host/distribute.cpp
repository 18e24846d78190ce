#include "distribute.hpp"

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>

namespace bddc_b200 {

std::vector<int> block_partition(const Decomposition& d, int world) {
    const index_t nsub = d.n_subdomains;
    if (world < 1) throw std::invalid_argument("distribute: world size must be positive");
    if (world > 64) throw std::invalid_argument("distribute: at most 64 ranks");
    if (world > nsub) throw std::invalid_argument("distribute: more ranks than subdomains");
    std::vector<int> out(nsub);
    if (d.kx > 0 && d.ky > 0 && d.kx * d.ky == nsub) {
        int best_px = 0;
        double best = 1e300;
        for (int px = 1; px <= world; ++px) {
            if (world % px) continue;
            const int py = world / px;
            if (d.kx % px || d.ky % py) continue;
            const double bx = static_cast<double>(d.kx) / px, by = static_cast<double>(d.ky) / py;
            const double score = std::abs(bx - by) + 1e-3 * px;  // squarest blocks, fewer columns
            if (score < best) { best = score; best_px = px; }
        }
        if (best_px) {
            const int px = best_px, py = world / px;
            const index_t bx = d.kx / px, by = d.ky / py;
            for (index_t sy = 0; sy < d.ky; ++sy)
                for (index_t sx = 0; sx < d.kx; ++sx)
                    out[sy * d.kx + sx] = static_cast<int>((sy / by) * px + sx / bx);
            return out;
        }
    }
    for (index_t j = 0; j < nsub; ++j) out[j] = static_cast<int>((static_cast<std::int64_t>(j) * world) / nsub);
    return out;
}

RankPlan make_rank_plan(const ProblemData& G, int rank, int world, const int* sub_rank_in) {
    const Decomposition& d = G.decomposition;
    const index_t nsub = d.n_subdomains, n = d.global_dofs;
    if (rank < 0 || rank >= world) throw std::invalid_argument("distribute: rank out of range");
    RankPlan P;
    P.rank = rank;
    P.world = world;
    if (sub_rank_in) {
        P.sub_rank.assign(sub_rank_in, sub_rank_in + nsub);
        for (int q : P.sub_rank)
            if (q < 0 || q >= world) throw std::invalid_argument("distribute: subdomain rank out of range");
    } else {
        P.sub_rank = block_partition(d, world);
    }
    if (world > 64) throw std::invalid_argument("distribute: at most 64 ranks");
    std::vector<std::vector<index_t>> subs_of(world);
    for (index_t j = 0; j < nsub; ++j) subs_of[P.sub_rank[j]].push_back(j);
    for (int q = 0; q < world; ++q)
        if (subs_of[q].empty()) throw std::invalid_argument("distribute: rank " + std::to_string(q) + " owns no subdomain");
    P.subdomains = subs_of[rank];

    // ranks containing each dof, and its lowest subdomain
    std::vector<std::uint64_t> mask(n, 0);
    std::vector<index_t> min_sub(n, nsub);
    for (index_t j = 0; j < nsub; ++j)
        for (index_t g : d.subdomain_dofs[j]) {
            mask[g] |= std::uint64_t(1) << P.sub_rank[j];
            min_sub[g] = std::min(min_sub[g], j);
        }
    auto owner = [&](index_t g) { return P.sub_rank[min_sub[g]]; };
    const std::uint64_t me = std::uint64_t(1) << rank;

    // halo: columns of rows a rank holds that the rank does not hold itself
    std::vector<std::vector<index_t>> recv_from(world), send_to(world);
    const CsrMatrix& A = G.global_matrix;
    for (index_t g = 0; g < n; ++g) {
        const std::uint64_t mg = mask[g];
        if (!mg) throw std::invalid_argument("distribute: dof " + std::to_string(g) + " in no subdomain");
        for (index_t p = A.row_offsets[g]; p < A.row_offsets[g + 1]; ++p) {
            const index_t c = A.col_indices[p];
            std::uint64_t missing = mg & ~mask[c];
            if (!missing) continue;
            const int oc = owner(c);
            if (missing & me) recv_from[oc].push_back(c);
            if (oc == rank)
                for (int q = 0; q < world; ++q)
                    if (missing >> q & 1) send_to[q].push_back(c);
        }
    }
    for (int q = 0; q < world; ++q) {
        for (auto* v : {&recv_from[q], &send_to[q]}) {
            std::sort(v->begin(), v->end());
            v->erase(std::unique(v->begin(), v->end()), v->end());
        }
    }

    // rank-local ordering: owned | held, not owned | halo by owner rank
    std::vector<index_t> g2l(n, -1);
    for (index_t g = 0; g < n; ++g)
        if ((mask[g] & me) && owner(g) == rank) P.local_to_global.push_back(g);
    P.n_owned = static_cast<index_t>(P.local_to_global.size());
    for (index_t g = 0; g < n; ++g)
        if ((mask[g] & me) && owner(g) != rank) P.local_to_global.push_back(g);
    P.n_rows = static_cast<index_t>(P.local_to_global.size());
    P.halo_recv_off.push_back(0);
    P.halo_send_off.push_back(0);
    for (int q = 0; q < world; ++q) {
        if (q == rank || (recv_from[q].empty() && send_to[q].empty())) continue;
        P.halo_peers.push_back(q);
        P.local_to_global.insert(P.local_to_global.end(), recv_from[q].begin(), recv_from[q].end());
        P.halo_recv_off.push_back(static_cast<index_t>(P.local_to_global.size()) - P.n_rows);
    }
    P.n_local = static_cast<index_t>(P.local_to_global.size());
    for (index_t l = 0; l < P.n_local; ++l) g2l[P.local_to_global[l]] = l;
    for (int q : P.halo_peers) {
        for (index_t g : send_to[q]) {
            if (g2l[g] < 0 || g2l[g] >= P.n_owned) throw std::logic_error("distribute: halo send of a non-owned dof");
            P.halo_send_idx.push_back(g2l[g]);
        }
        P.halo_send_off.push_back(static_cast<index_t>(P.halo_send_idx.size()));
    }

    // interface exchange of h_i: (subdomain ascending, gamma ascending) on both sides
    std::vector<index_t> slot_base(nsub, -1);
    {
        index_t s = 0;
        for (index_t j : P.subdomains) {
            slot_base[j] = s;
            s += static_cast<index_t>(d.subdomain_dofs[j].size()) - d.interior_counts[j];
        }
        P.n_local_slots = s;
    }
    P.remote_owners.assign(P.n_rows, {});
    P.iface_send_off.push_back(0);
    P.iface_recv_off.push_back(0);
    for (int q = 0; q < world; ++q) {
        if (q == rank) continue;
        const std::uint64_t qb = std::uint64_t(1) << q;
        bool any = false;
        for (index_t j : P.subdomains) {
            const auto& dofs = d.subdomain_dofs[j];
            const index_t nI = d.interior_counts[j];
            for (index_t gm = 0; gm + nI < static_cast<index_t>(dofs.size()); ++gm)
                if (mask[dofs[nI + gm]] & qb) {
                    P.iface_send_slot.push_back(slot_base[j] + gm);
                    any = true;
                }
        }
        for (index_t j : subs_of[q]) {
            const auto& dofs = d.subdomain_dofs[j];
            const index_t nI = d.interior_counts[j];
            for (index_t gm = 0; gm + nI < static_cast<index_t>(dofs.size()); ++gm) {
                const index_t g = dofs[nI + gm];
                if (mask[g] & me) {
                    P.remote_owners[g2l[g]].push_back({j, P.n_remote_slots++});
                    any = true;
                }
            }
        }
        if (!any) continue;
        P.iface_peers.push_back(q);
        P.iface_send_off.push_back(static_cast<index_t>(P.iface_send_slot.size()));
        P.iface_recv_off.push_back(P.n_remote_slots);
    }

    // gathered coarse contributions
    const ConstraintSet& cs = G.constraints;
    P.primal_all = cs.primal_maps;
    std::vector<index_t> per_rank(world, 0);
    P.cbuf_offset.assign(nsub, 0);
    for (index_t j = 0; j < nsub; ++j) {
        P.cbuf_offset[j] = per_rank[P.sub_rank[j]];
        per_rank[P.sub_rank[j]] += static_cast<index_t>(cs.primal_maps[j].size());
    }
    P.cbuf_pad = *std::max_element(per_rank.begin(), per_rank.end());
    for (index_t j = 0; j < nsub; ++j) P.cbuf_offset[j] += P.sub_rank[j] * P.cbuf_pad;

    // rank-local problem
    ProblemData& L = P.local;
    Decomposition& ld = L.decomposition;
    ld.k = ld.kx = ld.ky = 0;
    ld.n_subdomains = static_cast<index_t>(P.subdomains.size());
    ld.global_dofs = P.n_local;
    ld.classes.resize(P.n_local);
    ld.multiplicity.resize(P.n_local);
    for (index_t l = 0; l < P.n_local; ++l) {
        ld.classes[l] = d.classes[P.local_to_global[l]];
        ld.multiplicity[l] = d.multiplicity[P.local_to_global[l]];
    }
    for (index_t j : P.subdomains) {
        std::vector<index_t> dofs(d.subdomain_dofs[j].size());
        for (std::size_t l = 0; l < dofs.size(); ++l) dofs[l] = g2l[d.subdomain_dofs[j][l]];
        ld.subdomain_dofs.push_back(std::move(dofs));
        ld.interior_counts.push_back(d.interior_counts[j]);
        ld.weights.push_back(d.weights[j]);
        L.local_matrices.push_back(G.local_matrices[j]);
        L.constraints.constraint_matrices.push_back(cs.constraint_matrices[j]);
        L.constraints.primal_maps.push_back(cs.primal_maps[j]);
    }
    L.constraints.n_coarse = cs.n_coarse;
    CsrMatrix& LA = L.global_matrix;
    LA.nrows = LA.ncols = P.n_local;
    LA.row_offsets.assign(1, 0);
    for (index_t l = 0; l < P.n_local; ++l) {
        if (l < P.n_rows) {
            const index_t g = P.local_to_global[l];
            for (index_t p = A.row_offsets[g]; p < A.row_offsets[g + 1]; ++p) {
                const index_t c = g2l[A.col_indices[p]];
                if (c < 0) throw std::logic_error("distribute: column outside the halo");
                LA.col_indices.push_back(c);  // global column order kept: same summation order
                LA.values.push_back(A.values[p]);
            }
        }
        LA.row_offsets.push_back(static_cast<index_t>(LA.values.size()));
    }
    if (!G.coords.empty()) {
        L.coords.resize(static_cast<std::size_t>(P.n_local) * 2);
        for (index_t l = 0; l < P.n_local; ++l) {
            L.coords[2 * l] = G.coords[2 * P.local_to_global[l]];
            L.coords[2 * l + 1] = G.coords[2 * P.local_to_global[l] + 1];
        }
    }
    return P;
}

}  // namespace bddc_b200
