#include "program.hpp"

#include <algorithm>
#include <map>
#include <numeric>
#include <stdexcept>
#include <string>

namespace bddc_b200 {
namespace {

struct Chunk {
    index_t snode;
    index_t start;  // row offset within the supernode
    index_t rows;
    std::vector<TileTask> tiles;      // m_off filled later (relative to tile data)
    std::vector<std::vector<double>> data;
    std::int64_t cost = 0;
};

struct PassBuilder {
    std::vector<TileTask>& tasks;
    std::vector<double>& stream;
    std::vector<std::int32_t>& phases;
    std::int64_t task_base, stream_base;
    std::int32_t n_phases = 0;
    std::int64_t values = 0;

    // Assign chunks of one phase to warps (LPT on cost) and append tasks + data.
    void emit_phase(std::vector<Chunk>& chunks) {
        if (chunks.empty()) return;
        std::vector<index_t> order(chunks.size());
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(),
                         [&](index_t a, index_t b) { return chunks[a].cost > chunks[b].cost; });
        std::vector<std::int64_t> load(kSolveWarps, 0);
        std::vector<std::vector<index_t>> per_warp(kSolveWarps);
        for (index_t c : order) {
            const int w = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
            load[w] += chunks[c].cost + 64;
            per_warp[w].push_back(c);
        }
        for (auto& v : per_warp) std::sort(v.begin(), v.end());
        phases.push_back(static_cast<std::int32_t>(tasks.size() - task_base));
        for (int w = 0; w < kSolveWarps; ++w) {
            for (index_t c : per_warp[w]) {
                Chunk& ch = chunks[c];
                for (std::size_t t = 0; t < ch.tiles.size(); ++t) {
                    TileTask task = ch.tiles[t];
                    task.m_off = static_cast<std::uint32_t>(stream.size() - stream_base);
                    stream.insert(stream.end(), ch.data[t].begin(), ch.data[t].end());
                    values += static_cast<std::int64_t>(ch.data[t].size());
                    if (stream.size() % 2) stream.push_back(0.0);  // 16-byte tile alignment
                    tasks.push_back(task);
                }
            }
            phases.push_back(static_cast<std::int32_t>(tasks.size() - task_base));
        }
        ++n_phases;
    }
};

}  // namespace

DeviceImage build_device_image(const Decomposition& d, const ConstraintSet& cs,
                               const std::vector<CsrMatrix>& locals, const CsrMatrix& global,
                               const BddcSetup& setup) {
    DeviceImage img;
    const index_t nsub = d.n_subdomains;
    img.n_vector = d.global_dofs;
    img.n_coarse = cs.n_coarse;
    img.subs.resize(nsub);

    // ---- global interface dofs and their interior-column rows of A
    std::vector<std::int32_t> gid_of(d.global_dofs, -1);
    for (index_t g = 0; g < d.global_dofs; ++g)
        if (d.classes[g].kind != DofKind::interior) {
            gid_of[g] = static_cast<std::int32_t>(img.gi_dof.size());
            img.gi_dof.push_back(g);
        }
    img.gi_row_ptr.push_back(0);
    for (std::int32_t g : img.gi_dof) {
        for (index_t p = global.row_offsets[g]; p < global.row_offsets[g + 1]; ++p) {
            const index_t c = global.col_indices[p];
            if (d.classes[c].kind == DofKind::interior) {
                img.gi_row_col.push_back(c);
                img.gi_row_val.push_back(global.values[p]);
            }
        }
        img.gi_row_ptr.push_back(static_cast<std::int32_t>(img.gi_row_col.size()));
    }
    std::vector<std::vector<std::int32_t>> gi_owners(img.gi_dof.size());
    std::vector<std::vector<std::int32_t>> c_owners(cs.n_coarse);

    for (index_t i = 0; i < nsub; ++i) {
        const SubdomainSetup& S = setup.subs[i];
        const InteriorFactor& F = S.factor;
        const auto& dofs = d.subdomain_dofs[i];
        const index_t nI = S.n_interior, ng = S.n_iface, np = S.n_primal, nl = S.n_local;
        if (nI > 65535 - 64) throw std::runtime_error("subdomain interior too large for the solve kernel");
        SubdomainDesc& sd = img.subs[i];
        sd.n_interior = nI;
        sd.n_iface = ng;
        sd.n_primal = np;
        sd.n_local = nl;
        img.max_interior = std::max<std::int32_t>(img.max_interior, nI);
        img.max_iface = std::max<std::int32_t>(img.max_iface, ng);
        img.max_primal = std::max<std::int32_t>(img.max_primal, np);
        img.factor_values += F.factor_values();

        // maps
        sd.gmap = static_cast<std::int64_t>(img.gmap.size());
        for (index_t p = 0; p < nI; ++p) img.gmap.push_back(dofs[F.perm[p]]);
        sd.local_dofs = static_cast<std::int64_t>(img.local_dofs.size());
        img.local_dofs.insert(img.local_dofs.end(), dofs.begin(), dofs.end());
        sd.iface = static_cast<std::int64_t>(img.iface_dof.size());
        sd.hbuf = img.hbuf_total;
        for (index_t gmm = 0; gmm < ng; ++gmm) {
            const index_t g = dofs[nI + gmm];
            img.iface_dof.push_back(g);
            img.iface_w.push_back(d.weights[i][nI + gmm]);
            const std::int32_t gid = gid_of[g];
            if (gid < 0) throw std::runtime_error("interface dof classified interior");
            img.iface_gid.push_back(gid);
            img.iface_writer.push_back(gi_owners[gid].empty() ? 1 : 0);
            gi_owners[gid].push_back(static_cast<std::int32_t>(img.hbuf_total + gmm));
        }
        img.hbuf_total += ng;
        sd.cbuf = img.cbuf_total;
        sd.primal = static_cast<std::int64_t>(img.primal.size());
        for (index_t j = 0; j < np; ++j) {
            const index_t q = cs.primal_maps[i][j];
            img.primal.push_back(q);
            c_owners[q].push_back(static_cast<std::int32_t>(img.cbuf_total + j));
        }
        img.cbuf_total += np;

        // dense interface blocks
        sd.kmat = static_cast<std::int64_t>(img.kmat.size());
        img.kmat.insert(img.kmat.end(), S.K.begin(), S.K.end());
        sd.phig = static_cast<std::int64_t>(img.phig.size());
        img.phig.insert(img.phig.end(), S.phi.begin() + static_cast<std::ptrdiff_t>(nI) * np, S.phi.end());
        sd.phi = static_cast<std::int64_t>(img.phi.size());
        img.phi.insert(img.phi.end(), S.phi.begin(), S.phi.end());

        // coupling A_IG in permuted interior order (for the second interior solve)
        const CsrMatrix& A = locals[i];
        sd.couple_ptr = static_cast<std::int64_t>(img.couple_ptr.size());
        sd.couple_ent = static_cast<std::int64_t>(img.couple_gamma.size());
        std::int32_t cnt = 0;
        img.couple_ptr.push_back(0);
        for (index_t p = 0; p < nI; ++p) {
            const index_t l = F.perm[p];
            for (index_t q = A.row_offsets[l]; q < A.row_offsets[l + 1]; ++q) {
                const index_t c = A.col_indices[q];
                if (c >= nI) {
                    img.couple_gamma.push_back(c - nI);
                    img.couple_val.push_back(A.values[q]);
                    ++cnt;
                }
            }
            img.couple_ptr.push_back(cnt);
        }

        // ---- interior solve program
        const auto& sn = F.snodes;
        const index_t nsn = static_cast<index_t>(sn.size());
        index_t H = 0;
        for (const auto& s : sn) H = std::max(H, s.height + 1);
        std::vector<index_t> owner(nI, -1);
        for (index_t s = 0; s < nsn; ++s)
            for (index_t c = sn[s].col_begin; c < sn[s].col_end; ++c) owner[c] = s;
        sd.idx_base = static_cast<std::int64_t>(img.idx.size());
        std::vector<std::int64_t> rows_idx(nsn, -1);  // index-list offsets of R_s^I
        for (index_t s = 0; s < nsn; ++s) {
            if (sn[s].n_interior_rows == 0) continue;
            rows_idx[s] = static_cast<std::int64_t>(img.idx.size()) - sd.idx_base;
            img.idx.insert(img.idx.end(), sn[s].rows.begin(), sn[s].rows.begin() + sn[s].n_interior_rows);
        }

        auto chunks_of_height = [&](index_t h) {
            std::vector<Chunk> out;
            std::map<std::pair<index_t, index_t>, index_t> at;  // (snode, chunk) -> index
            for (index_t s = 0; s < nsn; ++s) {
                if (sn[s].height != h) continue;
                for (index_t r0 = 0; r0 < sn[s].size(); r0 += 32) {
                    Chunk c;
                    c.snode = s;
                    c.start = r0;
                    c.rows = std::min<index_t>(32, sn[s].size() - r0);
                    at[{s, r0 / 32}] = static_cast<index_t>(out.size());
                    out.push_back(std::move(c));
                }
            }
            return std::make_pair(std::move(out), std::move(at));
        };

        // forward pass
        sd.fwd_stream = static_cast<std::int64_t>(img.stream.size());
        sd.fwd_tasks = static_cast<std::int64_t>(img.tasks.size());
        sd.fwd_phases = static_cast<std::int32_t>(img.phases.size());
        PassBuilder fwd{img.tasks, img.stream, img.phases, sd.fwd_tasks, sd.fwd_stream};
        for (index_t h = 0; h < H; ++h) {
            // phase A: gathers from descendants into height-h supernodes
            {
                auto [chunks, at] = chunks_of_height(h);
                for (index_t dsn = 0; dsn < nsn; ++dsn) {
                    const Supernode& D = sn[dsn];
                    const index_t nd = D.size();
                    index_t a = 0;
                    while (a < D.n_interior_rows) {
                        const index_t r = D.rows[a];
                        const index_t s = owner[r];
                        if (sn[s].height != h) { ++a; continue; }
                        const index_t rel = r - sn[s].col_begin;
                        const index_t chunk = rel / 32;
                        const index_t cstart = sn[s].col_begin + chunk * 32;
                        const index_t cend = std::min(sn[s].col_end, cstart + 32);
                        index_t k = 1;
                        while (a + k < D.n_interior_rows && D.rows[a + k] == r + k && r + k < cend) ++k;
                        Chunk& ch = chunks[at.at({s, chunk})];
                        TileTask t{};
                        t.in_ref = static_cast<std::uint32_t>(D.col_begin);
                        t.out_base = static_cast<std::uint16_t>(cstart);
                        t.ncols = static_cast<std::uint16_t>(nd);
                        t.nrows = static_cast<std::uint8_t>(k);
                        t.lane_off = static_cast<std::uint8_t>(r - cstart);
                        t.nvalid = static_cast<std::uint8_t>(cend - cstart);
                        std::vector<double> data(static_cast<std::size_t>(k) * nd);
                        for (index_t j = 0; j < nd; ++j)
                            for (index_t ii = 0; ii < k; ++ii)
                                data[static_cast<std::size_t>(j) * k + ii] =
                                    D.B[static_cast<std::size_t>(a + ii) * nd + j];
                        ch.cost += static_cast<std::int64_t>(k) * nd + 16;
                        ch.tiles.push_back(t);
                        ch.data.push_back(std::move(data));
                        a += k;
                    }
                }
                std::vector<Chunk> used;
                for (auto& c : chunks)
                    if (!c.tiles.empty()) {
                        c.tiles.front().flags |= kTaskFirst;
                        c.tiles.back().flags |= kTaskLast;
                        used.push_back(std::move(c));
                    }
                fwd.emit_phase(used);
            }
            // phase B: diagonal blocks x_s = L_ss^{-1} t_s
            {
                auto [chunks, at] = chunks_of_height(h);
                (void)at;
                for (Chunk& ch : chunks) {
                    const Supernode& s = sn[ch.snode];
                    const index_t ns = s.size(), r0 = ch.start, nr = ch.rows, nc = r0 + nr;
                    TileTask t{};
                    t.in_ref = static_cast<std::uint32_t>(s.col_begin);
                    t.out_base = static_cast<std::uint16_t>(s.col_begin + r0);
                    t.ncols = static_cast<std::uint16_t>(nc);
                    t.nrows = static_cast<std::uint8_t>(nr);
                    t.lane_off = 0;
                    t.nvalid = static_cast<std::uint8_t>(nr);
                    t.flags = kTaskFirst | kTaskLast | kTaskDiag;
                    std::vector<double> data(static_cast<std::size_t>(nr) * nc, 0.0);
                    for (index_t j = 0; j < nc; ++j)
                        for (index_t ii = 0; ii < nr; ++ii)
                            if (j <= r0 + ii)
                                data[static_cast<std::size_t>(j) * nr + ii] =
                                    s.Linv[static_cast<std::size_t>(r0 + ii) * ns + j];
                    ch.cost = static_cast<std::int64_t>(nr) * nc;
                    ch.tiles.push_back(t);
                    ch.data.push_back(std::move(data));
                }
                fwd.emit_phase(chunks);
            }
        }
        sd.n_fwd_phases = fwd.n_phases;
        img.fwd_values += fwd.values;

        // backward pass
        sd.bwd_stream = static_cast<std::int64_t>(img.stream.size());
        sd.bwd_tasks = static_cast<std::int64_t>(img.tasks.size());
        sd.bwd_phases = static_cast<std::int32_t>(img.phases.size());
        PassBuilder bwd{img.tasks, img.stream, img.phases, sd.bwd_tasks, sd.bwd_stream};
        for (index_t h = H - 1; h >= 0; --h) {
            // phase A: u_s = x_s - B_s^T y[R_s]
            {
                auto [chunks, at] = chunks_of_height(h);
                (void)at;
                std::vector<Chunk> used;
                for (Chunk& ch : chunks) {
                    const Supernode& s = sn[ch.snode];
                    const index_t mI = s.n_interior_rows;
                    if (mI == 0) continue;
                    const index_t ns = s.size(), q0 = ch.start, nq = ch.rows;
                    TileTask t{};
                    t.in_ref = static_cast<std::uint32_t>(rows_idx[ch.snode]);
                    t.out_base = static_cast<std::uint16_t>(s.col_begin + q0);
                    t.ncols = static_cast<std::uint16_t>(mI);
                    t.nrows = static_cast<std::uint8_t>(nq);
                    t.lane_off = 0;
                    t.nvalid = static_cast<std::uint8_t>(nq);
                    t.flags = kTaskFirst | kTaskLast | kTaskInIndexed;
                    std::vector<double> data(static_cast<std::size_t>(nq) * mI);
                    for (index_t j = 0; j < mI; ++j)
                        for (index_t ii = 0; ii < nq; ++ii)
                            data[static_cast<std::size_t>(j) * nq + ii] =
                                s.B[static_cast<std::size_t>(j) * ns + q0 + ii];
                    ch.cost = static_cast<std::int64_t>(nq) * mI;
                    ch.tiles.push_back(t);
                    ch.data.push_back(std::move(data));
                    used.push_back(std::move(ch));
                }
                bwd.emit_phase(used);
            }
            // phase B: y_s = L_ss^{-T} u_s
            {
                auto [chunks, at] = chunks_of_height(h);
                (void)at;
                for (Chunk& ch : chunks) {
                    const Supernode& s = sn[ch.snode];
                    const index_t ns = s.size(), q0 = ch.start, nq = ch.rows, nc = ns - q0;
                    TileTask t{};
                    t.in_ref = static_cast<std::uint32_t>(s.col_begin + q0);
                    t.out_base = static_cast<std::uint16_t>(s.col_begin + q0);
                    t.ncols = static_cast<std::uint16_t>(nc);
                    t.nrows = static_cast<std::uint8_t>(nq);
                    t.lane_off = 0;
                    t.nvalid = static_cast<std::uint8_t>(nq);
                    t.flags = kTaskFirst | kTaskLast | kTaskDiag;
                    std::vector<double> data(static_cast<std::size_t>(nq) * nc, 0.0);
                    for (index_t j = 0; j < nc; ++j)
                        for (index_t ii = 0; ii < nq; ++ii)
                            if (j >= ii)
                                data[static_cast<std::size_t>(j) * nq + ii] =
                                    s.Linv[static_cast<std::size_t>(q0 + j) * ns + q0 + ii];
                    ch.cost = static_cast<std::int64_t>(nq) * nc;
                    ch.tiles.push_back(t);
                    ch.data.push_back(std::move(data));
                }
                bwd.emit_phase(chunks);
            }
        }
        sd.n_bwd_phases = bwd.n_phases;
        img.bwd_values += bwd.values;
    }
    img.fwd_tasks_total = 0;
    img.bwd_tasks_total = static_cast<std::int64_t>(img.tasks.size());

    img.gi_own_ptr.push_back(0);
    for (auto& o : gi_owners) {
        img.gi_own_ref.insert(img.gi_own_ref.end(), o.begin(), o.end());
        img.gi_own_ptr.push_back(static_cast<std::int32_t>(img.gi_own_ref.size()));
    }
    img.c_own_ptr.push_back(0);
    for (auto& o : c_owners) {
        img.c_own_ref.insert(img.c_own_ref.end(), o.begin(), o.end());
        img.c_own_ptr.push_back(static_cast<std::int32_t>(img.c_own_ref.size()));
    }
    img.coarse_inv = setup.coarse_inverse;
    return img;
}

}  // namespace bddc_b200
