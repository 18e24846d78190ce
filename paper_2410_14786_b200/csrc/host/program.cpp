#include "program.hpp"

#include <algorithm>
#include <atomic>
#include <exception>
#include <mutex>
#include <thread>
#include <utility>

#include "distribute.hpp"
#include "gpu_setup.hpp"
#include <stdexcept>
#include <string>

namespace bddc_b200 {

DeviceImage build_device_image(const Decomposition& d, const ConstraintSet& cs,
                               const std::vector<CsrMatrix>& locals, const CsrMatrix& global,
                               const BddcSetup& setup, int parts, int unit_bytes, const RankPlan* plan,
                               bool harmonic, const std::vector<SetupClass>* classes) {
    DeviceImage img;
    const bool dev = classes != nullptr;
    img.device_values = dev;
    if (dev) {
        img.sub_class.assign(d.n_subdomains, -1);
        for (std::size_t c = 0; c < classes->size(); ++c)
            for (index_t i : (*classes)[c].members) img.sub_class[i] = static_cast<std::int32_t>(c);
    }
    const index_t nsub = d.n_subdomains;
    img.parts = parts;
    img.n_vector = d.global_dofs;
    img.n_coarse = cs.n_coarse;
    img.subs.resize(nsub);

    // ---- global interface dofs and their interior-column rows of A (r' = r - A u0 on G)
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
    // (global subdomain id, hbuf slot): sorted by subdomain before flattening
    std::vector<std::vector<std::pair<std::int32_t, std::int32_t>>> gi_owners(img.gi_dof.size());
    // every vector dof's owners as local-dof slots (ascending subdomain): a CSR built in two
    // passes (counts, then the slots in subdomain order) instead of a list per dof
    img.dof_own_ptr.assign(static_cast<std::size_t>(d.global_dofs) + 1, 0);
    for (index_t i = 0; i < nsub; ++i)
        for (index_t g : d.subdomain_dofs[i]) ++img.dof_own_ptr[g + 1];
    for (index_t g = 0; g < d.global_dofs; ++g) img.dof_own_ptr[g + 1] += img.dof_own_ptr[g];
    img.dof_own_ref.assign(static_cast<std::size_t>(img.dof_own_ptr.back()), 0);
    std::vector<std::int32_t> dof_fill(img.dof_own_ptr.begin(), img.dof_own_ptr.end() - 1);
    std::vector<std::vector<std::int32_t>> c_owners(cs.n_coarse);

    for (index_t i = 0; i < nsub; ++i) {
        const SubdomainSetup& S = setup.subs[i];
        const auto& dofs = d.subdomain_dofs[i];
        const index_t nI = S.n_interior, ng = S.n_iface, np = S.n_primal, nl = S.n_local;
        SubdomainDesc& sd = img.subs[i];
        sd.n_interior = nI;
        sd.n_iface = ng;
        sd.n_primal = np;
        sd.n_local = nl;
        img.max_interior = std::max<std::int32_t>(img.max_interior, nI);
        img.max_iface = std::max<std::int32_t>(img.max_iface, ng);
        img.max_primal = std::max<std::int32_t>(img.max_primal, np);
        img.factor_values += dev ? (*classes)[img.sub_class[i]].factor_values : S.factor.factor_values();

        sd.local_dofs = static_cast<std::int64_t>(img.local_dofs.size());
        for (index_t l = 0; l < nl; ++l) {
            img.dof_own_ref[dof_fill[dofs[l]]++] = static_cast<std::int32_t>(img.local_total + l);
            img.local_dofs.push_back(dofs[l]);
        }
        img.local_total += nl;
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
            const std::int32_t gsub = plan ? plan->subdomains[i] : i;
            gi_owners[gid].push_back({gsub, static_cast<std::int32_t>(img.hbuf_total + gmm)});
        }
        img.hbuf_total += ng;
        sd.cbuf = plan ? plan->cbuf_offset[plan->subdomains[i]] : img.cbuf_total;
        sd.primal = static_cast<std::int64_t>(img.primal.size());
        for (index_t j = 0; j < np; ++j) {
            const index_t q = cs.primal_maps[i][j];
            img.primal.push_back(q);
            if (!plan) c_owners[q].push_back(static_cast<std::int32_t>(img.cbuf_total + j));
        }
        img.cbuf_total += np;

        if (dev) {  // sizes only: the device setup writes the values
            sd.kmat = img.kmat_total;
            img.kmat_total += static_cast<std::int64_t>(ng) * ng;
            sd.phig = img.phig_total;
            img.phig_total += static_cast<std::int64_t>(ng) * np;
            sd.phi = img.phi_total;
            img.phi_total += static_cast<std::int64_t>(nl) * np;
            img.lambda_off.push_back(img.lambda_total);
            img.lambda_total += static_cast<std::int64_t>(np) * np;
        } else {
            sd.kmat = static_cast<std::int64_t>(img.kmat.size());
            img.kmat.insert(img.kmat.end(), S.K.begin(), S.K.end());
            sd.phig = static_cast<std::int64_t>(img.phig.size());
            img.phig.insert(img.phig.end(), S.phi.begin() + static_cast<std::ptrdiff_t>(nI) * np, S.phi.end());
            sd.phi = static_cast<std::int64_t>(img.phi.size());
            img.phi.insert(img.phi.end(), S.phi.begin(), S.phi.end());
        }

        // local A_GI rows of subdomain i (local_correction stage): interior cols as vector index
        const CsrMatrix& A = locals[i];
        sd.lrow_ptr = static_cast<std::int64_t>(img.lrow_ptr.size());
        img.lrow_ptr.push_back(static_cast<std::int32_t>(img.lrow_col.size()));
        for (index_t gmm = 0; gmm < ng; ++gmm) {
            const index_t l = nI + gmm;
            for (index_t p = A.row_offsets[l]; p < A.row_offsets[l + 1]; ++p)
                if (A.col_indices[p] < nI) {
                    img.lrow_col.push_back(dofs[A.col_indices[p]]);
                    img.lrow_val.push_back(A.values[p]);
                }
            img.lrow_ptr.push_back(static_cast<std::int32_t>(img.lrow_col.size()));
        }

    }

    if (dev) {
        // GPU setup: every subdomain's programs are its class's templates with the subdomain's
        // own dof map and coupling values; the stream values are filled on the device
        // offsets sequentially (cheap), then every subdomain's ranges filled on host threads
        for (int k = 0; k < (harmonic ? 3 : 1); ++k) {
            SolvePools& dst = k == 0 ? img.solve : (k == 1 ? img.harm : img.head);
            dst.stream_words = 0;
            struct At { std::size_t units, order, phases, gmap, cptr, cent, parts; };
            std::vector<At> at(nsub);
            std::size_t nu = 0, no = 0, nph = 0, ngm = 0, ncp = 0, nce = 0, npt = 0;
            for (index_t i = 0; i < nsub; ++i) {
                const SolvePools& T = (*classes)[img.sub_class[i]].prog[k];
                ncp += ncp & 1;  // int2 alignment of the parts' {row, end} pairs
                at[i] = {nu, no, nph, ngm, ncp, nce, npt};
                nu += T.units.size();
                no += T.order.size();
                nph += T.phases.size();
                ngm += T.gmap.size();
                ncp += T.couple_ptr.size();
                nce += T.couple_gamma.size();
                npt += T.parts.size();
                img.fills[k].push_back({dst.stream_words, T.words(), img.sub_class[i], k, i});
                dst.stream_words += T.words();
                dst.tile_values += T.tile_values;
                dst.fwd_factor_values += T.fwd_factor_values;
                dst.bwd_factor_values += T.bwd_factor_values;
                dst.n_tiles += T.n_tiles;
                dst.max_loc = std::max(dst.max_loc, T.max_loc);
                dst.max_top = std::max(dst.max_top, T.max_top);
                dst.max_phases = std::max(dst.max_phases, T.max_phases);
                dst.max_units = std::max(dst.max_units, T.max_units);
            }
            dst.units.resize(nu);
            dst.order.resize(no);
            dst.phases.resize(nph);
            dst.gmap.resize(ngm);
            dst.couple_ptr.assign(ncp, 0);
            dst.couple_gamma.resize(nce);
            dst.couple_val.resize(nce);
            dst.parts.resize(npt);
            auto fill = [&](index_t i) {
                const SolvePools& T = (*classes)[img.sub_class[i]].prog[k];
                const At& a = at[i];
                for (std::size_t q = 0; q < T.parts.size(); ++q) {
                    PartDesc pd = T.parts[q];
                    pd.stream += img.fills[k][i].dst;
                    pd.units += static_cast<std::int64_t>(a.units / 2);
                    pd.order += static_cast<std::int64_t>(a.order / 4);
                    pd.phases += static_cast<std::int32_t>(a.phases);
                    pd.gmap += static_cast<std::int64_t>(a.gmap);
                    pd.couple_ptr += static_cast<std::int64_t>(a.cptr);
                    pd.couple_ent += static_cast<std::int64_t>(a.cent);
                    pd.sub = static_cast<std::int32_t>(i);
                    dst.parts[a.parts + q] = pd;
                }
                std::copy(T.units.begin(), T.units.end(), dst.units.begin() + a.units);
                std::copy(T.order.begin(), T.order.end(), dst.order.begin() + a.order);
                std::copy(T.phases.begin(), T.phases.end(), dst.phases.begin() + a.phases);
                std::copy(T.couple_ptr.begin(), T.couple_ptr.end(), dst.couple_ptr.begin() + a.cptr);
                std::copy(T.couple_gamma.begin(), T.couple_gamma.end(), dst.couple_gamma.begin() + a.cent);
                const auto& dofs = d.subdomain_dofs[i];
                for (std::size_t q = 0; q < T.gmap.size(); ++q) dst.gmap[a.gmap + q] = dofs[T.gmap[q]];
                const auto& vals = locals[i].values;
                for (std::size_t q = 0; q < T.couple_src.size(); ++q) dst.couple_val[a.cent + q] = vals[T.couple_src[q]];
            };
            std::atomic<index_t> next{0};
            auto work = [&] {
                for (index_t i = next++; i < nsub; i = next++) fill(i);
            };
            const int nt = std::max(1, std::min<int>(static_cast<int>(std::thread::hardware_concurrency()), nsub));
            std::vector<std::thread> th;
            for (int t = 1; t < nt; ++t) th.emplace_back(work);
            work();
            for (auto& t : th) t.join();
        }
    } else {
    // interior-solve programs (local dof -> vector index = the subdomain map), built per
    // subdomain on host threads and appended in subdomain order (deterministic image)
    {
        const int nprog = harmonic ? 3 : 1;
        std::vector<SolvePools> built(static_cast<std::size_t>(nsub) * nprog);
        std::atomic<index_t> next{0};
        std::exception_ptr err;
        std::mutex err_mu;
        auto work = [&] {
            for (index_t i = next++; i < nsub; i = next++) {
                try {
                    const SubdomainSetup& S = setup.subs[i];
                    const auto& dofs = d.subdomain_dofs[i];
                    build_solve_program(S.factor, locals[i], dofs, i, parts, unit_bytes, built[i * nprog]);
                    if (harmonic) {
                        build_solve_program(S.factor, locals[i], dofs, i, parts, unit_bytes, built[i * nprog + 1], true);
                        build_solve_program(S.factor, locals[i], dofs, i, parts, unit_bytes, built[i * nprog + 2], false,
                                            true);
                    }
                } catch (...) {
                    std::lock_guard<std::mutex> lk(err_mu);
                    if (!err) err = std::current_exception();
                }
            }
        };
        const int nt = std::max(1, std::min<int>(static_cast<int>(std::thread::hardware_concurrency()), nsub));
        std::vector<std::thread> th;
        for (int t = 1; t < nt; ++t) th.emplace_back(work);
        work();
        for (auto& t : th) t.join();
        if (err) std::rethrow_exception(err);
        for (int k = 0; k < nprog; ++k) {  // one allocation per pool
            SolvePools& dst = k == 0 ? img.solve : (k == 1 ? img.harm : img.head);
            std::size_t ns = 0, nu = 0, no = 0, ng = 0;
            for (index_t i = 0; i < nsub; ++i) {
                const SolvePools& b = built[i * nprog + k];
                ns += b.stream.size();
                nu += b.units.size();
                no += b.order.size();
                ng += b.gmap.size();
            }
            dst.stream.reserve(ns);
            dst.units.reserve(nu);
            dst.order.reserve(no);
            dst.gmap.reserve(ng);
        }
        for (index_t i = 0; i < nsub; ++i) {
            append_pools(img.solve, std::move(built[i * nprog]));
            if (harmonic) {
                append_pools(img.harm, std::move(built[i * nprog + 1]));
                append_pools(img.head, std::move(built[i * nprog + 2]));
            }
        }
    }

    }  // host-built programs

    if (plan) {
        // remote interface contributions (filled by the interface exchange) and the
        // gathered coarse buffer of all ranks
        if (img.hbuf_total != plan->n_local_slots) throw std::logic_error("rank plan: hbuf slot layout mismatch");
        for (index_t l = 0; l < plan->n_rows; ++l)
            for (const auto& [gsub, k] : plan->remote_owners[l]) {
                const std::int32_t gid = gid_of[l];
                if (gid < 0) throw std::logic_error("rank plan: remote owner of an interior dof");
                gi_owners[gid].push_back({gsub, static_cast<std::int32_t>(plan->n_local_slots + k)});
            }
        img.hbuf_total += plan->n_remote_slots;
        for (std::size_t j = 0; j < plan->primal_all.size(); ++j)
            for (std::size_t t = 0; t < plan->primal_all[j].size(); ++t)
                c_owners[plan->primal_all[j][t]].push_back(static_cast<std::int32_t>(plan->cbuf_offset[j] + t));
        img.cbuf_total = static_cast<std::int64_t>(plan->world) * plan->cbuf_pad;
    }
    for (auto& o : gi_owners) std::stable_sort(o.begin(), o.end());
    img.gi_own_ptr.assign(1, 0);
    for (const auto& o : gi_owners) {
        for (const auto& e : o) img.gi_own_ref.push_back(e.second);
        img.gi_own_ptr.push_back(static_cast<std::int32_t>(img.gi_own_ref.size()));
    }

    auto flatten = [](const std::vector<std::vector<std::int32_t>>& lists, std::vector<std::int32_t>& ptr,
                      std::vector<std::int32_t>& ref) {
        ptr.assign(1, 0);
        for (const auto& o : lists) {
            ref.insert(ref.end(), o.begin(), o.end());
            ptr.push_back(static_cast<std::int32_t>(ref.size()));
        }
    };
    flatten(c_owners, img.c_own_ptr, img.c_own_ref);
    img.coarse_inv = setup.coarse_inverse;
    return img;
}

}  // namespace bddc_b200
