#include "gpu_setup.hpp"

#include <algorithm>
#include <atomic>
#include <exception>
#include <mutex>
#include <numeric>
#include <stdexcept>
#include <thread>
#include <unordered_map>

namespace bddc_b200 {
namespace {

template <typename T>
void put(std::string& k, const T* p, std::size_t n) {
    k.append(reinterpret_cast<const char*>(p), n * sizeof(T));
}

// Multifrontal plan, Schur assembly and value layout of one class (from its representative).
void plan_class(SetupClass& C, const CsrMatrix& A, const CsrMatrix& Cm) {
    const InteriorFactor& F = C.sym;
    const index_t nI = F.n_interior, ng = F.n_iface;
    const index_t nsn = static_cast<index_t>(F.snodes.size());
    auto position = [&](index_t local) { return local < nI ? F.iperm[local] : local; };

    C.sn_nc.resize(nsn);
    C.sn_m.resize(nsn);
    C.sn_mi.resize(nsn);
    C.front_off.resize(nsn);
    C.layout.linv_off.resize(nsn);
    C.layout.bl_off.resize(nsn);
    std::int64_t off = 0, dv = 0;
    for (index_t s = 0; s < nsn; ++s) {
        const Supernode& S = F.snodes[s];
        const std::int64_t nc = S.size(), m = static_cast<std::int64_t>(S.rows.size()), f = nc + m;
        C.sn_nc[s] = static_cast<std::int32_t>(nc);
        C.sn_m[s] = static_cast<std::int32_t>(m);
        C.sn_mi[s] = static_cast<std::int32_t>(S.n_interior_rows);
        C.front_off[s] = off;
        off += f * f;
        C.max_front = std::max<std::int32_t>(C.max_front, static_cast<std::int32_t>(f));
        C.layout.linv_off[s] = dv;
        dv += nc * nc;
    }
    for (index_t s = 0; s < nsn; ++s) {
        C.layout.bl_off[s] = dv;
        dv += static_cast<std::int64_t>(C.sn_mi[s]) * C.sn_nc[s];
    }
    C.front_total = off;
    C.layout.total = dv;
    if (dv > (std::int64_t(1) << 31) - 1) throw std::runtime_error("gpu setup: subdomain value array too large");

    // front position of a position p within supernode s's front
    std::vector<std::int32_t> fpos(A.nrows, -1);
    auto bind = [&](index_t s) {
        const Supernode& S = F.snodes[s];
        for (index_t c = S.col_begin; c < S.col_end; ++c) fpos[c] = static_cast<std::int32_t>(c - S.col_begin);
        for (std::size_t a = 0; a < S.rows.size(); ++a) fpos[S.rows[a]] = static_cast<std::int32_t>(S.size() + a);
    };
    auto unbind = [&](index_t s) {
        const Supernode& S = F.snodes[s];
        for (index_t c = S.col_begin; c < S.col_end; ++c) fpos[c] = -1;
        for (index_t r : S.rows) fpos[r] = -1;
    };
    std::vector<std::vector<index_t>> children(nsn);
    for (index_t s = 0; s < nsn; ++s)
        if (F.snodes[s].parent >= 0) children[F.snodes[s].parent].push_back(s);
        else C.roots.push_back(static_cast<std::int32_t>(s));

    C.asc_ptr.assign(1, 0);
    C.ch_ptr.assign(1, 0);
    std::vector<std::vector<std::int32_t>> em(nsn);
    for (index_t s = 0; s < nsn; ++s) {
        const Supernode& S = F.snodes[s];
        const std::int64_t f = S.size() + static_cast<std::int64_t>(S.rows.size());
        bind(s);
        for (index_t c = S.col_begin; c < S.col_end; ++c) {
            const index_t v = F.perm[c];
            for (index_t q = A.row_offsets[v]; q < A.row_offsets[v + 1]; ++q) {
                const index_t pos = position(A.col_indices[q]);
                if (pos < c) continue;
                if (fpos[pos] < 0) throw std::logic_error("gpu setup: matrix entry outside its front");
                C.asc_pos.push_back(static_cast<std::int32_t>(fpos[c] * f + fpos[pos]));
                C.asc_csr.push_back(static_cast<std::int32_t>(q));
            }
        }
        C.asc_ptr.push_back(static_cast<std::int32_t>(C.asc_pos.size()));
        for (index_t ch : children[s]) {
            C.ch_id.push_back(static_cast<std::int32_t>(ch));
            for (index_t r : F.snodes[ch].rows) {
                if (fpos[r] < 0) throw std::logic_error("gpu setup: child row outside the parent front");
                em[ch].push_back(fpos[r]);
            }
        }
        C.ch_ptr.push_back(static_cast<std::int32_t>(C.ch_id.size()));
        unbind(s);
    }
    C.em_ptr.assign(1, 0);
    for (index_t s = 0; s < nsn; ++s) {
        C.em_pos.insert(C.em_pos.end(), em[s].begin(), em[s].end());
        C.em_ptr.push_back(static_cast<std::int32_t>(C.em_pos.size()));
    }
    // supernodes by height
    std::int32_t hmax = 0;
    for (const Supernode& S : F.snodes) hmax = std::max<std::int32_t>(hmax, S.height);
    C.level_ptr.assign(1, 0);
    for (std::int32_t h = 0; h <= hmax; ++h) {
        for (index_t s = 0; s < nsn; ++s)
            if (F.snodes[s].height == h) C.level_sn.push_back(static_cast<std::int32_t>(s));
        C.level_ptr.push_back(static_cast<std::int32_t>(C.level_sn.size()));
    }
    // Schur complement: A_GG entries, then the roots' updates (interface rows only)
    for (index_t l = nI; l < A.nrows; ++l)
        for (index_t q = A.row_offsets[l]; q < A.row_offsets[l + 1]; ++q) {
            const index_t c = A.col_indices[q];
            if (c < nI) continue;
            C.sgg_pos.push_back(static_cast<std::int32_t>((l - nI) * ng + (c - nI)));
            C.sgg_csr.push_back(static_cast<std::int32_t>(q));
        }
    C.root_gamma_ptr.assign(1, 0);
    for (std::int32_t r : C.roots) {
        for (index_t p : F.snodes[r].rows) {
            if (p < nI) throw std::logic_error("gpu setup: interior root update has interior rows");
            C.root_gamma.push_back(static_cast<std::int32_t>(p - nI));
        }
        C.root_gamma_ptr.push_back(static_cast<std::int32_t>(C.root_gamma.size()));
    }
    // constraints on the interface columns
    C.c_ptr.assign(1, 0);
    for (index_t r = 0; r < Cm.nrows; ++r) {
        for (index_t q = Cm.row_offsets[r]; q < Cm.row_offsets[r + 1]; ++q) {
            const index_t col = Cm.col_indices[q];
            if (col < nI) {
                if (Cm.values[q] != 0.0)
                    throw std::runtime_error("constraint row " + std::to_string(r) + " touches an interior dof");
                continue;
            }
            C.c_col.push_back(static_cast<std::int32_t>(col - nI));
            C.c_val.push_back(Cm.values[q]);
        }
        C.c_ptr.push_back(static_cast<std::int32_t>(C.c_col.size()));
    }
}

}  // namespace

std::string setup_pattern_key(const CsrMatrix& A, index_t nI, const CsrMatrix& C, const std::vector<index_t>& rel) {
    std::string k;
    put(k, &A.nrows, 1);
    put(k, &nI, 1);
    put(k, A.row_offsets.data(), A.row_offsets.size());
    put(k, A.col_indices.data(), A.col_indices.size());
    put(k, &C.nrows, 1);
    put(k, C.row_offsets.data(), C.row_offsets.size());
    put(k, C.col_indices.data(), C.col_indices.size());
    put(k, C.values.data(), C.values.size());
    put(k, rel.data(), rel.size());
    return k;
}

std::vector<SetupClass> plan_gpu_setup(const std::vector<CsrMatrix>& locals, const Decomposition& d,
                                       const ConstraintSet& cs, const index_t* coords, const FactorOptions& fopt,
                                       int parts, int unit_bytes, bool harmonic, int workers) {
    const index_t nsub = d.n_subdomains;
    if (static_cast<index_t>(locals.size()) != nsub || static_cast<index_t>(cs.constraint_matrices.size()) != nsub)
        throw std::invalid_argument("bddc setup: subdomain count mismatch");
    std::vector<std::vector<index_t>> rel(nsub);
    std::vector<SetupClass> classes;
    {
        std::unordered_map<std::string, std::size_t> seen;
        for (index_t i = 0; i < nsub; ++i) {
            const auto& dofs = d.subdomain_dofs[i];
            if (coords) {
                rel[i].resize(dofs.size() * 2);
                index_t mx = 1 << 30, my = 1 << 30;
                for (index_t g : dofs) {
                    mx = std::min(mx, coords[2 * g]);
                    my = std::min(my, coords[2 * g + 1]);
                }
                for (std::size_t l = 0; l < dofs.size(); ++l) {
                    rel[i][2 * l] = coords[2 * dofs[l]] - mx;
                    rel[i][2 * l + 1] = coords[2 * dofs[l] + 1] - my;
                }
            }
            const CsrMatrix& A = locals[i];
            if (A.nrows != A.ncols || cs.constraint_matrices[i].ncols != A.nrows)
                throw std::invalid_argument("bddc setup: subdomain " + std::to_string(i) +
                                            ": setup_subdomain: dimension mismatch");
            const auto key = setup_pattern_key(A, d.interior_counts[i], cs.constraint_matrices[i], rel[i]);
            auto it = seen.find(key);
            if (it == seen.end()) {
                it = seen.emplace(key, classes.size()).first;
                classes.emplace_back();
                classes.back().rep = i;
            }
            classes[it->second].members.push_back(i);
        }
    }
    // two parallel passes: the symbolic factor + plan of every class, then the class x program
    // templates (the three programs of a class are independent)
    std::exception_ptr err;
    std::mutex mu;
    auto run = [&](std::size_t n_tasks, auto&& task) {
        std::atomic<std::size_t> next{0};
        auto work = [&] {
            for (std::size_t t = next++; t < n_tasks; t = next++) {
                const index_t i = classes[t % classes.size()].rep;
                try {
                    task(t);
                } catch (const std::exception& e) {
                    std::lock_guard<std::mutex> lk(mu);
                    if (!err)
                        err = std::make_exception_ptr(
                            std::runtime_error("bddc setup: subdomain " + std::to_string(i) + ": " + e.what()));
                }
            }
        };
        const int nt = std::max(1, std::min<int>(workers, static_cast<int>(n_tasks)));
        std::vector<std::thread> th;
        for (int t = 1; t < nt; ++t) th.emplace_back(work);
        work();
        for (auto& t : th) t.join();
        if (err) std::rethrow_exception(err);
    };
    run(classes.size(), [&](std::size_t c) {
        SetupClass& C = classes[c];
        const index_t i = C.rep;
        const CsrMatrix& A = locals[i];
        const index_t nI = d.interior_counts[i];
        C.n_local = A.nrows;
        C.n_interior = nI;
        C.n_iface = A.nrows - nI;
        C.n_primal = cs.constraint_matrices[i].nrows;
        C.nnz = A.nnz();
        C.sym = symbolic_factor(A, nI, coords ? rel[i].data() : nullptr, fopt);
        C.factor_values = C.sym.factor_values();
        plan_class(C, A, cs.constraint_matrices[i]);
    });
    const int nprog = harmonic ? 3 : 1;
    run(classes.size() * nprog, [&](std::size_t t) {
        SetupClass& C = classes[t % classes.size()];
        const int q = static_cast<int>(t / classes.size());
        const CsrMatrix& A = locals[C.rep];
        std::vector<index_t> ident(A.nrows);
        std::iota(ident.begin(), ident.end(), 0);
        // 0: full solve, 1: harmonic (pruned forward), 2: head (pruned backward)
        build_solve_program(C.sym, A, ident, C.rep, parts, unit_bytes, C.prog[q], q == 1, q == 2, &C.layout);
    });
    return classes;
}

}  // namespace bddc_b200
