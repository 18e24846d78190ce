#include "setup.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <mutex>
#include <stdexcept>
#include <thread>
#include <unordered_map>

namespace bddc_b200 {
namespace {

template <typename Fn>
void parallel_for(index_t n, index_t workers, Fn&& fn) {
    workers = std::max<index_t>(1, std::min(workers, n));
    if (workers == 1) {
        for (index_t i = 0; i < n; ++i) fn(i);
        return;
    }
    std::vector<std::thread> pool;
    std::exception_ptr err;
    std::mutex mu;
    for (index_t t = 0; t < workers; ++t)
        pool.emplace_back([&, t] {
            try {
                for (index_t i = t; i < n; i += workers) fn(i);
            } catch (...) {
                std::lock_guard<std::mutex> lk(mu);
                if (!err) err = std::current_exception();
            }
        });
    for (auto& th : pool) th.join();
    if (err) std::rethrow_exception(err);
}

std::uint64_t fnv(std::uint64_t h, const void* p, std::size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    for (std::size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ULL;
    return h;
}

// Key identifying a subdomain's setup inputs exactly (matrix, split, constraints,
// coordinates relative to the subdomain origin).
std::string setup_key(const CsrMatrix& A, index_t nI, const CsrMatrix& C,
                      const std::vector<index_t>& rel_coords) {
    std::string k;
    auto put = [&](const void* p, std::size_t n) { k.append(static_cast<const char*>(p), n); };
    put(&A.nrows, sizeof A.nrows);
    put(&nI, sizeof nI);
    put(A.row_offsets.data(), A.row_offsets.size() * sizeof(index_t));
    put(A.col_indices.data(), A.col_indices.size() * sizeof(index_t));
    put(A.values.data(), A.values.size() * sizeof(double));
    put(&C.nrows, sizeof C.nrows);
    put(C.row_offsets.data(), C.row_offsets.size() * sizeof(index_t));
    put(C.col_indices.data(), C.col_indices.size() * sizeof(index_t));
    put(C.values.data(), C.values.size() * sizeof(double));
    put(rel_coords.data(), rel_coords.size() * sizeof(index_t));
    return k;
}

SubdomainSetup setup_one(const CsrMatrix& A, index_t nI, const CsrMatrix& C, const index_t* coords,
                         const FactorOptions& fopt) {
    if (A.nrows != A.ncols || C.ncols != A.nrows)
        throw std::invalid_argument("setup_subdomain: dimension mismatch");
    if (nI < 0 || nI > A.nrows) throw std::invalid_argument("setup_subdomain: interior count out of range");
    SubdomainSetup S;
    S.n_local = A.nrows;
    S.n_interior = nI;
    S.n_iface = A.nrows - nI;
    S.n_primal = C.nrows;
    const index_t ng = S.n_iface, np = S.n_primal, nl = S.n_local;
    for (index_t r = 0; r < C.nrows; ++r)
        for (index_t p = C.row_offsets[r]; p < C.row_offsets[r + 1]; ++p)
            if (C.col_indices[p] < nI && C.values[p] != 0.0)
                throw std::runtime_error("constraint row " + std::to_string(r) +
                                         " touches an interior dof");

    S.factor = factor_subdomain(A, nI, coords, fopt);

    // Reduced saddle [[S, C_G^T], [C_G, 0]] and its inverse.
    const index_t ns = ng + np;
    std::vector<double> M(static_cast<std::size_t>(ns) * ns, 0.0);
    for (index_t r = 0; r < ng; ++r)
        std::memcpy(&M[static_cast<std::size_t>(r) * ns], &S.factor.schur[static_cast<std::size_t>(r) * ng],
                    sizeof(double) * ng);
    for (index_t r = 0; r < np; ++r)
        for (index_t p = C.row_offsets[r]; p < C.row_offsets[r + 1]; ++p) {
            const index_t g = C.col_indices[p] - nI;
            M[static_cast<std::size_t>(ng + r) * ns + g] += C.values[p];
            M[static_cast<std::size_t>(g) * ns + ng + r] += C.values[p];
        }
    dense_inverse(M, ns, "singular saddle system");
    S.K.resize(static_cast<std::size_t>(ng) * ng);
    for (index_t r = 0; r < ng; ++r)
        for (index_t c = 0; c < ng; ++c)
            S.K[static_cast<std::size_t>(r) * ng + c] = M[static_cast<std::size_t>(r) * ns + c];
    S.lambda.resize(static_cast<std::size_t>(np) * np);
    for (index_t r = 0; r < np; ++r)
        for (index_t c = 0; c < np; ++c)
            S.lambda[static_cast<std::size_t>(r) * np + c] = M[static_cast<std::size_t>(ng + r) * ns + ng + c];

    // Coarse basis: Phi_G from the inverse, Phi_I = -A_II^{-1} A_IG Phi_G.
    S.phi.assign(static_cast<std::size_t>(nl) * np, 0.0);
    for (index_t g = 0; g < ng; ++g)
        for (index_t j = 0; j < np; ++j)
            S.phi[static_cast<std::size_t>(nI + g) * np + j] = M[static_cast<std::size_t>(g) * ns + ng + j];
    if (nI > 0) {
        std::vector<double> X(static_cast<std::size_t>(nI) * np, 0.0);
        for (index_t i = 0; i < nI; ++i)
            for (index_t p = A.row_offsets[i]; p < A.row_offsets[i + 1]; ++p) {
                const index_t c = A.col_indices[p];
                if (c < nI) continue;
                for (index_t j = 0; j < np; ++j)
                    X[static_cast<std::size_t>(i) * np + j] -= A.values[p] * S.phi[static_cast<std::size_t>(c) * np + j];
            }
        factor_solve(S.factor, X.data(), np);
        for (index_t i = 0; i < nI; ++i)
            for (index_t j = 0; j < np; ++j)
                S.phi[static_cast<std::size_t>(i) * np + j] = X[static_cast<std::size_t>(i) * np + j];
    }
    // A_ci = Phi^T A Phi in the reference's loop order (dense_matrix.cpp:32-55).
    std::vector<double> T(static_cast<std::size_t>(nl) * np, 0.0);
    for (index_t i = 0; i < nl; ++i)
        for (index_t p = A.row_offsets[i]; p < A.row_offsets[i + 1]; ++p) {
            const index_t k = A.col_indices[p];
            const double a = A.values[p];
            for (index_t j = 0; j < np; ++j)
                T[static_cast<std::size_t>(i) * np + j] += a * S.phi[static_cast<std::size_t>(k) * np + j];
        }
    S.aci.assign(static_cast<std::size_t>(np) * np, 0.0);
    for (index_t i = 0; i < nl; ++i)
        for (index_t r = 0; r < np; ++r) {
            const double pv = S.phi[static_cast<std::size_t>(i) * np + r];
            if (pv == 0.0) continue;
            for (index_t j = 0; j < np; ++j)
                S.aci[static_cast<std::size_t>(r) * np + j] += pv * T[static_cast<std::size_t>(i) * np + j];
        }
    return S;
}

}  // namespace

void dense_inverse(std::vector<double>& a, index_t n, const char* what) {
    std::vector<double> inv(static_cast<std::size_t>(n) * n, 0.0);
    for (index_t i = 0; i < n; ++i) inv[static_cast<std::size_t>(i) * n + i] = 1.0;
    double scale = 0.0;
    for (double v : a) scale = std::max(scale, std::abs(v));
    auto A = [&](index_t r, index_t c) -> double& { return a[static_cast<std::size_t>(r) * n + c]; };
    auto I = [&](index_t r, index_t c) -> double& { return inv[static_cast<std::size_t>(r) * n + c]; };
    for (index_t k = 0; k < n; ++k) {
        index_t piv = k;
        double best = std::abs(A(k, k));
        for (index_t i = k + 1; i < n; ++i)
            if (std::abs(A(i, k)) > best) { best = std::abs(A(i, k)); piv = i; }
        if (!(best > 1e-13 * scale) || !std::isfinite(best))
            throw std::runtime_error(std::string(what) + " (zero pivot at step " + std::to_string(k) + ")");
        if (piv != k) {
            for (index_t c = 0; c < n; ++c) {
                std::swap(A(k, c), A(piv, c));
                std::swap(I(k, c), I(piv, c));
            }
        }
        const double d = A(k, k);
        for (index_t i = k + 1; i < n; ++i) {
            const double f = A(i, k) / d;
            if (f == 0.0) continue;
            A(i, k) = 0.0;
            double* ai = &A(i, 0);
            const double* ak = &A(k, 0);
            for (index_t c = k + 1; c < n; ++c) ai[c] -= f * ak[c];
            double* ii = &I(i, 0);
            const double* ik = &I(k, 0);
            for (index_t c = 0; c < n; ++c) ii[c] -= f * ik[c];
        }
    }
    for (index_t k = n - 1; k >= 0; --k) {
        const double d = A(k, k);
        double* ik = &I(k, 0);
        for (index_t c = 0; c < n; ++c) ik[c] /= d;
        for (index_t i = 0; i < k; ++i) {
            const double f = A(i, k);
            if (f == 0.0) continue;
            double* ii = &I(i, 0);
            for (index_t c = 0; c < n; ++c) ii[c] -= f * ik[c];
        }
    }
    a.swap(inv);
}

void spd_inverse(std::vector<double>& a, index_t n, const char* what) {
    // Cholesky a = L L^T (lower, row-major), then inv = L^-T L^-1.
    auto A = [&](index_t r, index_t c) -> double& { return a[static_cast<std::size_t>(r) * n + c]; };
    for (index_t j = 0; j < n; ++j) {
        double d = A(j, j);
        for (index_t k = 0; k < j; ++k) d -= A(j, k) * A(j, k);
        if (!(d > 0.0)) throw std::runtime_error(std::string(what) + ": not positive definite");
        d = std::sqrt(d);
        A(j, j) = d;
        for (index_t i = j + 1; i < n; ++i) {
            double s = A(i, j);
            const double* ai = &A(i, 0);
            const double* aj = &A(j, 0);
            for (index_t k = 0; k < j; ++k) s -= ai[k] * aj[k];
            A(i, j) = s / d;
        }
    }
    // W = L^{-1} (lower)
    std::vector<double> W(static_cast<std::size_t>(n) * n, 0.0);
    for (index_t c = 0; c < n; ++c)
        for (index_t r = c; r < n; ++r) {
            double acc = r == c ? 1.0 : 0.0;
            for (index_t k = c; k < r; ++k) acc -= A(r, k) * W[static_cast<std::size_t>(k) * n + c];
            W[static_cast<std::size_t>(r) * n + c] = acc / A(r, r);
        }
    // inv = W^T W
    for (index_t i = 0; i < n; ++i)
        for (index_t j = 0; j <= i; ++j) {
            double s = 0.0;
            for (index_t k = i; k < n; ++k)
                s += W[static_cast<std::size_t>(k) * n + i] * W[static_cast<std::size_t>(k) * n + j];
            A(i, j) = s;
            A(j, i) = s;
        }
}

// assemble_coarse (preconditioner.cpp:68-98): triplets in ascending subdomain order, then
// from_triplets (duplicates summed in input order); plus the dense inverse for the GEMV.
void assemble_coarse(BddcSetup& out, const std::vector<const std::vector<double>*>& aci,
                     const std::vector<std::vector<index_t>>& primal_maps, index_t n_coarse,
                     bool dense_inverse) {
    std::vector<Triplet> entries;
    const index_t nsub = static_cast<index_t>(aci.size());
    for (index_t i = 0; i < nsub; ++i) {
        const auto& blk = *aci[i];
        const auto& map = primal_maps[i];
        const index_t np = static_cast<index_t>(map.size());
        if (static_cast<index_t>(blk.size()) != np * np)
            throw std::invalid_argument("assemble_coarse: primal map size mismatch at subdomain " +
                                        std::to_string(i));
        for (index_t r = 0; r < np; ++r)
            for (index_t c = 0; c < np; ++c) {
                if (map[r] < 0 || map[r] >= n_coarse || map[c] < 0 || map[c] >= n_coarse)
                    throw std::out_of_range("assemble_coarse: primal index out of range at subdomain " +
                                            std::to_string(i));
                const double v = blk[static_cast<std::size_t>(r) * np + c];
                if (v != 0.0) entries.push_back({map[r], map[c], v});
            }
    }
    out.coarse_matrix = CsrMatrix::from_triplets(n_coarse, n_coarse, std::move(entries));
    out.coarse_inverse.clear();
    if (!dense_inverse) return;
    const index_t nc = n_coarse;
    out.coarse_inverse.assign(static_cast<std::size_t>(nc) * nc, 0.0);
    for (index_t r = 0; r < nc; ++r)
        for (index_t p = out.coarse_matrix.row_offsets[r]; p < out.coarse_matrix.row_offsets[r + 1]; ++p)
            out.coarse_inverse[static_cast<std::size_t>(r) * nc + out.coarse_matrix.col_indices[p]] =
                out.coarse_matrix.values[p];
    try {
        spd_inverse(out.coarse_inverse, nc, "coarse matrix");
    } catch (const std::runtime_error&) {
        out.coarse_inverse.clear();  // not SPD: the caller falls back to the coarse CG
    }
}

BddcSetup bddc_setup(const std::vector<CsrMatrix>& locals, const Decomposition& d,
                     const ConstraintSet& cs, const index_t* coords, index_t workers,
                     const FactorOptions& fopt, bool assemble, bool dense_inverse) {
    const auto t0 = std::chrono::steady_clock::now();
    const index_t nsub = d.n_subdomains;
    if (static_cast<index_t>(locals.size()) != nsub ||
        static_cast<index_t>(cs.constraint_matrices.size()) != nsub ||
        static_cast<index_t>(cs.primal_maps.size()) != nsub)
        throw std::invalid_argument("bddc setup: subdomain count mismatch");
    BddcSetup out;
    out.subs.resize(nsub);

    // Local coordinates (relative to the subdomain's min corner) and dedup keys.
    std::vector<std::vector<index_t>> lcoords(nsub);
    std::vector<index_t> first_of(nsub, -1);
    {
        std::unordered_map<std::string, index_t> seen;
        for (index_t i = 0; i < nsub; ++i) {
            const auto& dofs = d.subdomain_dofs[i];
            if (coords) {
                lcoords[i].resize(dofs.size() * 2);
                index_t mx = 1 << 30, my = 1 << 30;
                for (index_t g : dofs) { mx = std::min(mx, coords[2 * g]); my = std::min(my, coords[2 * g + 1]); }
                for (std::size_t l = 0; l < dofs.size(); ++l) {
                    lcoords[i][2 * l] = coords[2 * dofs[l]] - mx;
                    lcoords[i][2 * l + 1] = coords[2 * dofs[l] + 1] - my;
                }
            }
            const std::string key =
                setup_key(locals[i], d.interior_counts[i], cs.constraint_matrices[i], lcoords[i]);
            auto it = seen.find(key);
            if (it == seen.end()) { seen.emplace(key, i); first_of[i] = i; }
            else first_of[i] = it->second;
        }
    }
    std::vector<index_t> uniques;
    for (index_t i = 0; i < nsub; ++i)
        if (first_of[i] == i) uniques.push_back(i);
    out.unique_subdomains = static_cast<index_t>(uniques.size());
    parallel_for(static_cast<index_t>(uniques.size()), workers, [&](index_t u) {
        const index_t i = uniques[u];
        try {
            out.subs[i] = setup_one(locals[i], d.interior_counts[i], cs.constraint_matrices[i],
                                    coords ? lcoords[i].data() : nullptr, fopt);
        } catch (const std::exception& e) {
            throw std::runtime_error("bddc setup: subdomain " + std::to_string(i) + ": " + e.what());
        }
    });
    for (index_t i = 0; i < nsub; ++i)
        if (first_of[i] != i) {
            out.subs[i] = out.subs[first_of[i]];
            out.subs[i].dedup_of = first_of[i];
        }

    if (assemble) {
        std::vector<const std::vector<double>*> blocks(nsub);
        for (index_t i = 0; i < nsub; ++i) blocks[i] = &out.subs[i].aci;
        assemble_coarse(out, blocks, cs.primal_maps, cs.n_coarse, dense_inverse);
    }
    out.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return out;
}

}  // namespace bddc_b200
