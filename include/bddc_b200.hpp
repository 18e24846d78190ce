// bddc_b200.hpp — header-only C++20 drop-in for the reference's BDDC API, over the C-ABI in
// bddc_b200.h (no CUDA or torch types; link with paper_2410_14786_b200/lib/libbddc_b200.so).
//
// Mirrors (file:line in /root/reference/proj):
//   bddc_b200::Preconditioner  bddc::Preconditioner   include/bddc/preconditioner.hpp:62-104
//   bddc_b200::pcg             bddc::pcg with M = Preconditioner::apply
//                                                    include/bddc/pcg.hpp:43-45, src/study.cpp:113-119
//   SolverOptions / SolveReport                      include/bddc/pcg.hpp:17-30
// The constructor is duck-typed on the reference's own CsrMatrix / Decomposition /
// ConstraintSet (include/bddc/csr_matrix.hpp:27-47, decomposition.hpp:29-48), so a caller
// of the reference passes the very objects it already has. Status codes become the
// reference's exception types with the messages verbatim (std::invalid_argument,
// std::out_of_range, std::runtime_error).
#ifndef BDDC_B200_HPP
#define BDDC_B200_HPP

#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "bddc_b200.h"

namespace bddc_b200 {

struct SolverOptions {
    double rel_tolerance = 1e-8;
    double abs_tolerance = 0.0;
    std::int32_t max_iterations = 1000;
    bool record_history = false;
};

struct SolveReport {
    std::int32_t iterations = 0;
    double final_relative_residual = 0.0;
    std::vector<double> residual_history;
    std::optional<double> condition_estimate;
    bool converged = false;
};

namespace detail {

inline void check(int code, const char* msg) {
    if (code == BDDC_OK) return;
    const std::string m = msg ? msg : "";
    if (code == BDDC_ERR_INVALID_ARGUMENT) throw std::invalid_argument(m);
    if (code == BDDC_ERR_OUT_OF_RANGE) throw std::out_of_range(m);
    throw std::runtime_error(m);
}

template <class Csr>
bddc_csr_view view(const Csr& A) {
    return {static_cast<int32_t>(A.nrows), static_cast<int32_t>(A.ncols), A.row_offsets.data(),
            A.col_indices.data(), A.values.data()};
}

}  // namespace detail

// Drop-in for bddc::Preconditioner: same constructor arguments, same apply / stage methods.
// The per-subdomain worker pool becomes host setup threads; the apply runs on a B200.
class Preconditioner {
public:
    template <class Csr, class Decomp, class Constraints, class Options = SolverOptions>
    Preconditioner(const Csr& global_matrix, const std::vector<Csr>& local_matrices, const Decomp& decomp,
                   const Constraints& constraints, std::int32_t worker_count = 1,
                   Options coarse_options = Options{1e-12, 0.0, 500, false}, std::int32_t device = 0) {
        const std::size_t ns = local_matrices.size();
        std::vector<bddc_csr_view> locals(ns), cons(ns);
        std::vector<std::int64_t> doff{0}, poff{0};
        std::vector<std::int32_t> dofs, primal, entity;
        std::vector<double> weights;
        std::vector<std::uint8_t> kind;
        for (std::size_t i = 0; i < ns; ++i) {
            locals[i] = detail::view(local_matrices[i]);
            cons[i] = detail::view(constraints.constraint_matrices[i]);
            dofs.insert(dofs.end(), decomp.subdomain_dofs[i].begin(), decomp.subdomain_dofs[i].end());
            weights.insert(weights.end(), decomp.weights[i].begin(), decomp.weights[i].end());
            doff.push_back(static_cast<std::int64_t>(dofs.size()));
            primal.insert(primal.end(), constraints.primal_maps[i].begin(), constraints.primal_maps[i].end());
            poff.push_back(static_cast<std::int64_t>(primal.size()));
        }
        for (const auto& c : decomp.classes) {
            kind.push_back(static_cast<std::uint8_t>(c.kind));
            entity.push_back(static_cast<std::int32_t>(c.entity));
        }
        bddc_problem_view v{};
        v.n_subdomains = static_cast<int32_t>(ns);
        v.global_dofs = static_cast<int32_t>(decomp.global_dofs);
        v.n_coarse = static_cast<int32_t>(constraints.n_coarse);
        v.global_matrix = detail::view(global_matrix);
        v.local_matrices = locals.data();
        v.constraint_matrices = cons.data();
        v.dof_offsets = doff.data();
        v.subdomain_dofs = dofs.data();
        v.weights = weights.data();
        v.interior_counts = decomp.interior_counts.data();
        v.primal_offsets = poff.data();
        v.primal_maps = primal.data();
        v.class_kind = kind.empty() ? nullptr : kind.data();
        v.class_entity = entity.empty() ? nullptr : entity.data();
        v.multiplicity = decomp.multiplicity.empty() ? nullptr : decomp.multiplicity.data();
        detail::check(bddc_problem_from_view(&v, &problem_), bddc_last_error());
        bddc_gpu_options o;
        bddc_default_gpu_options(&o);
        o.device = device;
        o.workers = worker_count;
        // the reference's default coarse CG (1e-12, 500) is replaced by the exact replicated
        // dense coarse solve; any other coarse options select the reference-faithful coarse CG
        const bool reference_default = coarse_options.rel_tolerance == 1e-12 &&
                                       coarse_options.abs_tolerance == 0.0 && coarse_options.max_iterations == 500;
        o.coarse_mode = reference_default ? BDDC_COARSE_DIRECT : BDDC_COARSE_CG;
        o.coarse_rel_tolerance = coarse_options.rel_tolerance;
        o.coarse_abs_tolerance = coarse_options.abs_tolerance;
        o.coarse_max_iterations = static_cast<int32_t>(coarse_options.max_iterations);
        const int rc = bddc_gpu_create(problem_, &o, &ctx_);
        if (rc != BDDC_OK) {
            const std::string msg = bddc_last_error();
            bddc_problem_destroy(problem_);
            detail::check(rc, msg.c_str());
        }
        n_ = v.global_dofs;
    }
    ~Preconditioner() {
        if (ctx_) bddc_gpu_destroy(ctx_);
        if (problem_) bddc_problem_destroy(problem_);
    }
    Preconditioner(const Preconditioner&) = delete;
    Preconditioner& operator=(const Preconditioner&) = delete;

    std::vector<double> apply(std::span<const double> r) const {
        size_check(r);
        std::vector<double> z(n_);
        detail::check(bddc_gpu_apply(ctx_, r.data(), z.data()), bddc_gpu_last_error(ctx_));
        return z;
    }
    std::vector<double> coarse_correction(std::span<const double> r) const { return stage(BDDC_STAGE_COARSE, r); }
    std::vector<double> local_correction(std::span<const double> r) const { return stage(BDDC_STAGE_LOCAL, r); }
    std::vector<double> interior_correction(std::span<const double> r) const { return stage(BDDC_STAGE_INTERIOR, r); }
    std::vector<double> static_condensation_correction(std::span<const double> r, std::span<const double> v1,
                                                       std::span<const double> v2) const {
        size_check(r);
        size_check(v1);
        size_check(v2);
        std::vector<double> out(n_);
        detail::check(bddc_gpu_stage(ctx_, BDDC_STAGE_STATIC_CONDENSATION, r.data(), v1.data(), v2.data(), out.data()),
                      bddc_gpu_last_error(ctx_));
        return out;
    }

    // pcg(A, b, M = this->apply, opts, x) with the whole loop on the device.
    SolveReport pcg(std::span<const double> b, const SolverOptions& opts, std::vector<double>& x,
                    bool precondition = true) const {
        size_check(b);
        x.assign(n_, 0.0);
        bddc_solver_options so{opts.rel_tolerance, opts.abs_tolerance, opts.max_iterations,
                               opts.record_history ? 1 : 0};
        bddc_solve_report rep{};
        std::vector<double> hist(static_cast<std::size_t>(opts.max_iterations) + 1);
        detail::check(bddc_gpu_pcg(ctx_, b.data(), &so, precondition ? 1 : 0, x.data(), &rep, hist.data(),
                                   static_cast<int32_t>(hist.size())),
                      bddc_gpu_last_error(ctx_));
        SolveReport out;
        out.iterations = rep.iterations;
        out.final_relative_residual = rep.final_relative_residual;
        out.residual_history.assign(hist.begin(), hist.begin() + rep.history_length);
        if (rep.has_condition_estimate) out.condition_estimate = rep.condition_estimate;
        out.converged = rep.converged != 0;
        return out;
    }

    std::int32_t size() const { return n_; }

private:
    void size_check(std::span<const double> r) const {
        if (static_cast<std::int32_t>(r.size()) != n_)
            throw std::invalid_argument("bddc apply: residual size mismatch");
    }
    std::vector<double> stage(int32_t st, std::span<const double> r) const {
        size_check(r);
        std::vector<double> out(n_);
        detail::check(bddc_gpu_stage(ctx_, st, r.data(), nullptr, nullptr, out.data()), bddc_gpu_last_error(ctx_));
        return out;
    }
    bddc_problem* problem_ = nullptr;
    bddc_gpu_ctx* ctx_ = nullptr;
    std::int32_t n_ = 0;
};

// Drop-in for bddc::pcg(A, b, M, opts, x) when M is the BDDC preconditioner (the reference
// harness's lambda, src/study.cpp:113-119): A is the preconditioner's global matrix.
inline SolveReport pcg(const Preconditioner& M, std::span<const double> b, const SolverOptions& opts,
                       std::vector<double>& x) {
    return M.pcg(b, opts, x);
}

}  // namespace bddc_b200

#endif  // BDDC_B200_HPP
