// dropin_check — TEST INFRASTRUCTURE ONLY. Demonstrates the drop-in boundary from the
// reference's side: a program written against the reference API (/root/reference/proj,
// compiled from its unmodified sources by oracle/Makefile) swaps bddc::Preconditioner +
// bddc::pcg for bddc_b200::Preconditioner + bddc_b200::pcg (include/bddc_b200.hpp) on the
// SAME objects, and checks that the results agree (iterations exact, histories and
// solutions within 1e-10). Runs on a B200 (tests/test_gpu_parity.py::test_reference_dropin).
//
//   dropin_check <k> <m>     prints one JSON line, exit 0 iff parity holds
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <span>
#include <vector>

#include "bddc/decomposition.hpp"
#include "bddc/grid.hpp"
#include "bddc/pcg.hpp"
#include "bddc/preconditioner.hpp"
#include "bddc/study.hpp"
#include "bddc_b200.hpp"

int main(int argc, char** argv) {
    const int k = argc > 1 ? std::atoi(argv[1]) : 4;
    const int m = argc > 2 ? std::atoi(argv[2]) : 16;
    try {
        // --- the reference caller's code (src/study.cpp:77-120), unchanged up to the swap
        const bddc::StructuredGrid grid(k * m);
        bddc::PoissonProblem p = bddc::assemble_poisson(grid, k);
        const bddc::ConstraintSet cs = bddc::build_constraints(p.decomposition);
        const std::vector<double> b = bddc::study_rhs(grid.free_dofs, 1);
        bddc::SolverOptions opts;
        opts.rel_tolerance = 1e-8;
        opts.max_iterations = 10000;
        opts.record_history = true;

        const bddc::Preconditioner ref(p.global_matrix, p.local_matrices, p.decomposition, cs, 1);
        std::vector<double> xr;
        const bddc::SolveReport rr = bddc::pcg(
            p.global_matrix, b,
            [&](std::span<const double> r, std::span<double> z) {
                const auto v = ref.apply(r);
                std::copy(v.begin(), v.end(), z.begin());
            },
            opts, xr);
        const std::vector<double> zr = ref.apply(b);

        // --- the swap: same objects into the B200 preconditioner
        const bddc_b200::Preconditioner gpu(p.global_matrix, p.local_matrices, p.decomposition, cs, 1);
        std::vector<double> xg;
        const bddc_b200::SolveReport rg =
            bddc_b200::pcg(gpu, b, {opts.rel_tolerance, opts.abs_tolerance, opts.max_iterations, true}, xg);
        const std::vector<double> zg = gpu.apply(b);

        double zerr = 0, zmax = 0, xerr = 0, xmax = 0, herr = 0;
        for (std::size_t i = 0; i < zr.size(); ++i) {
            zerr = std::max(zerr, std::abs(zr[i] - zg[i]));
            zmax = std::max(zmax, std::abs(zr[i]));
            xerr = std::max(xerr, std::abs(xr[i] - xg[i]));
            xmax = std::max(xmax, std::abs(xr[i]));
        }
        const std::size_t nh = std::min(rr.residual_history.size(), rg.residual_history.size());
        for (std::size_t i = 0; i < nh; ++i)
            herr = std::max(herr, std::abs(rr.residual_history[i] - rg.residual_history[i]) /
                                      std::max(rr.residual_history[i], 1e-6));
        const bool ok = rr.iterations == rg.iterations && rg.converged && zerr <= 1e-10 * zmax &&
                        xerr <= 1e-10 * xmax && herr <= 1e-10;
        std::printf("{\"k\": %d, \"m\": %d, \"iterations\": [%d, %d], \"apply_rel_err\": %.3e, "
                    "\"x_rel_err\": %.3e, \"history_err\": %.3e, \"ok\": %s}\n",
                    k, m, static_cast<int>(rg.iterations), static_cast<int>(rr.iterations), zerr / zmax,
                    xerr / xmax, herr, ok ? "true" : "false");
        // error mapping: a size mismatch is std::invalid_argument in both
        try {
            (void)gpu.apply(std::span<const double>(b.data(), b.size() - 1));
            std::printf("expected invalid_argument\n");
            return 1;
        } catch (const std::invalid_argument&) {
        }
        return ok ? 0 : 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "dropin_check error: %s\n", e.what());
        return 2;
    }
}
