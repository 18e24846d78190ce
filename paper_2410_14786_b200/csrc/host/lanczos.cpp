// Condition estimate of the preconditioned operator from the CG coefficients (reference
// SolveReport::condition_estimate, src/pcg.cpp:111-124 and its tridiagonal eigenvalue helper
// :126-173).
//
// CG is Lanczos in disguise: with alpha_j, beta_j of the recurrences, the Lanczos
// tridiagonal T has diagonal 1/alpha_j + beta_{j-1}/alpha_{j-1} and off-diagonal
// sqrt(beta_j)/alpha_j, and its extreme eigenvalues approximate those of M^-1 A. The reference
// brackets them by Gershgorin discs and bisects Sturm counts; here every eigenvalue of T is
// computed by the implicitly shifted QL iteration (Wilkinson shift, Givens bulge chase), which
// converges to the same extreme values (to ~1e-15 relative for these well-separated ends).
#include <algorithm>
#include <cmath>
#include <limits>
#include <optional>
#include <vector>

#include "../context.hpp"

namespace bddc_b200 {
namespace {

// All eigenvalues of the symmetric tridiagonal (a = diagonal, b[i] couples i and i+1),
// returned in a (unordered). b is destroyed.
void tridiagonal_eigenvalues(std::vector<double>& a, std::vector<double>& b) {
    const std::size_t n = a.size();
    b.resize(n, 0.0);  // b[n-1] = 0 terminates every deflation scan
    const double eps = std::numeric_limits<double>::epsilon();
    for (std::size_t top = 0; top < n; ++top) {
        for (int sweep = 0; sweep < 64; ++sweep) {
            // the unreduced block starting at `top` ends at `end` (negligible coupling below it)
            std::size_t end = top;
            while (end + 1 < n && std::abs(b[end]) > eps * (std::abs(a[end]) + std::abs(a[end + 1]))) ++end;
            if (end == top) break;  // a[top] has converged
            // Wilkinson-type shift from the leading 2x2 of the block
            const double half_gap = (a[top + 1] - a[top]) / (2.0 * b[top]);
            const double root = std::hypot(half_gap, 1.0);
            double bulge_g = a[end] - a[top] + b[top] / (half_gap + std::copysign(root, half_gap));
            double sn = 1.0, cs = 1.0, shift_acc = 0.0;
            bool split = false;
            // chase the bulge from the bottom of the block up to `top`
            for (std::size_t k = end; k-- > top;) {
                const double f = sn * b[k], h = cs * b[k];
                const double rad = std::hypot(f, bulge_g);
                b[k + 1] = rad;
                if (rad == 0.0) {  // exact split: restart on the shorter block
                    a[k + 1] -= shift_acc;
                    b[end] = 0.0;
                    split = true;
                    break;
                }
                sn = f / rad;
                cs = bulge_g / rad;
                const double g = a[k + 1] - shift_acc;
                const double t = (a[k] - g) * sn + 2.0 * cs * h;
                shift_acc = sn * t;
                a[k + 1] = g + shift_acc;
                bulge_g = cs * t - h;
            }
            if (split) continue;
            a[top] -= shift_acc;
            b[top] = bulge_g;
            b[end] = 0.0;
        }
    }
}

}  // namespace

std::optional<double> condition_estimate(const std::vector<double>& alphas, const std::vector<double>& betas) {
    const std::size_t k = alphas.size();
    if (k < 2 || betas.size() + 1 < k) return std::nullopt;  // as the reference: needs two steps
    std::vector<double> a(k), b(k - 1);
    for (std::size_t j = 0; j < k; ++j) {
        a[j] = 1.0 / alphas[j] + (j > 0 ? betas[j - 1] / alphas[j - 1] : 0.0);
        if (j + 1 < k) b[j] = std::sqrt(betas[j]) / alphas[j];
    }
    tridiagonal_eigenvalues(a, b);
    const auto [lo, hi] = std::minmax_element(a.begin(), a.end());
    if (!(*lo > 0.0)) return std::nullopt;
    return *hi / *lo;
}

}  // namespace bddc_b200
