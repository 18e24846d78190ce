// Condition estimate of the preconditioned operator from the CG coefficients (reference
// SolveReport::condition_estimate, src/pcg.cpp:111-124 and its tridiagonal eigenvalue helper
// :126-173).
//
// CG is Lanczos in disguise: with alpha_j, beta_j of the recurrences, the Lanczos
// tridiagonal T has diagonal 1/alpha_j + beta_{j-1}/alpha_{j-1} and off-diagonal
// sqrt(beta_j)/alpha_j, and its extreme eigenvalues approximate those of M^-1 A. Here they are
// located by bisection on the inertia of T - x I (the signs of its LDL^T pivots count the
// eigenvalues below x), bracketed by the infinity norm of T; O(n) per step, so the estimate
// stays cheap for the ~2,000-step plain-CG runs of C4 / C5.
#include <algorithm>
#include <cmath>
#include <limits>
#include <optional>
#include <vector>

#include "../context.hpp"

namespace bddc_b200 {
namespace {

// Eigenvalues of the symmetric tridiagonal (diagonal a, squared couplings b2[i] between i and
// i+1) strictly below x: the negative pivots of the LDL^T factorisation of T - x I (a zero
// pivot is nudged to the smallest positive normal number).
std::size_t count_below(const std::vector<double>& a, const std::vector<double>& b2, double x) {
    std::size_t neg = 0;
    double piv = 1.0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        piv = (a[i] - x) - (i > 0 ? b2[i - 1] / piv : 0.0);
        if (piv == 0.0) piv = std::numeric_limits<double>::min();
        neg += piv < 0.0 ? 1 : 0;
    }
    return neg;
}

// The k-th smallest eigenvalue (k = 1 .. n) by bisection of [lo, hi] down to 1e-15 relative.
double kth_eigenvalue(const std::vector<double>& a, const std::vector<double>& b2, std::size_t k, double lo,
                      double hi) {
    for (int step = 0; step < 256; ++step) {
        if (hi - lo <= 1e-15 * std::max(1.0, std::abs(hi))) break;
        const double mid = lo + 0.5 * (hi - lo);
        (count_below(a, b2, mid) >= k ? hi : lo) = mid;
    }
    return lo + 0.5 * (hi - lo);
}

}  // namespace

std::optional<double> condition_estimate(const std::vector<double>& alphas, const std::vector<double>& betas) {
    const std::size_t k = alphas.size();
    if (k < 2 || betas.size() + 1 < k) return std::nullopt;  // as the reference: needs two steps
    std::vector<double> a(k), b2(k - 1);
    double norm = 0.0;  // infinity norm of T: every eigenvalue lies in [-norm, norm]
    for (std::size_t j = 0; j < k; ++j) {
        a[j] = 1.0 / alphas[j] + (j > 0 ? betas[j - 1] / alphas[j - 1] : 0.0);
        if (j + 1 < k) {
            const double off = std::sqrt(betas[j]) / alphas[j];
            b2[j] = off * off;
        }
    }
    for (std::size_t j = 0; j < k; ++j)
        norm = std::max(norm, std::abs(a[j]) + (j > 0 ? std::sqrt(b2[j - 1]) : 0.0) + (j + 1 < k ? std::sqrt(b2[j]) : 0.0));
    const double lo = kth_eigenvalue(a, b2, 1, -norm, norm);
    const double hi = kth_eigenvalue(a, b2, k, -norm, norm);
    if (!(lo > 0.0)) return std::nullopt;
    return hi / lo;
}

}  // namespace bddc_b200
