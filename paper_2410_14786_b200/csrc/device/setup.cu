// GPU setup kernels (device/setup.cuh). Every kernel works on one class of identically
// patterned subdomains (host/gpu_setup.hpp): the plan arrays are shared, the values are per
// member. All reductions run in a fixed order (no atomics on values): the setup is
// deterministic run to run.
#include "setup.cuh"

#include <algorithm>
#include <cstdlib>

namespace bddc_b200 {
namespace {

constexpr int kMfThreads = 256;
constexpr int kPanel = 32;  // columns factored per shared-memory panel

__device__ __forceinline__ void report(int* status, int slot, int member, int info) {
    if (atomicCAS(status + slot, 0, member + 1) == 0) status[slot + 1] = info;
}

// One front per CTA: assemble (local matrix entries, then the children's update blocks in
// child order), then the partial Cholesky of its n_c leading columns in panels of kPanel
// columns: each panel is factored in shared memory (right-looking, column by column) and the
// trailing lower triangle of the front, rows and columns past the panel, is updated once per
// panel. Column-major f x f front; the first n_c columns end up holding L_ss (diagonal block)
// and L_{R_s,s}, the trailing m x m block the update matrix for the parent.
__global__ void __launch_bounds__(kMfThreads) mf_front_kernel(const MfPlanDev P, const MfBatch B, int lb) {
    extern __shared__ double pan[];
    const int s = P.level_sn[lb + blockIdx.x];
    const int b = blockIdx.y;
    const int nc = P.sn_nc[s], m = P.sn_m[s], f = nc + m;
    double* F = B.fronts + static_cast<long long>(b) * P.front_total + P.front_off[s];
    const double* av = B.aval + static_cast<long long>(b) * P.nnz;
    const int tid = threadIdx.x;
    const long long ff = static_cast<long long>(f) * f;
    for (long long i = tid; i < ff; i += blockDim.x) F[i] = 0.0;
    __syncthreads();
    for (int e = P.asc_ptr[s] + tid; e < P.asc_ptr[s + 1]; e += blockDim.x) F[P.asc_pos[e]] = av[P.asc_csr[e]];
    __syncthreads();
    for (int c = P.ch_ptr[s]; c < P.ch_ptr[s + 1]; ++c) {
        const int ch = P.ch_id[c];
        const int ncc = P.sn_nc[ch], mc = P.sn_m[ch], fc = ncc + mc;
        const double* U = B.fronts + static_cast<long long>(b) * P.front_total + P.front_off[ch];
        const std::int32_t* map = P.em_pos + P.em_ptr[ch];
        for (int idx = tid; idx < mc * mc; idx += blockDim.x) {
            const int a = idx % mc, bb = idx / mc;
            if (a < bb) continue;
            F[static_cast<long long>(map[bb]) * f + map[a]] += U[static_cast<long long>(ncc + bb) * fc + ncc + a];
        }
        __syncthreads();
    }
    for (int j0 = 0; j0 < nc; j0 += kPanel) {
        const int jn = min(kPanel, nc - j0), nr = f - j0;
        for (int idx = tid; idx < jn * nr; idx += blockDim.x) {
            const int jj = idx / nr, i = idx % nr;
            pan[idx] = F[static_cast<long long>(j0 + jj) * f + j0 + i];
        }
        __syncthreads();
        for (int jj = 0; jj < jn; ++jj) {
            double d = pan[jj * nr + jj];
            if (!(d > 0.0) || !isfinite(d)) {  // host checks the status: "not positive definite"
                if (tid == 0) report(B.status, 0, B.first + b, s * 4096 + j0 + jj);
                d = 1.0;
            }
            d = sqrt(d);
            __syncthreads();
            for (int i = jj + tid; i < nr; i += blockDim.x) pan[jj * nr + i] = i == jj ? d : pan[jj * nr + i] / d;
            __syncthreads();
            const int rest = jn - jj - 1;
            for (int idx = tid; idx < rest * nr; idx += blockDim.x) {
                const int kk = jj + 1 + idx / nr, i = idx % nr;
                if (i >= kk) pan[kk * nr + i] -= pan[jj * nr + i] * pan[jj * nr + kk];
            }
            __syncthreads();
        }
        for (int idx = tid; idx < jn * nr; idx += blockDim.x) {
            const int jj = idx / nr, i = idx % nr;
            if (i >= jj) F[static_cast<long long>(j0 + jj) * f + j0 + i] = pan[idx];
        }
        const int rem = nr - jn;
        for (long long idx = tid; idx < static_cast<long long>(rem) * rem; idx += blockDim.x) {
            const int i = jn + static_cast<int>(idx % rem), k = jn + static_cast<int>(idx / rem);
            if (i < k) continue;
            double acc = 0.0;
            for (int jj = 0; jj < jn; ++jj) acc = fma(pan[jj * nr + i], pan[jj * nr + k], acc);
            F[static_cast<long long>(j0 + k) * f + j0 + i] -= acc;
        }
        __syncthreads();
    }
}

// S = A_GG + the roots' update blocks (interface rows), roots in order (factor.cpp).
__global__ void __launch_bounds__(kMfThreads) schur_kernel(const MfPlanDev P, const MfBatch B) {
    const int b = blockIdx.x, ng = P.n_iface, tid = threadIdx.x;
    double* S = B.S + static_cast<long long>(b) * ng * ng;
    const double* av = B.aval + static_cast<long long>(b) * P.nnz;
    for (long long i = tid; i < static_cast<long long>(ng) * ng; i += blockDim.x) S[i] = 0.0;
    __syncthreads();
    for (int e = tid; e < P.sgg_n; e += blockDim.x) S[P.sgg_pos[e]] = av[P.sgg_csr[e]];
    __syncthreads();
    for (int q = 0; q < P.n_roots; ++q) {
        const int r = P.roots[q];
        const int nc = P.sn_nc[r], m = P.sn_m[r], f = nc + m;
        const double* Fr = B.fronts + static_cast<long long>(b) * P.front_total + P.front_off[r];
        const std::int32_t* gam = P.root_gamma + P.root_gamma_ptr[q];
        for (int idx = tid; idx < m * m; idx += blockDim.x) {
            const int a = idx % m, bb = idx / m;
            if (a < bb) continue;
            const double u = Fr[static_cast<long long>(nc + bb) * f + nc + a];
            S[static_cast<long long>(gam[a]) * ng + gam[bb]] += u;
            if (a != bb) S[static_cast<long long>(gam[bb]) * ng + gam[a]] += u;
        }
        __syncthreads();
    }
}

// L_ss^-1 (row-major, lower) and BL_s = L_{R_s,s} L_ss^-1 (interior rows) into D, in the loop
// orders of factor.cpp / solve_program.cpp.
__global__ void __launch_bounds__(128) linv_bl_kernel(const MfPlanDev P, const MfBatch B) {
    extern __shared__ double Ls[];
    const int s = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
    const int nc = P.sn_nc[s], m = P.sn_m[s], mi = P.sn_mi[s], f = nc + m;
    const double* F = B.fronts + static_cast<long long>(b) * P.front_total + P.front_off[s];
    double* D = B.D + static_cast<long long>(b) * P.d_total;
    for (int idx = tid; idx < nc * nc; idx += blockDim.x) {
        const int r = idx / nc, c = idx % nc;
        Ls[idx] = c <= r ? F[static_cast<long long>(c) * f + r] : 0.0;
    }
    __syncthreads();
    double* Li = D + P.linv_off[s];
    for (int c = tid; c < nc; c += blockDim.x) {
        for (int r = 0; r < c; ++r) Li[r * nc + c] = 0.0;
        for (int r = c; r < nc; ++r) {
            double acc = r == c ? 1.0 : 0.0;
            for (int k = c; k < r; ++k) acc -= Ls[r * nc + k] * Li[k * nc + c];
            Li[r * nc + c] = acc / Ls[r * nc + r];
        }
    }
    __syncthreads();
    double* BL = D + P.bl_off[s];
    for (int idx = tid; idx < mi * nc; idx += blockDim.x) {
        const int a = idx / nc, j = idx % nc;
        double acc = 0.0;
        for (int k = j; k < nc; ++k) acc += F[static_cast<long long>(k) * f + nc + a] * Li[k * nc + j];
        BL[idx] = acc;
    }
}

__global__ void fill_kernel(double* dst, const double* tmpl, const std::int32_t* srcmap, const double* D,
                            const FillJob* jobs) {
    const FillJob J = jobs[blockIdx.y];
    auto* out = reinterpret_cast<unsigned long long*>(dst + J.dst);
    const auto* tw = reinterpret_cast<const unsigned long long*>(tmpl + J.tmpl);
    const auto* dv = reinterpret_cast<const unsigned long long*>(D + J.d_off);
    const std::int32_t* code = srcmap + J.tmpl;
    for (long long w = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; w < J.words;
         w += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int c = code[w];
        unsigned long long v;
        if (c == -1) v = tw[w];        // kSrcCopy: header / index words
        else if (c == -2) v = 0ull;    // kSrcZero
        else if (c >= 0) v = dv[c];
        else v = dv[-c - 3] ^ 0x8000000000000000ull;  // negated value (sign bit)
        out[w] = v;
    }
}

constexpr int kSaddleThreads = 1024;

__device__ double block_max(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    v = l < (blockDim.x >> 5) ? red[l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// In-place Gauss-Jordan inverse of the saddle matrix [[S, C_G^T], [C_G, 0]] with row partial
// pivoting (the first row of largest |entry|, setup.cpp dense_inverse's rule; singular when the
// pivot is below 1e-13 of the largest entry), column interchanges undone at the end; then the
// blocks out to the image.
__global__ void __launch_bounds__(kSaddleThreads) saddle_kernel(const MfPlanDev P, const MfBatch B) {
    __shared__ double red[32];
    __shared__ int redi[32];
    __shared__ int s_piv;
    __shared__ double s_best;
    extern __shared__ double sh[];  // row k, column k
    const int b = blockIdx.x, tid = threadIdx.x;
    const int ng = P.n_iface, np = P.n_primal, ns = ng + np;
    double* M = B.M + static_cast<long long>(b) * ns * ns;
    int* piv = B.piv + static_cast<long long>(b) * 2 * ns + ns;  // (the row map's half: identity, below)
    const double* S = B.S + static_cast<long long>(b) * ng * ng;
    const long long nn = static_cast<long long>(ns) * ns;
    for (long long idx = tid; idx < nn; idx += blockDim.x) {
        const int r = static_cast<int>(idx / ns), c = static_cast<int>(idx % ns);
        M[idx] = r < ng && c < ng ? S[static_cast<long long>(r) * ng + c] : 0.0;
    }
    __syncthreads();
    for (int r = tid; r < np; r += blockDim.x)
        for (int e = P.c_ptr[r]; e < P.c_ptr[r + 1]; ++e) {
            const int g = P.c_col[e];
            M[static_cast<long long>(ng + r) * ns + g] += P.c_val[e];
            M[static_cast<long long>(g) * ns + ng + r] += P.c_val[e];
        }
    __syncthreads();
    double mx = 0.0;
    for (long long idx = tid; idx < nn; idx += blockDim.x) mx = fmax(mx, fabs(M[idx]));
    const double scale = block_max(mx, red);
    double* rk = sh;
    double* ck = sh + ns;
    bool failed = false;
    for (int k = 0; k < ns; ++k) {
        // pivot: the first row (>= k) of largest |M[i][k]|
        double best = -1.0;
        int bi = k;
        for (int i = k + tid; i < ns; i += blockDim.x) {
            const double a = fabs(M[static_cast<long long>(i) * ns + k]);
            if (a > best) { best = a; bi = i; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if ((tid & 31) == 0) { red[tid >> 5] = best; redi[tid >> 5] = bi; }
        __syncthreads();
        if (tid == 0) {
            double bb = red[0];
            int bx = redi[0];
            for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
                if (red[w] > bb || (red[w] == bb && redi[w] < bx)) { bb = red[w]; bx = redi[w]; }
            s_best = bb;
            s_piv = bx;
        }
        __syncthreads();
        const double pb = s_best;
        const int p = s_piv;
        if (!(pb > 1e-13 * scale) || !isfinite(pb)) {
            if (tid == 0) report(B.status, 2, B.first + b, k);
            failed = true;
            break;
        }
        if (tid == 0) piv[k] = p;
        if (p != k)
            for (int j = tid; j < ns; j += blockDim.x) {
                const double t = M[static_cast<long long>(k) * ns + j];
                M[static_cast<long long>(k) * ns + j] = M[static_cast<long long>(p) * ns + j];
                M[static_cast<long long>(p) * ns + j] = t;
            }
        __syncthreads();
        const double pv = M[static_cast<long long>(k) * ns + k];
        for (int j = tid; j < ns; j += blockDim.x) {
            rk[j] = j == k ? 1.0 / pv : M[static_cast<long long>(k) * ns + j] / pv;
            ck[j] = M[static_cast<long long>(j) * ns + k];
        }
        __syncthreads();
        // rank-1 update: one row per warp at a time, lanes along the row (coalesced, no index
        // division), four independent entries in flight per lane
        {
            const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
            for (int i = warp; i < ns; i += nw) {
                double* Mi = M + static_cast<long long>(i) * ns;
                if (i == k) {
                    for (int j = lane; j < ns; j += 32) Mi[j] = rk[j];
                    continue;
                }
                const double f = ck[i];
                for (int j0 = lane; j0 < ns; j0 += 128) {
                    double v[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) v[u] = j0 + 32 * u < ns ? Mi[j0 + 32 * u] : 0.0;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int j = j0 + 32 * u;
                        if (j < ns) Mi[j] = j == k ? -f * rk[k] : v[u] - f * rk[j];
                    }
                }
            }
        }
        __syncthreads();
    }
    if (failed) return;
    for (int k = ns - 1; k >= 0; --k) {
        const int p = piv[k];
        if (p != k)
            for (int i = tid; i < ns; i += blockDim.x) {
                const double t = M[static_cast<long long>(i) * ns + k];
                M[static_cast<long long>(i) * ns + k] = M[static_cast<long long>(i) * ns + p];
                M[static_cast<long long>(i) * ns + p] = t;
            }
        __syncthreads();
    }
    // rows and columns are in place: identity maps for the output kernel
    int* map = B.piv + static_cast<long long>(b) * 2 * ns;
    for (int i = tid; i < ns; i += blockDim.x) map[i] = i;
    __syncthreads();
    for (int i = tid; i < ns; i += blockDim.x) map[ns + i] = i;
}

// The same Gauss-Jordan inverse, blocked: the pivots of a block of KB columns are taken on a
// shared-memory copy of those columns (the panel), and the rest of the matrix receives the
// block's KB rank-1 updates in one pass afterwards. Each entry still gets saddle_kernel's
// updates in pivot order with its expressions (x - f rk[j]; the pivot row replaced by rk), so the
// inverse is bitwise the same; the matrix is read and written once per block instead of once
// per pivot. For pivot k of the block, the pivot row outside the panel is brought up to date
// from the block's earlier pivot rows (Rb) and multipliers (F). Row interchanges are a
// permutation (logical position -> physical row), column interchanges a composed map; the
// output kernel reads the inverse through both (map[0..ns) rows, map[ns..2ns) columns).
constexpr int kGjThreads = 512;

std::size_t gj_blocked_smem(int ns, int kb) {
    return sizeof(double) * 3 * static_cast<std::size_t>(ns) * kb + sizeof(int) * 3 * static_cast<std::size_t>(ns);
}

template <int KB>
__global__ void __launch_bounds__(kGjThreads) saddle_gj_blocked_kernel(const MfPlanDev P, const MfBatch B) {
    extern __shared__ double sh[];
    __shared__ double red[32];
    __shared__ int redi[32];
    __shared__ int s_piv;
    __shared__ double s_best;
    const int b = blockIdx.x, tid = threadIdx.x;
    const int ng = P.n_iface, np = P.n_primal, ns = ng + np;
    double* M = B.M + static_cast<long long>(b) * ns * ns;
    const double* S = B.S + static_cast<long long>(b) * ng * ng;
    double* Pn = sh;                                    // [ns][KB] panel, physical rows
    double* F = Pn + static_cast<std::size_t>(ns) * KB;  // [ns][KB] multipliers f of the block's pivots
    double* Rb = F + static_cast<std::size_t>(ns) * KB;  // [KB][ns] the block's pivot rows rk
    int* perm = reinterpret_cast<int*>(Rb + static_cast<std::size_t>(ns) * KB);
    int* pos = perm + ns;
    int* piv = pos + ns;
    const long long nn = static_cast<long long>(ns) * ns;
    for (int r = tid >> 5; r < ns; r += blockDim.x >> 5)
        for (int c = tid & 31; c < ns; c += 32)
            M[static_cast<long long>(r) * ns + c] = r < ng && c < ng ? S[static_cast<long long>(r) * ng + c] : 0.0;
    for (int i = tid; i < ns; i += blockDim.x) perm[i] = pos[i] = i;
    __syncthreads();
    for (int r = tid; r < np; r += blockDim.x)
        for (int e = P.c_ptr[r]; e < P.c_ptr[r + 1]; ++e) {
            const int g = P.c_col[e];
            M[static_cast<long long>(ng + r) * ns + g] += P.c_val[e];
            M[static_cast<long long>(g) * ns + ng + r] += P.c_val[e];
        }
    __syncthreads();
    double mx = 0.0;
    for (long long idx = tid; idx < nn; idx += blockDim.x) mx = fmax(mx, fabs(M[idx]));
    const double scale = block_max(mx, red);
    bool failed = false;
#ifdef GJ_PROF
    long long t_search = 0, t_rk = 0, t_panel = 0, t_trail = 0, t0p = clock64(), tq;
#define GJ_T(acc) do { __syncthreads(); tq = clock64(); acc += tq - t0p; t0p = tq; } while (0)
#else
#define GJ_T(acc) do { } while (0)
#endif
    for (int k0 = 0; k0 < ns && !failed; k0 += KB) {
        const int kb = min(KB, ns - k0);
        for (int idx = tid; idx < ns * KB; idx += blockDim.x) {
            const int r = idx / KB, c = idx % KB;
            if (c < kb) Pn[r * KB + c] = M[static_cast<long long>(r) * ns + k0 + c];
        }
        __syncthreads();
        for (int c = 0; c < kb; ++c) {
            const int k = k0 + c;
            double best = -1.0;
            int bi = k;
            for (int i = k + tid; i < ns; i += blockDim.x) {
                const double a = fabs(Pn[perm[i] * KB + c]);
                if (a > best) { best = a; bi = i; }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
            }
            if ((tid & 31) == 0) { red[tid >> 5] = best; redi[tid >> 5] = bi; }
            __syncthreads();
            if (tid == 0) {
                double bb = red[0];
                int bx = redi[0];
                for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
                    if (red[w] > bb || (red[w] == bb && redi[w] < bx)) { bb = red[w]; bx = redi[w]; }
                s_best = bb;
                s_piv = bx;
                if ((bb > 1e-13 * scale) && isfinite(bb)) {
                    piv[k] = bx;
                    const int qk = perm[k], qp = perm[bx];
                    perm[k] = qp;
                    perm[bx] = qk;
                    pos[qp] = k;
                    pos[qk] = bx;
                }
            }
            __syncthreads();
            if (!(s_best > 1e-13 * scale) || !isfinite(s_best)) {
                if (tid == 0) report(B.status, 2, B.first + b, k);
                failed = true;
                break;
            }
            GJ_T(t_search);
            const int q = perm[k];
            const double pv = Pn[q * KB + c];
            // the pivot row rk: panel entries current, the others brought up to date from the
            // block's earlier pivots (q was not one of them)
            double* rk = Rb + static_cast<std::size_t>(c) * ns;
            for (int j = tid; j < ns; j += blockDim.x) {
                double v;
                if (j >= k0 && j < k0 + kb) {
                    v = Pn[q * KB + (j - k0)];
                } else {
                    v = M[static_cast<long long>(q) * ns + j];
                    for (int cc = 0; cc < c; ++cc) v = v - F[q * KB + cc] * Rb[static_cast<std::size_t>(cc) * ns + j];
                }
                rk[j] = j == k ? 1.0 / pv : v / pv;
            }
            for (int r = tid; r < ns; r += blockDim.x) F[r * KB + c] = Pn[r * KB + c];
            __syncthreads();
            GJ_T(t_rk);
            // the panel's update (saddle_kernel's expressions)
            for (int idx = tid; idx < ns * KB; idx += blockDim.x) {
                const int r = idx / KB, cj = idx % KB, j = k0 + cj;
                if (cj >= kb) continue;
                if (r == q) {
                    Pn[r * KB + cj] = rk[j];
                } else {
                    const double f = F[r * KB + c];
                    Pn[r * KB + cj] = j == k ? -f * rk[k] : Pn[r * KB + cj] - f * rk[j];
                }
            }
            __syncthreads();
            GJ_T(t_panel);
        }
        if (failed) break;
        // the block's updates to the columns outside the panel, in pivot order; the panel back.
        // A warp per row (its multipliers in registers), lanes along the row, four columns in
        // flight per lane; the block's pivot rows take the replacing branch
        {
            const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
            for (int r = warp; r < ns; r += nw) {
                double* Mr = M + static_cast<long long>(r) * ns;
                const int pr = pos[r] - k0;  // the block step at which r was the pivot row, if any
                if (pr >= 0 && pr < kb) {
                    for (int j = lane; j < ns; j += 32) {
                        if (j >= k0 && j < k0 + kb) {
                            Mr[j] = Pn[r * KB + (j - k0)];
                            continue;
                        }
                        double v = Mr[j];
                        for (int cc = 0; cc < kb; ++cc) {
                            const double rj = Rb[static_cast<std::size_t>(cc) * ns + j];
                            v = cc == pr ? rj : v - F[r * KB + cc] * rj;
                        }
                        Mr[j] = v;
                    }
                    continue;
                }
                double f[KB];
#pragma unroll
                for (int cc = 0; cc < KB; ++cc) f[cc] = cc < kb ? F[r * KB + cc] : 0.0;
                constexpr int TW = KB == 16 ? 18 : 1;  // the whole row in registers (ns <= 32 TW)
                if (ns <= 32 * TW && TW > 1) {
                    double v[TW];
#pragma unroll
                    for (int t = 0; t < TW; ++t) {
                        const int j = lane + 32 * t;
                        v[t] = j < ns ? Mr[j] : 0.0;
                    }
#pragma unroll
                    for (int cc = 0; cc < KB; ++cc) {
                        if (cc < kb) {
                            const double* Rc = Rb + static_cast<std::size_t>(cc) * ns;
#pragma unroll
                            for (int t = 0; t < TW; ++t) {
                                const int j = lane + 32 * t;
                                if (j < ns) v[t] = v[t] - f[cc] * Rc[j];
                            }
                        }
                    }
#pragma unroll
                    for (int t = 0; t < TW; ++t) {
                        const int j = lane + 32 * t;
                        if (j < ns) Mr[j] = (j >= k0 && j < k0 + kb) ? Pn[r * KB + (j - k0)] : v[t];
                    }
                    continue;
                }
                for (int j0 = lane; j0 < ns; j0 += 128) {
                    double v[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int j = j0 + 32 * u;
                        v[u] = j < ns ? Mr[j] : 0.0;
                    }
#pragma unroll
                    for (int cc = 0; cc < KB; ++cc) {
                        if (cc < kb) {
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int j = j0 + 32 * u;
                                if (j < ns) v[u] = v[u] - f[cc] * Rb[static_cast<std::size_t>(cc) * ns + j];
                            }
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int j = j0 + 32 * u;
                        if (j < ns) Mr[j] = (j >= k0 && j < k0 + kb) ? Pn[r * KB + (j - k0)] : v[u];
                    }
                }
            }
        }
        __syncthreads();
        GJ_T(t_trail);
    }
#ifdef GJ_PROF
    if (tid == 0 && b == 0) printf("gj ns %d search %lld rk %lld panel %lld trail %lld\n", ns, t_search, t_rk, t_panel, t_trail);
#endif
    if (failed) return;
    // row map (logical -> physical) and the composed column interchanges (undone in reverse)
    int* map = B.piv + static_cast<long long>(b) * 2 * ns;
    for (int i = tid; i < ns; i += blockDim.x) map[i] = perm[i];
    if (tid == 0) {
        int* sig = map + ns;
        for (int c = 0; c < ns; ++c) sig[c] = c;
        for (int k = ns - 1; k >= 0; --k) {
            const int p = piv[k];
            if (p != k) {
                const int t = sig[k];
                sig[k] = sig[p];
                sig[p] = t;
            }
        }
    }
}

// The blocks of the saddle inverse out to the image (M: the inverse, logical row order), and
// A_ci = Phi^T A Phi = Phi_G^T (S Phi_G).
__global__ void __launch_bounds__(kSaddleThreads) saddle_out_kernel(const MfPlanDev P, const MfBatch B,
                                                                    const SaddleOut O) {
    extern __shared__ double sh[];
    const int b = blockIdx.x, tid = threadIdx.x;
    const int ng = P.n_iface, np = P.n_primal, ns = ng + np, nI = P.n_interior;
    const double* Mp = B.M + static_cast<long long>(b) * ns * ns;
    const double* S = B.S + static_cast<long long>(b) * ng * ng;
    if (B.status[2] != 0) return;  // a singular saddle matrix: the setup throws
    // the inverse's entry (r, c) through the row / column maps of the elimination
    const int* rmap = B.piv + static_cast<long long>(b) * 2 * ns;
    const int* cmap = rmap + ns;
    auto Minv = [&](int r, int c) { return Mp[static_cast<long long>(rmap[r]) * ns + cmap[c]]; };
    const std::int64_t* off = O.off + 5 * static_cast<long long>(b);
    double* K = O.kmat + off[0];
    for (long long idx = tid; idx < static_cast<long long>(ng) * ng; idx += blockDim.x) {
        const int r = static_cast<int>(idx / ng), c = static_cast<int>(idx % ng);
        K[idx] = Minv(r, c);
    }
    for (int idx = tid; idx < ng * np; idx += blockDim.x) {
        const int g = idx / np, j = idx % np;
        const double v = Minv(g, ng + j);
        O.phig[off[1] + idx] = v;
        O.phi[off[2] + static_cast<long long>(nI + g) * np + j] = v;
    }
    for (int idx = tid; idx < np * np; idx += blockDim.x) {
        const int r = idx / np, c = idx % np;
        O.lambda[off[3] + idx] = Minv(ng + r, ng + c);
    }
    // W = S Phi_G in shared memory (rows of S in order), then one warp per A_ci entry
    // (lane-strided over the interface, fixed butterfly)
    double* W = sh;
    for (int idx = tid; idx < ng * np; idx += blockDim.x) {
        const int g = idx / np, c = idx % np;
        const double* Sg = S + static_cast<long long>(g) * ng;
        double acc = 0.0;
        for (int h = 0; h < ng; ++h) acc = fma(Sg[h], Minv(h, ng + c), acc);
        W[idx] = acc;
    }
    __syncthreads();
    const int warp = tid >> 5, lane = tid & 31;
    for (int e = warp; e < np * np; e += blockDim.x >> 5) {
        const int r = e / np, c = e % np;
        double acc = 0.0;
        for (int g = lane; g < ng; g += 32) acc = fma(Minv(g, ng + r), W[g * np + c], acc);
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) O.aci[off[4] + e] = acc;
    }
}

__global__ void phi_to_hbuf_kernel(const SubdomainDesc* subs, const double* phig, double* hbuf, int j) {
    const SubdomainDesc sd = subs[blockIdx.x];
    for (int g = threadIdx.x; g < sd.n_iface; g += blockDim.x)
        hbuf[sd.hbuf + g] = j < sd.n_primal ? phig[sd.phig + static_cast<long long>(g) * sd.n_primal + j] : 0.0;
}

__global__ void phi_from_solution_kernel(const SubdomainDesc* subs, const std::int32_t* local_dofs, const double* x,
                                         double* phi, int j) {
    const SubdomainDesc sd = subs[blockIdx.x];
    if (j >= sd.n_primal) return;
    for (int l = threadIdx.x; l < sd.n_interior; l += blockDim.x)
        phi[sd.phi + static_cast<long long>(l) * sd.n_primal + j] = x[local_dofs[sd.local_dofs + l]];
}

// Dense SPD inverse, Gauss-Jordan without pivoting: per pivot k, (1) the normalised pivot row
// and the pivot column to scratch, (2) the rank-1 update of every entry (all SMs).
__global__ void gj_pivot_kernel(const double* A, int n, int k, double* rk, double* ck, int* status) {
    const double pv = A[static_cast<long long>(k) * n + k];
    if (!(pv > 0.0) || !isfinite(pv)) {
        if (threadIdx.x == 0 && blockIdx.x == 0 && status[0] == 0) status[0] = k + 1;
    }
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        rk[j] = j == k ? 1.0 / pv : A[static_cast<long long>(k) * n + j] / pv;
        ck[j] = A[static_cast<long long>(j) * n + k];
    }
}

__global__ void gj_update_kernel(double* A, int n, int k, const double* rk, const double* ck) {
    const long long nn = static_cast<long long>(n) * n;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < nn;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(idx / n), j = static_cast<int>(idx % n);
        if (i == k) A[idx] = rk[j];
        else A[idx] = j == k ? -ck[i] * rk[k] : A[idx] - ck[i] * rk[j];
    }
}

}  // namespace

void launch_mf_level(const MfPlanDev& P, const MfBatch& B, int lb, int le, int max_f, cudaStream_t s) {
    if (le <= lb || B.n <= 0) return;
    const std::size_t smem = sizeof(double) * static_cast<std::size_t>(max_f) * kPanel;
    BDDC_CUDA(cudaFuncSetAttribute(mf_front_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    mf_front_kernel<<<dim3(le - lb, B.n), kMfThreads, smem, s>>>(P, B, lb);
    BDDC_LAUNCHED();
}

void launch_schur(const MfPlanDev& P, const MfBatch& B, int, cudaStream_t s) {
    if (B.n <= 0) return;
    schur_kernel<<<B.n, kMfThreads, 0, s>>>(P, B);
    BDDC_LAUNCHED();
}

void launch_linv_bl(const MfPlanDev& P, const MfBatch& B, int max_nc, cudaStream_t s) {
    if (B.n <= 0 || P.n_sn <= 0) return;
    const std::size_t smem = sizeof(double) * static_cast<std::size_t>(max_nc) * max_nc;
    BDDC_CUDA(cudaFuncSetAttribute(linv_bl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    linv_bl_kernel<<<dim3(P.n_sn, B.n), 128, smem, s>>>(P, B);
    BDDC_LAUNCHED();
}

void launch_fill(double* dst, const double* tmpl, const std::int32_t* srcmap, const double* D, const FillJob* jobs,
                 int n_jobs, cudaStream_t s) {
    if (n_jobs <= 0) return;
    fill_kernel<<<dim3(64, n_jobs), 256, 0, s>>>(dst, tmpl, srcmap, D, jobs);
    BDDC_LAUNCHED();
}

void launch_saddle(const MfPlanDev& P, const MfBatch& B, const SaddleOut& O, cudaStream_t s) {
    if (B.n <= 0) return;
    const int ns = P.n_iface + P.n_primal;
    static const bool global_gj = std::getenv("BDDC_SADDLE_GLOBAL") && std::atoi(std::getenv("BDDC_SADDLE_GLOBAL")) == 1;
    constexpr std::size_t kMaxSmem = 220 * 1024;
    if (!global_gj && gj_blocked_smem(ns, 16) <= kMaxSmem) {
        const std::size_t smem = gj_blocked_smem(ns, 16);
        BDDC_CUDA(cudaFuncSetAttribute(saddle_gj_blocked_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        saddle_gj_blocked_kernel<16><<<B.n, kGjThreads, smem, s>>>(P, B);
    } else if (!global_gj && gj_blocked_smem(ns, 4) <= kMaxSmem) {
        const std::size_t smem = gj_blocked_smem(ns, 4);
        BDDC_CUDA(cudaFuncSetAttribute(saddle_gj_blocked_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        saddle_gj_blocked_kernel<4><<<B.n, kGjThreads, smem, s>>>(P, B);
    } else {
        const std::size_t smem = sizeof(double) * 2 * static_cast<std::size_t>(ns);
        if (smem > 48 * 1024)
            BDDC_CUDA(cudaFuncSetAttribute(saddle_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        saddle_kernel<<<B.n, kSaddleThreads, smem, s>>>(P, B);
    }
    BDDC_LAUNCHED();
    const std::size_t out_smem = sizeof(double) * std::max<std::size_t>(1, static_cast<std::size_t>(P.n_iface) * P.n_primal);
    if (out_smem > 48 * 1024)
        BDDC_CUDA(cudaFuncSetAttribute(saddle_out_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)out_smem));
    saddle_out_kernel<<<B.n, kSaddleThreads, out_smem, s>>>(P, B, O);
    BDDC_LAUNCHED();
}

void launch_phi_to_hbuf(const SubdomainDesc* subs, int n_sub, const double* phig, double* hbuf, int j,
                        cudaStream_t s) {
    phi_to_hbuf_kernel<<<n_sub, 256, 0, s>>>(subs, phig, hbuf, j);
    BDDC_LAUNCHED();
}

void launch_phi_from_solution(const SubdomainDesc* subs, int n_sub, const std::int32_t* local_dofs, const double* x,
                              double* phi, int j, cudaStream_t s) {
    phi_from_solution_kernel<<<n_sub, 256, 0, s>>>(subs, local_dofs, x, phi, j);
    BDDC_LAUNCHED();
}

void dense_spd_inverse(double* A, int n, double* scratch, int* status, cudaStream_t s) {
    BDDC_CUDA(cudaMemsetAsync(status, 0, sizeof(int), s));
    const int upd = std::max(1, std::min(148 * 8, static_cast<int>((static_cast<long long>(n) * n + 255) / 256)));
    for (int k = 0; k < n; ++k) {
        gj_pivot_kernel<<<std::max(1, std::min(16, (n + 255) / 256)), 256, 0, s>>>(A, n, k, scratch, scratch + n,
                                                                                   status);
        BDDC_LAUNCHED();
        gj_update_kernel<<<upd, 256, 0, s>>>(A, n, k, scratch, scratch + n);
        BDDC_LAUNCHED();
    }
}

}  // namespace bddc_b200
