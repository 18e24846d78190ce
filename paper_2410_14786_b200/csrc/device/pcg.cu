// PCG vector kernels (reference src/pcg.cpp:40-109): SpMV fused with p.q, the
// x/r update fused with ||r||^2, deterministic grid-partial reductions.
#include "pcg.cuh"

namespace bddc_b200 {
namespace {

__device__ __forceinline__ double sum_partials(const double* part, int n, double* scratch) {
    double v = 0.0;
#pragma unroll 8  // independent loads in flight; the sum order is unchanged
    for (int i = threadIdx.x; i < n; i += blockDim.x) v += part[i];
    return block_sum<kVecThreads>(v, scratch);
}

// Sum over ranks in rank order (same arithmetic as sum_partials over the gathered buffer): my
// own value from red[me], the peers' from the LL scalar row (seq null: gathered buffer).
__device__ __forceinline__ double sum_ranks(const PcgDevice& D, const double* red, int n, int row,
                                            const std::uint64_t* seq, double* scratch) {
    if (!seq) return sum_partials(red, n, scratch);
    const std::uint32_t tag = ll_tag(seq);
    double v = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        v += i == D.me ? red[i] : ll_get(D.ll_sc + 2 * (static_cast<std::int64_t>(row) * n + i), tag);
    return block_sum<kVecThreads>(v, scratch);
}

// column of sliced-ELL entry k of row i: 32-bit columns, or 16-bit offsets from the row (the
// kernels are instantiated for both; the launch picks the matrix's)
__device__ __forceinline__ int ell_column(const std::int32_t* __restrict__ c, std::int64_t k, int) { return c[k]; }
__device__ __forceinline__ int ell_column(const std::int16_t* __restrict__ c, std::int64_t k, int i) {
    return i + static_cast<int>(c[k]);
}
template <typename COL>
__device__ __forceinline__ const COL* ell_cols(const PcgDevice& D);
template <>
__device__ __forceinline__ const std::int32_t* ell_cols<std::int32_t>(const PcgDevice& D) { return D.ell_col; }
template <>
__device__ __forceinline__ const std::int16_t* ell_cols<std::int16_t>(const PcgDevice& D) { return D.ell_d16; }

__global__ void __launch_bounds__(kVecThreads) dot_kernel(int n, const double* __restrict__ a,
                                                          const double* __restrict__ b, double* part) {
    __shared__ double scratch[kVecThreads / 32];
    double acc = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        acc = fma(a[i], b[i], acc);
    acc = block_sum<kVecThreads>(acc, scratch);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(kVecThreads) finalize_kernel(const double* part, int n, double* out,
                                                               int take_sqrt) {
    __shared__ double scratch[kVecThreads / 32];
    const double v = sum_partials(part, n, scratch);
    if (threadIdx.x == 0) *out = take_sqrt ? sqrt(v) : v;
}

template <typename COL>
__global__ void __launch_bounds__(kVecThreads, 4) spmv_dot_kernel(const PcgDevice D) {
    __shared__ double scratch[kVecThreads / 32];
    pdl_trigger();
    pdl_wait();
    if (blockIdx.x == 0 && threadIdx.x == 0) *D.iter += 1;  // read by the later kernels of this iteration
    const double* __restrict__ p = D.p;
    double* __restrict__ q = D.q;
    double acc = 0.0;
    // sliced ELL: a warp's 32 rows are one slice, so every entry load of the warp is one
    // contiguous 256-byte (values) / 128-byte (columns) access
    const COL* __restrict__ ec = ell_cols<COL>(D);
    const double* __restrict__ ev = D.ell_val;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < D.n; i += gridDim.x * blockDim.x) {
        const std::int64_t base = D.ell_off[i >> 5] + (i & 31);
        const int len = D.ell_len[i];
        double y = 0.0;
        int j = 0;
        for (; j + 7 < len; j += 8) {  // eight entries' loads in flight; the sum stays in CSR order
            double v[8], x[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) v[t] = ev[base + 32 * (j + t)];
#pragma unroll
            for (int t = 0; t < 8; ++t) x[t] = p[ell_column(ec, base + 32 * (j + t), i)];
#pragma unroll
            for (int t = 0; t < 8; ++t) y += v[t] * x[t];
        }
        for (; j + 3 < len; j += 4) {  // four entries' loads in flight; the sum stays in CSR order
            const double v0 = ev[base + 32 * j], v1 = ev[base + 32 * (j + 1)];
            const double v2 = ev[base + 32 * (j + 2)], v3 = ev[base + 32 * (j + 3)];
            const double x0 = p[ell_column(ec, base + 32 * j, i)], x1 = p[ell_column(ec, base + 32 * (j + 1), i)];
            const double x2 = p[ell_column(ec, base + 32 * (j + 2), i)], x3 = p[ell_column(ec, base + 32 * (j + 3), i)];
            y += v0 * x0;
            y += v1 * x1;
            y += v2 * x2;
            y += v3 * x3;
        }
        for (; j < len; ++j) y += ev[base + 32 * j] * p[ell_column(ec, base + 32 * j, i)];
        q[i] = y;
        if (i < D.n_dot) acc = fma(p[i], y, acc);
    }
    acc = block_sum<kVecThreads>(acc, scratch);
    if (threadIdx.x == 0) D.part_a[blockIdx.x] = acc;
    publish<kVecThreads>(D.pub_pq);
}

// pcg.cpp:94-100: relative residual, history, convergence / failure flags (one thread)
__device__ __forceinline__ void check_scalar(const PcgDevice& D, int it, double rr) {
    if (D.scal[3] != 1.0) {
        const double normb = D.scal[0];
        const double rel = sqrt(rr) / normb;
        D.hist[it] = rel;
        D.scal[1] = rel;
        // 2 = this iteration's residual norm is not finite (the host decides: the reference
        // throws only from the next apply's ensure_finite, preconditioner.cpp:229)
        D.scal[3] = isfinite(rel) ? 0.0 : 2.0;
        if (rel <= D.rtol || (D.atol > 0.0 && rel * normb <= D.atol)) D.scal[2] = 1.0;
    }
    if (D.host_scal) {
        volatile double* h = D.host_scal;
        for (int k = 0; k < 4; ++k) h[k] = D.scal[k];
    }
}

// pcg.cpp:101-104 + 74: beta = rz / rho, p_k = z + beta p_{k-1} (p_1 = z), q = A p_k, p.q.
// Every row forms the p entries of its columns from z and p_{k-1} (the same expression as
// xpay_kernel, so the iterates are bitwise those of the unfused loop); the distributed halo of
// z comes from the LL buffer. The iteration counter is advanced by the grid's last CTA, after
// every CTA has read it.
template <typename COL>
__global__ void __launch_bounds__(kVecThreads) dir_spmv_kernel(const PcgDevice D) {
    __shared__ double scratch[kVecThreads / 32];
    pdl_trigger();
    pdl_wait();
    const int km1 = *D.iter;  // k - 1
    const int k = km1 + 1;
    double* pn = (k & 1) ? D.p_alt : D.p;
    const double* po = (k & 1) ? D.p : D.p_alt;
    double beta = 0.0;
    const double rz = sum_ranks(D, D.red_c, D.red_c_n, 2, D.seq_rz, scratch);
    if (km1 > 0) beta = rz / D.rho[km1 - 1];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        D.rho[km1] = rz;
        if (km1 > 0) D.beta[km1 - 1] = beta;
    }
    const std::uint32_t tag = D.ll_z ? ll_tag(D.seq_rz) : 0u;
    auto p_at = [&](int j) {
        const double zj = (D.ll_z && j >= D.n) ? ll_get(D.ll_z + 2 * static_cast<std::int64_t>(j - D.n), tag) : D.z[j];
        return km1 > 0 ? zj + beta * po[j] : zj;
    };
    double acc = 0.0;
    const COL* __restrict__ ec = ell_cols<COL>(D);
    const double* __restrict__ ev = D.ell_val;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < D.n; i += gridDim.x * blockDim.x) {
        // sliced ELL (CSR order), four entries' loads in flight
        const std::int64_t base = D.ell_off[i >> 5] + (i & 31);
        const int len = D.ell_len[i];
        double y = 0.0;
        int j = 0;
        for (; j + 3 < len; j += 4) {
            const double v0 = ev[base + 32 * j], v1 = ev[base + 32 * (j + 1)];
            const double v2 = ev[base + 32 * (j + 2)], v3 = ev[base + 32 * (j + 3)];
            const double x0 = p_at(ell_column(ec, base + 32 * j, i));
            const double x1 = p_at(ell_column(ec, base + 32 * (j + 1), i));
            const double x2 = p_at(ell_column(ec, base + 32 * (j + 2), i));
            const double x3 = p_at(ell_column(ec, base + 32 * (j + 3), i));
            y += v0 * x0;
            y += v1 * x1;
            y += v2 * x2;
            y += v3 * x3;
        }
        for (; j < len; ++j) y += ev[base + 32 * j] * p_at(ell_column(ec, base + 32 * j, i));
        const double pi = p_at(i);
        pn[i] = pi;
        D.q[i] = y;
        if (i < D.n_dot) acc = fma(pi, y, acc);
    }
    for (int i = D.n + blockIdx.x * blockDim.x + threadIdx.x; i < D.n_dir; i += gridDim.x * blockDim.x)
        pn[i] = p_at(i);  // the halo of p_k (read as p_{k-1} next iteration)
    acc = block_sum<kVecThreads>(acc, scratch);
    if (threadIdx.x == 0) D.part_a[blockIdx.x] = acc;
    if (publish<kVecThreads>(D.pub_pq) && threadIdx.x == 0) *D.iter = k;
}

__global__ void __launch_bounds__(kVecThreads) update_kernel(const PcgDevice D, int) {
    __shared__ double scratch[kVecThreads / 32];
    pdl_trigger();
    pdl_wait();
    const int it = *D.iter;
    const double* __restrict__ p = (D.fuse_dir && (it & 1)) ? D.p_alt : D.p;
    const double* __restrict__ q = D.q;
    double* __restrict__ x = D.x;
    double* __restrict__ r = D.r;
    // the thread's first two entries are loaded before the p.q reduction, so their latency hides
    // behind it (the vectors do not depend on alpha)
    const int stride = gridDim.x * blockDim.x, i0 = blockIdx.x * blockDim.x + threadIdx.x, i1 = i0 + stride;
    const bool h0 = i0 < D.n, h1 = i1 < D.n;
    const double p0 = h0 ? p[i0] : 0.0, q0 = h0 ? q[i0] : 0.0, x0 = h0 ? x[i0] : 0.0, r0 = h0 ? r[i0] : 0.0;
    const double p1 = h1 ? p[i1] : 0.0, q1 = h1 ? q[i1] : 0.0, x1 = h1 ? x[i1] : 0.0, r1 = h1 ? r[i1] : 0.0;
    const double pq = sum_ranks(D, D.red_a, D.red_a_n, 0, D.seq_pq, scratch);
    if (pq <= 0.0) {  // pcg.cpp:75-78 "matrix not SPD" (a NaN curvature carries on, like the reference)
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            D.scal[3] = 1.0;
            if (D.host_scal) reinterpret_cast<volatile double*>(D.host_scal)[3] = 1.0;
        }
        return;
    }
    const double alpha = D.rho[it - 1] / pq;
    if (blockIdx.x == 0 && threadIdx.x == 0) D.alpha[it - 1] = alpha;
    double acc = 0.0;
    if (h0) {
        x[i0] = x0 + alpha * p0;
        const double ri = r0 - alpha * q0;
        r[i0] = ri;
        if (i0 < D.n_dot) acc = fma(ri, ri, acc);
    }
    if (h1) {
        x[i1] = x1 + alpha * p1;
        const double ri = r1 - alpha * q1;
        r[i1] = ri;
        if (i1 < D.n_dot) acc = fma(ri, ri, acc);
    }
#pragma unroll 2
    for (int i = i0 + 2 * stride; i < D.n; i += stride) {
        x[i] += alpha * p[i];
        const double ri = r[i] - alpha * q[i];
        r[i] = ri;
        if (i < D.n_dot) acc = fma(ri, ri, acc);
    }
    acc = block_sum<kVecThreads>(acc, scratch);
    if (threadIdx.x == 0) D.part_b[blockIdx.x] = acc;
    const bool last = publish<kVecThreads>(D.pub_rr);
    if (D.fuse_check && last) {  // check_kernel's work, in the grid's last CTA
        const double rr = D.seq_rr ? sum_ranks(D, D.red_b, D.red_b_n, 1, D.seq_rr, scratch) : D.pub_rr.red[0];
        if (threadIdx.x == 0) check_scalar(D, it, rr);
    }
}

__global__ void __launch_bounds__(kVecThreads) check_kernel(const PcgDevice D, int) {
    // (fuse_check: done by update_kernel's last CTA)
    __shared__ double scratch[kVecThreads / 32];
    pdl_trigger();
    pdl_wait();
    const int it = *D.iter;
    if (D.scal[3] == 1.0) return;
    const double rr = sum_ranks(D, D.red_b, D.red_b_n, 1, D.seq_rr, scratch);
    if (threadIdx.x == 0) check_scalar(D, it, rr);
}

__global__ void __launch_bounds__(kVecThreads) init_rho_kernel(const PcgDevice D) {
    __shared__ double scratch[kVecThreads / 32];
    pdl_trigger();
    pdl_wait();
    const double rz = sum_ranks(D, D.red_c, D.red_c_n, 2, D.seq_rz, scratch);
    if (blockIdx.x == 0 && threadIdx.x == 0) D.rho[0] = rz;
    const std::uint32_t tag = D.ll_z ? ll_tag(D.seq_rz) : 0u;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < D.n_dir; i += gridDim.x * blockDim.x)
        D.p[i] = (D.ll_z && i >= D.n) ? ll_get(D.ll_z + 2 * static_cast<std::int64_t>(i - D.n), tag) : D.z[i];
}

__global__ void __launch_bounds__(kVecThreads) xpay_kernel(const PcgDevice D, int) {
    __shared__ double scratch[kVecThreads / 32];
    pdl_trigger();
    pdl_wait();
    const int it = *D.iter;
    const double* __restrict__ z = D.z;
    double* __restrict__ p = D.p;
    // the thread's first two rows (not the LL halo) are loaded before the r.z reduction
    const int stride = gridDim.x * blockDim.x, i0 = blockIdx.x * blockDim.x + threadIdx.x, i1 = i0 + stride;
    const double z0 = i0 < D.n ? z[i0] : 0.0, p0 = i0 < D.n ? p[i0] : 0.0;
    const double z1 = i1 < D.n ? z[i1] : 0.0, p1 = i1 < D.n ? p[i1] : 0.0;
    const double rz = sum_ranks(D, D.red_c, D.red_c_n, 2, D.seq_rz, scratch);
    const double beta = rz / D.rho[it - 1];
    const std::uint32_t tag = D.ll_z ? ll_tag(D.seq_rz) : 0u;
    auto z_at = [&](int i) {
        return (D.ll_z && i >= D.n) ? ll_get(D.ll_z + 2 * static_cast<std::int64_t>(i - D.n), tag) : z[i];
    };
    if (i0 < D.n) p[i0] = z0 + beta * p0;
    else if (i0 < D.n_dir) p[i0] = z_at(i0) + beta * p[i0];
    if (i1 < D.n) p[i1] = z1 + beta * p1;
    else if (i1 < D.n_dir) p[i1] = z_at(i1) + beta * p[i1];
#pragma unroll 2
    for (int i = i0 + 2 * stride; i < D.n_dir; i += stride) p[i] = z_at(i) + beta * p[i];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        D.beta[it - 1] = beta;
        D.rho[it] = rz;
    }
}

// Grid-wide barrier of a cooperative (all CTAs resident) launch: a monotonic arrival counter,
// released by each CTA's thread 0 after the CTA's writes, acquired before the CTA proceeds.
__device__ __forceinline__ void grid_barrier(unsigned int* ctr, unsigned int& target) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        fence_acq_rel_gpu();
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        unsigned int v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

// Plain CG on one GPU (pcg.cpp:61-109 with z = r): the whole iteration loop in ONE cooperative
// launch, two grid barriers per iteration instead of four kernels and a host read-back of the
// convergence flags. Phase 1 is dir_spmv's: p_k = r + beta p_{k-1} formed on the fly for the
// columns each row reads (p_k in p_alt for odd k, p for even k), q = A p_k, p.q; phase 2 is
// update's. The partials and their fixed-order sums (every CTA sums the same grid partials in the
// same order, so every CTA takes the same decisions) and every expression are those of the
// launch-per-kernel loop, so the iterates are bitwise identical. The vectors change inside the
// launch and are read through the coherent path (no __restrict__ / non-coherent loads); only
// the matrix is. scal[4] = iterations done.
template <typename COL>
__global__ void __launch_bounds__(kVecThreads, 4) plain_cg_kernel(const PcgDevice D, int max_it, unsigned int* bar) {
    __shared__ double scratch[kVecThreads / 32];
    unsigned int target = 0;
    const int stride = gridDim.x * blockDim.x, i0 = blockIdx.x * blockDim.x + threadIdx.x;
    const COL* __restrict__ ec = ell_cols<COL>(D);
    const double* __restrict__ ev = D.ell_val;
    double* q = D.q;
    double* x = D.x;
    double* r = D.r;
    const double normb = D.scal[0];
    double rho = D.rho[0];
    double beta = 0.0;
    for (int it = 1;; ++it) {
        double* pn = (it & 1) ? D.p_alt : D.p;
        const double* po = (it & 1) ? D.p : D.p_alt;
        const bool first = it == 1;  // p_1 = z = r
        auto p_at = [&](int j) { return first ? r[j] : r[j] + beta * po[j]; };
        double acc = 0.0;
        for (int i = i0; i < D.n; i += stride) {
            const std::int64_t base = D.ell_off[i >> 5] + (i & 31);
            const int len = D.ell_len[i];
            double y = 0.0;
            int j = 0;
            for (; j + 7 < len; j += 8) {  // eight entries' loads in flight, CSR-order sum
                double v[8], x[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) v[t] = ev[base + 32 * (j + t)];
#pragma unroll
                for (int t = 0; t < 8; ++t) x[t] = p_at(ell_column(ec, base + 32 * (j + t), i));
#pragma unroll
                for (int t = 0; t < 8; ++t) y += v[t] * x[t];
            }
            for (; j + 3 < len; j += 4) {
                const double v0 = ev[base + 32 * j], v1 = ev[base + 32 * (j + 1)];
                const double v2 = ev[base + 32 * (j + 2)], v3 = ev[base + 32 * (j + 3)];
                const double x0 = p_at(ell_column(ec, base + 32 * j, i));
                const double x1 = p_at(ell_column(ec, base + 32 * (j + 1), i));
                const double x2 = p_at(ell_column(ec, base + 32 * (j + 2), i));
                const double x3 = p_at(ell_column(ec, base + 32 * (j + 3), i));
                y += v0 * x0;
                y += v1 * x1;
                y += v2 * x2;
                y += v3 * x3;
            }
            for (; j < len; ++j) y += ev[base + 32 * j] * p_at(ell_column(ec, base + 32 * j, i));
            const double pi = p_at(i);
            pn[i] = pi;
            q[i] = y;
            if (i < D.n_dot) acc = fma(pi, y, acc);
        }
        acc = block_sum<kVecThreads>(acc, scratch);
        if (threadIdx.x == 0) D.part_a[blockIdx.x] = acc;
        grid_barrier(bar, target);
        // alpha, x += alpha p, r -= alpha q, r.r (update_kernel; p_k[i] of the thread's own rows)
        const double pq = sum_partials(D.part_a, gridDim.x, scratch);
        if (pq <= 0.0) {  // pcg.cpp:75-78 "matrix not SPD"
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                D.scal[3] = 1.0;
                D.scal[4] = it;
            }
            return;
        }
        const double alpha = rho / pq;
        if (blockIdx.x == 0 && threadIdx.x == 0) D.alpha[it - 1] = alpha;
        acc = 0.0;
        for (int i = i0; i < D.n; i += stride) {
            x[i] += alpha * pn[i];
            const double ri = r[i] - alpha * q[i];
            r[i] = ri;
            if (i < D.n_dot) acc = fma(ri, ri, acc);
        }
        acc = block_sum<kVecThreads>(acc, scratch);
        if (threadIdx.x == 0) D.part_b[blockIdx.x] = acc;
        grid_barrier(bar, target);
        // convergence (check_scalar), beta for the next direction (xpay_kernel)
        const double rr = sum_partials(D.part_b, gridDim.x, scratch);
        const double rel = sqrt(rr) / normb;
        const bool done = rel <= D.rtol || (D.atol > 0.0 && rel * normb <= D.atol);
        beta = rr / rho;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            D.hist[it] = rel;
            D.scal[1] = rel;
            D.scal[3] = isfinite(rel) ? 0.0 : 2.0;  // a non-finite residual carries on (no apply)
            if (done) D.scal[2] = 1.0;
            D.scal[4] = it;
            if (!done && it < max_it) {
                D.beta[it - 1] = beta;
                D.rho[it] = rr;
            }
        }
        if (done || it == max_it) return;
        rho = rr;
    }
}

// Grid barrier on a monotonic 64-bit counter (no reset between launches): the k-th arrival of
// a barrier round falls in [m * grid, (m + 1) * grid) for one m, the round ends at (m + 1) * grid.
__device__ __forceinline__ void grid_sync_mono(unsigned long long* ctr) {
    __syncthreads();
    if (threadIdx.x == 0) {
        fence_acq_rel_gpu();
        const unsigned long long v = atomicAdd(ctr, 1ull);
        const unsigned long long target = (v / gridDim.x + 1) * gridDim.x;
        unsigned long long c;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(c) : "l"(ctr) : "memory");
        } while (c < target);
    }
    __syncthreads();
}

// One BDDC-PCG iteration's vector work on one GPU as ONE cooperative launch (pcg.cpp:65-104):
// phase 0 is xpay_kernel's (beta = r.z / rho from the harmonic solve's partials, p = z + beta p;
// p = z and rho_0 for the first direction), phase 1 spmv_dot_kernel's (q = A p, p.q), phase 2
// update_kernel's (alpha, x += alpha p, r -= alpha q, r.r, the fused convergence check in the
// grid's last CTA, which also advances the iteration counter). Grid barriers between the phases
// instead of kernel boundaries; every expression and fixed-order partial sum is the per-kernel
// loop's, so the iterates are bitwise identical to it.
template <typename COL>
__global__ void __launch_bounds__(kVecThreads, 4) pcg_step_kernel(const PcgDevice D, unsigned long long* bar) {
    __shared__ double scratch[kVecThreads / 32];
    const int km1 = *D.iter, k = km1 + 1;
    const int stride = gridDim.x * blockDim.x, i0 = blockIdx.x * blockDim.x + threadIdx.x;
    {
        // phase 0: the direction (the thread's first rows' loads before the r.z reduction)
        double* p = D.p;
        const double* z = D.z;
        const double z0 = i0 < D.n ? z[i0] : 0.0, p0 = i0 < D.n && km1 > 0 ? p[i0] : 0.0;
        const double rz = sum_partials(D.red_c, D.red_c_n, scratch);
        const double beta = km1 > 0 ? rz / D.rho[km1 - 1] : 0.0;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            D.rho[km1] = rz;
            if (km1 > 0) D.beta[km1 - 1] = beta;
        }
        if (i0 < D.n) p[i0] = km1 > 0 ? z0 + beta * p0 : z0;
        for (int i = i0 + stride; i < D.n; i += stride) p[i] = km1 > 0 ? z[i] + beta * p[i] : z[i];
    }
    grid_sync_mono(bar);
    {
        // phase 1: q = A p (sliced ELL, CSR order), p.q
        const double* p = D.p;
        double* q = D.q;
        const COL* __restrict__ ec = ell_cols<COL>(D);
        const double* __restrict__ ev = D.ell_val;
        double acc = 0.0;
        for (int i = i0; i < D.n; i += stride) {
            const std::int64_t base = D.ell_off[i >> 5] + (i & 31);
            const int len = D.ell_len[i];
            double y = 0.0;
            int j = 0;
            for (; j + 3 < len; j += 4) {
                const double v0 = ev[base + 32 * j], v1 = ev[base + 32 * (j + 1)];
                const double v2 = ev[base + 32 * (j + 2)], v3 = ev[base + 32 * (j + 3)];
                const double x0 = p[ell_column(ec, base + 32 * j, i)];
                const double x1 = p[ell_column(ec, base + 32 * (j + 1), i)];
                const double x2 = p[ell_column(ec, base + 32 * (j + 2), i)];
                const double x3 = p[ell_column(ec, base + 32 * (j + 3), i)];
                y += v0 * x0;
                y += v1 * x1;
                y += v2 * x2;
                y += v3 * x3;
            }
            for (; j < len; ++j) y += ev[base + 32 * j] * p[ell_column(ec, base + 32 * j, i)];
            q[i] = y;
            if (i < D.n_dot) acc = fma(p[i], y, acc);
        }
        acc = block_sum<kVecThreads>(acc, scratch);
        if (threadIdx.x == 0) D.part_a[blockIdx.x] = acc;
    }
    grid_sync_mono(bar);
    {
        // phase 2: update_kernel's
        const double* p = D.p;
        const double* q = D.q;
        double* x = D.x;
        double* r = D.r;
        const double pq = sum_partials(D.part_a, gridDim.x, scratch);
        if (pq <= 0.0) {  // pcg.cpp:75-78 "matrix not SPD"
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                D.scal[3] = 1.0;
                if (D.host_scal) reinterpret_cast<volatile double*>(D.host_scal)[3] = 1.0;
                *D.iter = k;
            }
            return;
        }
        const double alpha = D.rho[km1] / pq;
        if (blockIdx.x == 0 && threadIdx.x == 0) D.alpha[km1] = alpha;
        double acc = 0.0;
        for (int i = i0; i < D.n; i += stride) {
            x[i] += alpha * p[i];
            const double ri = r[i] - alpha * q[i];
            r[i] = ri;
            if (i < D.n_dot) acc = fma(ri, ri, acc);
        }
        acc = block_sum<kVecThreads>(acc, scratch);
        if (threadIdx.x == 0) D.part_b[blockIdx.x] = acc;
        if (publish<kVecThreads>(D.pub_rr) && threadIdx.x == 0) {  // the grid's last CTA
            check_scalar(D, k, D.pub_rr.red[0]);
            *D.iter = k;
        }
    }
}

__global__ void __launch_bounds__(kVecThreads) spmv_kernel(int n, const std::int32_t* __restrict__ ptr,
                                                           const std::int32_t* __restrict__ col,
                                                           const double* __restrict__ val,
                                                           const double* __restrict__ x, double* y) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int e = ptr[i]; e < ptr[i + 1]; ++e) acc += val[e] * x[col[e]];
        y[i] = acc;
    }
}

__global__ void __launch_bounds__(kVecThreads) axpby_kernel(int n, double a, const double* x, double b,
                                                            const double* y, double* out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = a * x[i] + b * y[i];
}

__global__ void __launch_bounds__(kVecThreads) nonfinite_kernel(int n, const double* x, int* res) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (!isfinite(x[i])) atomicMin(res, i);
}

__global__ void __launch_bounds__(kVecThreads) csr_to_ell_kernel(int n, const std::int32_t* __restrict__ ptr,
                                                                const std::int32_t* __restrict__ col,
                                                                const double* __restrict__ val,
                                                                const std::int64_t* __restrict__ off,
                                                                std::int32_t* ell_col, double* ell_val,
                                                                std::int16_t* d16, int* overflow) {
    bool over = false;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const std::int64_t base = off[i >> 5] + (i & 31);
        for (int e = ptr[i], j = 0; e < ptr[i + 1]; ++e, ++j) {
            ell_col[base + 32 * j] = col[e];
            ell_val[base + 32 * j] = val[e];
            const int d = col[e] - i;
            over |= d < -32768 || d > 32767;
            if (d16) d16[base + 32 * j] = static_cast<std::int16_t>(d);
        }
    }
    if (over && overflow) atomicOr(overflow, 1);
}

int vec_grid(int n) { return std::max(1, std::min((n + kVecThreads - 1) / kVecThreads, 148 * 4)); }

}  // namespace

void pcg_dot(const PcgDevice& D, const double* a, const double* b, double* part, cudaStream_t s) {
    dot_kernel<<<D.grid, kVecThreads, 0, s>>>(D.n_dot, a, b, part);
    BDDC_LAUNCHED();
}
void pcg_finalize(const PcgDevice& D, const double* part, int slot, bool take_sqrt, cudaStream_t s) {
    finalize_kernel<<<1, kVecThreads, 0, s>>>(part, D.grid, D.scal + slot, take_sqrt ? 1 : 0);
    BDDC_LAUNCHED();
}
void pcg_spmv_dot(const PcgDevice& D, cudaStream_t s) {
    if (D.ell_d16) launch_pdl(spmv_dot_kernel<std::int16_t>, D.grid, kVecThreads, 0, s, D);
    else launch_pdl(spmv_dot_kernel<std::int32_t>, D.grid, kVecThreads, 0, s, D);
    BDDC_LAUNCHED();
}
void pcg_dir_spmv(const PcgDevice& D, cudaStream_t s) {
    if (D.ell_d16) launch_pdl(dir_spmv_kernel<std::int16_t>, D.grid, kVecThreads, 0, s, D);
    else launch_pdl(dir_spmv_kernel<std::int32_t>, D.grid, kVecThreads, 0, s, D);
    BDDC_LAUNCHED();
}
void pcg_update(const PcgDevice& D, int it, cudaStream_t s) {
    launch_pdl(update_kernel, D.grid, kVecThreads, 0, s, D, it);
    BDDC_LAUNCHED();
}
void pcg_check(const PcgDevice& D, int it, cudaStream_t s) {
    launch_pdl(check_kernel, 1, kVecThreads, 0, s, D, it);
    BDDC_LAUNCHED();
}
void pcg_init_rho(const PcgDevice& D, cudaStream_t s) {
    launch_pdl(init_rho_kernel, D.grid, kVecThreads, 0, s, D);
    BDDC_LAUNCHED();
}
void pcg_xpay(const PcgDevice& D, int it, cudaStream_t s) {
    launch_pdl(xpay_kernel, D.grid, kVecThreads, 0, s, D, it);
    BDDC_LAUNCHED();
}
void device_spmv(int n, const std::int32_t* ptr, const std::int32_t* col, const double* val,
                 const double* x, double* y, cudaStream_t s) {
    spmv_kernel<<<vec_grid(n), kVecThreads, 0, s>>>(n, ptr, col, val, x, y);
    BDDC_LAUNCHED();
}
void device_axpby(int n, double a, const double* x, double b, const double* y, double* out,
                  cudaStream_t s) {
    axpby_kernel<<<vec_grid(n), kVecThreads, 0, s>>>(n, a, x, b, y, out);
    BDDC_LAUNCHED();
}
void device_first_nonfinite(int n, const double* x, int* dev_result, cudaStream_t s) {
    const int init = 0x7fffffff;
    BDDC_CUDA(cudaMemcpyAsync(dev_result, &init, sizeof(int), cudaMemcpyHostToDevice, s));
    nonfinite_kernel<<<vec_grid(n), kVecThreads, 0, s>>>(n, x, dev_result);
    BDDC_LAUNCHED();
}

int pcg_grid_for(int n) { return vec_grid(n); }
void device_csr_to_sliced_ell(int n, const std::int32_t* ptr, const std::int32_t* col, const double* val,
                              const std::int64_t* off, std::int32_t* ell_col, double* ell_val, std::int16_t* d16,
                              int* overflow, cudaStream_t s) {
    if (n <= 0) return;
    csr_to_ell_kernel<<<vec_grid(n), kVecThreads, 0, s>>>(n, ptr, col, val, off, ell_col, ell_val, d16, overflow);
    BDDC_LAUNCHED();
}
bool pcg_step_fits(int grid) {
    int dev = 0, sms = 0, per_sm = 0;
    BDDC_CUDA(cudaGetDevice(&dev));
    BDDC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    BDDC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcg_step_kernel<std::int32_t>, kVecThreads, 0));
    return grid <= per_sm * sms;
}
void pcg_step(const PcgDevice& D, unsigned long long* barrier, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(D.grid);
    cfg.blockDim = dim3(kVecThreads);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    BDDC_CUDA(D.ell_d16 ? cudaLaunchKernelEx(&cfg, pcg_step_kernel<std::int16_t>, D, barrier)
                             : cudaLaunchKernelEx(&cfg, pcg_step_kernel<std::int32_t>, D, barrier));
    BDDC_LAUNCHED();
}
bool pcg_plain_loop_fits(int grid) {
    int dev = 0, sms = 0, per_sm = 0;
    BDDC_CUDA(cudaGetDevice(&dev));
    BDDC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    BDDC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, plain_cg_kernel<std::int32_t>, kVecThreads, 0));
    return grid <= per_sm * sms;
}
void pcg_plain_loop(const PcgDevice& D, int max_iterations, unsigned int* barrier, cudaStream_t s) {
    BDDC_CUDA(cudaMemsetAsync(barrier, 0, sizeof(unsigned int), s));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(D.grid);
    cfg.blockDim = dim3(kVecThreads);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    BDDC_CUDA(D.ell_d16 ? cudaLaunchKernelEx(&cfg, plain_cg_kernel<std::int16_t>, D, max_iterations, barrier)
                             : cudaLaunchKernelEx(&cfg, plain_cg_kernel<std::int32_t>, D, max_iterations, barrier));
    BDDC_LAUNCHED();
}


}  // namespace bddc_b200
