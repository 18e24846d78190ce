// Interface-side steps of the BDDC apply (everything between the two interior solves).
//
// With the interior pre-solve u0 = B r, the statically condensed residual r' = r - A u0
// vanishes on interior dofs, so the coarse and local corrections only see
// g_i = W_i R_i r' on the interface, and v3 makes z_I the discrete harmonic
// extension of z_G.  Exact algebra of reference src/preconditioner.cpp:225-249:
//   r_c  = sum_i R_ci^T Phi_Gi^T g_i                (coarse_correction :135-147)
//   x_c  = A_c^{-1} r_c                             (:149-151, dense replicated inverse)
//   h_i  = W_i (Phi_Gi x_c[map_i] + K_i g_i)         (:159-167 and local_correction :177-188)
//   z_G  = sum_i R_i^T h_i  (ascending i, fused into the second interior solve)
#include "iface.cuh"

#include <algorithm>

namespace bddc_b200 {
namespace {

constexpr int kRestrictThreads = 512;  // one interface dof per thread at C2 (n_G <= 400)

__global__ void __launch_bounds__(kRestrictThreads)
iface_restrict_kernel(const IfaceParams P, const double* __restrict__ r, const double* __restrict__ u0) {
    pdl_trigger();
    pdl_wait();
    if (skip_launch(P.skip)) return;
    const std::uint32_t tag_u = P.ll_u ? ll_tag(P.seq_u) : 0u;
    extern __shared__ double sg[];
    const SubdomainDesc& sd = P.subs[blockIdx.x];
    const int ng = sd.n_iface, np = sd.n_primal;
    for (int g = threadIdx.x; g < ng; g += blockDim.x) {
        // the slot's A_GI row range, its r entry and weight: independent loads, issued together
        const int2 er = __ldg(reinterpret_cast<const int2*>(P.slot_rows) + sd.iface + g);
        const double rg = r[P.iface_dof[sd.iface + g]];
        const double wg = P.iface_w[sd.iface + g];
        double acc = 0.0;
        // four entries per round: their column / value / u0 loads issue back to back; the sum
        // stays sequential in CSR order
        const int e0 = er.x, e1 = er.y;
        for (int e = e0; e < e1; e += 4) {
            int col[4];
            double val[4], u[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                col[q] = e + q < e1 ? P.gi_row_col[e + q] : -1;
                val[q] = e + q < e1 ? P.gi_row_val[e + q] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                u[q] = col[q] < 0 ? 0.0
                       : (P.ll_u && col[q] >= P.ll_u_base)
                           ? ll_get(P.ll_u + 2 * static_cast<std::int64_t>(col[q] - P.ll_u_base), tag_u)
                           : u0[col[q]];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (col[q] >= 0) acc += val[q] * u[q];
        }
        const double v = wg * (rg - acc);
        sg[g] = v;
        P.gbuf[sd.hbuf + g] = v;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double* phig = P.phig + sd.phig;
    for (int j = warp; j < np; j += kRestrictThreads / 32) {
        double acc = 0.0;
        for (int g = lane; g < ng; g += 32) acc = fma(phig[g * np + j], sg[g], acc);
        acc = warp_sum(acc);
        if (lane == 0) P.cbuf[sd.cbuf + j] = acc;
    }
    publish<kRestrictThreads>(P.pub_c);
}

constexpr int kCoarseThreads = 512;
constexpr int kCoarseRows = 16;

__global__ void __launch_bounds__(kCoarseThreads)
coarse_direct_kernel(const IfaceParams P) {
    if (skip_launch(P.skip)) return;
    extern __shared__ double rc[];
    const int nc = P.n_coarse;
    for (int q = threadIdx.x; q < nc; q += blockDim.x) {
        double acc = 0.0;
        for (int o = P.c_own_ptr[q]; o < P.c_own_ptr[q + 1]; ++o) acc += P.cbuf[P.c_own_ref[o]];
        rc[q] = acc;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int q = blockIdx.x * kCoarseRows + warp; q < min(nc, (blockIdx.x + 1) * kCoarseRows);
         q += kCoarseThreads / 32) {
        const double* row = P.coarse_inv + static_cast<std::size_t>(q) * nc;
        double acc = 0.0;
        for (int k = lane; k < nc; k += 32) acc = fma(row[k], rc[k], acc);
        acc = warp_sum(acc);
        if (lane == 0) P.xc[q] = acc;
    }
}

constexpr int kLocalThreads = 256;
#ifndef BDDC_LOCAL_ROWS
#define BDDC_LOCAL_ROWS 4
#endif
constexpr int kLocalRows = BDDC_LOCAL_ROWS;  // rows per warp in flight (2 * kLocalRows independent loads per lane)

// h_i = W_i (Phi_Gi x_c[map_i] + K_i g_i) (with_coarse) or h_i = K_i g_i. Each streaming warp
// handles kLocalRows rows of K_i at once so every lane keeps 2 * kLocalRows loads in flight;
// the K_i g_i rows go to shared memory. With the fused coarse solve (with_coarse == 2, a
// cooperative launch) r_c is formed once per GPU: the last warp of every CTA sums its share of
// the coarse entries (latency-bound owner gathers, each entry in its fixed owner order) while
// the other warps stream K_i; after a grid barrier every CTA reads the whole r_c, forms this
// subdomain's x_c rows, and every warp finishes its rows with Phi_G x_c.
__device__ __forceinline__ double coarse_entry(const IfaceParams& P, int q, std::uint32_t tag_c) {
    double acc = 0.0;
    int o0 = 0, o1 = 0;
    if (P.c_own4) {  // the entry's owners (<= 4) in one 16-byte load: no owner-list walk
        const int4 o4 = __ldg(reinterpret_cast<const int4*>(P.c_own4) + q);
        if (o4.x <= -2) {  // more than four owners: the owner list
            o0 = P.c_own_ptr[q];
            o1 = P.c_own_ptr[q + 1];
        } else {
            const int ref[4] = {o4.x, o4.y, o4.z, o4.w};
            double c[4];
#pragma unroll
            for (int t = 0; t < 4; ++t)
                c[t] = ref[t] < 0 ? 0.0
                       : (P.ll_c && (ref[t] < P.c_own_lo || ref[t] >= P.c_own_hi))
                           ? ll_get(P.ll_c + 2 * static_cast<std::int64_t>(ref[t]), tag_c)
                           : P.cbuf[ref[t]];
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (ref[t] >= 0) acc += c[t];
        }
    } else {
        o0 = P.c_own_ptr[q];
        o1 = P.c_own_ptr[q + 1];
    }
    for (int o = o0; o < o1; o += 4) {  // the owners' loads of a round back to back
        int ref[4];
        double c[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) ref[t] = o + t < o1 ? P.c_own_ref[o + t] : -1;
#pragma unroll
        for (int t = 0; t < 4; ++t)
            c[t] = ref[t] < 0 ? 0.0
                   : (P.ll_c && (ref[t] < P.c_own_lo || ref[t] >= P.c_own_hi))
                       ? ll_get(P.ll_c + 2 * static_cast<std::int64_t>(ref[t]), tag_c)
                       : P.cbuf[ref[t]];
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (ref[t] >= 0) acc += c[t];
    }
    return acc;
}

// h rows rb, rb + stride, ... (< r1) for n_primal > 32: lane-strided Phi_G x_c partial sums
__device__ __noinline__ void wide_phi_rows(const IfaceParams& P, const SubdomainDesc& sd, const double* phig,
                                           const double* xl, const double* kg, int rb, int r1, int r0, int stride,
                                           int count, int lane) {
    const int np = sd.n_primal;
    for (int q = 0; q < count; ++q) {
        const int row = rb + q * stride;
        if (row >= r1) break;  // warp-uniform
        double part = 0.0;
        for (int j = lane; j < np; j += 32) part = fma(phig[row * np + j], xl[j], part);
        const double c = warp_sum(part);
        if (lane == 0) P.hbuf[sd.hbuf + row] = P.iface_w[sd.iface + row] * (c + kg[row - r0]);
    }
}

__global__ void __launch_bounds__(kLocalThreads)
iface_local_kernel(const IfaceParams P, int blocks_per_sub, int with_coarse) {
    pdl_trigger();
    pdl_wait();
    if (skip_launch(P.skip)) return;
    extern __shared__ double sm[];
    const int sub = blockIdx.x / blocks_per_sub, part = blockIdx.x % blocks_per_sub;
    const SubdomainDesc& sd = P.subs[sub];
    const int ng = sd.n_iface, np = sd.n_primal;
    const int nc = P.n_coarse;
    double* g = sm;
    double* xl = sm + ((ng + 1) & ~1);
    double* rc = xl + ((P.max_primal + 1) & ~1);
    double* kg = rc + (with_coarse == 2 ? ((nc + 1) & ~1) : 0);  // this CTA's rows of K_i g_i
    __shared__ int next_q;  // local r_c (grid not co-resident): next entry to form
    for (int k = threadIdx.x; k < ng; k += blockDim.x) g[k] = P.gbuf[sd.hbuf + k];
    if (threadIdx.x == 0) next_q = 0;
    __syncthreads();
    const int rows_per = (ng + blocks_per_sub - 1) / blocks_per_sub;
    const int r0 = part * rows_per, r1 = min(ng, r0 + rows_per);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double* K = P.kmat + sd.kmat;
    constexpr int kWarps = kLocalThreads / 32;
    const std::uint32_t tag_c = with_coarse == 2 && P.ll_c ? ll_tag(P.seq_c) : 0u;
    const int cw = with_coarse == 2 ? 1 : 0;  // coarse warps
    const int sw = kWarps - cw;               // streaming warps
    if (warp < sw) {
        for (int row0 = r0 + warp * kLocalRows; row0 < r1; row0 += sw * kLocalRows) {
            const double* kr[kLocalRows];
            bool live[kLocalRows];
#pragma unroll
            for (int q = 0; q < kLocalRows; ++q) {
                live[q] = row0 + q < r1;
                kr[q] = K + static_cast<std::size_t>(live[q] ? row0 + q : row0) * ng;
            }
            double a[kLocalRows][2] = {};
            int k = lane;
            for (; k + 32 < ng; k += 64) {
                const double g0 = g[k], g1 = g[k + 32];
#pragma unroll
                for (int q = 0; q < kLocalRows; ++q)
                    if (live[q]) {
                        a[q][0] = fma(ld_stream(kr[q] + k), g0, a[q][0]);
                        a[q][1] = fma(ld_stream(kr[q] + k + 32), g1, a[q][1]);
                    }
            }
            if (k < ng) {
                const double g0 = g[k];
#pragma unroll
                for (int q = 0; q < kLocalRows; ++q)
                    if (live[q]) a[q][0] = fma(ld_stream(kr[q] + k), g0, a[q][0]);
            }
#pragma unroll
            for (int q = 0; q < kLocalRows; ++q) {
                if (!live[q]) continue;  // warp-uniform
                const double acc = warp_sum(a[q][0] + a[q][1]);
                if (lane == 0) {
                    if (with_coarse) kg[row0 + q - r0] = acc;
                    else P.hbuf[sd.hbuf + row0 + q] = acc;
                }
            }
        }
    } else if (P.coarse_ctr) {
        // this CTA's share of r_c (every owner's c_i, ascending subdomain), to rc_g, then arrive
        const int q0 = static_cast<int>(static_cast<long long>(nc) * blockIdx.x / gridDim.x);
        const int q1 = static_cast<int>(static_cast<long long>(nc) * (blockIdx.x + 1) / gridDim.x);
        for (int q = q0 + lane; q < q1; q += 32) P.rc_g[q] = coarse_entry(P, q, tag_c);
        __syncwarp();
        if (lane == 0) {
            fence_acq_rel_gpu();
            atomicAdd(P.coarse_ctr, 1ull);
        }
    } else {
        for (int q = atomicAdd(&next_q, 1); q < nc; q = atomicAdd(&next_q, 1)) rc[q] = coarse_entry(P, q, tag_c);
    }
    if (with_coarse == 2 && !P.coarse_ctr) {
        // grid too large to be co-resident: every CTA forms the whole r_c itself (the coarse
        // warp started during the stream, the streaming warps join it through the counter)
        for (int q = atomicAdd(&next_q, 1); q < nc; q = atomicAdd(&next_q, 1)) rc[q] = coarse_entry(P, q, tag_c);
        __syncthreads();
    } else if (with_coarse == 2) {
        __syncthreads();
        if (threadIdx.x == 0) {  // grid barrier: every CTA's share of r_c is in rc_g
            // the counter only grows (gridDim.x per launch): the target is the end of this launch's
            // block of arrivals, which this CTA's own arrival falls into
            const unsigned long long seen = *reinterpret_cast<volatile unsigned long long*>(P.coarse_ctr);
            const unsigned long long target = (seen + gridDim.x - 1) / gridDim.x * gridDim.x;
            while (*reinterpret_cast<volatile unsigned long long*>(P.coarse_ctr) < target) {
            }
            fence_acq_rel_gpu();
        }
        __syncthreads();
        for (int q = threadIdx.x; q < nc; q += blockDim.x) rc[q] = __ldcg(P.rc_g + q);
        __syncthreads();
    }
    if (with_coarse == 2) {
        // only the rows of x_c = A_c^{-1} r_c this subdomain needs, in coarse_direct_kernel's order
        for (int j = warp; j < np; j += kWarps) {
            const double* row = P.coarse_inv + static_cast<std::size_t>(P.primal[sd.primal + j]) * nc;
            double acc = 0.0;
            for (int k = lane; k < nc; k += 32) acc = fma(row[k], rc[k], acc);
            acc = warp_sum(acc);
            if (lane == 0) xl[j] = acc;
        }
    }
    if (with_coarse == 1)
        for (int j = threadIdx.x; j < np; j += blockDim.x) xl[j] = P.xc[P.primal[sd.primal + j]];
    if (with_coarse) {
        __syncthreads();
        const double* phig = P.phig + sd.phig;
        constexpr int kB = 8;  // rows per batch: their Phi_G / weight loads issue together
        for (int rb = r0 + warp; rb < r1; rb += kB * kWarps) {
            if (np > 32) {  // general constraint sets: more than one primal column per lane
                wide_phi_rows(P, sd, phig, xl, kg, rb, r1, r0, kWarps, kB, lane);
                continue;
            }
            double ph[kB], w[kB];
#pragma unroll
            for (int q = 0; q < kB; ++q) {
                const int row = rb + q * kWarps;
                ph[q] = row < r1 && lane < np ? phig[row * np + lane] : 0.0;
                w[q] = row < r1 ? P.iface_w[sd.iface + row] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < kB; ++q) {
                const int row = rb + q * kWarps;
                if (row >= r1) break;  // warp-uniform
                const double c = warp_sum(lane < np ? ph[q] * xl[lane] : 0.0);
                if (lane == 0) P.hbuf[sd.hbuf + row] = w[q] * (c + kg[row - r0]);
            }
        }
    }
    publish<kLocalThreads>(P.pub_h);
}


// Packed symmetric K_i (kpacked): a cluster of kcluster CTAs per subdomain streams the stored
// tiles (a, b), a <= b, of the 32 x 32 tiling of K_i once each (K_i is symmetric: the lower tiles
// are the upper ones transposed) and forms both of their products: u_ab = K_ab g_b for the rows
// of block a and, off the diagonal, v_ab = K_ab^T g_a for the rows of block b. A warp holds a
// tile's 32 rows (lane = column: every row load is one coalesced 256-byte read); v is a
// lane-local column sum, u a reduce-scatter of the 32 row products over the lanes (recursive
// halving, 31 shuffles). The partials go to kpart; after a cluster barrier each CTA sums, for its
// row blocks (sym_rows_begin), the partials in a fixed order (b ascending: v_ba for b < a, u_ab
// for b >= a), so the result is deterministic. Half the K_i bytes of a row-major GEMV. r_c is
// formed by all threads while the first tiles' loads are in flight; every CTA of the cluster
// forms the x_c rows its Phi_G rows need.
constexpr int kSymThreads = 512;
constexpr int kSymWarps = kSymThreads / 32;

__device__ __forceinline__ int sym_tile(int a, int b, int nt) { return a * nt - a * (a - 1) / 2 + (b - a); }

// xl[j] = (A_c^{-1} r_c)[primal j] for j = first, first + stride, ... (a warp per row)
__device__ __forceinline__ void coarse_rows(const IfaceParams& P, const SubdomainDesc& sd, const double* rc, double* xl,
                                            int first, int stride, int lane) {
    const int nc = P.n_coarse;
    for (int j = first; j < sd.n_primal; j += stride) {
        const double* row = P.coarse_inv + static_cast<std::size_t>(P.primal[sd.primal + j]) * nc;
        double acc = 0.0;
        for (int k = lane; k < nc; k += 32) acc = fma(row[k], rc[k], acc);
        acc = warp_sum(acc);
        if (lane == 0) xl[j] = acc;
    }
}

#ifdef SYM_PROF
#define SYM_T(i) do { ts_[i] = clock64() - t0_; } while (0)
#else
#define SYM_T(i) do { } while (0)
#endif
template <int CLUSTER>
__global__ void __launch_bounds__(kSymThreads) iface_local_sym_kernel(const IfaceParams P, int with_coarse) {
    const long long t0_ = clock64();
    long long ts_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    (void)t0_;
    (void)ts_;
    pdl_trigger();
    pdl_wait();
    if (skip_launch(P.skip)) return;  // uniform over the cluster
    extern __shared__ double sm[];
    const int sub = blockIdx.x / CLUSTER, crank = blockIdx.x % CLUSTER;
    const SubdomainDesc& sd = P.subs[sub];
    const int ng = sd.n_iface, np = sd.n_primal, nc = P.n_coarse;
    const int nt = (ng + 31) >> 5;
    double* g = sm;                                   // nt * 32, zero padded
    double* xl = g + nt * 32;
    double* rc = xl + ((P.max_primal + 1) & ~1);
    double* kg = rc + (with_coarse == 2 ? ((nc + 1) & ~1) : 0);  // K_i g_i (nt * 32)
    for (int k = threadIdx.x; k < nt * 32; k += blockDim.x) g[k] = k < ng ? P.gbuf[sd.hbuf + k] : 0.0;
    __syncthreads();
    SYM_T(0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double* K = P.kmat + sd.kmat;
    double* part = P.kpart + sd.kmat / 16;
    const int ntiles = nt * (nt + 1) / 2;
    const std::uint32_t tag_c = with_coarse == 2 && P.ll_c ? ll_tag(P.seq_c) : 0u;
    constexpr int kStride = CLUSTER * kSymWarps;
    int t = crank * kSymWarps + warp;
    double x[32];
    if (t < ntiles) {  // the first tile's loads, in flight while r_c is formed
#pragma unroll
        for (int r = 0; r < 32; ++r) x[r] = ld_stream(K + static_cast<std::int64_t>(t) * 1024 + 32 * r + lane);
    }
    if (with_coarse == 2) {
        if (P.coarse_ctr) {
            // this CTA's share of r_c (every owner's c_i, ascending subdomain) to rc_g, then arrive
            const int q0 = static_cast<int>(static_cast<long long>(nc) * blockIdx.x / gridDim.x);
            const int q1 = static_cast<int>(static_cast<long long>(nc) * (blockIdx.x + 1) / gridDim.x);
            for (int q = q0 + threadIdx.x; q < q1; q += kSymThreads) P.rc_g[q] = coarse_entry(P, q, tag_c);
            fence_acq_rel_gpu();  // each writer's entries visible GPU-wide before the CTA arrives
        } else {
            for (int q = threadIdx.x; q < nc; q += kSymThreads) rc[q] = coarse_entry(P, q, tag_c);
        }
    }
    SYM_T(1);
    int a = 0, row_end = nt;  // tile t = (a, b): the tiles of row a are [row_end - (nt - a), row_end)
    for (; t < ntiles; t += kStride) {
        while (t >= row_end) row_end += nt - ++a;
        const int b = a + (t - (row_end - (nt - a)));
        if (a != b) {
            const double* ga = g + a * 32;
            double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
#pragma unroll
            for (int r = 0; r < 32; r += 4) {
                v0 = fma(x[r], ga[r], v0);
                v1 = fma(x[r + 1], ga[r + 1], v1);
                v2 = fma(x[r + 2], ga[r + 2], v2);
                v3 = fma(x[r + 3], ga[r + 3], v3);
            }
            part[static_cast<std::int64_t>(t) * 64 + 32 + lane] = (v0 + v1) + (v2 + v3);
        }
        const double gb = g[b * 32 + lane];
#pragma unroll
        for (int r = 0; r < 32; ++r) x[r] *= gb;
        // reduce-scatter: after the step of width w a lane keeps the half of its 2w values
        // selected by its bit w, plus the partner's copy of that half; lane l ends with row l
#pragma unroll
        for (int w = 16; w >= 1; w >>= 1) {
            const bool up = lane & w;
#pragma unroll
            for (int i = 0; i < w; ++i) {
                const double send = up ? x[i] : x[i + w];
                const double keep = up ? x[i + w] : x[i];
                x[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
            }
        }
        part[static_cast<std::int64_t>(t) * 64 + lane] = x[0];
        if (t + kStride < ntiles) {
#pragma unroll
            for (int r = 0; r < 32; ++r)
                x[r] = ld_stream(K + static_cast<std::int64_t>(t + kStride) * 1024 + 32 * r + lane);
        }
    }
    SYM_T(2);
    // every partial of the subdomain written (and this CTA's r_c complete)
    if (CLUSTER > 1) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
        __syncthreads();
    }
    SYM_T(3);
    if (with_coarse == 2 && P.coarse_ctr) {
        if (threadIdx.x == 0) {  // grid barrier (monotonic counter, see iface_local_kernel)
            fence_acq_rel_gpu();
            atomicAdd(P.coarse_ctr, 1ull);
            const unsigned long long seen = *reinterpret_cast<volatile unsigned long long*>(P.coarse_ctr);
            const unsigned long long target = (seen + gridDim.x - 1) / gridDim.x * gridDim.x;
            while (*reinterpret_cast<volatile unsigned long long*>(P.coarse_ctr) < target) {
            }
            fence_acq_rel_gpu();
        }
        __syncthreads();
        for (int q = threadIdx.x; q < nc; q += blockDim.x) rc[q] = __ldcg(P.rc_g + q);
        __syncthreads();
    }
    // this CTA's row blocks: K_i g_i from the partials in a fixed order, and the x_c rows
    const int a0 = sym_rows_begin(ng, CLUSTER, crank) / 32, a1 = (sym_rows_begin(ng, CLUSTER, crank + 1) + 31) / 32;
    for (int ab = a0 + warp; ab < a1; ab += kSymWarps) {
        double acc = 0.0;
        for (int bb = 0; bb < nt; ++bb)
            acc += bb < ab ? part[static_cast<std::int64_t>(sym_tile(bb, ab, nt)) * 64 + 32 + lane]
                           : part[static_cast<std::int64_t>(sym_tile(ab, bb, nt)) * 64 + lane];
        kg[ab * 32 + lane] = acc;
    }
    if (with_coarse == 2) coarse_rows(P, sd, rc, xl, warp, kSymWarps, lane);
    if (with_coarse == 1)
        for (int j = threadIdx.x; j < np; j += blockDim.x) xl[j] = P.xc[P.primal[sd.primal + j]];
    __syncthreads();
    SYM_T(4);
    const int r0 = sym_rows_begin(ng, CLUSTER, crank), r1 = sym_rows_begin(ng, CLUSTER, crank + 1);
    if (!with_coarse) {
        for (int k = r0 + threadIdx.x; k < r1; k += blockDim.x) P.hbuf[sd.hbuf + k] = kg[k];
    } else {
        // h = W (Phi_G x_c + K g): a thread per row (its Phi_G row's loads in flight together)
        const double* phig = P.phig + sd.phig;
        for (int row = r0 + threadIdx.x; row < r1; row += kSymThreads) {
            const double* ph = phig + static_cast<std::int64_t>(row) * np;
            double c = 0.0;
            for (int j = 0; j < np; ++j) c = fma(ph[j], xl[j], c);
            P.hbuf[sd.hbuf + row] = P.iface_w[sd.iface + row] * (c + kg[row]);
        }
    }
    SYM_T(5);
    // the partials stay alive until every CTA of the cluster has read them
    if (CLUSTER > 1) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    publish<kSymThreads>(P.pub_h);
    SYM_T(6);
#ifdef SYM_PROF
    if ((blockIdx.x / CLUSTER == 0 || blockIdx.x / CLUSTER == 27) && (threadIdx.x & 31) == 0)
        printf("sym cta %d warp %d: %lld %lld %lld %lld %lld %lld %lld\n", blockIdx.x, threadIdx.x >> 5, ts_[0], ts_[1],
               ts_[2], ts_[3], ts_[4], ts_[5], ts_[6]);
#endif
}

__global__ void pack_sym_k_kernel(const double* __restrict__ full, const std::int64_t* __restrict__ full_off,
                                  double* packed, const std::int64_t* __restrict__ sym_off,
                                  const std::int32_t* __restrict__ ngs) {
    const int sub = blockIdx.x, ng = ngs[sub], nt = (ng + 31) >> 5;
    const double* K = full + full_off[sub];
    double* out = packed + sym_off[sub];
    for (int a = 0, t = 0; a < nt; ++a)
        for (int b = a; b < nt; ++b, ++t)
            for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
                const int row = a * 32 + (e >> 5), col = b * 32 + (e & 31);
                out[static_cast<std::int64_t>(t) * 1024 + e] =
                    row < ng && col < ng ? K[static_cast<std::int64_t>(row) * ng + col] : 0.0;
            }
}

// ---------------------------------------------------------------- stage hooks
constexpr int kStageThreads = 256;

// c_i = Phi_i^T (W_i R_i r)   (coarse_correction restriction, preconditioner.cpp:135-140)
__global__ void __launch_bounds__(kStageThreads) stage_phi_restrict_kernel(const StageParams P, const double* r) {
    const SubdomainDesc& sd = P.subs[blockIdx.x];
    const int nl = sd.n_local, np = sd.n_primal;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double* phi = P.phi + sd.phi;
    for (int j = warp; j < np; j += kStageThreads / 32) {
        double acc = 0.0;
        for (int l = lane; l < nl; l += 32)
            acc = fma(phi[l * np + j], P.weights_local[sd.local_dofs + l] * r[P.local_dofs[sd.local_dofs + l]], acc);
        acc = warp_sum(acc);
        if (lane == 0) P.cbuf[sd.cbuf + j] = acc;
    }
}

// lbuf_i = W_i Phi_i x_c[map_i]   (preconditioner.cpp:159-167)
__global__ void __launch_bounds__(kStageThreads) stage_phi_prolong_kernel(const StageParams P) {
    const SubdomainDesc& sd = P.subs[blockIdx.x];
    const int nl = sd.n_local, np = sd.n_primal;
    const double* phi = P.phi + sd.phi;
    for (int l = threadIdx.x; l < nl; l += blockDim.x) {
        double acc = 0.0;
        for (int j = 0; j < np; ++j) acc += phi[l * np + j] * P.xc[P.primal[sd.primal + j]];
        P.lbuf[sd.local_dofs + l] = P.weights_local[sd.local_dofs + l] * acc;
    }
}

// out[g] = sum over owners (ascending subdomain) of lbuf   (prolong_add loop order)
__global__ void __launch_bounds__(kStageThreads) stage_gather_local_kernel(const StageParams P, double* out) {
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < P.n_vector; g += gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int o = P.dof_own_ptr[g]; o < P.dof_own_ptr[g + 1]; ++o) acc += P.lbuf[P.dof_own_ref[o]];
        out[g] = acc;
    }
}

// g_i = W_G r_G - A_GI^(i) y_I   (interface rhs of the local saddle solve)
__global__ void __launch_bounds__(kStageThreads) stage_local_g_kernel(const StageParams P, const double* r,
                                                                    const double* y) {
    const SubdomainDesc& sd = P.subs[blockIdx.x];
    const int ng = sd.n_iface;
    const std::int32_t* rp = P.lrow_ptr + sd.lrow_ptr;
    for (int g = threadIdx.x; g < ng; g += blockDim.x) {
        double acc = 0.0;
        for (int e = rp[g]; e < rp[g + 1]; ++e) acc += P.lrow_val[e] * y[P.lrow_col[e]];
        P.gbuf[sd.hbuf + g] = P.iface_w[sd.iface + g] * r[P.iface_dof[sd.iface + g]] - acc;
    }
}

// out[G] = sum over owners of w * h   (local_correction interface prolongation)
__global__ void __launch_bounds__(kStageThreads) stage_iface_gather_kernel(const StageParams P, const double* h,
                                                                         double* out) {
    for (int gid = blockIdx.x * blockDim.x + threadIdx.x; gid < P.n_gi; gid += gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int o = P.gi_own_ptr[gid]; o < P.gi_own_ptr[gid + 1]; ++o) {
            const int slot = P.gi_own_ref[o];
            acc += P.iface_w[slot] * h[slot];
        }
        out[P.gi_dof[gid]] = acc;
    }
}

constexpr int kCgThreads = 1024;

__global__ void __launch_bounds__(kCgThreads) coarse_cg_kernel(const CoarseCgParams P) {
    extern __shared__ double sh[];
    __shared__ double scratch[kCgThreads / 32];
    const int n = P.n;
    const int ld = (n + 1) & ~1;
    double* x = sh;
    double* r = x + ld;
    double* p = r + ld;
    double* q = p + ld;
    double bb = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double acc = 0.0;
        for (int o = P.c_own_ptr[i]; o < P.c_own_ptr[i + 1]; ++o) acc += P.cbuf[P.c_own_ref[o]];
        r[i] = acc;
        p[i] = acc;
        x[i] = 0.0;
        bb += acc * acc;
    }
    const double norm_b = sqrt(block_sum<kCgThreads>(bb, scratch));
    int iterations = 0;
    double rel = 1.0;
    bool converged = false;
    if (norm_b == 0.0) {
        converged = true;
    } else {
        double rho = block_sum<kCgThreads>(bb, scratch);
        for (int it = 1; it <= P.max_it; ++it) {
            double pq = 0.0;
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                double acc = 0.0;
                for (int e = P.ptr[i]; e < P.ptr[i + 1]; ++e) acc += P.val[e] * p[P.col[e]];
                q[i] = acc;
                pq += p[i] * acc;
            }
            pq = block_sum<kCgThreads>(pq, scratch);
            if (!(pq > 0.0)) { iterations = -it; break; }
            const double alpha = rho / pq;
            double rr = 0.0;
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                x[i] += alpha * p[i];
                r[i] -= alpha * q[i];
                rr += r[i] * r[i];
            }
            rr = block_sum<kCgThreads>(rr, scratch);
            rel = sqrt(rr) / norm_b;
            iterations = it;
            if (rel <= P.rtol || (P.atol > 0.0 && rel * norm_b <= P.atol)) { converged = true; break; }
            if (it == P.max_it) break;
            const double beta = rr / rho;
            rho = rr;
            for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = r[i] + beta * p[i];
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) P.xc[i] = x[i];
    if (threadIdx.x == 0) {
        P.status[0] = iterations;
        P.status[1] = rel;
        P.status[2] = converged ? 1.0 : 0.0;
    }
}

}  // namespace

void launch_coarse_cg(const CoarseCgParams& P, cudaStream_t s) {
    const std::size_t smem = sizeof(double) * 4 * ((P.n + 1) & ~1);
    if (smem > 48 * 1024)
        BDDC_CUDA(cudaFuncSetAttribute(coarse_cg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    coarse_cg_kernel<<<1, kCgThreads, smem, s>>>(P);
    BDDC_LAUNCHED();
}

static int stage_grid(int n) { return std::max(1, std::min((n + kStageThreads - 1) / kStageThreads, 148 * 8)); }

void launch_stage_phi_restrict(const StageParams& P, const double* r, cudaStream_t s) {
    stage_phi_restrict_kernel<<<P.n_subdomains, kStageThreads, 0, s>>>(P, r);
    BDDC_LAUNCHED();
}
void launch_stage_phi_prolong(const StageParams& P, cudaStream_t s) {
    stage_phi_prolong_kernel<<<P.n_subdomains, kStageThreads, 0, s>>>(P);
    BDDC_LAUNCHED();
}
void launch_stage_gather_local(const StageParams& P, double* out, cudaStream_t s) {
    stage_gather_local_kernel<<<stage_grid(P.n_vector), kStageThreads, 0, s>>>(P, out);
    BDDC_LAUNCHED();
}
void launch_stage_local_g(const StageParams& P, const double* r, const double* y, cudaStream_t s) {
    stage_local_g_kernel<<<P.n_subdomains, kStageThreads, 0, s>>>(P, r, y);
    BDDC_LAUNCHED();
}
void launch_stage_iface_gather(const StageParams& P, const double* h, double* out, cudaStream_t s) {
    stage_iface_gather_kernel<<<stage_grid(P.n_gi), kStageThreads, 0, s>>>(P, h, out);
    BDDC_LAUNCHED();
}

namespace {
}  // namespace

void launch_iface_restrict(const IfaceParams& P, const double* r, const double* u0, cudaStream_t s) {
    const std::size_t smem = sizeof(double) * (P.max_iface + 2);
    if (smem > 48 * 1024)
        BDDC_CUDA(cudaFuncSetAttribute(iface_restrict_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    launch_pdl(iface_restrict_kernel, P.n_subdomains, kRestrictThreads, smem, s, P, r, u0);
    BDDC_LAUNCHED();
}

void launch_coarse_direct(const IfaceParams& P, cudaStream_t s) {
    const int blocks = (P.n_coarse + kCoarseRows - 1) / kCoarseRows;
    const std::size_t smem = sizeof(double) * (P.n_coarse + 2);
    if (smem > 48 * 1024)
        BDDC_CUDA(cudaFuncSetAttribute(coarse_direct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    coarse_direct_kernel<<<blocks, kCoarseThreads, smem, s>>>(P);
    BDDC_LAUNCHED();
}

std::size_t sym_smem(const IfaceParams& P, int coarse) {
    const std::size_t nt = (P.max_iface + 31) / 32;
    return sizeof(double) * (64 * nt + P.max_primal + 4 + (coarse == 2 ? static_cast<std::size_t>(P.n_coarse) : 0));
}

std::int64_t sym_k_values(int ng) {
    const std::int64_t nt = (ng + 31) / 32;
    return nt * (nt + 1) / 2 * 1024;
}

void launch_pack_sym_k(const double* full, const std::int64_t* full_off, double* packed, const std::int64_t* sym_off,
                       const std::int32_t* ng, int n_subdomains, cudaStream_t s) {
    if (n_subdomains <= 0) return;
    pack_sym_k_kernel<<<n_subdomains, 256, 0, s>>>(full, full_off, packed, sym_off, ng);
    BDDC_LAUNCHED();
}

bool iface_local_cooperative_fits(const IfaceParams& P, int blocks_per_sub, int device) {
    if (P.kpacked) {  // the cooperative K_i grid runs one CTA per subdomain
        const std::size_t smem = sym_smem(P, 2);
        if (smem > 48 * 1024)
            BDDC_CUDA(cudaFuncSetAttribute(iface_local_sym_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0, nsm = 0, coop = 0;
        BDDC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, iface_local_sym_kernel<1>, kSymThreads, smem));
        BDDC_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
        BDDC_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
        return coop && static_cast<long long>(per_sm) * nsm >= P.n_subdomains;
    }
    const std::size_t smem =
        sizeof(double) * (P.max_iface + P.max_primal + 6 + static_cast<std::size_t>(P.n_coarse) +
                          (P.max_iface + blocks_per_sub - 1) / blocks_per_sub);
    if (smem > 48 * 1024)
        BDDC_CUDA(cudaFuncSetAttribute(iface_local_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0, nsm = 0, coop = 0;
    BDDC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, iface_local_kernel, kLocalThreads, smem));
    BDDC_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
    BDDC_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
    return coop && static_cast<long long>(per_sm) * nsm >= static_cast<long long>(P.n_subdomains) * blocks_per_sub;
}

void launch_iface_local(const IfaceParams& P, int blocks_per_sub, cudaStream_t s, int coarse) {
    if (P.kpacked) {  // kcluster CTAs per subdomain (blocks_per_sub does not apply)
        const std::size_t smem = sym_smem(P, coarse);
        const bool coop = coarse == 2 && P.coarse_ctr;
        auto go = [&](auto kern) {
            if (smem > 48 * 1024) BDDC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(P.n_subdomains * P.kcluster);
            cfg.blockDim = dim3(kSymThreads);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = s;
            cudaLaunchAttribute attr[2];
            int na = 0;
            if (coop) {
                attr[na].id = cudaLaunchAttributeCooperative;
                attr[na++].val.cooperative = 1;
            } else if (P.kcluster > 1) {
                attr[na].id = cudaLaunchAttributeClusterDimension;
                attr[na].val.clusterDim.x = P.kcluster;
                attr[na].val.clusterDim.y = 1;
                attr[na++].val.clusterDim.z = 1;
            }
            if (!coop && pdl_enabled()) {
                attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                attr[na++].val.programmaticStreamSerializationAllowed = 1;
            }
            cfg.attrs = attr;
            cfg.numAttrs = na;
            BDDC_CUDA(cudaLaunchKernelEx(&cfg, kern, P, coarse));
        };
        if (P.kcluster == 2) go(iface_local_sym_kernel<2>);
        else go(iface_local_sym_kernel<1>);
        BDDC_LAUNCHED();
        return;
    }
    const std::size_t smem =
        sizeof(double) * (P.max_iface + P.max_primal + 6 + (coarse == 2 ? static_cast<std::size_t>(P.n_coarse) : 0) +
                          (P.max_iface + blocks_per_sub - 1) / blocks_per_sub);
    if (smem > 48 * 1024)
        BDDC_CUDA(cudaFuncSetAttribute(iface_local_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    if (coarse == 2 && P.coarse_ctr) {  // grid barrier inside: all CTAs co-resident (cooperative launch)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(P.n_subdomains * blocks_per_sub);
        cfg.blockDim = dim3(kLocalThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        BDDC_CUDA(cudaLaunchKernelEx(&cfg, iface_local_kernel, P, blocks_per_sub, coarse));
    } else {
        launch_pdl(iface_local_kernel, P.n_subdomains * blocks_per_sub, kLocalThreads, smem, s, P, blocks_per_sub, coarse);
    }
    BDDC_LAUNCHED();
}

}  // namespace bddc_b200
