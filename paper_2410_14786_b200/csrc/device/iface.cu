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

namespace bddc_b200 {
namespace {

constexpr int kRestrictThreads = 256;

__global__ void __launch_bounds__(kRestrictThreads)
iface_restrict_kernel(const IfaceParams P, const double* __restrict__ r, const double* __restrict__ u0) {
    extern __shared__ double sg[];
    const SubdomainDesc& sd = P.subs[blockIdx.x];
    const int ng = sd.n_iface, np = sd.n_primal;
    for (int g = threadIdx.x; g < ng; g += blockDim.x) {
        const int gid = P.iface_gid[sd.iface + g];
        double acc = 0.0;
        for (int e = P.gi_row_ptr[gid]; e < P.gi_row_ptr[gid + 1]; ++e)
            acc += P.gi_row_val[e] * u0[P.gi_row_col[e]];
        const double v = P.iface_w[sd.iface + g] * (r[P.iface_dof[sd.iface + g]] - acc);
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
}

constexpr int kCoarseThreads = 512;
constexpr int kCoarseRows = 16;

__global__ void __launch_bounds__(kCoarseThreads)
coarse_direct_kernel(const IfaceParams P) {
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

__global__ void __launch_bounds__(kLocalThreads)
iface_local_kernel(const IfaceParams P, int blocks_per_sub) {
    extern __shared__ double sm[];
    const int sub = blockIdx.x / blocks_per_sub, part = blockIdx.x % blocks_per_sub;
    const SubdomainDesc& sd = P.subs[sub];
    const int ng = sd.n_iface, np = sd.n_primal;
    double* g = sm;
    double* xl = sm + ((ng + 1) & ~1);
    for (int k = threadIdx.x; k < ng; k += blockDim.x) g[k] = P.gbuf[sd.hbuf + k];
    for (int j = threadIdx.x; j < np; j += blockDim.x) xl[j] = P.xc[P.primal[sd.primal + j]];
    __syncthreads();
    const int rows_per = (ng + blocks_per_sub - 1) / blocks_per_sub;
    const int r0 = part * rows_per, r1 = min(ng, r0 + rows_per);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double* K = P.kmat + sd.kmat;
    const double* phig = P.phig + sd.phig;
    for (int row = r0 + warp; row < r1; row += kLocalThreads / 32) {
        const double* krow = K + static_cast<std::size_t>(row) * ng;
        double a0 = 0.0, a1 = 0.0;
        int k = lane;
        for (; k + 32 < ng; k += 64) {
            a0 = fma(ld_stream(krow + k), g[k], a0);
            a1 = fma(ld_stream(krow + k + 32), g[k + 32], a1);
        }
        if (k < ng) a0 = fma(ld_stream(krow + k), g[k], a0);
        double acc = warp_sum(a0 + a1);
        if (lane == 0) {
            double coarse = 0.0;
            for (int j = 0; j < np; ++j) coarse = fma(phig[row * np + j], xl[j], coarse);
            P.hbuf[sd.hbuf + row] = P.iface_w[sd.iface + row] * (coarse + acc);
        }
    }
}

}  // namespace

void launch_iface_restrict(const IfaceParams& P, const double* r, const double* u0, cudaStream_t s) {
    const std::size_t smem = sizeof(double) * (P.max_iface + 2);
    if (smem > 48 * 1024)
        BDDC_CUDA(cudaFuncSetAttribute(iface_restrict_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    iface_restrict_kernel<<<P.n_subdomains, kRestrictThreads, smem, s>>>(P, r, u0);
    BDDC_CUDA(cudaGetLastError());
}

void launch_coarse_direct(const IfaceParams& P, cudaStream_t s) {
    const int blocks = (P.n_coarse + kCoarseRows - 1) / kCoarseRows;
    const std::size_t smem = sizeof(double) * (P.n_coarse + 2);
    if (smem > 48 * 1024)
        BDDC_CUDA(cudaFuncSetAttribute(coarse_direct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    coarse_direct_kernel<<<blocks, kCoarseThreads, smem, s>>>(P);
    BDDC_CUDA(cudaGetLastError());
}

void launch_iface_local(const IfaceParams& P, int blocks_per_sub, cudaStream_t s) {
    const std::size_t smem = sizeof(double) * (P.max_iface + P.max_primal + 4);
    if (smem > 48 * 1024)
        BDDC_CUDA(cudaFuncSetAttribute(iface_local_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    iface_local_kernel<<<P.n_subdomains * blocks_per_sub, kLocalThreads, smem, s>>>(P, blocks_per_sub);
    BDDC_CUDA(cudaGetLastError());
}

}  // namespace bddc_b200
