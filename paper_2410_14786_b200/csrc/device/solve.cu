// Batched interior solve A_II^{-1} b for every subdomain: one CTA per subdomain,
// the whole permuted interior vector resident in shared memory (two arrays T, X),
// the supernodal factor streamed once per sweep as coalesced column-major tiles.
//
// Replaces reference interior_correction (src/preconditioner.cpp:194-213) and the
// lu_solve it calls (src/sparse_lu.cpp:203-237).
#include "solve.cuh"

namespace bddc_b200 {
namespace {

struct PassArgs {
    const double* stream;
    const TileTask* tasks;
    const std::int32_t* phases;  // (kSolveWarps+1) per phase
    int n_phases;
    const std::int32_t* idx;
};

// One sweep. own/other: see device_format.hpp (forward own=T, backward own=X).
__device__ __forceinline__ void run_pass(const PassArgs a, double* __restrict__ own,
                                         double* __restrict__ other) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int ph = 0; ph < a.n_phases; ++ph) {
        const std::int32_t* tab = a.phases + ph * (kSolveWarps + 1);
        const int t0 = tab[warp], t1 = tab[warp + 1];
        double acc = 0.0;
        for (int t = t0; t < t1; ++t) {
            const int4 raw = __ldg(reinterpret_cast<const int4*>(a.tasks) + t);
            TileTask task;
            *reinterpret_cast<int4*>(&task) = raw;
            if (task.flags & kTaskFirst) acc = 0.0;
            const double* in = (task.flags & kTaskDiag) ? own : other;
            const int row = lane - task.lane_off;
            const int nrows = task.nrows, ncols = task.ncols;
            if (row >= 0 && row < nrows) {
                const double* M = a.stream + task.m_off + row;
                double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
                int j = 0;
                if (task.flags & kTaskInIndexed) {
                    const std::int32_t* ix = a.idx + task.in_ref;
                    for (; j + 4 <= ncols; j += 4) {
                        const double m0 = ld_stream(M + (j + 0) * nrows);
                        const double m1 = ld_stream(M + (j + 1) * nrows);
                        const double m2 = ld_stream(M + (j + 2) * nrows);
                        const double m3 = ld_stream(M + (j + 3) * nrows);
                        s0 = fma(m0, in[__ldg(ix + j + 0)], s0);
                        s1 = fma(m1, in[__ldg(ix + j + 1)], s1);
                        s2 = fma(m2, in[__ldg(ix + j + 2)], s2);
                        s3 = fma(m3, in[__ldg(ix + j + 3)], s3);
                    }
                    for (; j < ncols; ++j) s0 = fma(ld_stream(M + j * nrows), in[__ldg(ix + j)], s0);
                } else {
                    const double* v = in + task.in_ref;
                    for (; j + 4 <= ncols; j += 4) {
                        const double m0 = ld_stream(M + (j + 0) * nrows);
                        const double m1 = ld_stream(M + (j + 1) * nrows);
                        const double m2 = ld_stream(M + (j + 2) * nrows);
                        const double m3 = ld_stream(M + (j + 3) * nrows);
                        s0 = fma(m0, v[j + 0], s0);
                        s1 = fma(m1, v[j + 1], s1);
                        s2 = fma(m2, v[j + 2], s2);
                        s3 = fma(m3, v[j + 3], s3);
                    }
                    for (; j < ncols; ++j) s0 = fma(ld_stream(M + j * nrows), v[j], s0);
                }
                acc += (s0 + s1) + (s2 + s3);
            }
            if (task.flags & kTaskLast) {
                if (lane < task.nvalid) {
                    if (task.flags & kTaskDiag) other[task.out_base + lane] = acc;
                    else own[task.out_base + lane] -= acc;
                }
            }
        }
        __syncthreads();
    }
}

template <int MODE>
__global__ void __launch_bounds__(kSolveWarps * 32, 1)
interior_solve_kernel(const SolveParams P) {
    extern __shared__ double smem[];
    const int sub = blockIdx.x + P.first_subdomain;
    const SubdomainDesc& sd = P.subs[sub];
    const int nI = sd.n_interior;
    const int ldn = (nI + 1) & ~1;
    double* T = smem;
    double* X = smem + ldn;
    double* ZG = X + ldn;  // interface values (MODE 1)
    const std::int32_t* gmap = P.gmap + sd.gmap;

    for (int p = threadIdx.x; p < nI; p += blockDim.x) T[p] = P.in[gmap[p]];
    if (MODE == 1) {
        // z_G = sum over the subdomains sharing each interface dof of their h
        // contributions, ascending subdomain (reference prolong_add order,
        // preconditioner.cpp:168-169,189-190); writes the interface part of z.
        const int ng = sd.n_iface;
        for (int g = threadIdx.x; g < ng; g += blockDim.x) {
            const int gid = P.iface_gid[sd.iface + g];
            double z = 0.0;
            for (int o = P.gi_own_ptr[gid]; o < P.gi_own_ptr[gid + 1]; ++o) z += P.hbuf[P.gi_own_ref[o]];
            ZG[g] = z;
            if (P.iface_writer[sd.iface + g]) P.out[P.iface_dof[sd.iface + g]] = z;
        }
        __syncthreads();
        // b_I = r_I - A_IG z_G
        const std::int32_t* cp = P.couple_ptr + sd.couple_ptr;
        for (int p = threadIdx.x; p < nI; p += blockDim.x) {
            double acc = 0.0;
            for (int e = cp[p]; e < cp[p + 1]; ++e)
                acc += P.couple_val[sd.couple_ent + e] * ZG[P.couple_gamma[sd.couple_ent + e]];
            T[p] -= acc;
        }
    }
    __syncthreads();

    const PassArgs fwd{P.stream + sd.fwd_stream, P.tasks + sd.fwd_tasks, P.phases + sd.fwd_phases,
                       sd.n_fwd_phases, P.idx + sd.idx_base};
    run_pass(fwd, T, X);
    const PassArgs bwd{P.stream + sd.bwd_stream, P.tasks + sd.bwd_tasks, P.phases + sd.bwd_phases,
                       sd.n_bwd_phases, P.idx + sd.idx_base};
    run_pass(bwd, X, T);

    for (int p = threadIdx.x; p < nI; p += blockDim.x) P.out[gmap[p]] = T[p];
}

}  // namespace

std::size_t interior_solve_smem(int max_interior, int max_iface) {
    const int ldn = (max_interior + 1) & ~1;
    return sizeof(double) * (2 * static_cast<std::size_t>(ldn) + max_iface + 2);
}

void launch_interior_solve(const SolveParams& P, int mode, int n_subdomains, std::size_t smem,
                           cudaStream_t stream) {
    if (n_subdomains <= 0) return;
    if (mode == 0) {
        BDDC_CUDA(cudaFuncSetAttribute(interior_solve_kernel<0>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        interior_solve_kernel<0><<<n_subdomains, kSolveWarps * 32, smem, stream>>>(P);
    } else {
        BDDC_CUDA(cudaFuncSetAttribute(interior_solve_kernel<1>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        interior_solve_kernel<1><<<n_subdomains, kSolveWarps * 32, smem, stream>>>(P);
    }
    BDDC_CUDA(cudaGetLastError());
}

}  // namespace bddc_b200
