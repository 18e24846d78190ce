#pragma once

#include "fused_comm.cuh"

namespace bddc_b200 {

// Device-resident CG state. Scalars live in device memory; kernels derive alpha/beta
// from fixed-order partial sums, so results are deterministic run to run.
struct PcgDevice {
    int n;                    // rows updated (single GPU: all; distributed: the rank's dofs)
    int n_dot;                // leading entries that enter dot products (distributed: owned dofs)
    int n_dir;                // entries p = z (+ beta p) updates (distributed peer-memory mode: rows +
                              // halo, the halo of z arriving with the r.z exchange)
    int grid;                 // blocks of the vector kernels (fixed => fixed reduction order)
    const std::int32_t* A_ptr;
    const std::int32_t* A_col;
    const double* A_val;
    // the same matrix as sliced ELL (SpMV of the PCG loop): slices of 32 consecutive rows, each
    // slice column-major (entry j of the slice's lane-th row at ell_off[slice] + 32 j + lane), row
    // lengths in ell_len; entries keep their CSR order, so every row sum is the CSR sum
    const std::int64_t* ell_off;
    const std::uint16_t* ell_len;
    const std::int32_t* ell_col;
    // the same columns as 16-bit offsets from the row (column = row + offset) when every entry's
    // offset fits (2D stencils: about one grid line); null: ell_col
    const std::int16_t* ell_d16;
    const double* ell_val;
    double* x;
    double* r;
    double* z;
    double* p;
    double* q;
    double* part_a;   // grid partials
    double* part_b;
    // what the consumers of p.q / r.z (red_a) and r.r (red_b) sum, in order: the grid
    // partials on one GPU; the gathered per-rank totals (rank order) when distributed
    const double* red_a;      // p.q   (update)
    int red_a_n;
    const double* red_b;      // r.r   (check)
    int red_b_n;
    const double* red_c;      // r.z   (init_rho, xpay)
    int red_c_n;
    double* rho;      // [max_it + 1]
    double* alpha;    // [max_it]
    double* beta;     // [max_it]
    double* hist;     // [max_it + 1]
    double* scal;     // [0]=||b||, [1]=rel, [2]=converged flag, [3]=error code
    int* iter;        // device iteration counter: spmv_dot advances it, update/check/xpay read it
                      // (so one captured graph serves every iteration)
    // multi-GPU, fused LL exchanges (null on one GPU): p.q published by spmv_dot and read by
    // update, r.r published by update and read by check, r.z (+ the halo of z, entries >= n)
    // published by the harmonic-extension solve and read by init_rho / xpay. ll_sc: scalar
    // rows [p.q | r.r | r.z][rank] (word pairs); seq_*: the tags (null: gathered buffers)
    Publish pub_pq, pub_rr;
    const ll_word* ll_sc;
    const ll_word* ll_z;
    const std::uint64_t* seq_pq;
    const std::uint64_t* seq_rr;
    const std::uint64_t* seq_rz;
    int me;
    // convergence check fused into update's last CTA (r.r reduced there; peers' r.r from the LL
    // row), scal[0..3] written straight to mapped pinned host memory (null: check kernel + copy)
    double* host_scal;
    int fuse_check;
    // p = z + beta p fused into the next SpMV (pcg_dir_spmv; no xpay pass): p_k lives in p (k
    // even) / p_alt (k odd), each row forms the p entries it reads on the fly from z and
    // p_{k-1}; the grid's last CTA advances the iteration counter
    double* p_alt;
    int fuse_dir;
    double rtol, atol;
};

constexpr int kVecThreads = 512;  // 4 CTAs per SM (vec_grid): 592 grid partials per reduction

void pcg_dot(const PcgDevice& D, const double* a, const double* b, double* part, cudaStream_t s);
// scal[slot] = sqrt(sum part) (sqrt=true) or sum part
void pcg_finalize(const PcgDevice& D, const double* part, int slot, bool take_sqrt, cudaStream_t s);
void pcg_spmv_dot(const PcgDevice& D, cudaStream_t s);           // q = A p ; part_a = p.q (owned rows)
void pcg_dir_spmv(const PcgDevice& D, cudaStream_t s);           // p = z + beta p ; q = A p ; part_a = p.q
void pcg_update(const PcgDevice& D, int it, cudaStream_t s);     // x += a p ; r -= a q ; part_b = r.r
void pcg_check(const PcgDevice& D, int it, cudaStream_t s);      // hist[it], converged flag
void pcg_init_rho(const PcgDevice& D, cudaStream_t s);           // rho[0] = sum part_a ; p = z
void pcg_xpay(const PcgDevice& D, int it, cudaStream_t s);       // beta from part_a ; p = z + beta p
void device_spmv(int n, const std::int32_t* ptr, const std::int32_t* col, const double* val,
                 const double* x, double* y, cudaStream_t s);
void device_axpby(int n, double a, const double* x, double b, const double* y, double* out,
                  cudaStream_t s);  // out = a x + b y
int pcg_grid_for(int n);
// sliced ELL from CSR (entry j of row i at off[i / 32] + 32 j + i % 32, CSR order kept)
// (and, with d16, the column offsets col - row as int16; *overflow set when one does not fit)
void device_csr_to_sliced_ell(int n, const std::int32_t* ptr, const std::int32_t* col, const double* val,
                              const std::int64_t* off, std::int32_t* ell_col, double* ell_val, std::int16_t* d16,
                              int* overflow, cudaStream_t s);
// plain CG (no preconditioner, one GPU) as one cooperative launch over D.grid CTAs: iterations
// 1..max_iterations from rho[0] and p = r; scal[1..4] = rel, converged, error code, iterations
// one BDDC-PCG iteration's xpay + SpMV + update (+ fused check) on one GPU as one cooperative
// launch over D.grid CTAs (monotonic grid-barrier counter, zeroed once)
bool pcg_step_fits(int grid);
void pcg_step(const PcgDevice& D, unsigned long long* barrier, cudaStream_t s);
bool pcg_plain_loop_fits(int grid);
void pcg_plain_loop(const PcgDevice& D, int max_iterations, unsigned int* barrier, cudaStream_t s);
// Smallest index of a non-finite entry, or -1 (writes to *dev_result).
void device_first_nonfinite(int n, const double* x, int* dev_result, cudaStream_t s);

}  // namespace bddc_b200
