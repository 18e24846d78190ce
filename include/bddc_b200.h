/* bddc_b200.h — C-ABI of the B200-native BDDC-PCG hot path.
 *
 * Drop-in boundary for the reference's C++ solver/preconditioner API
 * (/root/reference/proj). Plain pointers and sizes only; every
 * function returns a status code (BDDC_OK = 0) and never lets an exception cross
 * the ABI. The message of the last failure on the calling thread is available
 * from bddc_last_error(); the reference's exception types map to the codes below
 * and its messages are preserved verbatim (e.g. "matrix not SPD",
 * "coarse CG did not converge: ...", "bddc setup: subdomain i: ...").
 *
 * Reference interface each entry point replaces (file:line in /root/reference/proj):
 *   bddc_problem_poisson        assemble_poisson + build_constraints + study_rhs
 *                               (src/decomposition.cpp:161-203, :112-159; src/study.cpp:69-75)
 *   bddc_problem_from_view      the in-memory PoissonProblem / IngestedProblem handed to the
 *                               Preconditioner ctor (include/bddc/decomposition.hpp:29-57,
 *                               include/bddc/bundle.hpp:18-24)
 *   bddc_gpu_create             Preconditioner::Preconditioner (include/bddc/preconditioner.hpp:62-66,
 *                               src/preconditioner.cpp:100-127)
 *   bddc_gpu_apply[_device]     Preconditioner::apply (src/preconditioner.cpp:225-249)
 *   bddc_gpu_stage              coarse_correction / local_correction / interior_correction /
 *                               static_condensation_correction (src/preconditioner.cpp:129-223)
 *   bddc_gpu_pcg[_device]       pcg (include/bddc/pcg.hpp:43-45, src/pcg.cpp:40-109) with
 *                               M = Preconditioner::apply (src/study.cpp:113-119)
 *   bddc_gpu_subdomain_blocks   SubdomainData::coarse_basis / multipliers / coarse_block
 *                               (include/bddc/preconditioner.hpp:27-35)
 *   bddc_gpu_coarse_matrix      Preconditioner::coarse().matrix (include/bddc/preconditioner.hpp:92)
 *   bddc_gpu_create_dist        Preconditioner ctor, one rank per B200: the reference's only
 *                               parallelism is the parallel_for worker pool over subdomains
 *                               (include/bddc/parallel.hpp:19-45, src/preconditioner.cpp:114-123);
 *                               here subdomain blocks go to ranks and cross-subdomain sums keep its
 *                               ascending-subdomain order (src/preconditioner.cpp:141-147,168-169)
 *   bddc_rank_plan_*            host-only view of one rank's partition (CPU tests, tooling)
 */
#ifndef BDDC_B200_H
#define BDDC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BDDC_OK 0
#define BDDC_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument in the reference */
#define BDDC_ERR_RUNTIME 2          /* std::runtime_error */
#define BDDC_ERR_OUT_OF_RANGE 3     /* std::out_of_range */
#define BDDC_ERR_CUDA 4             /* CUDA runtime failure */
#define BDDC_ERR_NO_DEVICE 5        /* no B200 visible: there is no CPU fallback */

#define BDDC_STAGE_INTERIOR 0            /* interior_correction(r) */
#define BDDC_STAGE_COARSE 1              /* coarse_correction(r) */
#define BDDC_STAGE_LOCAL 2               /* local_correction(r) */
#define BDDC_STAGE_STATIC_CONDENSATION 3 /* static_condensation_correction(r, v1, v2) */

#define BDDC_COARSE_DIRECT 0 /* replicated dense A_c^{-1} GEMV (default) */
#define BDDC_COARSE_CG 1     /* reference-faithful coarse CG (src/preconditioner.cpp:149-157) */

/* Host CSR view (reference CsrMatrix, include/bddc/csr_matrix.hpp:27-47). */
typedef struct {
    int32_t nrows, ncols;
    const int32_t* row_offsets; /* nrows + 1 */
    const int32_t* col_indices; /* nnz */
    const double* values;       /* nnz */
} bddc_csr_view;

/* Borrowed view of a decomposed problem (Decomposition + ConstraintSet + matrices). */
typedef struct {
    int32_t n_subdomains;
    int32_t global_dofs;
    int32_t n_coarse;
    bddc_csr_view global_matrix;
    const bddc_csr_view* local_matrices;      /* [n_subdomains], interior dofs first */
    const bddc_csr_view* constraint_matrices; /* [n_subdomains] */
    const int64_t* dof_offsets;               /* [n_subdomains+1] into subdomain_dofs / weights */
    const int32_t* subdomain_dofs;            /* local -> global dof, interior first, ascending */
    const double* weights;                    /* 1/multiplicity per local dof */
    const int32_t* interior_counts;           /* [n_subdomains] */
    const int64_t* primal_offsets;            /* [n_subdomains+1] into primal_maps */
    const int32_t* primal_maps;               /* strictly increasing coarse ids per subdomain */
    const uint8_t* class_kind;                /* [global_dofs] 0 interior, 1 edge, 2 corner */
    const int32_t* class_entity;              /* [global_dofs] */
    const int32_t* multiplicity;              /* [global_dofs] */
    const int32_t* coords;                    /* optional [2*global_dofs] (x,y) grid coords, or NULL */
    const double* rhs;                        /* optional [global_dofs], or NULL */
} bddc_problem_view;

typedef struct {
    int32_t device;                /* CUDA device ordinal */
    int32_t workers;               /* host setup threads; 0 = all cores */
    int32_t coarse_mode;           /* BDDC_COARSE_DIRECT | BDDC_COARSE_CG */
    double coarse_rel_tolerance;   /* reference default 1e-12 */
    double coarse_abs_tolerance;   /* 0 */
    int32_t coarse_max_iterations; /* 500 */
    int32_t leaf_size;             /* nested-dissection leaf size (default 24) */
    int32_t local_blocks;          /* CTAs per subdomain of the row-major K_i GEMV (default 8; only with
                                      BDDC_K_FULL=1 - the default packed-symmetric K_i kernel runs a
                                      2-CTA cluster per subdomain) */
    int32_t solve_parts;           /* CTAs (cluster size) per subdomain in the interior solve: 0 auto, 1, 2 */
    int32_t setup_mode;            /* BDDC_SETUP_DEVICE (default): factorisation, Schur complements, K_i,
                                      Phi, A_ci and A_c^-1 on the GPU; BDDC_SETUP_HOST: host numeric setup */
} bddc_gpu_options;

enum { BDDC_SETUP_DEVICE = 0, BDDC_SETUP_HOST = 1 };

/* Reference SolverOptions (include/bddc/pcg.hpp:17-22). */
typedef struct {
    double rel_tolerance;
    double abs_tolerance;
    int32_t max_iterations;
    int32_t record_history;
} bddc_solver_options;

/* Reference SolveReport (include/bddc/pcg.hpp:24-30). */
typedef struct {
    int32_t iterations;
    double final_relative_residual;
    int32_t history_length; /* entries written to the caller's history buffer */
    int32_t has_condition_estimate;
    double condition_estimate;
    int32_t converged;
} bddc_solve_report;

typedef struct {
    double setup_seconds;
    int64_t factor_values;        /* stored FP64 values of all interior factors */
    int64_t interior_solve_bytes; /* FP64 bytes streamed by one batched interior solve */
    int64_t apply_bytes;          /* algorithmic FP64 bytes of one apply */
    int32_t n_subdomains;
    int32_t global_dofs;
    int32_t n_coarse;
    int32_t unique_subdomains;    /* distinct setup problems after exact deduplication */
    int32_t max_interior;
    int32_t max_interface;
    int64_t interior_dofs;        /* sum of n_I over subdomains */
    int64_t interior_apply_bytes; /* algorithmic FP64 bytes of the two interior solves of one apply */
    int64_t graph_captures;       /* PCG iteration graphs captured so far (a repeated identical solve
                                     re-uses them; host setup contexts: 0) */
    int32_t coarse_mode;          /* coarse solve in effect: 0 dense replicated A_c^-1, 1 coarse CG */
    int32_t switches;             /* bit mask of the BDDC_* environment switches set at creation
                                     (bit i = bddc_switch_name(i)); 0 = all defaults */
    double setup_device_seconds;  /* part of setup_seconds spent in device setup kernels */
} bddc_stats;

typedef struct {
    double interior_ms; /* summed over profiled applies: both batched interior solves */
    int64_t interior_launches;
    double iface_ms;    /* interface restrict + coarse + local */
    double apply_ms;
    int64_t applies;
} bddc_kernel_times;

typedef struct bddc_problem bddc_problem;
typedef struct bddc_host_setup bddc_host_setup;
typedef struct bddc_gpu_ctx bddc_gpu_ctx;
typedef struct bddc_rank_plan bddc_rank_plan;

/* Multi-GPU: this process is `rank` of `world` (one process per B200, NCCL over NVLink). */
typedef struct {
    int32_t rank;
    int32_t world;
    uint8_t nccl_id[128];            /* from bddc_dist_unique_id() on rank 0, broadcast by the caller */
    const int32_t* subdomain_rank;   /* optional [n_subdomains]; NULL = rectangular blocks */
} bddc_dist_options;

/* One rank's partition. Rank-local vector layout: [0, n_owned) owned dofs (dot products),
 * [0, n_rows) every dof of the rank's subdomains, [n_rows, n_local) halo. */
typedef struct {
    int32_t rank, world, n_local, n_rows, n_owned, n_subdomains_global;
    const int32_t* local_to_global;  /* [n_local] */
    const int32_t* subdomain_rank;   /* [n_subdomains_global] */
    int32_t n_local_subdomains;
    const int32_t* subdomains;       /* global ids, ascending */
    int32_t n_halo_peers;
    const int32_t* halo_peers;       /* ranks */
    const int32_t* halo_send_off;    /* [n_halo_peers+1] into halo_send_idx */
    const int32_t* halo_send_idx;    /* rank-local indices packed per peer */
    const int32_t* halo_recv_off;    /* [n_halo_peers+1]: received into n_rows + off */
    int32_t n_iface_peers;
    const int32_t* iface_peers;
    const int32_t* iface_send_off;   /* [n_iface_peers+1] into iface_send_slot */
    const int32_t* iface_send_slot;  /* local h slots (subdomain-major, interface order) */
    const int32_t* iface_recv_off;   /* [n_iface_peers+1]: remote slot ranges */
    int32_t n_local_slots, n_remote_slots;
    const int32_t* remote_ptr;       /* [n_rows+1]: remote interface owners per local row */
    const int32_t* remote_subdomain; /* global subdomain of each remote owner */
    const int32_t* remote_slot;      /* its remote slot */
    int32_t cbuf_pad;                /* gathered coarse contributions: rank q at q*cbuf_pad */
    const int32_t* cbuf_offset;      /* [n_subdomains_global] */
    const bddc_problem* local_problem; /* rank-local problem (borrowed; lives with the plan) */
} bddc_rank_plan_view;

const char* bddc_last_error(void);
int32_t bddc_abi_version(void);
/* Name of environment switch bit i of bddc_stats.switches (NULL past the last). */
const char* bddc_switch_name(int32_t i);
/* Kernel launches issued by this library in this process so far (all contexts). */
int64_t bddc_kernel_launches(void);
void bddc_default_gpu_options(bddc_gpu_options* opt);
void bddc_default_solver_options(bddc_solver_options* opt);

/* ---- problem layer (host) ---- */
int bddc_problem_poisson(int32_t cells_x, int32_t cells_y, int32_t kx, int32_t ky,
                         double kappa_decades, uint64_t kappa_seed, uint64_t rhs_seed,
                         bddc_problem** out);
int bddc_problem_from_view(const bddc_problem_view* view, bddc_problem** out);
int bddc_problem_get_view(const bddc_problem* p, bddc_problem_view* view);
int bddc_problem_export_bundle(const bddc_problem* p, const char* directory);
/* Reads a reference bundle (manifest + Matrix Market locals + maps + classes + rhs) into a
 * problem: replaces bddc::ingest_bundle (include/bddc/bundle.hpp, src/bundle.cpp:113-290) with
 * the same validation messages; no coordinates (the factorisation orders by graph). */
int bddc_problem_ingest_bundle(const char* manifest_path, bddc_problem** out);
void bddc_problem_destroy(bddc_problem* p);

/* ---- host setup only (no GPU; used by CPU tests and tooling) ---- */
int bddc_host_setup_create(const bddc_problem* p, const bddc_gpu_options* opt, bddc_host_setup** out);
int bddc_host_setup_blocks(const bddc_host_setup* s, int32_t subdomain, double* phi, double* lambda,
                           double* aci);
int bddc_host_setup_coarse(const bddc_host_setup* s, int32_t* nnz, int32_t* row_offsets,
                           int32_t* col_indices, double* values);
int bddc_host_setup_interior_solve(const bddc_host_setup* s, int32_t subdomain, double* x);
int bddc_host_setup_stats(const bddc_host_setup* s, bddc_stats* stats);
void bddc_host_setup_destroy(bddc_host_setup* s);

/* ---- multi-GPU ---- */
int bddc_dist_unique_id(uint8_t* id128);
int bddc_gpu_create_dist(const bddc_problem* global_problem, const bddc_gpu_options* opt,
                         const bddc_dist_options* dist, bddc_gpu_ctx** out);
/* Device vector layout of a context (identity on one GPU); local_to_global may be NULL. */
int bddc_gpu_layout(const bddc_gpu_ctx* ctx, int32_t* n_local, int32_t* n_rows, int32_t* n_owned,
                    int32_t* local_to_global);
int bddc_rank_plan_create(const bddc_problem* p, int32_t rank, int32_t world,
                          const int32_t* subdomain_rank, bddc_rank_plan** out);
int bddc_rank_plan_get_view(const bddc_rank_plan* plan, bddc_rank_plan_view* view);
void bddc_rank_plan_destroy(bddc_rank_plan* plan);

/* ---- GPU hot path ----
 * On a distributed context the host entry points take GLOBAL vectors and each rank writes
 * the entries of its own subdomains; the *_device entry points take rank-local vectors
 * (bddc_gpu_layout). Every rank must make the same calls in the same order.
 * A context shares the problem's (immutable) data with the handle it was created from: the
 * problem handle may be destroyed before the context, the data lives until both are gone. */
int bddc_gpu_create(const bddc_problem* p, const bddc_gpu_options* opt, bddc_gpu_ctx** out);
int bddc_gpu_apply(bddc_gpu_ctx* ctx, const double* r, double* z);
int bddc_gpu_apply_device(bddc_gpu_ctx* ctx, const double* r_dev, double* z_dev, void* cuda_stream);
int bddc_gpu_stage(bddc_gpu_ctx* ctx, int32_t stage, const double* in0, const double* in1,
                   const double* in2, double* out);
int bddc_gpu_pcg(bddc_gpu_ctx* ctx, const double* b, const bddc_solver_options* opt,
                 int32_t precondition, double* x, bddc_solve_report* report, double* history,
                 int32_t history_capacity);
int bddc_gpu_pcg_device(bddc_gpu_ctx* ctx, const double* b_dev, const bddc_solver_options* opt,
                        int32_t precondition, double* x_dev, bddc_solve_report* report,
                        double* history, int32_t history_capacity, void* cuda_stream);
int bddc_gpu_subdomain_blocks(const bddc_gpu_ctx* ctx, int32_t subdomain, double* phi,
                              double* lambda, double* aci);
int bddc_gpu_coarse_matrix(const bddc_gpu_ctx* ctx, int32_t* nnz, int32_t* row_offsets,
                           int32_t* col_indices, double* values);
int bddc_gpu_get_stats(const bddc_gpu_ctx* ctx, bddc_stats* stats);
int bddc_gpu_set_profile(bddc_gpu_ctx* ctx, int32_t on);
int bddc_gpu_kernel_times(const bddc_gpu_ctx* ctx, bddc_kernel_times* times, int32_t reset);
int bddc_gpu_synchronize(bddc_gpu_ctx* ctx);
/* Diagnostics: per-CTA, per-warp cycle accounting {total, wait, barrier, units} of the last
 * interior solve; only recorded when the context was created with BDDC_SOLVE_STATS set.
 * Returns the number of int64 values written (0 when not recorded). */
int64_t bddc_gpu_solve_profile(bddc_gpu_ctx* ctx, int64_t* out, int64_t capacity);
const char* bddc_gpu_last_error(const bddc_gpu_ctx* ctx);
void bddc_gpu_destroy(bddc_gpu_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* BDDC_B200_H */
