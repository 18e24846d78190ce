// Device context: owns the uploaded device image, scratch vectors and the stream;
// runs the BDDC apply and the device-resident PCG loop. No CUDA types leak out of
// this header (the C-ABI layer in capi.cpp includes it from plain C++).
#pragma once

#include <atomic>
#include <cstdlib>
#include <cstdint>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "host/problem.hpp"
#include "host/setup.hpp"

namespace bddc_b200 {

// Kernel launches issued by this library in this process (defined in device/context.cu).
extern std::atomic<std::int64_t> g_kernel_launches;

struct GpuOptions {
    int device = 0;
    int workers = 0;              // host setup threads (0 = hardware concurrency)
    int coarse_mode = 0;          // 0: dense replicated A_c^{-1}; 1: reference-faithful coarse CG
    double coarse_rtol = 1e-12;   // reference preconditioner.hpp:42
    double coarse_atol = 0.0;
    int coarse_max_iterations = 500;
    int leaf_size = 24;           // measured best on B200 (tools/leaf_sweep.sh)
    int local_blocks = 8;         // CTAs per subdomain for the K_i GEMV (measured: 8 > 4, = 16)
    int solve_parts = 0;          // CTAs per subdomain in the interior solve (0 = auto)
    bool profile = false;         // record per-kernel CUDA events in apply()
    bool setup_on_device = true;  // GPU setup (device/setup.cu); false: host numeric setup (host/setup.cpp)
    // second interior solve of the apply as the harmonic extension u0 - A_II^{-1} A_IG z_G with a
    // pruned forward sweep (BDDC_HARMONIC=0 selects the full solve of r_I - A_IG z_G)
    bool harmonic = !(std::getenv("BDDC_HARMONIC") && std::string(std::getenv("BDDC_HARMONIC")) == "0");
};

struct SolverOpts {
    double rel_tolerance = 1e-8;
    double abs_tolerance = 0.0;
    int max_iterations = 1000;
    bool record_history = false;
};

struct SolveResult {
    int iterations = 0;
    double final_relative_residual = 0.0;
    std::vector<double> history;
    std::optional<double> condition_estimate;
    bool converged = false;
};

struct ProblemData {
    Decomposition decomposition;
    ConstraintSet constraints;
    CsrMatrix global_matrix;
    std::vector<CsrMatrix> local_matrices;
    std::vector<index_t> coords;  // optional (empty => graph ordering)
};

struct KernelTimes {
    double interior_ms = 0.0;   // both interior solves
    std::int64_t interior_launches = 0;
    double iface_ms = 0.0;      // restrict + coarse + local
    double apply_ms = 0.0;
    std::int64_t applies = 0;
};

// Multi-GPU: this process is rank `rank` of `world` (one per B200); the context is built
// from the GLOBAL problem and keeps the rank's block of subdomains (host/distribute.hpp).
struct DistSpec {
    int rank = 0;
    int world = 1;
    char nccl_id[128] = {};     // ncclUniqueId from rank 0, broadcast by the caller
    std::vector<int> sub_rank;  // optional subdomain -> rank (empty: rectangular blocks)
};

// 128-byte ncclUniqueId for a new distributed job (rank 0 calls this).
void dist_nccl_id(char out[128]);

enum class Stage : int { interior = 0, coarse = 1, local = 2, static_condensation = 3 };

class GpuContext {
public:
    GpuContext(ProblemData problem, const GpuOptions& opt, const DistSpec* dist = nullptr);
    // shares the (immutable) problem instead of copying it
    GpuContext(std::shared_ptr<const ProblemData> problem, const GpuOptions& opt, const DistSpec* dist = nullptr);
    ~GpuContext();
    GpuContext(const GpuContext&) = delete;
    GpuContext& operator=(const GpuContext&) = delete;

    index_t n() const;         // device vector length (distributed: the rank-local layout)
    index_t n_global() const;  // host vector length of apply_host / pcg_host
    // distributed layout: [0, n_owned) owned, [0, n_rows) the rank's dofs, then the halo
    index_t n_owned() const;
    index_t n_rows() const;
    int rank() const;
    int world() const;
    const std::vector<index_t>& local_to_global() const;  // empty on one GPU
    // Device pointers (n() doubles each) on the context's device; stream may be null.
    // Host entry points take global vectors; a distributed rank reads and writes only
    // the entries of its own subdomains.
    void apply_device(const double* r, double* z, void* stream);
    void apply_host(const double* r, double* z);
    SolveResult pcg_host(const double* b, const SolverOpts& o, double* x, bool precondition);
    SolveResult pcg_device(const double* b, const SolverOpts& o, double* x, bool precondition,
                           void* stream);
    void stage_host(Stage st, const double* in0, const double* in1, const double* in2, double* out);

    const BddcSetup& setup() const;
    const ProblemData& problem() const;
    double setup_seconds() const;
    // Phi_i (n_local x n_primal), Lambda_i, A_ci (n_primal^2) host copies; null pointers skipped
    void subdomain_blocks(int i, double* phi, double* lambda, double* aci) const;
    double setup_device_seconds() const;
    std::int64_t graph_captures() const;
    int coarse_mode() const;  // in effect (direct mode falls back to coarse CG above the dense cap)
    int switches() const;     // env_switch_mask() at creation
    std::int64_t apply_bytes() const;       // algorithmic FP64 bytes per apply
    std::int64_t interior_apply_bytes() const;  // algorithmic bytes of the two interior solves of an apply
    std::int64_t interior_pass_bytes() const;  // stream bytes of one batched interior solve
    int solve_parts() const;
    std::int64_t factor_values() const;
    KernelTimes kernel_times();
    void reset_kernel_times();
    void set_profile(bool on);
    int device() const;
    void synchronize();
    std::int64_t solve_profile(std::int64_t* out, std::int64_t cap);

private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
};

// BDDC_* environment switches: bit i of the mask = switch i is set.
const char* env_switch_name(int i);
int env_switch_mask();

std::optional<double> condition_estimate(const std::vector<double>& alphas,
                                         const std::vector<double>& betas);

}  // namespace bddc_b200
