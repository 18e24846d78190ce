// GpuContext: uploads the device image and orchestrates the apply / PCG on one B200.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <thread>

#include "../context.hpp"
#include "../host/distribute.hpp"
#include "../host/program.hpp"
#include "../host/gpu_setup.hpp"
#include "setup.cuh"
#include "comm.cuh"
#include "iface.cuh"
#include "pcg.cuh"
#include "solve.cuh"

namespace bddc_b200 {

std::atomic<std::int64_t> g_kernel_launches{0};
// BDDC_PDL=1: programmatic dependent launch for the PCG loop's kernels. Off by default:
// measured on B200 inside the per-iteration CUDA graph it changed nothing (within noise).
bool pdl_enabled() {
    static const bool on = std::getenv("BDDC_PDL") && std::atoi(std::getenv("BDDC_PDL")) == 1;
    return on;
}

namespace {

template <typename T>
struct DBuf {
    T* p = nullptr;
    std::size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { if (p) cudaFree(p); }
    void alloc(std::size_t count) {
        if (p) { cudaFree(p); p = nullptr; }
        n = count;
        if (count) BDDC_CUDA(cudaMalloc(&p, sizeof(T) * count));
    }
    void upload(const std::vector<T>& v) {
        alloc(std::max<std::size_t>(v.size(), 1));
        if (!v.empty()) BDDC_CUDA(cudaMemcpy(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
    }
};

// Non-owning view into a scratch block.
template <typename T>
struct Span {
    T* p = nullptr;
    std::size_t n = 0;
};

// The device setup's numeric scratch (supernode fronts, Schur blocks, saddle matrices: ~1-2 GB at
// C2) as one block that is kept for the process's next setup on the same device, like a caching
// allocator: freeing and re-mapping GBs costs 20-200 ms of host time per construction, more than
// the setup's kernels. BDDC_SETUP_SCRATCH_CACHE=0 frees it after every setup.
std::mutex g_scratch_mu;
std::vector<std::pair<char*, std::size_t>> g_scratch(64, {nullptr, 0});

struct SetupScratch {
    char* p = nullptr;
    std::size_t bytes = 0;
    int dev = 0;
    SetupScratch(int device, std::size_t need) : dev(device) {
        char* stale = nullptr;
        {
            std::lock_guard<std::mutex> g(g_scratch_mu);
            auto& c = g_scratch.at(static_cast<std::size_t>(dev));
            if (c.first && c.second >= need) {
                p = c.first;
                bytes = c.second;
            } else {
                stale = c.first;
            }
            if (p || stale) c = {nullptr, 0};
        }
        if (stale) BDDC_CUDA(cudaFree(stale));
        if (!p) {
            bytes = need;
            BDDC_CUDA(cudaMalloc(&p, bytes));
        }
    }
    SetupScratch(const SetupScratch&) = delete;
    SetupScratch& operator=(const SetupScratch&) = delete;
    ~SetupScratch() {
        static const bool keep = !(std::getenv("BDDC_SETUP_SCRATCH_CACHE") && std::atoi(std::getenv("BDDC_SETUP_SCRATCH_CACHE")) == 0);
        cudaDeviceSynchronize();  // no setup work may still use the block
        char* drop = p;
        if (keep) {
            std::lock_guard<std::mutex> g(g_scratch_mu);
            auto& c = g_scratch[static_cast<std::size_t>(dev)];
            if (!c.first || c.second < bytes) {
                std::swap(c.first, drop);
                std::swap(c.second, bytes);
            }
        }
        if (drop) cudaFree(drop);
    }
    template <typename T>
    Span<T> span(std::size_t off, std::size_t n) const { return {reinterpret_cast<T*>(p + off), n}; }
};

struct Event {
    cudaEvent_t e = nullptr;
    Event() { BDDC_CUDA(cudaEventCreate(&e)); }
    ~Event() { if (e) cudaEventDestroy(e); }
};

struct ApplyEvents {  // interior solve | interface steps | interior solve of one apply
    Event e[4];
};

// Host passes over rank-sized vectors (multi-GPU host entry points): split over a few threads.
template <typename F>
void host_parallel(std::size_t n, F&& f, std::size_t min_items = std::size_t(1) << 16) {
    static const int nt = std::max(1, std::getenv("BDDC_HOST_THREADS") ? std::atoi(std::getenv("BDDC_HOST_THREADS")) : 4);
    if (nt == 1 || n < min_items) {
        f(std::size_t(0), n);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back([&, t] { f(n * t / nt, n * (t + 1) / nt); });
    f(std::size_t(0), n / nt);
    for (auto& x : th) x.join();
}

void ensure_finite(const double* x, index_t n, const char* context) {
    std::atomic<bool> bad{false};
    host_parallel(static_cast<std::size_t>(n), [&](std::size_t a, std::size_t b) {
        bool any = false;  // branch-free, vectorisable pass; the index search only on failure
        for (std::size_t i = a; i < b; ++i) any |= !(std::fabs(x[i]) <= 1.7976931348623157e308);
        if (any) bad = true;
    });
    if (!bad) return;
    for (index_t i = 0; i < n; ++i)
        if (!std::isfinite(x[i]))
            throw std::invalid_argument(std::string(context) + ": non-finite entry at index " + std::to_string(i));
}

// Multi-GPU host entry points with a pinned (device-mapped) user buffer: the rank's runs
// {local, global, length} are read from / written to host memory directly over PCIe by one
// warp per run, with no host-side staging pass (gather_host / scatter_host).
__global__ void __launch_bounds__(256) gather_runs_kernel(const index_t* __restrict__ runs, int n_runs,
                                                          const double* __restrict__ g, double* __restrict__ l) {
    const int lane = threadIdx.x & 31;
    for (int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < n_runs; k += (gridDim.x * blockDim.x) >> 5) {
        const index_t lo = runs[3 * k], go = runs[3 * k + 1], len = runs[3 * k + 2];
        for (index_t i = lane; i < len; i += 32) l[lo + i] = g[go + i];
    }
}

__global__ void __launch_bounds__(256) scatter_runs_kernel(const index_t* __restrict__ runs, int n_runs, index_t n_rows,
                                                           const double* __restrict__ l, double* __restrict__ g) {
    const int lane = threadIdx.x & 31;
    for (int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < n_runs; k += (gridDim.x * blockDim.x) >> 5) {
        const index_t lo = runs[3 * k], go = runs[3 * k + 1], len = runs[3 * k + 2];
        if (lo >= n_rows) continue;
        for (index_t i = lane; i < len; i += 32) g[go + i] = l[lo + i];
    }
}

// Device address of a pinned, device-mapped host buffer (nullptr for pageable memory).
const void* mapped_host_pointer(const void* p) {
    static const bool on = !std::getenv("BDDC_ZERO_COPY") || std::atoi(std::getenv("BDDC_ZERO_COPY")) != 0;
    if (!on) return nullptr;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return nullptr;
    }
    return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

// pcg.cpp:21-36
void sampled_symmetry_check(const CsrMatrix& A) {
    if (A.nrows != A.ncols) throw std::invalid_argument("pcg: matrix must be square");
    const index_t stride = std::max<index_t>(1, A.nrows / 16);
    for (index_t i = 0; i < A.nrows; i += stride) {
        if (A.row_offsets[i] == A.row_offsets[i + 1]) continue;
        const index_t p = A.row_offsets[i];
        const index_t j = A.col_indices[p];
        const double a = A.values[p];
        double b = 0.0;
        for (index_t q = A.row_offsets[j]; q < A.row_offsets[j + 1]; ++q)
            if (A.col_indices[q] == i) { b = A.values[q]; break; }
        if (std::abs(a - b) > 1e-12 * (std::abs(a) + std::abs(b)) + 1e-300)
            throw std::invalid_argument("pcg: matrix is not symmetric");
    }
}

// Every BDDC_* environment switch the library reads, in mask-bit order.
const char* const kEnvSwitches[] = {
    "BDDC_SPLIT", "BDDC_HARMONIC", "BDDC_GRAPH", "BDDC_FUSED_EX", "BDDC_P2P", "BDDC_COOP_COARSE",
    "BDDC_DIR_SPMV", "BDDC_PDL", "BDDC_PROFILE_STRIDE", "BDDC_ZERO_COPY", "BDDC_HOST_THREADS",
    "BDDC_UNIT_BYTES", "BDDC_MIN_CHUNK_ROWS", "BDDC_TILE_COST", "BDDC_JOBS_PER_WARP", "BDDC_SOLVE_STATS",
    "BDDC_EXCH_STATS", "BDDC_FUSED_TRACE", "BDDC_NO_EXCHANGE", "BDDC_EXPERIMENTS", "BDDC_SETUP_TIMES",
    "BDDC_PRUNED_JOBS", "BDDC_PLAIN_LOOP", "BDDC_SADDLE_GLOBAL", "BDDC_PAIR_TILES", "BDDC_K_FULL", "BDDC_STEP", "BDDC_MAX_CHAIN", "BDDC_QUAD_TILES",
    "BDDC_SETUP_SCRATCH_CACHE", "BDDC_ELL16"};
constexpr int kNumEnvSwitches = sizeof(kEnvSwitches) / sizeof(kEnvSwitches[0]);

// Diagnostics (BDDC_SETUP_TIMES=1): wall time of each setup phase on stderr.
struct SetupTimer {
    bool on = std::getenv("BDDC_SETUP_TIMES") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        cudaDeviceSynchronize();
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[setup] %-34s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

// Largest coarse dimension served by the dense replicated A_c^-1 (n_c^2 doubles per GPU, n_c
// doubles of r_c in the K_i kernel's shared memory, and an O(n_c^3) Gauss-Jordan inverse whose
// rank-1 passes stream n_c^2 doubles each); above it the coarse solve is the coarse CG.
constexpr index_t kDenseCoarseMax = 4096;
}  // namespace

struct GpuContext::Impl {
    // the problem, shared with the caller's handle (read-only: no per-construction deep copy)
    std::shared_ptr<const ProblemData> pbs;
    const ProblemData& pb() const { return *pbs; }
    GpuOptions opt;
    BddcSetup setup;
    int device = 0;
    cudaStream_t stream = nullptr;
    std::mutex mu;  // the reference apply() is callable concurrently; serialise here

    // interior-solve programs: the full solve, and the harmonic extension A_II^{-1} A_IG z_G of
    // the second solve of the apply (pruned forward sweep; BDDC_HARMONIC=0 disables)
    struct SolveProgram {
        DBuf<PartDesc> parts;
        DBuf<double> stream;
        DBuf<std::int32_t> units, phases, gmap, couple_ptr, couple_gamma;
        DBuf<double> couple_val;
        std::int64_t stream_bytes = 0;
        bool valid = false;
        void upload(const SolvePools& sp) {
            parts.alloc(std::max<std::size_t>(sp.parts.size(), 1));
            if (!sp.parts.empty())
                BDDC_CUDA(cudaMemcpy(parts.p, sp.parts.data(), sizeof(PartDesc) * sp.parts.size(), cudaMemcpyHostToDevice));
            if (sp.stream_words >= 0) stream.alloc(std::max<std::int64_t>(sp.stream_words, 1));  // device fill
            else stream.upload(sp.stream);
            units.upload(sp.units);
            phases.upload(sp.phases);
            gmap.upload(sp.gmap);
            couple_ptr.upload(sp.couple_ptr);
            couple_gamma.upload(sp.couple_gamma);
            couple_val.upload(sp.couple_val);
            for (const PartDesc& pd : sp.parts) stream_bytes += pd.stream_bytes;
            valid = !sp.parts.empty();
        }
    };
    SolveProgram prog, harm, head;
    // fused coarse solve: r_c formed once per GPU inside the cooperative K_i grid (large n_c),
    // else (or when the grid cannot be co-resident) every CTA forms r_c itself
    DBuf<double> rc_g;
    DBuf<unsigned long long> coarse_ctr;
    bool coop_coarse = false;
    // split apply (head + harmonic programs, device/solve.cuh y_out / y_in): y0 = L^-1 r_I per
    // part in local order; BDDC_SPLIT=0 keeps u0 from a full solve
    DBuf<double> ybuf;
    bool use_split = !(std::getenv("BDDC_SPLIT") && std::atoi(std::getenv("BDDC_SPLIT")) == 0);
    bool split() const { return use_split && harm.valid && head.valid; }
    SolveLaunch launch;
    // interface data
    DBuf<SubdomainDesc> subs;
    DBuf<std::int32_t> slot_rows;  // per local interface slot: {begin, end} of its global A_GI row
    DBuf<std::int32_t> iface_dof, iface_gid, iface_writer, primal, local_dofs, gi_dof, gi_row_ptr, gi_row_col,
        gi_own_ptr, gi_own_ref, dof_own_ptr, dof_own_ref, c_own_ptr, c_own_ref, lrow_ptr, lrow_col, iface_own4, c_own4;
    DBuf<double> iface_w, kmat, phig, phi, gi_row_val, coarse_inv, lrow_val, weights_local;
    // coarse matrix (CG mode)
    DBuf<std::int32_t> Ac_ptr, Ac_col;
    DBuf<double> Ac_val, coarse_status;
    // global matrix
    DBuf<std::int32_t> A_ptr, A_col;
    DBuf<double> A_val;
    DBuf<std::int64_t> ell_off;  // the global (rank) matrix as sliced ELL (PcgDevice)
    DBuf<std::uint16_t> ell_len;
    DBuf<std::int32_t> ell_col;
    DBuf<std::int16_t> ell_d16;  // column offsets from the row, when they all fit (else empty)
    DBuf<double> ell_val;
    // scratch
    DBuf<double> U, gbuf, hbuf, cbuf, xc, lbuf, vin, vout, vtmp, vtmp2;
    // pcg
    DBuf<double> x, r, z, p, q, part_a, part_b, rho, alpha, beta, hist, scal;
    DBuf<int> iter_ctr;
    double* pinned = nullptr;
    double* pinned_dev = nullptr;  // the same buffer, mapped (update's fused check writes it)
    DBuf<std::uint64_t> solo_seq;  // one GPU: grid tickets of update's fused check and dir_spmv
    DBuf<unsigned int> solo_ticket;
    DBuf<unsigned int> plain_bar;  // grid barrier of the one-launch plain CG
    // plain CG on one GPU as one cooperative launch (BDDC_PLAIN_LOOP=0: the per-kernel loop)
    bool use_plain_loop = !(std::getenv("BDDC_PLAIN_LOOP") && std::atoi(std::getenv("BDDC_PLAIN_LOOP")) == 0);
    // K_i stored as packed symmetric 32 x 32 tiles, one CTA per subdomain (BDDC_K_FULL=1: the
    // row-major K_i and local_blocks CTAs per subdomain)
    bool kpacked = !(std::getenv("BDDC_K_FULL") && std::atoi(std::getenv("BDDC_K_FULL")) == 1);
    // BDDC_STEP=1 (experiment, measured slower: two grid barriers over 592 CTAs cost more than
    // the graph's kernel boundaries): xpay + SpMV + update of a BDDC-PCG iteration on one GPU as
    // one cooperative launch
    bool use_step = std::getenv("BDDC_STEP") && std::atoi(std::getenv("BDDC_STEP")) == 1;
    int step_ok = -1;
    DBuf<unsigned long long> step_bar;
    DBuf<double> kpart;  // packed K_i: per tile two 32-vectors of partial sums
    int plain_loop_ok = -1;  // occupancy check, once
    DBuf<double> p_alt;            // second direction buffer (pcg_dir_spmv)
    // BDDC_DIR_SPMV=1: fuse p = z + beta p into the SpMV. Off by default: measured on B200 the
    // on-the-fly p entries (two extra gathers per nonzero) cost more than the xpay pass saves
    bool use_dir_spmv = std::getenv("BDDC_DIR_SPMV") && std::atoi(std::getenv("BDDC_DIR_SPMV")) == 1;
    int max_it_alloc = 0;

    std::int32_t max_iface = 0, max_primal = 0, n_coarse = 0, n_gi = 0;
    std::int64_t solve_stream_bytes = 0, harm_stream_bytes = 0, factor_vals = 0, harm_fwd_values = 0,
                 head_bwd_values = 0;
    std::int64_t k_values = 0, phig_values = 0, ginnz = 0, couple_nnz = 0;

    KernelTimes times;
    const double* apply_skip = nullptr;  // set while the pipelined PCG enqueues speculative applies
    // set by pcg(): the harmonic-extension launch also forms the per-CTA partials of r.z
    const double* apply_dot_r = nullptr;
    int apply_dot_n = 0;
    DBuf<double> part_rz;

    // CUDA graphs of the PCG iteration (BDDC_GRAPH=0 disables): A = spmv/update/check and the
    // convergence read-back, B = the speculative apply, r.z and the new direction. The device
    // iteration counter and exchange sequence counters make one capture valid for every
    // iteration; with profiling on, B's four event-record nodes are rebound to fresh pool
    // events before each launch so the per-kernel timing stays live.
    struct IterGraphs {
        cudaGraphExec_t a = nullptr, b = nullptr;
        cudaGraphExec_t b_plain = nullptr;  // profiling on: the same iteration without event nodes
        cudaGraph_t b_graph = nullptr;  // kept alive: its event-record nodes are rebound per launch
        std::int64_t a_kernels = 0, b_kernels = 0;
        cudaGraphNode_t ev_nodes[4] = {};
        PcgDevice key{};
        bool precondition = false, profile = false, valid = false;
        void reset() {
            if (a) cudaGraphExecDestroy(a);
            if (b) cudaGraphExecDestroy(b);
            if (b_plain) cudaGraphExecDestroy(b_plain);
            b_plain = nullptr;
            if (b_graph) cudaGraphDestroy(b_graph);
            a = b = nullptr;
            b_graph = nullptr;
            valid = false;
        }
        ~IterGraphs() { reset(); }
    } graphs;
    ApplyEvents* capture_events = nullptr;
    bool suppress_profile = false;  // capturing the unprofiled iteration graph
    // profiling samples one pipelined iteration in BDDC_PROFILE_STRIDE (default 8): rebinding the
    // event nodes costs host time inside the host-driven loop (~6% of the solve if every iteration)
    int profile_stride = std::getenv("BDDC_PROFILE_STRIDE") ? std::max(1, std::atoi(std::getenv("BDDC_PROFILE_STRIDE"))) : 8;
    std::unique_ptr<ApplyEvents> graph_events;
    bool use_graphs = !(std::getenv("BDDC_GRAPH") && std::atoi(std::getenv("BDDC_GRAPH")) == 0);

    template <typename Body>
    cudaGraphExec_t capture(cudaStream_t s, Body&& body, std::int64_t* kernels, cudaGraph_t* keep = nullptr) {
        cudaGraph_t g = nullptr;
        const std::int64_t l0 = g_kernel_launches.load();
        BDDC_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
        try {
            body();
        } catch (...) {
            cudaStreamEndCapture(s, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        BDDC_CUDA(cudaStreamEndCapture(s, &g));
        // captured launches run at every graph launch: count them there, not here
        *kernels = g_kernel_launches.load() - l0;
        g_kernel_launches.fetch_sub(*kernels);
        cudaGraphExec_t e = nullptr;
        BDDC_CUDA(cudaGraphInstantiate(&e, g, 0));
        if (keep) *keep = g;
        else cudaGraphDestroy(g);
        return e;
    }
    Event check_ev;  // convergence read-back of the pipelined PCG loop
    Event norm_ev;   // ||b|| read-back

    // ---- multi-GPU (null / unused on one GPU)
    std::unique_ptr<RankPlan> plan;
    std::unique_ptr<Comm> comm;
    DBuf<std::int32_t> halo_idx, iface_idx;
    DBuf<double> halo_send, iface_send, gath_a, gath_b, gath_c, gath_d;  // p.q, r.r, r.z, b.b per rank
    // peer-memory exchanges (default): IPC mappings, one descriptor + sequence per type
    enum ExType { kExU = 0, kExP = 1, kExH = 2, kExC = 3, kExPQ = 4, kExRR = 5, kExRZ = 6, kExNB = 7, kExZ = 8 };
    std::unique_ptr<PeerLinks> links;
    std::vector<ExchangeDesc> ex_host;  // passed by value (kernel parameters)
    DBuf<std::uint64_t> ex_flags, ex_seq;  // flags [type][src]; per-type sequence counters
    DBuf<unsigned long long> ex_stats;
    DBuf<double*> ex_item_dst;
    DBuf<std::int32_t> ex_item_src;
    // fused LL exchanges (device/fused_comm.cuh): a per-rank LL receive buffer (exported to the
    // peers), the sent items bucketed by producing CTA, one grid ticket per type. BDDC_FUSED_EX
    // bit mask (default 7): 1 = the p.q / r.r scalars, 2 = the apply's u0 halo / c_i / h_i,
    // 4 = z's halo with r.z; 0 keeps the separate exchange launches
    DBuf<ll_word> ll_buf;
    std::int64_t ll_off[5] = {};  // my regions (words): u0 halo, z halo, h_i, c_i, scalars
    DBuf<std::int32_t> ll_src, ll_cta;
    DBuf<ll_word*> ll_dst, ll_sc_dst;  // item destinations; scalar destinations [row][peer != me]
    std::int64_t ll_cta_off[kFlagTypes] = {};
    bool ll_has[kFlagTypes] = {};
    DBuf<unsigned int> ex_ticket;
    int fused_ex = std::getenv("BDDC_FUSED_EX") ? std::atoi(std::getenv("BDDC_FUSED_EX")) : 7;
    bool pub_rz = false;  // set by pcg(): the harmonic-extension launch publishes z's halo + r.z
    bool p2p() const { return static_cast<bool>(links); }
    // the apply's exchanges ride on its kernels (u0 halo, c_i gather, h_i) when peer-memory
    bool fused_apply() const {
        return dist() && p2p() && (fused_ex & 2) && !no_exchange && harm.valid && opt.coarse_mode == 0;
    }
    bool fused_pcg() const { return dist() && p2p() && (fused_ex & 1) && !no_exchange; }
    DBuf<unsigned long long> fused_trace;  // diagnostics: BDDC_FUSED_TRACE=1 (event ring)
    // kernel ids of the trace: 0 solve0, 1 restrict, 2 K_i, 3 harmonic solve, 5 spmv_dot, 6 update
    Publish ll_publish(int t, int kid, const double* src) const {
        Publish P;
        P.seq = ex_seq.p + t;
        P.ticket = ex_ticket.p + t;
        P.trace = fused_trace.p;
        P.kid = kid;
        if (ll_has[t]) {
            P.cta_ptr = ll_cta.p + ll_cta_off[t];
            P.item_src = ll_src.p;
            P.item_dst = ll_dst.p;
            P.src = src;
        }
        return P;
    }
    // scalar row (0 p.q, 1 r.r, 2 r.z): part[0..grid) -> red[rank] -> every peer's row slot
    void ll_scalar(Publish& P, int row, const double* part, int grid, double* red) const {
        P.part = part;
        P.red = red;
        P.grid = grid;
        P.slot = comm->rank();
        P.sc_dst = ll_sc_dst.p + static_cast<std::int64_t>(row) * (comm->world() - 1);
        P.n_sc = comm->world() - 1;
    }
    // timing experiments only (wrong results): BDDC_NO_EXCHANGE=1 skips every exchange
    bool no_exchange = std::getenv("BDDC_NO_EXCHANGE") && std::atoi(std::getenv("BDDC_NO_EXCHANGE")) == 1;
    std::int64_t graph_captures = 0;  // PCG iteration graphs captured (stats)
    int switch_mask = 0;              // env_switch_mask() at creation (stats)
    double setup_device_s = 0.0;      // device setup kernels (stats)
    std::vector<std::int32_t> halo_soff, halo_roff, iface_soff, iface_roff;
    index_t n_global = 0, n_rows = 0, n_owned = 0;
    std::string symmetry_error;  // distributed: global symmetry check done once at creation
    // host entry points: the rank-local layout as runs {local, global, length} of consecutive
    // indices (split at n_rows, and into pieces of at most kRunPiece entries: a warp copies one
    // piece, so a rank whose rows are one contiguous block of the global vector still spreads
    // its PCIe reads over the whole GPU), copied through a pinned staging buffer
    static constexpr index_t kRunPiece = 1024;
    std::vector<std::array<index_t, 3>> runs;
    double* stage = nullptr;
    void build_runs() {
        const auto& l2g = plan->local_to_global;
        const index_t n = static_cast<index_t>(l2g.size());
        for (index_t l = 0; l < n;) {
            index_t e = l + 1;
            while (e < n && e != n_rows && e - l < kRunPiece && l2g[e] == l2g[e - 1] + 1) ++e;
            runs.push_back({l, l2g[l], e - l});
            l = e;
        }
        BDDC_CUDA(cudaMallocHost(&stage, sizeof(double) * std::max<index_t>(n, 1)));
        std::vector<index_t> flat;
        for (const auto& r : runs) flat.insert(flat.end(), r.begin(), r.end());
        runs_dev.upload(flat);
    }
    DBuf<index_t> runs_dev;
    int runs_grid() const { return std::max(1, std::min<int>(148 * 4, static_cast<int>((runs.size() + 7) / 8))); }
    // global (host, device-mapped) -> dst (device, all local entries)
    void gather_mapped(const double* g, double* dst, cudaStream_t s) const {
        gather_runs_kernel<<<runs_grid(), 256, 0, s>>>(runs_dev.p, static_cast<int>(runs.size()), g, dst);
        BDDC_LAUNCHED();
    }
    // src rows (device) -> global (host, device-mapped)
    void scatter_mapped(const double* src, double* g, cudaStream_t s) const {
        scatter_runs_kernel<<<runs_grid(), 256, 0, s>>>(runs_dev.p, static_cast<int>(runs.size()), n_rows, src, g);
        BDDC_LAUNCHED();
    }
    void gather_host(const double* g) const {  // global -> stage (all local entries)
        host_parallel(runs.size(), [&](std::size_t a, std::size_t b) {
            for (std::size_t k = a; k < b; ++k) std::memcpy(stage + runs[k][0], g + runs[k][1], sizeof(double) * runs[k][2]);
        }, 64);
    }
    void scatter_host(double* g) const {  // stage rows -> global
        host_parallel(runs.size(), [&](std::size_t a, std::size_t b) {
            for (std::size_t k = a; k < b; ++k)
                if (runs[k][0] < n_rows) std::memcpy(g + runs[k][1], stage + runs[k][0], sizeof(double) * runs[k][2]);
        }, 64);
    }

    bool dist() const { return static_cast<bool>(comm); }

    // u0 / p halo: owners send their entries, the halo region [n_rows, n) is overwritten
    void halo_exchange(double* v, cudaStream_t s) {
        if (!dist() || no_exchange) return;
        if (p2p()) {
            const int t = v == U.p ? kExU : kExP;
            launch_exchange(ex_host[t], v, nullptr, 0, 0, s);
            return;
        }
        launch_pack(static_cast<int>(plan->halo_send_idx.size()), halo_idx.p, v, halo_send.p, s);
        comm->exchange(plan->halo_peers, halo_send.p, halo_soff, v + n_rows, halo_roff, s);
    }
    // h_i of interface dofs shared with other ranks -> remote hbuf slots
    void iface_exchange(cudaStream_t s) {
        if (!dist() || no_exchange) return;
        if (p2p()) {
            launch_exchange(ex_host[kExH], hbuf.p, nullptr, 0, 0, s);
            return;
        }
        launch_pack(static_cast<int>(plan->iface_send_slot.size()), iface_idx.p, hbuf.p, iface_send.p, s);
        comm->exchange(plan->iface_peers, iface_send.p, iface_soff, hbuf.p + plan->n_local_slots, iface_roff, s);
    }
    // every rank's c_i (padded blocks, rank order) for the ordered r_c sum
    void gather_cbuf(cudaStream_t s) {
        if (!dist() || no_exchange) return;
        if (p2p()) launch_exchange(ex_host[kExC], cbuf.p, nullptr, 0, 0, s);
        else comm->allgather_inplace(cbuf.p, static_cast<std::size_t>(plan->cbuf_pad), s);
    }
    // r.z gather fused with the halo of z (peer-memory mode, preconditioned): the new direction
    // p = z + beta p is then formed on the halo locally, bit-identical to its owner's values
    void gather_rz_with_z_halo(const double* part, int grid, cudaStream_t s) {
        if (no_exchange) return;
        launch_exchange2(ex_host[kExZ], z.p, ex_host[kExRZ], gath_c.p, part, grid, comm->rank(), s);
    }

    // part[0..grid) -> gath[rank], then gathered over ranks (consumers sum in rank order)
    void gather_partial(const double* part, int grid, double* gath, cudaStream_t s) {
        if (!dist() || no_exchange) return;
        if (p2p()) {
            const int t = gath == gath_a.p ? kExPQ : gath == gath_b.p ? kExRR : gath == gath_c.p ? kExRZ : kExNB;
            launch_exchange(ex_host[t], gath, part, grid, comm->rank(), s);
            return;
        }
        launch_reduce_to(part, grid, gath + comm->rank(), false, s);
        comm->allgather_inplace(gath, 1, s);
    }

    SolveParams solve_params(const double* in, double* out, const SolveProgram* pg = nullptr) const {
        const SolveProgram& G = pg ? *pg : prog;
        SolveParams P{};
        P.skip = apply_skip;
        P.parts = G.parts.p;
        P.subs = subs.p;
        P.stream = G.stream.p;
        P.units = G.units.p;
        P.phases = G.phases.p;
        P.gmap = G.gmap.p;
        P.couple_ptr = G.couple_ptr.p;
        P.couple_gamma = G.couple_gamma.p;
        P.couple_val = G.couple_val.p;
        P.u0 = U.p;
        P.iface_gid = iface_gid.p;
        P.iface_dof = iface_dof.p;
        P.iface_writer = iface_writer.p;
        P.gi_own_ptr = gi_own_ptr.p;
        P.gi_own_ref = gi_own_ref.p;
        P.iface_own4 = iface_own4.p;
        P.hbuf = hbuf.p;
        P.in = in;
        P.out = out;
        P.max_loc = max_loc;
        P.max_top = max_top;
        P.max_iface = max_iface;
        P.stats = dbg_buf.p;
        return P;
    }
    std::int32_t max_loc = 0, max_top = 0;
    DBuf<long long> dbg_buf;

    // K_i (row-major, written by the setup) -> packed symmetric tiles (iface.cu); the subdomain
    // descriptors' kmat offsets then index the packed array
    void pack_k(const DeviceImage& img) {
        const int nsub = static_cast<int>(img.subs.size());
        std::vector<SubdomainDesc> subs_h = img.subs;
        std::vector<std::int64_t> full_off(nsub), sym_off(nsub);
        std::vector<std::int32_t> ngs(nsub);
        std::int64_t total = 0;
        for (int i = 0; i < nsub; ++i) {
            full_off[i] = subs_h[i].kmat;
            ngs[i] = subs_h[i].n_iface;
            sym_off[i] = total;
            subs_h[i].kmat = total;
            total += sym_k_values(ngs[i]);
        }
        DBuf<std::int64_t> d_full, d_sym;
        DBuf<std::int32_t> d_ng;
        d_full.upload(full_off);
        d_sym.upload(sym_off);
        d_ng.upload(ngs);
        DBuf<double> packed;
        packed.alloc(std::max<std::int64_t>(total, 1));
        launch_pack_sym_k(kmat.p, d_full.p, packed.p, d_sym.p, d_ng.p, nsub, nullptr);
        BDDC_CUDA(cudaDeviceSynchronize());
        std::swap(kmat.p, packed.p);
        std::swap(kmat.n, packed.n);
        kpart.alloc(std::max<std::int64_t>(total / 16, 1) + 1024);  // (+ diagnostics slots)
        if (nsub) BDDC_CUDA(cudaMemcpy(subs.p, subs_h.data(), sizeof(SubdomainDesc) * nsub, cudaMemcpyHostToDevice));
        k_values = total;
    }

    IfaceParams iface_params() const {
        IfaceParams P{};
        P.skip = apply_skip;
        P.subs = subs.p;
        P.n_subdomains = pb().decomposition.n_subdomains;
        P.max_iface = max_iface;
        P.max_primal = max_primal;
        P.iface_dof = iface_dof.p;
        P.iface_w = iface_w.p;
        P.iface_gid = iface_gid.p;
        P.gi_row_ptr = gi_row_ptr.p;
        P.slot_rows = slot_rows.p;
        P.gi_row_col = gi_row_col.p;
        P.gi_row_val = gi_row_val.p;
        P.kmat = kmat.p;
        P.kpacked = kpacked ? 1 : 0;
        P.kcluster = coop_coarse ? 1 : 2;
        P.kpart = kpart.p;
        P.phig = phig.p;
        P.primal = primal.p;
        P.n_coarse = n_coarse;
        P.c_own_ptr = c_own_ptr.p;
        P.c_own_ref = c_own_ref.p;
        P.c_own4 = c_own4.p;
        P.coarse_inv = coarse_inv.p;
        if (coop_coarse) {
            P.rc_g = rc_g.p;
            P.coarse_ctr = coarse_ctr.p;
        }
        P.gbuf = gbuf.p;
        P.hbuf = hbuf.p;
        P.cbuf = cbuf.p;
        P.xc = xc.p;
        return P;
    }

    StageParams stage_params() const {
        StageParams P{};
        P.subs = subs.p;
        P.n_subdomains = pb().decomposition.n_subdomains;
        P.n_vector = pb().decomposition.global_dofs;
        P.max_primal = max_primal;
        P.local_dofs = local_dofs.p;
        P.phi = phi.p;
        P.iface_w = iface_w.p;
        P.iface_dof = iface_dof.p;
        P.gi_dof = gi_dof.p;
        P.n_gi = n_gi;
        P.gi_own_ptr = gi_own_ptr.p;
        P.gi_own_ref = gi_own_ref.p;
        P.dof_own_ptr = dof_own_ptr.p;
        P.dof_own_ref = dof_own_ref.p;
        P.lrow_ptr = lrow_ptr.p;
        P.lrow_col = lrow_col.p;
        P.lrow_val = lrow_val.p;
        P.primal = primal.p;
        P.weights_local = weights_local.p;
        P.lbuf = lbuf.p;
        P.gbuf = gbuf.p;
        P.cbuf = cbuf.p;
        P.xc = xc.p;
        return P;
    }

    void coarse_solve(cudaStream_t s) {
        if (opt.coarse_mode == 0) {
            launch_coarse_direct(iface_params(), s);
        } else {
            CoarseCgParams C{};
            C.n = n_coarse;
            C.ptr = Ac_ptr.p;
            C.col = Ac_col.p;
            C.val = Ac_val.p;
            C.c_own_ptr = c_own_ptr.p;
            C.c_own_ref = c_own_ref.p;
            C.cbuf = cbuf.p;
            C.xc = xc.p;
            C.status = coarse_status.p;
            C.rtol = opt.coarse_rtol;
            C.atol = opt.coarse_atol;
            C.max_it = opt.coarse_max_iterations;
            launch_coarse_cg(C, s);
        }
    }

    // Reference-faithful coarse CG: surface non-convergence like preconditioner.cpp:152-157.
    void check_coarse(cudaStream_t s) {
        if (opt.coarse_mode == 0) return;
        double st[3];
        BDDC_CUDA(cudaMemcpyAsync(st, coarse_status.p, sizeof st, cudaMemcpyDeviceToHost, s));
        BDDC_CUDA(cudaStreamSynchronize(s));
        if (st[0] < 0) throw std::runtime_error("matrix not SPD");
        if (st[2] == 0.0)
            throw std::runtime_error("coarse CG did not converge: " + std::to_string(static_cast<int>(st[0])) +
                                     " iterations, relative residual " + std::to_string(st[1]));
    }

    // Profiling: CUDA events recorded on the launching stream around the two interior
    // solves and the interface steps of every apply, without synchronising; they are
    // resolved lazily (kernel_times()), so profiling does not perturb the timed region.
    std::vector<std::unique_ptr<ApplyEvents>> ev_pool;
    std::size_t ev_used = 0;

    void resolve_events() {
        for (std::size_t i = 0; i < ev_used; ++i) {
            ApplyEvents& E = *ev_pool[i];
            BDDC_CUDA(cudaEventSynchronize(E.e[3].e));
            float a = 0, b = 0, c = 0, t = 0;
            BDDC_CUDA(cudaEventElapsedTime(&a, E.e[0].e, E.e[1].e));
            BDDC_CUDA(cudaEventElapsedTime(&b, E.e[1].e, E.e[2].e));
            BDDC_CUDA(cudaEventElapsedTime(&c, E.e[2].e, E.e[3].e));
            BDDC_CUDA(cudaEventElapsedTime(&t, E.e[0].e, E.e[3].e));
            times.interior_ms += a + c;
            times.interior_launches += 2;
            times.iface_ms += b;
            times.apply_ms += t;
            times.applies += 1;
        }
        ev_used = 0;
    }

    // inside a graph capture an event record must be an explicit (external) node
    void record(cudaEvent_t e, cudaStream_t s) {
        if (capture_events) BDDC_CUDA(cudaEventRecordWithFlags(e, s, cudaEventRecordExternal));
        else BDDC_CUDA(cudaEventRecord(e, s));
    }

    // ------------------------------------------------------------------ GPU setup (f1)
    DBuf<double> lambda_dev;               // Lambda_i of every subdomain (device setup)
    std::vector<std::int64_t> lambda_off;  // per subdomain

    // Numeric setup of every subdomain on the device (device/setup.cuh), class by class, in
    // member batches bounded by a scratch budget: multifrontal factorisation, Schur complement,
    // L_ss^-1 / BL, program fill, saddle inverse -> K_i / Phi_G / Lambda_i / A_ci; then Phi_I
    // (one interior solve per primal column, all subdomains at once). A handful of allocations
    // in total: every class's plan goes up in one blob per element type, the scratch buffers are
    // sized for the largest batch and reused, the jobs of all batches go up at once.
    // every class x program template (stream words + source codes) in two device buffers; run on
    // a host thread of its own while the device image is built (a pageable copy of ~100 MB)
    struct Templates {
        DBuf<double> word;
        DBuf<std::int32_t> code;
        std::vector<std::array<std::int64_t, 3>> off;
        std::exception_ptr error;
    };
    static void upload_templates(const std::vector<SetupClass>& classes, int device, Templates& T) {
        try {
            BDDC_CUDA(cudaSetDevice(device));
            cudaStream_t us = nullptr;
            BDDC_CUDA(cudaStreamCreateWithFlags(&us, cudaStreamNonBlocking));
            const std::size_t ncls = classes.size();
            T.off.assign(ncls, {});
            std::int64_t total = 0;
            for (std::size_t k = 0; k < ncls; ++k)
                for (int q = 0; q < 3; ++q) {
                    T.off[k][q] = total;
                    total += static_cast<std::int64_t>(classes[k].prog[q].stream.size());
                }
            T.word.alloc(std::max<std::int64_t>(total, 1));
            T.code.alloc(std::max<std::int64_t>(total, 1));
            for (std::size_t k = 0; k < ncls; ++k)
                for (int q = 0; q < 3; ++q) {
                    const SolvePools& P = classes[k].prog[q];
                    if (P.stream.empty()) continue;
                    BDDC_CUDA(cudaMemcpyAsync(T.word.p + T.off[k][q], P.stream.data(), sizeof(double) * P.stream.size(),
                                              cudaMemcpyHostToDevice, us));
                    BDDC_CUDA(cudaMemcpyAsync(T.code.p + T.off[k][q], P.srcmap.data(),
                                              sizeof(std::int32_t) * P.srcmap.size(), cudaMemcpyHostToDevice, us));
                }
            BDDC_CUDA(cudaStreamSynchronize(us));
            cudaStreamDestroy(us);
        } catch (...) {
            T.error = std::current_exception();
        }
    }

    void device_setup(const std::vector<SetupClass>& classes, const DeviceImage& img, const Templates& T) {
        const auto t0 = std::chrono::steady_clock::now();
        SetupTimer tm;
        cudaStream_t s = stream;
        const Decomposition& d = pb().decomposition;
        const index_t nsub = d.n_subdomains;
        SolveProgram* pools[3] = {&prog, &harm, &head};
        int nprog = 0;
        while (nprog < 3 && !img.fills[nprog].empty()) ++nprog;
        const std::size_t ncls = classes.size();

        // ---- templates (word + source code per stream word): uploaded by upload_templates
        const auto& toff = T.off;
        const DBuf<double>& tword = T.word;
        const DBuf<std::int32_t>& tcode = T.code;
        tm.mark("    templates upload");
        // ---- every class's plan in three blobs (int32 / int64 / double) with per-class offsets
        std::vector<std::int32_t> bi;
        std::vector<std::int64_t> bl;
        std::vector<double> bd;
        struct Ofs { std::size_t i[18], l[3], d; };
        std::vector<Ofs> of(ncls);
        for (std::size_t k = 0; k < ncls; ++k) {
            const SetupClass& C = classes[k];
            const std::vector<std::int32_t>* iv[18] = {&C.sn_nc, &C.sn_m, &C.sn_mi, &C.level_sn, &C.asc_ptr, &C.asc_pos,
                                                       &C.asc_csr, &C.ch_ptr, &C.ch_id, &C.em_ptr, &C.em_pos, &C.sgg_pos,
                                                       &C.sgg_csr, &C.roots, &C.root_gamma_ptr, &C.root_gamma, &C.c_ptr,
                                                       &C.c_col};
            for (int t = 0; t < 18; ++t) {
                of[k].i[t] = bi.size();
                bi.insert(bi.end(), iv[t]->begin(), iv[t]->end());
            }
            const std::vector<std::int64_t>* lv[3] = {&C.front_off, &C.layout.linv_off, &C.layout.bl_off};
            for (int t = 0; t < 3; ++t) {
                of[k].l[t] = bl.size();
                bl.insert(bl.end(), lv[t]->begin(), lv[t]->end());
            }
            of[k].d = bd.size();
            bd.insert(bd.end(), C.c_val.begin(), C.c_val.end());
        }
        DBuf<std::int32_t> pi;
        DBuf<std::int64_t> pl;
        DBuf<double> pdv;
        pi.upload(bi);
        pl.upload(bl);
        pdv.upload(bd);
        tm.mark("    plan blobs upload");
        // ---- batches: members per batch from a scratch budget. When every class's first batch
        // fits the budget at once, the classes get disjoint scratch and a stream each and run
        // concurrently (their pipelines are independent); otherwise they share the scratch in turn.
        const std::size_t budget = std::size_t(6) << 30;
        struct Batch { std::size_t cls; int m0, nb; };
        std::vector<Batch> batches;
        std::vector<int> bsz(ncls);
        std::vector<std::array<std::size_t, 6>> need(ncls);  // aval, fronts, S, D, M, row/column maps per class
        std::size_t total_bytes = 0;
        for (std::size_t k = 0; k < ncls; ++k) {
            const SetupClass& C = classes[k];
            const std::size_t ns = static_cast<std::size_t>(C.n_iface + C.n_primal);
            const std::size_t per = static_cast<std::size_t>(C.front_total) + C.layout.total +
                                    static_cast<std::size_t>(C.n_iface) * C.n_iface + ns * ns + C.nnz;
            const int nmem = static_cast<int>(C.members.size());
            bsz[k] = std::max(1, std::min<int>(nmem, static_cast<int>(budget / (8 * std::max<std::size_t>(per, 1)))));
            for (int m0 = 0; m0 < nmem; m0 += bsz[k]) batches.push_back({k, m0, std::min(bsz[k], nmem - m0)});
            const std::size_t b = static_cast<std::size_t>(bsz[k]);
            need[k] = {b * C.nnz, b * C.front_total, b * C.n_iface * C.n_iface, b * C.layout.total, b * ns * ns, 2 * b * ns};
            total_bytes += 8 * (need[k][0] + need[k][1] + need[k][2] + need[k][3] + need[k][4]) + 4 * need[k][5];
        }
        const bool concurrent = total_bytes <= budget && ncls > 1;
        std::vector<std::array<std::size_t, 6>> base(ncls, std::array<std::size_t, 6>{});
        std::array<std::size_t, 6> tot{1, 1, 1, 1, 1, 1};
        for (std::size_t k = 0; k < ncls; ++k)
            for (int t = 0; t < 6; ++t) {
                if (concurrent) {
                    base[k][t] = tot[t] - 1;
                    tot[t] += need[k][t];
                } else {
                    tot[t] = std::max(tot[t], need[k][t] + 1);
                }
            }
        std::vector<std::int64_t> aci_off(nsub);
        std::int64_t aci_total = 0;
        for (index_t i = 0; i < nsub; ++i) {
            aci_off[i] = aci_total;
            aci_total += static_cast<std::int64_t>(setup.subs[i].n_primal) * setup.subs[i].n_primal;
        }
        // one scratch block, 256-byte aligned pieces
        std::size_t sbytes = 0;
        auto carve = [&sbytes](std::size_t b) {
            const std::size_t o = sbytes;
            sbytes += (b + 255) & ~std::size_t(255);
            return o;
        };
        const std::size_t n_aci = static_cast<std::size_t>(std::max<std::int64_t>(aci_total, 1));
        const std::size_t o_aval = carve(8 * tot[0]), o_fronts = carve(8 * tot[1]), o_S = carve(8 * tot[2]),
                          o_D = carve(8 * tot[3]), o_M = carve(8 * tot[4]), o_aci = carve(8 * n_aci),
                          o_piv = carve(4 * tot[5]), o_status = carve(16 * batches.size());
        SetupScratch scratch(device, sbytes);
        const Span<double> aval = scratch.span<double>(o_aval, tot[0]), fronts = scratch.span<double>(o_fronts, tot[1]),
                           Sb = scratch.span<double>(o_S, tot[2]), Db = scratch.span<double>(o_D, tot[3]),
                           Mb = scratch.span<double>(o_M, tot[4]), aci_dev = scratch.span<double>(o_aci, n_aci);
        const Span<int> piv = scratch.span<int>(o_piv, tot[5]), status = scratch.span<int>(o_status, 4 * batches.size());
        BDDC_CUDA(cudaMemsetAsync(status.p, 0, sizeof(int) * status.n, s));
        tm.mark("    scratch");
        struct Streams {
            std::vector<cudaStream_t> v;
            ~Streams() {
                for (cudaStream_t q : v) cudaStreamDestroy(q);
            }
        } cs;
        cs.v.resize(concurrent ? ncls : 1);
        for (auto& q : cs.v) BDDC_CUDA(cudaStreamCreateWithFlags(&q, cudaStreamNonBlocking));
        Event ready;  // the class streams start after the work queued on s so far
        BDDC_CUDA(cudaEventRecord(ready.e, s));
        for (cudaStream_t q : cs.v) BDDC_CUDA(cudaStreamWaitEvent(q, ready.e, 0));
        // ---- jobs of every batch: fills and saddle output offsets
        std::vector<std::vector<const DeviceImage::Fill*>> fill_of(nprog, std::vector<const DeviceImage::Fill*>(nsub));
        for (int q = 0; q < nprog; ++q)
            for (const auto& f : img.fills[q]) fill_of[q][f.sub] = &f;
        std::vector<FillJob> jobs;
        std::vector<std::int64_t> outs;
        std::vector<std::size_t> job0(batches.size() * nprog + 1), out0(batches.size());
        for (std::size_t bt = 0; bt < batches.size(); ++bt) {
            const Batch& Bt = batches[bt];
            const SetupClass& C = classes[Bt.cls];
            for (int q = 0; q < nprog; ++q) {
                job0[bt * nprog + q] = jobs.size();
                for (int b = 0; b < Bt.nb; ++b) {
                    const DeviceImage::Fill* f = fill_of[q][C.members[Bt.m0 + b]];
                    jobs.push_back({f->dst, toff[Bt.cls][q], f->words, static_cast<std::int64_t>(b) * C.layout.total});
                }
            }
            out0[bt] = outs.size();
            for (int b = 0; b < Bt.nb; ++b) {
                const index_t i = C.members[Bt.m0 + b];
                outs.insert(outs.end(), {img.subs[i].kmat, img.subs[i].phig, img.subs[i].phi, lambda_off[i], aci_off[i]});
            }
        }
        job0.back() = jobs.size();
        DBuf<FillJob> jobs_dev;
        DBuf<std::int64_t> outs_dev;
        jobs_dev.upload(jobs);
        outs_dev.upload(outs);
        tm.mark("  templates, plans, scratch");

        double acc_t[4] = {};  // diagnostics: factor, schur + linv, fill, saddle
        static const bool lap_on = std::getenv("BDDC_SETUP_TIMES") && std::atoi(std::getenv("BDDC_SETUP_TIMES")) >= 2;
        auto lap = [&](int k, std::chrono::steady_clock::time_point& t) {
            if (!lap_on) return;  // BDDC_SETUP_TIMES=2: per-kernel-kind laps (serialise the classes)
            BDDC_CUDA(cudaDeviceSynchronize());  // (diagnostics: serialises the class streams)
            const auto now = std::chrono::steady_clock::now();
            acc_t[k] += std::chrono::duration<double, std::milli>(now - t).count();
            t = now;
        };
        std::vector<std::vector<double>> avs(ncls);
        for (std::size_t bt = 0; bt < batches.size(); ++bt) {
            const Batch& Bt = batches[bt];
            const SetupClass& C = classes[Bt.cls];
            const Ofs& o = of[Bt.cls];
            cudaStream_t s = cs.v[concurrent ? Bt.cls : 0];  // this class's stream
            const auto& bk = base[Bt.cls];
            std::vector<double>& av = avs[Bt.cls];
            MfPlanDev P{};
            const std::int32_t* ib = pi.p;
            P.sn_nc = ib + o.i[0]; P.sn_m = ib + o.i[1]; P.sn_mi = ib + o.i[2]; P.level_sn = ib + o.i[3];
            P.asc_ptr = ib + o.i[4]; P.asc_pos = ib + o.i[5]; P.asc_csr = ib + o.i[6]; P.ch_ptr = ib + o.i[7];
            P.ch_id = ib + o.i[8]; P.em_ptr = ib + o.i[9]; P.em_pos = ib + o.i[10]; P.sgg_pos = ib + o.i[11];
            P.sgg_csr = ib + o.i[12]; P.roots = ib + o.i[13]; P.root_gamma_ptr = ib + o.i[14];
            P.root_gamma = ib + o.i[15]; P.c_ptr = ib + o.i[16]; P.c_col = ib + o.i[17];
            P.front_off = pl.p + o.l[0]; P.linv_off = pl.p + o.l[1]; P.bl_off = pl.p + o.l[2];
            P.c_val = pdv.p + o.d;
            P.front_total = C.front_total;
            P.d_total = C.layout.total;
            P.nnz = C.nnz;
            P.n_local = C.n_local;
            P.n_interior = C.n_interior;
            P.n_iface = C.n_iface;
            P.n_primal = C.n_primal;
            P.n_roots = static_cast<int>(C.roots.size());
            P.n_sn = static_cast<int>(C.sym.snodes.size());
            P.sgg_n = static_cast<int>(C.sgg_pos.size());
            int max_nc = 1;
            for (int v : C.sn_nc) max_nc = std::max(max_nc, v);
            av.resize(static_cast<std::size_t>(Bt.nb) * C.nnz);
            for (int b = 0; b < Bt.nb; ++b) {
                const CsrMatrix& A = pb().local_matrices[C.members[Bt.m0 + b]];
                std::copy(A.values.begin(), A.values.end(), av.begin() + static_cast<std::ptrdiff_t>(b) * C.nnz);
            }
            // (pageable source: the call returns once av is staged, so the next batch may refill it)
            BDDC_CUDA(cudaMemcpyAsync(aval.p + bk[0], av.data(), sizeof(double) * av.size(), cudaMemcpyHostToDevice, s));
            auto tl = std::chrono::steady_clock::now();
            MfBatch B{};
            B.aval = aval.p + bk[0];
            B.fronts = fronts.p + bk[1];
            B.S = Sb.p + bk[2];
            B.D = Db.p + bk[3];
            B.M = Mb.p + bk[4];
            B.piv = piv.p + bk[5];
            B.status = status.p + 4 * bt;
            B.n = Bt.nb;
            B.first = Bt.m0;
            for (std::size_t h = 0; h + 1 < C.level_ptr.size(); ++h) {
                int fmax = 1;
                for (int q = C.level_ptr[h]; q < C.level_ptr[h + 1]; ++q) {
                    const int sn = C.level_sn[q];
                    fmax = std::max(fmax, C.sn_nc[sn] + C.sn_m[sn]);
                }
                launch_mf_level(P, B, C.level_ptr[h], C.level_ptr[h + 1], fmax, s);
            }
            lap(0, tl);
            launch_schur(P, B, 0, s);
            launch_linv_bl(P, B, max_nc, s);
            lap(1, tl);
            for (int q = 0; q < nprog; ++q)
                launch_fill(pools[q]->stream.p, tword.p, tcode.p, B.D, jobs_dev.p + job0[bt * nprog + q],
                            static_cast<int>(job0[bt * nprog + q + 1] - job0[bt * nprog + q]), s);
            lap(2, tl);
            SaddleOut O{outs_dev.p + out0[bt], kmat.p, phig.p, phi.p, lambda_dev.p, aci_dev.p};
            launch_saddle(P, B, O, s);
            lap(3, tl);
        }
        for (cudaStream_t q : cs.v) {  // join the class streams back into s
            Event done;
            BDDC_CUDA(cudaEventRecord(done.e, q));
            BDDC_CUDA(cudaStreamWaitEvent(s, done.e, 0));
        }
        std::vector<int> st(status.n);
        BDDC_CUDA(cudaMemcpyAsync(st.data(), status.p, sizeof(int) * st.size(), cudaMemcpyDeviceToHost, s));
        BDDC_CUDA(cudaStreamSynchronize(s));
        for (std::size_t bt = 0; bt < batches.size(); ++bt) {
            const SetupClass& C = classes[batches[bt].cls];
            const int* sb = st.data() + 4 * bt;
            if (sb[0]) {
                const index_t i = C.members[sb[0] - 1];
                const int sn = sb[1] / 4096, j = sb[1] % 4096;
                throw std::runtime_error("bddc setup: subdomain " + std::to_string(global_sub(i)) +
                                         ": interior block not positive definite at pivot " +
                                         std::to_string(C.sym.snodes[sn].col_begin + j));
            }
            if (sb[2]) {
                const index_t i = C.members[sb[2] - 1];
                throw std::runtime_error("bddc setup: subdomain " + std::to_string(global_sub(i)) +
                                         ": singular saddle system (zero pivot at step " + std::to_string(sb[3]) + ")");
            }
        }
        if (lap_on)
            std::fprintf(stderr, "[setup]     factor %.1f, schur+linv %.1f, fill %.1f, saddle %.1f ms\n", acc_t[0],
                         acc_t[1], acc_t[2], acc_t[3]);
        tm.mark("  classes (factor, fill, saddle)");
        // Phi_I = -A_II^-1 A_IG Phi_G, column j of every subdomain in one interior solve (MODE 2:
        // rhs 0 - A_IG h with h = Phi_G[:, j] in the hbuf slots)
        BDDC_CUDA(cudaMemsetAsync(vin.p, 0, sizeof(double) * vin.n, s));
        for (int j = 0; j < max_primal; ++j) {
            launch_phi_to_hbuf(subs.p, static_cast<int>(nsub), phig.p, hbuf.p, j, s);
            launch_interior_solve(solve_params(vin.p, vtmp.p), launch, 2, s);
            launch_phi_from_solution(subs.p, static_cast<int>(nsub), local_dofs.p, vtmp.p, phi.p, j, s);
        }
        std::vector<double> aci(std::max<std::int64_t>(aci_total, 1));
        BDDC_CUDA(cudaMemcpyAsync(aci.data(), aci_dev.p, sizeof(double) * aci.size(), cudaMemcpyDeviceToHost, s));
        BDDC_CUDA(cudaStreamSynchronize(s));
        for (index_t i = 0; i < nsub; ++i) {
            const std::int64_t np = setup.subs[i].n_primal;
            setup.subs[i].aci.assign(aci.begin() + aci_off[i], aci.begin() + aci_off[i] + np * np);
        }
        tm.mark("  Phi_I interior solves, A_ci");
        setup_device_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }

    index_t global_sub(index_t local) const { return plan ? plan->subdomains[local] : local; }

    // A_c from every subdomain's A_ci (gathered over the ranks), then its dense inverse (device
    // setup: on the GPU; host setup: setup.cpp) unless the coarse CG is in effect
    void finish_coarse(const DistSpec* dist) {
        const index_t nc = pb().constraints.n_coarse;
        const bool host_inverse = opt.coarse_mode == 0 && !opt.setup_on_device;
        if (plan) {
            // gather the padded per-rank blocks over NCCL, then assemble in ascending global
            // subdomain order exactly like one GPU would
            const RankPlan& P = *plan;
            const index_t nsub = static_cast<index_t>(P.sub_rank.size());
            std::vector<std::int64_t> per_rank(dist->world, 0), off(nsub, 0);
            for (index_t j = 0; j < nsub; ++j) {
                const std::int64_t np = static_cast<std::int64_t>(P.primal_all[j].size());
                off[j] = per_rank[P.sub_rank[j]];
                per_rank[P.sub_rank[j]] += np * np;
            }
            const std::int64_t pad = std::max<std::int64_t>(1, *std::max_element(per_rank.begin(), per_rank.end()));
            std::vector<double> host(static_cast<std::size_t>(pad) * dist->world, 0.0);
            for (std::size_t li = 0; li < P.subdomains.size(); ++li) {
                const index_t j = P.subdomains[li];
                const auto& a = setup.subs[li].aci;
                std::copy(a.begin(), a.end(), host.begin() + dist->rank * pad + off[j]);
            }
            DBuf<double> buf;
            buf.upload(host);
            comm->allgather_inplace(buf.p, static_cast<std::size_t>(pad), nullptr);
            BDDC_CUDA(cudaDeviceSynchronize());
            BDDC_CUDA(cudaMemcpy(host.data(), buf.p, sizeof(double) * host.size(), cudaMemcpyDeviceToHost));
            std::vector<std::vector<double>> aci(nsub);
            std::vector<const std::vector<double>*> blocks(nsub);
            for (index_t j = 0; j < nsub; ++j) {
                const std::int64_t np = static_cast<std::int64_t>(P.primal_all[j].size());
                const auto b0 = host.begin() + P.sub_rank[j] * pad + off[j];
                aci[j].assign(b0, b0 + np * np);
                blocks[j] = &aci[j];
            }
            assemble_coarse(setup, blocks, P.primal_all, nc, host_inverse);
        } else {
            std::vector<const std::vector<double>*> blocks(setup.subs.size());
            for (std::size_t i = 0; i < blocks.size(); ++i) blocks[i] = &setup.subs[i].aci;
            assemble_coarse(setup, blocks, pb().constraints.primal_maps, nc, host_inverse);
        }
        if (opt.coarse_mode == 0) {
            if (opt.setup_on_device) {
                std::vector<double> dense(static_cast<std::size_t>(nc) * nc, 0.0);
                const CsrMatrix& Ac = setup.coarse_matrix;
                for (index_t r = 0; r < nc; ++r)
                    for (index_t q = Ac.row_offsets[r]; q < Ac.row_offsets[r + 1]; ++q)
                        dense[static_cast<std::size_t>(r) * nc + Ac.col_indices[q]] = Ac.values[q];
                coarse_inv.upload(dense);
                DBuf<double> scr;
                scr.alloc(2 * static_cast<std::size_t>(std::max<index_t>(nc, 1)));
                DBuf<int> st;
                st.alloc(1);
                dense_spd_inverse(coarse_inv.p, nc, scr.p, st.p, stream);
                int bad = 0;
                BDDC_CUDA(cudaMemcpyAsync(&bad, st.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
                BDDC_CUDA(cudaStreamSynchronize(stream));
                // A_c not SPD: no dense inverse; the coarse CG then fails inside the apply
                // exactly like the reference's (preconditioner.cpp:141-157 -> "matrix not SPD")
                if (bad) opt.coarse_mode = 1;
            } else if (setup.coarse_inverse.empty()) {
                opt.coarse_mode = 1;
            } else {
                coarse_inv.upload(setup.coarse_inverse);
            }
        }
        if (opt.coarse_mode != 0) coarse_inv.alloc(1);
        Ac_ptr.upload(setup.coarse_matrix.row_offsets);
        Ac_col.upload(setup.coarse_matrix.col_indices);
        Ac_val.upload(setup.coarse_matrix.values);
    }

    void apply(const double* r_dev, double* z_dev, cudaStream_t s) {
        ApplyEvents* E = capture_events;  // graph capture: fixed events, rebound per launch
        if (opt.profile && !E && !suppress_profile) {
            if (ev_used == 4096) resolve_events();
            if (ev_used == ev_pool.size()) ev_pool.emplace_back(new ApplyEvents);
            E = ev_pool[ev_used++].get();
        }
        const bool fused = fused_apply();
        if (E) record(E->e[0].e, s);
        const bool spl = split();
        SolveParams sp = solve_params(r_dev, U.p, spl ? &head : nullptr);
        if (spl) sp.y_out = ybuf.p;  // u0 only where A_GI reads it (pruned backward sweep)
        if (fused) sp.pub = ll_publish(kExU, 0, U.p);
        launch_interior_solve(sp, launch, 0, s);
        if (E) record(E->e[1].e, s);
        IfaceParams ip = iface_params();
        if (fused) {
            ip.ll_u = ll_buf.p + ll_off[0];
            ip.seq_u = ex_seq.p + kExU;
            ip.ll_u_base = static_cast<int>(n_rows);
            ip.pub_c = ll_publish(kExC, 1, cbuf.p);
            ip.ll_c = ll_buf.p + ll_off[3];
            ip.seq_c = ex_seq.p + kExC;
            ip.c_own_lo = comm->rank() * plan->cbuf_pad;
            ip.c_own_hi = ip.c_own_lo + plan->cbuf_pad;
            ip.pub_h = ll_publish(kExH, 2, hbuf.p);
        } else {
            halo_exchange(U.p, s);
        }
        launch_iface_restrict(ip, r_dev, U.p, s);
        if (!fused) gather_cbuf(s);
        if (opt.coarse_mode == 0) {
            launch_iface_local(ip, opt.local_blocks, s, 2);  // coarse GEMV rows fused in
        } else {
            coarse_solve(s);
            launch_iface_local(ip, opt.local_blocks, s, 1);
        }
        if (!fused) iface_exchange(s);
        if (E) record(E->e[2].e, s);
        if (harm.valid) {  // z_I = u0 - A_II^-1 A_IG z_G
            SolveParams hp = solve_params(r_dev, z_dev, &harm);
            if (spl) hp.y_in = ybuf.p;  // z_I = L^-T (y0 - L^-1 A_IG z_G)
            if (apply_dot_r) {
                hp.dot_r = apply_dot_r;
                hp.dot_part = part_rz.p;
                hp.n_dot = apply_dot_n;
            }
            if (fused) {
                hp.ll_h = ll_buf.p + ll_off[2];
                hp.seq_h = ex_seq.p + kExH;
                hp.ll_h_base = static_cast<int>(plan->n_local_slots);
                if (pub_rz) {  // z's halo + this rank's r.z, as gather_rz_with_z_halo
                    hp.pub = ll_publish(kExZ, 3, z_dev);
                    ll_scalar(hp.pub, 2, part_rz.p, launch.n_parts, gath_c.p);
                }
            }
            launch_interior_solve(hp, launch, 3, s);
        }
        else launch_interior_solve(solve_params(r_dev, z_dev), launch, 1, s);
        if (E) record(E->e[3].e, s);
    }

    void ensure_pcg(int max_it) {
        const index_t n = pb().decomposition.global_dofs;
        if (!x.p) {
            for (DBuf<double>* b : {&x, &r, &z, &p, &q, &p_alt}) b->alloc(n);
            const int g = pcg_grid_for(dist() ? n_rows : n);
            part_a.alloc(g);
            part_b.alloc(g);
            for (DBuf<double>* gb : {&gath_a, &gath_b, &gath_c, &gath_d}) {
                gb->alloc(dist() ? comm->world() : 1);
                BDDC_CUDA(cudaMemset(gb->p, 0, sizeof(double) * gb->n));
            }
            scal.alloc(8);
            iter_ctr.alloc(1);
            BDDC_CUDA(cudaMallocHost(&pinned, sizeof(double) * 8));
            BDDC_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&pinned_dev), pinned, 0));
            solo_seq.alloc(2);
            BDDC_CUDA(cudaMemset(solo_seq.p, 0, sizeof(std::uint64_t) * 2));
            solo_ticket.alloc(2);
            BDDC_CUDA(cudaMemset(solo_ticket.p, 0, sizeof(unsigned int) * 2));
        }
        if (max_it > max_it_alloc) {
            rho.alloc(max_it + 1);
            alpha.alloc(max_it);
            beta.alloc(max_it);
            hist.alloc(max_it + 1);
            max_it_alloc = max_it;
        }
    }

    PcgDevice pcg_device(const SolverOpts& o, double* xd, double* rd, double* zd) const {
        PcgDevice D{};
        D.n = dist() ? n_rows : pb().decomposition.global_dofs;
        D.n_dot = dist() ? n_owned : D.n;
        D.n_dir = D.n;  // pcg() widens it to the halo when z's halo arrives with r.z
        D.grid = pcg_grid_for(D.n);
        D.A_ptr = A_ptr.p;
        D.A_col = A_col.p;
        D.A_val = A_val.p;
        D.ell_off = ell_off.p;
        D.ell_len = ell_len.p;
        D.ell_col = ell_col.p;
        D.ell_d16 = ell_d16.p;
        D.ell_val = ell_val.p;
        D.x = xd;
        D.r = rd;
        D.z = zd;
        D.p = p.p;
        D.q = q.p;
        D.part_a = part_a.p;
        D.part_b = part_b.p;
        D.red_a = dist() ? gath_a.p : part_a.p;
        D.red_a_n = dist() ? comm->world() : D.grid;
        D.red_b = dist() ? gath_b.p : part_b.p;
        D.red_b_n = dist() ? comm->world() : D.grid;
        D.red_c = dist() ? gath_c.p : part_a.p;
        D.red_c_n = dist() ? comm->world() : D.grid;
        D.rho = rho.p;
        D.alpha = alpha.p;
        D.beta = beta.p;
        D.hist = hist.p;
        D.scal = scal.p;
        D.iter = iter_ctr.p;
        D.rtol = o.rel_tolerance;
        D.atol = o.abs_tolerance;
        return D;
    }

    // Peer-memory exchange descriptors (see device/comm.cuh). Buffers exported, in order:
    // U, p, hbuf, cbuf, gath_a, gath_b, gath_c, gath_d, flags, z.
    void setup_peer_links(const DeviceImage& img) {
        const RankPlan& P = *plan;
        const int me = comm->rank(), world = comm->world();
        ex_flags.alloc(static_cast<std::size_t>(kFlagTypes) * kMaxPeers);
        BDDC_CUDA(cudaMemset(ex_flags.p, 0, sizeof(std::uint64_t) * ex_flags.n));
        ex_seq.alloc(kFlagTypes);
        BDDC_CUDA(cudaMemset(ex_seq.p, 0, sizeof(std::uint64_t) * ex_seq.n));
        // where each peer receives this rank's halo / interface values: rank r publishes
        // (n_rows + halo_recv_off, n_local_slots + iface_recv_off) for every source q
        // (+ the same offsets relative to the receive regions, and the LL region offsets)
        constexpr int kCols = 4, kLLRegions = 5;
        const std::int64_t n_halo = static_cast<std::int64_t>(U.n) - n_rows;
        const std::int64_t n_hrecv = img.hbuf_total - P.n_local_slots;
        ll_off[0] = 0;
        ll_off[1] = 2 * n_halo;
        ll_off[2] = 4 * n_halo;
        ll_off[3] = ll_off[2] + 2 * n_hrecv;
        ll_off[4] = ll_off[3] + 2 * static_cast<std::int64_t>(world) * P.cbuf_pad;
        ll_buf.alloc(ll_off[4] + 2 * 3 * static_cast<std::int64_t>(world));
        BDDC_CUDA(cudaMemset(ll_buf.p, 0, sizeof(ll_word) * ll_buf.n));
        const std::size_t row = static_cast<std::size_t>(world) * kCols + kLLRegions;
        std::vector<double> tbl(row * world, -1.0);
        for (std::size_t k = 0; k < P.halo_peers.size(); ++k) {
            tbl[me * row + P.halo_peers[k] * kCols] = P.n_rows + P.halo_recv_off[k];
            tbl[me * row + P.halo_peers[k] * kCols + 2] = P.halo_recv_off[k];
        }
        for (std::size_t k = 0; k < P.iface_peers.size(); ++k) {
            tbl[me * row + P.iface_peers[k] * kCols + 1] = P.n_local_slots + P.iface_recv_off[k];
            tbl[me * row + P.iface_peers[k] * kCols + 3] = P.iface_recv_off[k];
        }
        for (int r = 0; r < kLLRegions; ++r) tbl[me * row + world * kCols + r] = static_cast<double>(ll_off[r]);
        {
            DBuf<double> d;
            d.upload(tbl);
            comm->allgather_inplace(d.p, row, nullptr);
            BDDC_CUDA(cudaDeviceSynchronize());
            BDDC_CUDA(cudaMemcpy(tbl.data(), d.p, sizeof(double) * tbl.size(), cudaMemcpyDeviceToHost));
        }
        links = std::make_unique<PeerLinks>(*comm, std::vector<void*>{U.p, p.p, hbuf.p, cbuf.p, gath_a.p, gath_b.p,
                                                                      gath_c.p, gath_d.p, ex_flags.p, z.p, ll_buf.p});
        std::vector<ExchangeDesc> desc(kFlagTypes);
        auto flag_of = [&](int q, int type) {
            return static_cast<std::uint64_t*>(links->peer(q, 8)) + type * kMaxPeers + me;
        };
        auto neighbour = [&](ExchangeDesc& D, int type, int buffer, const std::vector<int>& peers,
                             const std::vector<index_t>& soff, const std::int32_t* idx, int col) {
            D.idx = idx;
            for (std::size_t k = 0; k < peers.size(); ++k) {
                const int q = peers[k];
                const double at = tbl[q * row + me * kCols + col];
                if (at < 0) throw std::logic_error("rank plan: peer does not expect this rank's values");
                PeerPut& pp = D.put[D.n_put++];
                pp.dst = static_cast<double*>(links->peer(q, buffer)) + static_cast<std::int64_t>(at);
                pp.flag = flag_of(q, type);
                pp.off = soff[k];
                pp.cnt = soff[k + 1] - soff[k];
                D.wait[D.n_wait++] = ex_flags.p + type * kMaxPeers + q;
            }
        };
        neighbour(desc[kExU], kExU, 0, P.halo_peers, P.halo_send_off, halo_idx.p, 0);
        neighbour(desc[kExP], kExP, 1, P.halo_peers, P.halo_send_off, halo_idx.p, 0);
        neighbour(desc[kExH], kExH, 2, P.iface_peers, P.iface_send_off, iface_idx.p, 1);
        neighbour(desc[kExZ], kExZ, 9, P.halo_peers, P.halo_send_off, halo_idx.p, 0);
        auto all_to_all = [&](ExchangeDesc& D, int type, int buffer, std::int32_t off, std::int32_t cnt) {
            for (int q = 0; q < world; ++q) {
                if (q == me) continue;
                PeerPut& pp = D.put[D.n_put++];
                pp.dst = static_cast<double*>(links->peer(q, buffer)) + off;
                pp.flag = flag_of(q, type);
                pp.off = off;
                pp.cnt = cnt;
                D.wait[D.n_wait++] = ex_flags.p + type * kMaxPeers + q;
            }
        };
        all_to_all(desc[kExC], kExC, 3, me * P.cbuf_pad, P.cbuf_pad);
        all_to_all(desc[kExPQ], kExPQ, 4, me, 1);
        all_to_all(desc[kExRR], kExRR, 5, me, 1);
        all_to_all(desc[kExRZ], kExRZ, 6, me, 1);
        all_to_all(desc[kExNB], kExNB, 7, me, 1);
        for (int t = 0; t < kFlagTypes; ++t) desc[t].seq = ex_seq.p + t;
        if (std::getenv("BDDC_EXCH_STATS")) {  // diagnostics: per-type {count, total ns, wait ns}
            ex_stats.alloc(8 * kFlagTypes);
            BDDC_CUDA(cudaMemset(ex_stats.p, 0, sizeof(unsigned long long) * ex_stats.n));
            for (int t = 0; t < kFlagTypes; ++t) desc[t].stats = ex_stats.p + 8 * t;
        }
        // flatten every descriptor's puts over its peers (one parallel loop in the kernel)
        std::vector<double*> dst_all;
        std::vector<std::int32_t> src_all;
        std::vector<std::size_t> first(desc.size() + 1, 0);
        for (std::size_t t = 0; t < desc.size(); ++t) {
            const ExchangeDesc& D = desc[t];
            const std::vector<index_t>* ids = D.idx == halo_idx.p ? &P.halo_send_idx
                                              : D.idx == iface_idx.p ? &P.iface_send_slot : nullptr;
            for (int k = 0; k < D.n_put; ++k)
                for (int i = 0; i < D.put[k].cnt; ++i) {
                    dst_all.push_back(D.put[k].dst + i);
                    src_all.push_back(ids ? (*ids)[D.put[k].off + i] : D.put[k].off + i);
                }
            first[t + 1] = dst_all.size();
        }
        // fused LL exchanges: every sent value's destination word pair in the peer's LL buffer,
        // bucketed by the CTA of the producing kernel that writes its source value
        {
            auto peer_ll = [&](int q, int region, std::int64_t word) {
                return static_cast<ll_word*>(links->peer(q, 10)) +
                       static_cast<std::int64_t>(tbl[q * row + world * kCols + region]) + word;
            };
            std::vector<std::int32_t> all_src, all_cta;
            std::vector<ll_word*> all_dst;
            auto add_type = [&](int t, const std::vector<std::int32_t>& src, const std::vector<ll_word*>& dst,
                                const std::vector<std::int32_t>& writer, int grid, bool need_writer) {
                std::vector<std::int32_t> cta(src.size());
                for (std::size_t i = 0; i < src.size(); ++i) {
                    std::int32_t w = src[i] >= 0 && src[i] < static_cast<std::int32_t>(writer.size()) ? writer[src[i]] : -1;
                    if (w < 0) {
                        if (need_writer) throw std::logic_error("fused exchange: a sent value has no producing CTA");
                        w = 0;  // never written (constant): any CTA may send it
                    }
                    cta[i] = w;
                }
                std::vector<std::size_t> ord(src.size());
                for (std::size_t i = 0; i < ord.size(); ++i) ord[i] = i;
                std::stable_sort(ord.begin(), ord.end(), [&](std::size_t x, std::size_t y) { return cta[x] < cta[y]; });
                const std::int32_t base = static_cast<std::int32_t>(all_src.size());
                std::vector<std::int32_t> ptr(grid + 1, 0);
                for (std::size_t i : ord) {
                    all_src.push_back(src[i]);
                    all_dst.push_back(dst[i]);
                    ++ptr[cta[i] + 1];
                }
                ptr[0] = base;
                for (int b = 0; b < grid; ++b) ptr[b + 1] += ptr[b];
                ll_cta_off[t] = static_cast<std::int64_t>(all_cta.size());
                all_cta.insert(all_cta.end(), ptr.begin(), ptr.end());
                ll_has[t] = true;
            };
            auto neighbour_items = [&](int region, const std::vector<int>& peers, const std::vector<index_t>& soff,
                                       const std::vector<index_t>& ids, int col, std::vector<std::int32_t>& src,
                                       std::vector<ll_word*>& dst) {
                for (std::size_t k = 0; k < peers.size(); ++k) {
                    const int q = peers[k];
                    const double rel = tbl[q * row + me * kCols + col];
                    if (rel < 0) throw std::logic_error("rank plan: peer does not expect this rank's values");
                    for (index_t i = soff[k]; i < soff[k + 1]; ++i) {
                        src.push_back(static_cast<std::int32_t>(ids[i]));
                        dst.push_back(peer_ll(q, region, 2 * (static_cast<std::int64_t>(rel) + i - soff[k])));
                    }
                }
            };
            // writers: solve0 CTAs (u0), harmonic-solve CTAs (z, incl. the interface values
            // written by the lowest owner's first CTA), restrict CTAs (c_i), K_i CTAs (h_i)
            const std::size_t nvec = U.n;
            std::vector<std::int32_t> wu(nvec, -1), wz(nvec, -1);
            for (std::size_t q = 0; q < img.solve.parts.size(); ++q) {
                const PartDesc& pd = img.solve.parts[q];
                for (int l = 0; l < pd.n_write; ++l) wu[img.solve.gmap[pd.gmap + l]] = static_cast<std::int32_t>(q);
            }
            for (std::size_t q = 0; q < img.harm.parts.size(); ++q) {
                const PartDesc& pd = img.harm.parts[q];
                for (int l = 0; l < pd.n_write; ++l) wz[img.harm.gmap[pd.gmap + l]] = static_cast<std::int32_t>(q);
                if (pd.rank != 0) continue;
                const SubdomainDesc& sd = img.subs[pd.sub];
                for (int g = 0; g < sd.n_iface; ++g)
                    if (img.iface_writer[sd.iface + g]) wz[img.iface_dof[sd.iface + g]] = static_cast<std::int32_t>(q);
            }
            std::vector<std::int32_t> wc(std::max<std::int64_t>(img.cbuf_total, 1), -1);
            std::vector<std::int32_t> wh(std::max<std::int64_t>(img.hbuf_total, 1), -1);
            // CTAs per subdomain of the K_i kernel and the h rows each produces
            const int bps = kpacked ? iface_params().kcluster : opt.local_blocks;
            for (std::size_t b = 0; b < img.subs.size(); ++b) {
                const SubdomainDesc& sd = img.subs[b];
                for (int j = 0; j < sd.n_primal; ++j) wc[sd.cbuf + j] = static_cast<std::int32_t>(b);
                const int rows_per = (sd.n_iface + bps - 1) / bps;
                for (int g = 0; g < sd.n_iface; ++g) {
                    int c = g / rows_per;
                    if (kpacked) {
                        c = 0;
                        while (c + 1 < bps && g >= sym_rows_begin(sd.n_iface, bps, c + 1)) ++c;
                    }
                    wh[sd.hbuf + g] = static_cast<std::int32_t>(b * bps + c);
                }
            }
            const int nsub = static_cast<int>(img.subs.size());
            {
                std::vector<std::int32_t> src;
                std::vector<ll_word*> dst;
                neighbour_items(0, P.halo_peers, P.halo_send_off, P.halo_send_idx, 2, src, dst);
                add_type(kExU, src, dst, wu, static_cast<int>(img.solve.parts.size()), false);
            }
            if (!img.harm.parts.empty()) {
                std::vector<std::int32_t> src;
                std::vector<ll_word*> dst;
                neighbour_items(1, P.halo_peers, P.halo_send_off, P.halo_send_idx, 2, src, dst);
                add_type(kExZ, src, dst, wz, static_cast<int>(img.harm.parts.size()), true);
            }
            {
                std::vector<std::int32_t> src;
                std::vector<ll_word*> dst;
                neighbour_items(2, P.iface_peers, P.iface_send_off, P.iface_send_slot, 3, src, dst);
                add_type(kExH, src, dst, wh, nsub * bps, true);
            }
            {
                std::vector<std::int32_t> src;
                std::vector<ll_word*> dst;
                for (int q = 0; q < world; ++q) {
                    if (q == me) continue;
                    for (std::int32_t i = 0; i < P.cbuf_pad; ++i) {
                        src.push_back(me * P.cbuf_pad + i);
                        dst.push_back(peer_ll(q, 3, 2 * (static_cast<std::int64_t>(me) * P.cbuf_pad + i)));
                    }
                }
                add_type(kExC, src, dst, wc, nsub, false);
            }
            std::vector<ll_word*> sc;
            for (int r = 0; r < 3; ++r)
                for (int q = 0; q < world; ++q)
                    if (q != me) sc.push_back(peer_ll(q, 4, 2 * (static_cast<std::int64_t>(r) * world + me)));
            ll_src.upload(all_src);
            ll_cta.upload(all_cta);
            ll_dst.alloc(std::max<std::size_t>(all_dst.size(), 1));
            if (!all_dst.empty())
                BDDC_CUDA(cudaMemcpy(ll_dst.p, all_dst.data(), sizeof(ll_word*) * all_dst.size(), cudaMemcpyHostToDevice));
            ll_sc_dst.alloc(std::max<std::size_t>(sc.size(), 1));
            if (!sc.empty())
                BDDC_CUDA(cudaMemcpy(ll_sc_dst.p, sc.data(), sizeof(ll_word*) * sc.size(), cudaMemcpyHostToDevice));
        }
        ex_item_dst.alloc(std::max<std::size_t>(dst_all.size(), 1));
        if (!dst_all.empty())
            BDDC_CUDA(cudaMemcpy(ex_item_dst.p, dst_all.data(), sizeof(double*) * dst_all.size(), cudaMemcpyHostToDevice));
        ex_item_src.upload(src_all);
        for (std::size_t t = 0; t < desc.size(); ++t) {
            desc[t].n_items = static_cast<std::int32_t>(first[t + 1] - first[t]);
            desc[t].item_dst = ex_item_dst.p + first[t];
            desc[t].item_src = ex_item_src.p + first[t];
        }
        ex_host = desc;
        if (std::getenv("BDDC_FUSED_TRACE")) {
            fused_trace.alloc(1 + 2 * (std::size_t(1) << 20));
            BDDC_CUDA(cudaMemset(fused_trace.p, 0, sizeof(unsigned long long) * fused_trace.n));
        }
        ex_ticket.alloc(kFlagTypes);
        BDDC_CUDA(cudaMemset(ex_ticket.p, 0, sizeof(unsigned int) * ex_ticket.n));
        BDDC_CUDA(cudaDeviceSynchronize());
    }

    // smallest global index of a non-finite entry of v over the owned rows of every rank (a
    // collective in the distributed case), 1e300 if there is none
    double first_nonfinite_global(const double* v, cudaStream_t s) {
        DBuf<int> bad;
        bad.alloc(1);
        device_first_nonfinite(dist() ? static_cast<int>(n_owned) : static_cast<int>(pb().decomposition.global_dofs), v,
                               bad.p, s);
        int idx = 0;
        BDDC_CUDA(cudaMemcpyAsync(&idx, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        BDDC_CUDA(cudaStreamSynchronize(s));
        double first = idx != 0x7fffffff ? static_cast<double>(global_index(idx)) : 1e300;
        if (dist()) {  // each rank owns its rows
            DBuf<double> all;
            all.alloc(comm->world());
            BDDC_CUDA(cudaMemcpy(all.p + comm->rank(), &first, sizeof(double), cudaMemcpyHostToDevice));
            comm->allgather_inplace(all.p, 1, s);
            std::vector<double> h(comm->world());
            BDDC_CUDA(cudaMemcpyAsync(h.data(), all.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s));
            BDDC_CUDA(cudaStreamSynchronize(s));
            first = *std::min_element(h.begin(), h.end());
        }
        return first;
    }
    index_t global_index(int local) const {
        return dist() && local >= 0 && local < static_cast<int>(plan->local_to_global.size()) ? plan->local_to_global[local]
                                                                                               : local;
    }

    // pcg.cpp:40-109 with every vector on the device; b and x are device pointers.
    SolveResult pcg(const double* b, const SolverOpts& o, double* xout, bool precondition, cudaStream_t s) {
        if (!(o.rel_tolerance > 0.0) || o.abs_tolerance < 0.0)
            throw std::invalid_argument("pcg: tolerances must be positive");
        if (o.max_iterations < 1) throw std::invalid_argument("pcg: max_iterations must be at least 1");
        if (dist()) {
            if (!symmetry_error.empty()) throw std::invalid_argument(symmetry_error);
        } else {
            sampled_symmetry_check(pb().global_matrix);
        }
        const index_t n = pb().decomposition.global_dofs;
        ensure_pcg(o.max_iterations);
        SolveResult rep;
        double* xd = xout;
        double* rd = r.p;
        double* zd = precondition ? z.p : r.p;
        PcgDevice D = pcg_device(o, xd, rd, zd);
        const bool fused_dir = dist() && p2p() && precondition;  // z halo arrives with r.z
        if (fused_dir) D.n_dir = static_cast<int>(n);
        // r.z formed inside the harmonic-extension launch (per-CTA partials) instead of a dot pass
        const bool fused_dot = precondition && harm.valid;
        if (fused_dot) {
            if (part_rz.n < static_cast<std::size_t>(launch.n_parts)) part_rz.alloc(launch.n_parts);
            if (!dist()) {
                D.red_c = part_rz.p;
                D.red_c_n = launch.n_parts;
            }
        }
        auto apply_rz = [&]() {  // apply + the r.z partials for the following reduction
            if (fused_dot) {
                apply_dot_r = rd;
                apply_dot_n = D.n_dot;
            }
            apply(rd, zd, s);
            apply_dot_r = nullptr;
        };
        // exchanges riding on the producing / consuming kernels (device/fused_comm.cuh)
        const bool fpcg = fused_pcg();
        const bool frz = fused_dir && fused_dot && fused_apply() && (fused_ex & 4);
        if (fpcg || frz) {
            D.ll_sc = ll_buf.p + ll_off[4];
            D.me = comm->rank();
        }
        if (fpcg) {
            D.pub_pq = ll_publish(kExPQ, 5, nullptr);
            ll_scalar(D.pub_pq, 0, part_a.p, D.grid, gath_a.p);
            D.seq_pq = ex_seq.p + kExPQ;
            D.pub_rr = ll_publish(kExRR, 6, nullptr);
            ll_scalar(D.pub_rr, 1, part_b.p, D.grid, gath_b.p);
            D.seq_rr = ex_seq.p + kExRR;
        }
        if (frz) {
            D.seq_rz = ex_seq.p + kExZ;  // r.z travels with z's halo, under its tag
            D.ll_z = ll_buf.p + ll_off[1];
        }
        // convergence check in update's last CTA, flags straight to pinned host memory
        const bool fcheck = !dist() || fpcg;
        if (fcheck) {
            D.fuse_check = 1;
            D.host_scal = pinned_dev;
            if (!dist()) {  // grid ticket + the r.r reduction only (no peers)
                D.pub_rr.seq = solo_seq.p;
                D.pub_rr.ticket = solo_ticket.p;
                D.pub_rr.part = part_b.p;
                D.pub_rr.red = gath_b.p;
                D.pub_rr.grid = D.grid;
                D.pub_rr.slot = 0;
            }
        }
        // p = z + beta p fused into the next iteration's SpMV (no xpay pass, no init_rho)
        const bool dirspmv = use_dir_spmv && precondition && fused_dot && (!dist() || frz);
        if (step_ok < 0) step_ok = pcg_step_fits(D.grid) ? 1 : 0;
        const bool stepfuse = use_step && step_ok == 1 && !dist() && precondition && fused_dot && fcheck && !dirspmv;
        if (stepfuse && !step_bar.p) {
            step_bar.alloc(1);
            BDDC_CUDA(cudaMemset(step_bar.p, 0, sizeof(unsigned long long)));
        }
        if (dirspmv) {
            D.fuse_dir = 1;
            D.p_alt = p_alt.p;
            if (!D.pub_pq.seq) {  // grid ticket only: the last CTA advances the iteration counter
                D.pub_pq.seq = solo_seq.p + 1;
                D.pub_pq.ticket = solo_ticket.p + 1;
            }
        }
        pub_rz = frz;
        struct ResetPub {
            bool& f;
            ~ResetPub() { f = false; }
        } reset_pub{pub_rz};
        const double* rz_part = fused_dot ? part_rz.p : part_a.p;
        const int rz_grid = fused_dot ? launch.n_parts : D.grid;
        BDDC_CUDA(cudaMemsetAsync(xd, 0, sizeof(double) * n, s));
        BDDC_CUDA(cudaMemsetAsync(scal.p, 0, sizeof(double) * 8, s));
        BDDC_CUDA(cudaMemsetAsync(iter_ctr.p, 0, sizeof(int), s));
        BDDC_CUDA(cudaMemcpyAsync(rd, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
        pcg_dot(D, b, b, part_b.p, s);
        if (dist()) {
            gather_partial(part_b.p, D.grid, gath_d.p, s);
            launch_reduce_to(gath_d.p, comm->world(), scal.p, true, s);
        } else {
            pcg_finalize(D, part_b.p, 0, true, s);
        }
        BDDC_CUDA(cudaMemcpyAsync(pinned, scal.p, sizeof(double) * 4, cudaMemcpyDeviceToHost, s));
        // z_0 = M r_0 and rho_0 are queued before the host looks at ||b|| (pipelined mode): the
        // checks below can only discard them (a zero rhs converges at once, a non-finite one
        // throws on every rank alike), so the device never waits for that round trip
        auto first_direction = [&]() {
            if (precondition) {
                // graphed loop + profiling: only the sampled graph iterations are timed (steady
                // state); the eager pre-loop apply is not
                const bool graph_loop = use_graphs && (opt.coarse_mode == 0) && (!dist() || p2p());
                suppress_profile = graph_loop && opt.profile;
                try {
                    apply_rz();
                } catch (...) {
                    suppress_profile = false;
                    throw;
                }
                suppress_profile = false;
                check_coarse(s);
            }
            if (!fused_dot) pcg_dot(D, rd, zd, part_a.p, s);
            if (dirspmv || stepfuse) {
                // rho[0] and p_1 = z are formed by the first dir_spmv / pcg_step
            } else if (fused_dir) {
                if (!frz) gather_rz_with_z_halo(rz_part, rz_grid, s);
                pcg_init_rho(D, s);
            } else {
                gather_partial(rz_part, rz_grid, gath_c.p, s);
                pcg_init_rho(D, s);
                halo_exchange(p.p, s);
            }
        };
        const bool early = precondition && opt.coarse_mode == 0;
        if (early) {
            BDDC_CUDA(cudaEventRecord(norm_ev.e, s));
            first_direction();
            BDDC_CUDA(cudaEventSynchronize(norm_ev.e));
        } else {
            BDDC_CUDA(cudaStreamSynchronize(s));
        }
        const double normb = pinned[0];
        if (!std::isfinite(normb)) {  // every rank sees the same ||b||: the decision is collective
            const double first = first_nonfinite_global(b, s);
            if (first < 1e300)  // else: finite entries whose squares overflow (the reference carries on)
                throw std::invalid_argument("pcg rhs: non-finite entry at index " +
                                            std::to_string(static_cast<long long>(first)));
        }
        if (o.record_history) rep.history.push_back(1.0);
        if (normb == 0.0) {
            rep.converged = true;
            return rep;
        }
        if (!early) first_direction();
        auto finish = [&](double rel) -> SolveResult {
            rep.final_relative_residual = rel;
            const int k = rep.iterations;
            std::vector<double> al(k), be(std::max(0, k - 1));
            if (k) BDDC_CUDA(cudaMemcpyAsync(al.data(), alpha.p, sizeof(double) * k, cudaMemcpyDeviceToHost, s));
            if (k > 1) BDDC_CUDA(cudaMemcpyAsync(be.data(), beta.p, sizeof(double) * (k - 1), cudaMemcpyDeviceToHost, s));
            if (o.record_history && k) {
                rep.history.resize(k + 1);
                BDDC_CUDA(cudaMemcpyAsync(rep.history.data() + 1, hist.p + 1, sizeof(double) * k, cudaMemcpyDeviceToHost, s));
            }
            BDDC_CUDA(cudaStreamSynchronize(s));
            rep.condition_estimate = condition_estimate(al, be);
            return rep;
        };
        double rel = 1.0;
        if (!precondition && !dist() && use_plain_loop) {
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            BDDC_CUDA(cudaStreamIsCapturing(s, &cs));
            if (plain_loop_ok < 0) plain_loop_ok = pcg_plain_loop_fits(D.grid) ? 1 : 0;
            if (cs == cudaStreamCaptureStatusNone && plain_loop_ok == 1) {
                if (!plain_bar.p) plain_bar.alloc(1);
                D.p_alt = p_alt.p;  // p_k alternates between p and p_alt
                pcg_plain_loop(D, o.max_iterations, plain_bar.p, s);
                BDDC_CUDA(cudaMemcpyAsync(pinned, scal.p, sizeof(double) * 5, cudaMemcpyDeviceToHost, s));
                BDDC_CUDA(cudaStreamSynchronize(s));
                if (pinned[3] == 1.0) throw std::runtime_error("matrix not SPD");
                rel = pinned[1];
                rep.iterations = static_cast<int>(pinned[4]);
                rep.converged = pinned[2] != 0.0;
                return finish(rel);
            }
        }
        // The convergence test of iteration `it` is read back while the GPU already runs the
        // next iteration's apply / dot / xpay (speculatively: they only touch z, p, rho, beta,
        // which are unused once the loop stops), so the host round trip leaves no bubble.
        // The reference-faithful coarse CG (check_coarse reads its status after every apply)
        // keeps the synchronous order.
        const bool pipelined = opt.coarse_mode == 0 || !precondition;
        // graphs: pipelined loop, peer-memory (or no) exchanges, not under an outer capture
        cudaStreamCaptureStatus cap_status = cudaStreamCaptureStatusNone;
        BDDC_CUDA(cudaStreamIsCapturing(s, &cap_status));
        const bool graphed = use_graphs && pipelined && (!dist() || p2p()) && cap_status == cudaStreamCaptureStatusNone;
        auto next_direction = [&](int it) {
            apply_skip = scal.p;  // no-op once iteration `it` has converged or failed
            if (precondition) apply_rz();
            apply_skip = nullptr;
            if (!fused_dot) pcg_dot(D, rd, zd, part_a.p, s);
            if (dirspmv || stepfuse) {
                // p = z + beta p happens inside the next dir_spmv / pcg_step
            } else if (fused_dir) {
                if (!frz) gather_rz_with_z_halo(rz_part, rz_grid, s);
                pcg_xpay(D, it, s);
            } else {
                gather_partial(rz_part, rz_grid, gath_c.p, s);
                pcg_xpay(D, it, s);
                halo_exchange(p.p, s);
            }
        };
        auto check_part = [&](int it) {
            if (stepfuse) {
                pcg_step(D, step_bar.p, s);  // xpay + SpMV + update + check
                return;
            }
            if (dirspmv) pcg_dir_spmv(D, s);
            else pcg_spmv_dot(D, s);
            if (!fpcg) gather_partial(part_a.p, D.grid, gath_a.p, s);
            pcg_update(D, it, s);
            if (fcheck) return;
            if (!fpcg) gather_partial(part_b.p, D.grid, gath_b.p, s);
            pcg_check(D, it, s);
            BDDC_CUDA(cudaMemcpyAsync(pinned, scal.p, sizeof(double) * 4, cudaMemcpyDeviceToHost, s));
        };
        if (graphed) {
            const bool prof = opt.profile;
            // the cached graphs are keyed by the kernels' parameter block; its padding bytes (and
            // those of the nested Publish blocks) are indeterminate, so they are zeroed first
            PcgDevice key = D;
            __builtin_clear_padding(&key);
            if (!graphs.valid || std::memcmp(&graphs.key, &key, sizeof key) != 0 || graphs.precondition != precondition ||
                graphs.profile != prof) {
                graphs.reset();
                graphs.a = capture(s, [&] { check_part(0); }, &graphs.a_kernels);
                cudaGraph_t gb = nullptr;
                if (prof) {
                    if (!graph_events) graph_events = std::make_unique<ApplyEvents>();
                    capture_events = graph_events.get();
                }
                try {
                    // one graph per pipelined iteration: check part, the read-back event (a
                    // record node), then the speculative next direction
                    graphs.b = capture(
                        s,
                        [&] {
                            check_part(0);
                            BDDC_CUDA(cudaEventRecordWithFlags(check_ev.e, s, cudaEventRecordExternal));
                            next_direction(0);
                        },
                        &graphs.b_kernels, &gb);
                } catch (...) {
                    capture_events = nullptr;
                    throw;
                }
                capture_events = nullptr;
                if (prof) {  // the same iteration without the apply's event nodes
                    suppress_profile = true;
                    std::int64_t plain_kernels = 0;
                    try {
                        graphs.b_plain = capture(
                            s,
                            [&] {
                                check_part(0);
                                BDDC_CUDA(cudaEventRecordWithFlags(check_ev.e, s, cudaEventRecordExternal));
                                next_direction(0);
                            },
                            &plain_kernels);
                    } catch (...) {
                        suppress_profile = false;
                        throw;
                    }
                    suppress_profile = false;
                }
                if (prof && precondition) {  // locate the event-record nodes of the apply
                    std::size_t nn = 0;
                    BDDC_CUDA(cudaGraphGetNodes(gb, nullptr, &nn));
                    std::vector<cudaGraphNode_t> nodes(nn);
                    BDDC_CUDA(cudaGraphGetNodes(gb, nodes.data(), &nn));
                    for (cudaGraphNode_t nd : nodes) {
                        cudaGraphNodeType ty;
                        BDDC_CUDA(cudaGraphNodeGetType(nd, &ty));
                        if (ty != cudaGraphNodeTypeEventRecord) continue;
                        cudaEvent_t ev = nullptr;
                        BDDC_CUDA(cudaGraphEventRecordNodeGetEvent(nd, &ev));
                        for (int k = 0; k < 4; ++k)
                            if (ev == graph_events->e[k].e) graphs.ev_nodes[k] = nd;
                    }
                }
                graphs.b_graph = gb;
                std::memcpy(&graphs.key, &key, sizeof key);
                ++graph_captures;
                graphs.precondition = precondition;
                graphs.profile = prof;
                graphs.valid = true;
            }
        }
        int profiled_it = -1;  // iteration whose graph launch carries the apply's timing events
        auto launch_b = [&](int it) {
            cudaGraphExec_t g = graphs.b;
            if (graphs.profile && precondition) {
                if (graphs.b_plain && (it - 1) % profile_stride != 0) {
                    g = graphs.b_plain;  // unsampled iteration
                } else {  // bind this launch's timing events
                    if (ev_used == 4096) resolve_events();
                    if (ev_used == ev_pool.size()) ev_pool.emplace_back(new ApplyEvents);
                    ApplyEvents* E = ev_pool[ev_used++].get();
                    for (int k = 0; k < 4; ++k)
                        BDDC_CUDA(cudaGraphExecEventRecordNodeSetEvent(graphs.b, graphs.ev_nodes[k], E->e[k].e));
                    profiled_it = it;
                }
            }
            BDDC_CUDA(cudaGraphLaunch(g, s));
            g_kernel_launches.fetch_add(graphs.b_kernels);
        };
        for (int it = 1; it <= o.max_iterations; ++it) {
            const bool spec = pipelined && it < o.max_iterations;
            if (graphed && spec) {
                launch_b(it);  // check part + read-back event + speculative next direction
            } else {
                if (graphed) {
                    BDDC_CUDA(cudaGraphLaunch(graphs.a, s));
                    g_kernel_launches.fetch_add(graphs.a_kernels);
                } else {
                    check_part(it);
                }
                BDDC_CUDA(cudaEventRecord(check_ev.e, s));
                if (spec) next_direction(it);
            }
            BDDC_CUDA(cudaEventSynchronize(check_ev.e));
            if (pinned[3] == 1.0) {
                BDDC_CUDA(cudaStreamSynchronize(s));
                throw std::runtime_error("matrix not SPD");
            }
            if (pinned[3] == 2.0 && precondition && !(pinned[2] != 0.0) && it < o.max_iterations) {
                // the reference's next M(r) rejects a non-finite r (ensure_finite,
                // preconditioner.cpp:229); a finite r whose norm overflowed carries on, and so
                // does plain CG (no apply)
                BDDC_CUDA(cudaStreamSynchronize(s));
                const double first = first_nonfinite_global(rd, s);  // collective over the ranks
                if (first < 1e300)
                    throw std::invalid_argument("bddc apply: non-finite entry at index " +
                                                std::to_string(static_cast<long long>(first)));
            }
            rel = pinned[1];
            rep.iterations = it;
            if (pinned[2] != 0.0) {
                rep.converged = true;
                // the speculative apply launched with this iteration is skipped on the device:
                // not an apply sample
                if (profiled_it == it && ev_used > 0) {
                    BDDC_CUDA(cudaStreamSynchronize(s));
                    --ev_used;
                }
                break;
            }
            if (it == o.max_iterations) break;
            if (!spec) {
                if (precondition) {
                    apply_rz();
                    check_coarse(s);
                }
                if (!fused_dot) pcg_dot(D, rd, zd, part_a.p, s);
                if (!dirspmv && !stepfuse) {
                    gather_partial(rz_part, rz_grid, gath_c.p, s);
                    pcg_xpay(D, it, s);
                    halo_exchange(p.p, s);
                }
            }
        }
        return finish(rel);
    }
};

GpuContext::GpuContext(ProblemData problem, const GpuOptions& opt, const DistSpec* dist)
    : GpuContext(std::make_shared<const ProblemData>(std::move(problem)), opt, dist) {}

GpuContext::GpuContext(std::shared_ptr<const ProblemData> problem, const GpuOptions& opt, const DistSpec* dist) {
    if (!problem) throw std::invalid_argument("bddc setup: null problem");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw std::runtime_error("no CUDA device available (the B200 path has no CPU fallback)");
    if (opt.device < 0 || opt.device >= ndev) throw std::invalid_argument("bad device index");
    BDDC_CUDA(cudaSetDevice(opt.device));
    impl_.reset(new Impl);
    Impl& I = *impl_;
    I.n_global = problem->decomposition.global_dofs;
    if (dist && dist->world > 1) {
        try {
            sampled_symmetry_check(problem->global_matrix);
        } catch (const std::invalid_argument& e) {
            I.symmetry_error = e.what();
        }
        I.plan = std::make_unique<RankPlan>(make_rank_plan(
            *problem, dist->rank, dist->world, dist->sub_rank.empty() ? nullptr : dist->sub_rank.data()));
        I.pbs = std::make_shared<const ProblemData>(std::move(I.plan->local));
        I.plan->local = ProblemData{};
        I.n_rows = I.plan->n_rows;
        I.n_owned = I.plan->n_owned;
    } else {
        I.pbs = std::move(problem);
    }
    I.opt = opt;
    I.device = opt.device;
    I.switch_mask = env_switch_mask();
    if (I.no_exchange && !(std::getenv("BDDC_EXPERIMENTS") && std::atoi(std::getenv("BDDC_EXPERIMENTS")) == 1))
        throw std::invalid_argument(
            "BDDC_NO_EXCHANGE=1 skips every inter-GPU exchange (timing experiments, wrong results); "
            "it needs BDDC_EXPERIMENTS=1");
    // the dense replicated A_c^-1 only up to kDenseCoarseMax coarse dofs; the coarse CG beyond
    if (I.opt.coarse_mode == 0 && I.pb().constraints.n_coarse > kDenseCoarseMax) I.opt.coarse_mode = 1;
    BDDC_CUDA(cudaSetDevice(I.device));
    const Decomposition& d = I.pb().decomposition;
    if (static_cast<index_t>(I.pb().local_matrices.size()) != d.n_subdomains ||
        static_cast<index_t>(I.pb().constraints.constraint_matrices.size()) != d.n_subdomains)
        throw std::invalid_argument("bddc setup: subdomain count mismatch");
    const int workers = opt.workers > 0 ? opt.workers : std::max(1u, std::thread::hardware_concurrency());
    FactorOptions fo;
    fo.leaf_size = opt.leaf_size;
    const auto t_setup0 = std::chrono::steady_clock::now();
    SetupTimer tm;
    const bool on_device = I.opt.setup_on_device;
    const index_t* coords = I.pb().coords.empty() ? nullptr : I.pb().coords.data();
    if (I.plan) I.comm = std::make_unique<Comm>(dist->nccl_id, dist->rank, dist->world);
    if (on_device) {
        // GPU setup: the host keeps only the per-subdomain sizes (the class planner below does the
        // pattern-only work; device/setup.cu the numeric work)
        I.setup.subs.resize(d.n_subdomains);
        for (index_t i = 0; i < d.n_subdomains; ++i) {
            SubdomainSetup& S = I.setup.subs[i];
            S.n_local = I.pb().local_matrices[i].nrows;
            S.n_interior = d.interior_counts[i];
            S.n_iface = S.n_local - S.n_interior;
            S.n_primal = I.pb().constraints.constraint_matrices[i].nrows;
        }
    } else {
        I.setup = bddc_setup(I.pb().local_matrices, d, I.pb().constraints, coords, workers, fo, /*assemble=*/false,
                             /*dense_inverse=*/false);
    }
    int nsm = 148;
    BDDC_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, I.device));
    // CTA pairs always: with more subdomains than SMs they run in waves, and halving the shared-
    // memory vectors keeps 4 KB TMA units (a one-CTA subdomain at C3 would fall back to 1 KB)
    const int parts = opt.solve_parts > 0 ? opt.solve_parts : 2;
    (void)nsm;
    // TMA unit size: the largest for which every warp gets at least two ring slots next to
    // the vectors (BDDC_UNIT_BYTES overrides, for experiments)
    // four parts per subdomain aim at two co-resident CTAs per SM (the SM's 228 KB shared)
    const int ctas_per_sm = parts >= 4 ? 2 : 1;
    const int max_smem = std::min(max_solve_smem(I.device), 228 * 1024 / ctas_per_sm - 1024) - kSolveStaticSmemReserve;
    DeviceImage img;
    // candidate unit sizes (multiples of 128 bytes, largest first); BDDC_UNIT_BYTES pins one
    std::vector<int> units = {4096, 3584, 3072, 2560, 2048, 1920, 1792, 1536, 1280, 1024};
    if (std::getenv("BDDC_UNIT_BYTES")) units = {std::atoi(std::getenv("BDDC_UNIT_BYTES"))};
    std::size_t ui = 0;
    int unit = units[0];
    int spw = 0;
    tm.mark("host numeric setup (host path)");
    std::vector<SetupClass> classes;
    std::unique_ptr<Impl::Templates> tmpl;
    // joined before the classes go away, also when the setup throws
    struct Joiner {
        std::thread t;
        bool joinable() const { return t.joinable(); }
        void join() { t.join(); }
        Joiner& operator=(std::thread&& o) {
            t = std::move(o);
            return *this;
        }
        ~Joiner() {
            if (t.joinable()) t.join();
        }
    } tup;
    for (;; unit = units[++ui]) {
        if (on_device) {
            if (tup.joinable()) tup.join();  // a previous unit size's upload still reads the classes
            classes = plan_gpu_setup(I.pb().local_matrices, d, I.pb().constraints, coords, fo, parts, unit,
                                     I.opt.harmonic, workers);
            tm.mark("  class plan (symbolic, templates)");
            tmpl = std::make_unique<Impl::Templates>();
            tup = std::thread(Impl::upload_templates, std::cref(classes), I.device, std::ref(*tmpl));
            img = build_device_image(d, I.pb().constraints, I.pb().local_matrices, I.pb().global_matrix, I.setup, parts,
                                     unit, I.plan.get(), I.opt.harmonic, &classes);
            tm.mark("  device image");
        } else {
            img = build_device_image(d, I.pb().constraints, I.pb().local_matrices, I.pb().global_matrix, I.setup, parts,
                                     unit, I.plan.get(), I.opt.harmonic);
        }
        const std::size_t fixed = interior_solve_smem(img.solve.max_loc, img.solve.max_top, img.max_iface, unit, 0);
        spw = 0;
        if (fixed < static_cast<std::size_t>(max_smem)) {
            const std::size_t fit = (max_smem - fixed) / (static_cast<std::size_t>(kSolveWarps) * unit);
            spw = fit >= 8 ? 8 : fit >= 4 ? 4 : fit >= 2 ? 2 : 0;
        }
        if (spw >= 2) break;
        if (ui + 1 >= units.size())
            throw std::runtime_error("subdomain interior (" + std::to_string(img.solve.max_loc) +
                                     " dofs per CTA) exceeds the shared-memory solve capacity");
    }
    tm.mark("class plan + device image");
    if (on_device) I.setup.unique_subdomains = static_cast<index_t>(classes.size());
    I.max_iface = img.max_iface;
    I.max_primal = img.max_primal;
    I.n_coarse = img.n_coarse;
    I.n_gi = static_cast<std::int32_t>(img.gi_dof.size());
    I.max_loc = img.solve.max_loc;
    I.max_top = img.solve.max_top;
    I.factor_vals = img.factor_values;
    for (const PartDesc& pd : img.solve.parts) I.solve_stream_bytes += pd.stream_bytes;
    for (const PartDesc& pd : img.harm.parts) I.harm_stream_bytes += pd.stream_bytes;
    I.harm_fwd_values = img.harm.parts.empty() ? I.factor_vals : img.harm.fwd_factor_values;
    I.k_values = img.device_values ? img.kmat_total : static_cast<std::int64_t>(img.kmat.size());
    I.phig_values = img.device_values ? img.phig_total : static_cast<std::int64_t>(img.phig.size());
    I.ginnz = static_cast<std::int64_t>(img.gi_row_val.size());
    for (const auto& v : img.solve.couple_val) (void)v;
    I.couple_nnz = static_cast<std::int64_t>(img.solve.couple_val.size());
    I.launch.n_parts = static_cast<int>(img.solve.parts.size());
    I.launch.cluster = parts;
    I.launch.unit_bytes = unit;
    I.launch.slot_shift = spw == 8 ? 3 : spw == 4 ? 2 : 1;
    I.launch.smem = interior_solve_smem(I.max_loc, I.max_top, I.max_iface, unit, spw);

    BDDC_CUDA(cudaStreamCreateWithFlags(&I.stream, cudaStreamNonBlocking));
    auto upload_pod = [](auto& buf, const auto& vec) {
        using T = typename std::decay_t<decltype(vec)>::value_type;
        buf.alloc(std::max<std::size_t>(vec.size(), 1));
        if (!vec.empty()) BDDC_CUDA(cudaMemcpy(buf.p, vec.data(), sizeof(T) * vec.size(), cudaMemcpyHostToDevice));
    };
    I.prog.upload(img.solve);
    I.harm.upload(img.harm);
    I.head.upload(img.head);
    tm.mark("program uploads");
    if (I.head.valid) {
        if (img.head.parts.size() != img.harm.parts.size()) throw std::logic_error("head/harmonic programs differ in parts");
        for (std::size_t q = 0; q < img.head.parts.size(); ++q)
            if (img.head.parts[q].gmap != img.harm.parts[q].gmap || img.head.parts[q].n_loc != img.harm.parts[q].n_loc)
                throw std::logic_error("head/harmonic programs differ in local layout");
        I.ybuf.alloc(std::max<std::size_t>(img.head.gmap.size(), 1));
        BDDC_CUDA(cudaMemset(I.ybuf.p, 0, sizeof(double) * I.ybuf.n));
        I.head_bwd_values = img.head.bwd_factor_values;
    }
    if (std::getenv("BDDC_SOLVE_STATS")) {
        I.dbg_buf.alloc(static_cast<std::size_t>(img.solve.parts.size()) * kSolveWarps * 8 + 256 + 5 * 256 * kSolveWarps + 8 + 4 * kSolveWarps + 512 * 6);
        BDDC_CUDA(cudaMemset(I.dbg_buf.p, 0, sizeof(long long) * I.dbg_buf.n));
    }
    upload_pod(I.subs, img.subs);
    I.iface_dof.upload(img.iface_dof);
    I.iface_w.upload(img.iface_w);
    I.iface_gid.upload(img.iface_gid);
    {
        // the solve kernel reads the written dof directly: the slot's dof if it is the writer, -1
        std::vector<std::int32_t> wdof(img.iface_writer.size());
        for (std::size_t k = 0; k < wdof.size(); ++k) wdof[k] = img.iface_writer[k] ? img.iface_dof[k] : -1;
        I.iface_writer.upload(wdof);
    }
    if (img.device_values) {  // written by the device setup
        I.kmat.alloc(std::max<std::int64_t>(img.kmat_total, 1));
        I.phig.alloc(std::max<std::int64_t>(img.phig_total, 1));
        I.phi.alloc(std::max<std::int64_t>(img.phi_total, 1));
        BDDC_CUDA(cudaMemset(I.phi.p, 0, sizeof(double) * I.phi.n));
        I.lambda_dev.alloc(std::max<std::int64_t>(img.lambda_total, 1));
        I.lambda_off = img.lambda_off;
    } else {
        I.kmat.upload(img.kmat);
        I.phig.upload(img.phig);
        I.phi.upload(img.phi);
    }
    I.primal.upload(img.primal);
    I.local_dofs.upload(img.local_dofs);
    I.lrow_ptr.upload(img.lrow_ptr);
    I.lrow_col.upload(img.lrow_col);
    I.lrow_val.upload(img.lrow_val);
    I.gi_dof.upload(img.gi_dof);
    I.gi_row_ptr.upload(img.gi_row_ptr);
    {
        std::vector<std::int32_t> sr(2 * std::max<std::size_t>(img.iface_gid.size(), 1), 0);
        for (std::size_t k = 0; k < img.iface_gid.size(); ++k) {
            sr[2 * k] = img.gi_row_ptr[img.iface_gid[k]];
            sr[2 * k + 1] = img.gi_row_ptr[img.iface_gid[k] + 1];
        }
        I.slot_rows.upload(sr);
    }
    I.gi_row_col.upload(img.gi_row_col);
    I.gi_row_val.upload(img.gi_row_val);
    tm.mark("subdomain / K / Phi buffers");
    I.gi_own_ptr.upload(img.gi_own_ptr);
    I.gi_own_ref.upload(img.gi_own_ref);
    {
        // each local interface slot's owners as one int4 (the interior solve's z_G gather)
        std::vector<std::int32_t> own4(4 * std::max<std::size_t>(img.iface_gid.size(), 1), -1);
        for (std::size_t k = 0; k < img.iface_gid.size(); ++k) {
            const int gid = img.iface_gid[k];
            const int o0 = img.gi_own_ptr[gid], o1 = img.gi_own_ptr[gid + 1];
            if (o1 - o0 > 4) {
                own4[4 * k] = -2 - gid;
                continue;
            }
            for (int o = o0; o < o1; ++o) own4[4 * k + (o - o0)] = img.gi_own_ref[o];
        }
        I.iface_own4.upload(own4);
    }
    I.dof_own_ptr.upload(img.dof_own_ptr);
    I.dof_own_ref.upload(img.dof_own_ref);
    I.c_own_ptr.upload(img.c_own_ptr);
    I.c_own_ref.upload(img.c_own_ref);
    {
        const std::size_t nc = img.c_own_ptr.empty() ? 0 : img.c_own_ptr.size() - 1;
        std::vector<std::int32_t> c4(4 * std::max<std::size_t>(nc, 1), -1);
        for (std::size_t q = 0; q < nc; ++q) {
            const int o0 = img.c_own_ptr[q], o1 = img.c_own_ptr[q + 1];
            if (o1 - o0 > 4) {
                c4[4 * q] = -2;
                continue;
            }
            for (int o = o0; o < o1; ++o) c4[4 * q + (o - o0)] = img.c_own_ref[o];
        }
        I.c_own4.upload(c4);
    }
    I.rc_g.alloc(std::max(img.n_coarse, 1));
    I.coarse_ctr.alloc(1);
    BDDC_CUDA(cudaMemset(I.coarse_ctr.p, 0, sizeof(unsigned long long)));
    {
        std::vector<double> wl;
        for (const auto& w : d.weights) wl.insert(wl.end(), w.begin(), w.end());
        I.weights_local.upload(wl);
    }
    I.coarse_status.alloc(4);
    tm.mark("  coarse-owner maps, weights");
    I.A_ptr.upload(I.pb().global_matrix.row_offsets);
    I.A_col.upload(I.pb().global_matrix.col_indices);
    I.A_val.upload(I.pb().global_matrix.values);
    {
        // sliced ELL copy for the PCG SpMV: slices of 32 rows, width = the slice's longest row,
        // entries column-major within the slice in CSR order (padding never read: row lengths)
        const CsrMatrix& A = I.pb().global_matrix;
        const index_t nr = A.nrows, ns = (nr + 31) / 32;
        std::vector<std::int64_t> off(static_cast<std::size_t>(ns) + 1, 0);
        std::vector<std::uint16_t> len(static_cast<std::size_t>(ns) * 32, 0);
        for (index_t sl = 0; sl < ns; ++sl) {
            index_t w = 0;
            for (index_t i = sl * 32; i < std::min(nr, sl * 32 + 32); ++i) {
                const index_t l = A.row_offsets[i + 1] - A.row_offsets[i];
                if (l > 65535) throw std::runtime_error("global matrix row longer than 65535 entries");
                len[i] = static_cast<std::uint16_t>(l);
                w = std::max(w, l);
            }
            off[sl + 1] = off[sl] + static_cast<std::int64_t>(w) * 32;
        }
        // the entries are scattered on the device from the CSR upload above
        const std::size_t words = static_cast<std::size_t>(std::max<std::int64_t>(off[ns], 1));
        I.ell_off.upload(off);
        I.ell_len.upload(len);
        I.ell_col.alloc(words);
        I.ell_val.alloc(words);
        BDDC_CUDA(cudaMemsetAsync(I.ell_col.p, 0, sizeof(std::int32_t) * words, I.stream));
        BDDC_CUDA(cudaMemsetAsync(I.ell_val.p, 0, sizeof(double) * words, I.stream));
        // 16-bit column offsets (half the column bytes of the SpMV) unless one does not fit
        I.ell_d16.alloc(words);
        DBuf<int> over;
        over.alloc(1);
        BDDC_CUDA(cudaMemsetAsync(I.ell_d16.p, 0, sizeof(std::int16_t) * words, I.stream));
        BDDC_CUDA(cudaMemsetAsync(over.p, 0, sizeof(int), I.stream));
        device_csr_to_sliced_ell(static_cast<int>(nr), I.A_ptr.p, I.A_col.p, I.A_val.p, I.ell_off.p, I.ell_col.p,
                                 I.ell_val.p, I.ell_d16.p, over.p, I.stream);
        int over_h = 0;
        BDDC_CUDA(cudaMemcpyAsync(&over_h, over.p, sizeof(int), cudaMemcpyDeviceToHost, I.stream));
        BDDC_CUDA(cudaStreamSynchronize(I.stream));
        const char* e16 = std::getenv("BDDC_ELL16");
        if (over_h || (e16 && std::atoi(e16) == 0)) I.ell_d16.alloc(0);
    }
    tm.mark("  global matrix, sliced ELL");
    const std::size_t n = d.global_dofs;
    I.U.alloc(n);
    BDDC_CUDA(cudaMemset(I.U.p, 0, sizeof(double) * n));
    I.gbuf.alloc(std::max<std::int64_t>(img.hbuf_total, 1));
    I.hbuf.alloc(std::max<std::int64_t>(img.hbuf_total, 1));
    I.cbuf.alloc(std::max<std::int64_t>(img.cbuf_total, 1));
    I.lbuf.alloc(std::max<std::int64_t>(img.local_total, 1));
    I.xc.alloc(std::max(img.n_coarse, 1));
    {
        // measured on B200: at n_c = 161 / 337 the grid barrier costs more than the redundant
        // per-CTA r_c (3-4 us per apply), at 705 they tie; it pays from ~1,000 coarse dofs (C2 at
        // N=8: 1,441). BDDC_COOP_COARSE=0/1 forces it.
        const char* e = std::getenv("BDDC_COOP_COARSE");
        const bool want = e ? std::atoi(e) == 1 : img.n_coarse >= 1024;
        if (want) I.coop_coarse = iface_local_cooperative_fits(I.iface_params(), I.opt.local_blocks, I.device);
    }
    I.vin.alloc(n);
    I.vout.alloc(n);
    I.vtmp.alloc(n);
    I.vtmp2.alloc(n);
    if (I.plan) {
        const RankPlan& P = *I.plan;
        I.build_runs();
        I.halo_idx.upload(P.halo_send_idx);
        I.iface_idx.upload(P.iface_send_slot);
        I.halo_send.alloc(std::max<std::size_t>(P.halo_send_idx.size(), 1));
        I.iface_send.alloc(std::max<std::size_t>(P.iface_send_slot.size(), 1));
        I.halo_soff.assign(P.halo_send_off.begin(), P.halo_send_off.end());
        I.halo_roff.assign(P.halo_recv_off.begin(), P.halo_recv_off.end());
        I.iface_soff.assign(P.iface_send_off.begin(), P.iface_send_off.end());
        I.iface_roff.assign(P.iface_recv_off.begin(), P.iface_recv_off.end());
        BDDC_CUDA(cudaMemset(I.hbuf.p, 0, sizeof(double) * I.hbuf.n));
        BDDC_CUDA(cudaMemset(I.cbuf.p, 0, sizeof(double) * I.cbuf.n));
        I.ensure_pcg(1);
        BDDC_CUDA(cudaDeviceSynchronize());
        const char* p2p_env = std::getenv("BDDC_P2P");
        if (!(p2p_env && std::atoi(p2p_env) == 0)) I.setup_peer_links(img);
    }
    tm.mark("uploads + buffers");
    if (tup.joinable()) tup.join();
    if (tmpl && tmpl->error) std::rethrow_exception(tmpl->error);
    if (on_device) I.device_setup(classes, img, *tmpl);
    tm.mark("device numeric setup");
    if (I.kpacked) I.pack_k(img);
    I.finish_coarse(dist);
    tm.mark("coarse");
    BDDC_CUDA(cudaDeviceSynchronize());
    I.setup.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_setup0).count();
}

GpuContext::~GpuContext() {
    if (impl_) {
        cudaSetDevice(impl_->device);
        if (impl_->pinned) cudaFreeHost(impl_->pinned);
        if (impl_->stage) cudaFreeHost(impl_->stage);
        if (impl_->stream) cudaStreamDestroy(impl_->stream);
    }
}

void dist_nccl_id(char out[128]) { nccl_unique_id(out); }

index_t GpuContext::n() const { return impl_->pb().decomposition.global_dofs; }
index_t GpuContext::n_global() const { return impl_->n_global; }
index_t GpuContext::n_owned() const { return impl_->dist() ? impl_->n_owned : n(); }
index_t GpuContext::n_rows() const { return impl_->dist() ? impl_->n_rows : n(); }
int GpuContext::rank() const { return impl_->dist() ? impl_->comm->rank() : 0; }
int GpuContext::world() const { return impl_->dist() ? impl_->comm->world() : 1; }
const std::vector<index_t>& GpuContext::local_to_global() const {
    static const std::vector<index_t> none;
    return impl_->plan ? impl_->plan->local_to_global : none;
}

void GpuContext::apply_device(const double* r, double* z, void* stream) {
    std::lock_guard<std::mutex> lk(impl_->mu);
    BDDC_CUDA(cudaSetDevice(impl_->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : impl_->stream;
    impl_->apply(r, z, s);
    impl_->check_coarse(s);
}

void GpuContext::apply_host(const double* r, double* z) {
    std::lock_guard<std::mutex> lk(impl_->mu);
    Impl& I = *impl_;
    const index_t n = I.pb().decomposition.global_dofs;
    ensure_finite(r, I.n_global, "bddc apply");
    BDDC_CUDA(cudaSetDevice(I.device));
    if (I.dist()) {
        const void* rm = mapped_host_pointer(r);
        void* zm = const_cast<void*>(mapped_host_pointer(z));
        if (rm && zm) {  // pinned user buffers: zero-copy gather / scatter over PCIe
            I.gather_mapped(static_cast<const double*>(rm), I.vin.p, I.stream);
            I.apply(I.vin.p, I.vout.p, I.stream);
            I.scatter_mapped(I.vout.p, static_cast<double*>(zm), I.stream);
            BDDC_CUDA(cudaStreamSynchronize(I.stream));
            I.check_coarse(I.stream);
            return;
        }
        I.gather_host(r);
        BDDC_CUDA(cudaMemcpyAsync(I.vin.p, I.stage, sizeof(double) * n, cudaMemcpyHostToDevice, I.stream));
        I.apply(I.vin.p, I.vout.p, I.stream);
        BDDC_CUDA(cudaMemcpyAsync(I.stage, I.vout.p, sizeof(double) * I.n_rows, cudaMemcpyDeviceToHost, I.stream));
        BDDC_CUDA(cudaStreamSynchronize(I.stream));
        I.check_coarse(I.stream);
        I.scatter_host(z);
        return;
    }
    BDDC_CUDA(cudaMemcpyAsync(I.vin.p, r, sizeof(double) * n, cudaMemcpyHostToDevice, I.stream));
    I.apply(I.vin.p, I.vout.p, I.stream);
    I.check_coarse(I.stream);
    BDDC_CUDA(cudaMemcpyAsync(z, I.vout.p, sizeof(double) * n, cudaMemcpyDeviceToHost, I.stream));
    BDDC_CUDA(cudaStreamSynchronize(I.stream));
}

SolveResult GpuContext::pcg_host(const double* b, const SolverOpts& o, double* x, bool precondition) {
    std::lock_guard<std::mutex> lk(impl_->mu);
    Impl& I = *impl_;
    const index_t n = I.pb().decomposition.global_dofs;
    BDDC_CUDA(cudaSetDevice(I.device));
    if (I.dist()) {  // non-finite rhs entries: found on the devices, agreed over the ranks (pcg)
        const void* bm = mapped_host_pointer(b);
        void* xm = const_cast<void*>(mapped_host_pointer(x));
        if (bm && xm) {  // pinned user buffers: zero-copy gather / scatter over PCIe
            I.gather_mapped(static_cast<const double*>(bm), I.vin.p, I.stream);
            SolveResult rep = I.pcg(I.vin.p, o, I.vout.p, precondition, I.stream);
            I.scatter_mapped(I.vout.p, static_cast<double*>(xm), I.stream);
            BDDC_CUDA(cudaStreamSynchronize(I.stream));
            return rep;
        }
        I.gather_host(b);
        BDDC_CUDA(cudaMemcpyAsync(I.vin.p, I.stage, sizeof(double) * n, cudaMemcpyHostToDevice, I.stream));
        SolveResult rep = I.pcg(I.vin.p, o, I.vout.p, precondition, I.stream);
        BDDC_CUDA(cudaMemcpyAsync(I.stage, I.vout.p, sizeof(double) * I.n_rows, cudaMemcpyDeviceToHost, I.stream));
        BDDC_CUDA(cudaStreamSynchronize(I.stream));
        I.scatter_host(x);
        return rep;
    }
    // one GPU: non-finite rhs entries are found on the device (pcg: ||b|| check + first index)
    BDDC_CUDA(cudaMemcpyAsync(I.vin.p, b, sizeof(double) * n, cudaMemcpyHostToDevice, I.stream));
    SolveResult rep = I.pcg(I.vin.p, o, I.vout.p, precondition, I.stream);
    BDDC_CUDA(cudaMemcpyAsync(x, I.vout.p, sizeof(double) * n, cudaMemcpyDeviceToHost, I.stream));
    BDDC_CUDA(cudaStreamSynchronize(I.stream));
    return rep;
}

SolveResult GpuContext::pcg_device(const double* b, const SolverOpts& o, double* x, bool precondition, void* stream) {
    std::lock_guard<std::mutex> lk(impl_->mu);
    BDDC_CUDA(cudaSetDevice(impl_->device));
    return impl_->pcg(b, o, x, precondition, stream ? static_cast<cudaStream_t>(stream) : impl_->stream);
}

void GpuContext::stage_host(Stage st, const double* in0, const double* in1, const double* in2, double* out) {
    std::lock_guard<std::mutex> lk(impl_->mu);
    Impl& I = *impl_;
    const index_t n = I.pb().decomposition.global_dofs;
    BDDC_CUDA(cudaSetDevice(I.device));
    if (I.dist()) throw std::invalid_argument("stage hooks are single-GPU parity hooks");
    cudaStream_t s = I.stream;
    const StageParams sp = I.stage_params();
    auto h2d = [&](double* dst, const double* src) {
        BDDC_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    };
    switch (st) {
        case Stage::interior:  // preconditioner.cpp:194-213
            h2d(I.vin.p, in0);
            BDDC_CUDA(cudaMemsetAsync(I.vout.p, 0, sizeof(double) * n, s));
            launch_interior_solve(I.solve_params(I.vin.p, I.vout.p), I.launch, 0, s);
            break;
        case Stage::coarse:  // preconditioner.cpp:129-171
            h2d(I.vin.p, in0);
            launch_stage_phi_restrict(sp, I.vin.p, s);
            I.coarse_solve(s);
            I.check_coarse(s);
            launch_stage_phi_prolong(sp, s);
            launch_stage_gather_local(sp, I.vout.p, s);
            break;
        case Stage::local: {  // preconditioner.cpp:173-192, saddle solve by interior/interface blocks
            h2d(I.vin.p, in0);
            BDDC_CUDA(cudaMemsetAsync(I.vtmp.p, 0, sizeof(double) * n, s));
            launch_interior_solve(I.solve_params(I.vin.p, I.vtmp.p), I.launch, 0, s);  // y = A_II^-1 f_I
            launch_stage_local_g(sp, I.vin.p, I.vtmp.p, s);                             // g = f_G - A_GI y
            launch_iface_local(I.iface_params(), I.opt.local_blocks, s, 0);             // z_G = K g
            BDDC_CUDA(cudaMemsetAsync(I.vout.p, 0, sizeof(double) * n, s));
            launch_interior_solve(I.solve_params(I.vin.p, I.vout.p), I.launch, 2, s);  // z_I
            launch_stage_iface_gather(sp, I.hbuf.p, I.vout.p, s);                       // sum_i w z_G
            break;
        }
        case Stage::static_condensation: {  // preconditioner.cpp:215-223
            h2d(I.vin.p, in1);
            h2d(I.vtmp.p, in2);
            device_axpby(n, 1.0, I.vin.p, 1.0, I.vtmp.p, I.vtmp2.p, s);
            device_spmv(n, I.A_ptr.p, I.A_col.p, I.A_val.p, I.vtmp2.p, I.vtmp.p, s);
            h2d(I.vin.p, in0);
            device_axpby(n, 1.0, I.vin.p, -1.0, I.vtmp.p, I.vtmp2.p, s);
            BDDC_CUDA(cudaMemsetAsync(I.vout.p, 0, sizeof(double) * n, s));
            launch_interior_solve(I.solve_params(I.vtmp2.p, I.vout.p), I.launch, 0, s);
            break;
        }
    }
    BDDC_CUDA(cudaMemcpyAsync(out, I.vout.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    BDDC_CUDA(cudaStreamSynchronize(s));
}

const BddcSetup& GpuContext::setup() const { return impl_->setup; }
const ProblemData& GpuContext::problem() const { return impl_->pb(); }
double GpuContext::setup_seconds() const { return impl_->setup.seconds; }
double GpuContext::setup_device_seconds() const { return impl_->setup_device_s; }

void GpuContext::subdomain_blocks(int i, double* phi, double* lambda, double* aci) const {
    const Impl& I = *impl_;
    const SubdomainSetup& S = I.setup.subs.at(i);
    const std::size_t np = S.n_primal;
    if (aci) std::memcpy(aci, S.aci.data(), sizeof(double) * S.aci.size());
    if (!I.opt.setup_on_device) {
        if (phi) std::memcpy(phi, S.phi.data(), sizeof(double) * S.phi.size());
        if (lambda) std::memcpy(lambda, S.lambda.data(), sizeof(double) * S.lambda.size());
        return;
    }
    BDDC_CUDA(cudaSetDevice(I.device));
    BDDC_CUDA(cudaDeviceSynchronize());
    std::vector<SubdomainDesc> sd(1);
    BDDC_CUDA(cudaMemcpy(sd.data(), I.subs.p + i, sizeof(SubdomainDesc), cudaMemcpyDeviceToHost));
    if (phi) BDDC_CUDA(cudaMemcpy(phi, I.phi.p + sd[0].phi, sizeof(double) * S.n_local * np, cudaMemcpyDeviceToHost));
    if (lambda)
        BDDC_CUDA(cudaMemcpy(lambda, I.lambda_dev.p + I.lambda_off[i], sizeof(double) * np * np, cudaMemcpyDeviceToHost));
}
std::int64_t GpuContext::graph_captures() const { return impl_->graph_captures; }
int GpuContext::coarse_mode() const { return impl_->opt.coarse_mode; }
int GpuContext::switches() const { return impl_->switch_mask; }

const char* env_switch_name(int i) { return i >= 0 && i < kNumEnvSwitches ? kEnvSwitches[i] : nullptr; }
int env_switch_mask() {
    int m = 0;
    for (int i = 0; i < kNumEnvSwitches; ++i)
        if (std::getenv(kEnvSwitches[i])) m |= 1 << i;
    return m;
}
std::int64_t GpuContext::factor_values() const { return impl_->factor_vals; }
std::int64_t GpuContext::interior_pass_bytes() const { return impl_->solve_stream_bytes; }
int GpuContext::solve_parts() const { return impl_->launch.cluster; }
std::int64_t GpuContext::apply_bytes() const {
    const Impl& I = *impl_;
    const std::int64_t n = I.pb().decomposition.global_dofs;
    // algorithmic FP64 bytes: the two interior solves (forward + backward over every factor
    // value; the harmonic extension's forward sweep only over its active supernodes), K_i,
    // Phi_G (restrict + prolong), the coarse inverse, interface rows and coupling, plus vector
    // traffic (r read twice, u0 written/read, z written)
    return interior_apply_bytes() +
           8 * (I.k_values + 2 * I.phig_values + static_cast<std::int64_t>(I.n_coarse) * I.n_coarse + I.ginnz +
                I.couple_nnz + 5 * n);
}
std::int64_t GpuContext::interior_apply_bytes() const {
    const Impl& I = *impl_;
    std::int64_t ni = 0;
    for (const auto& sub : I.setup.subs) ni += sub.n_interior;
    // solve 1: 2F values + rhs gather + solution write; solve 2: F + F_fwd(active) values + u0 read
    // + z write (its rhs comes from the interface coupling, counted in couple_nnz). Split apply:
    // solve 1 = F + F_bwd(active) + rhs gather + u0 write + y0 write, solve 2 = F_fwd + F + y0
    // read + z write.
    if (I.use_split && I.harm.valid && I.head.valid)
        return 8 * (I.factor_vals + I.head_bwd_values + 3 * ni) + 8 * (I.harm_fwd_values + I.factor_vals + 2 * ni);
    return 8 * (2 * I.factor_vals + 2 * ni) + 8 * (I.factor_vals + I.harm_fwd_values + 2 * ni);
}
KernelTimes GpuContext::kernel_times() {
    std::lock_guard<std::mutex> lk(impl_->mu);
    BDDC_CUDA(cudaSetDevice(impl_->device));
    impl_->resolve_events();
    return impl_->times;
}
void GpuContext::reset_kernel_times() {
    std::lock_guard<std::mutex> lk(impl_->mu);
    impl_->resolve_events();
    impl_->times = KernelTimes{};
}
void GpuContext::set_profile(bool on) { impl_->opt.profile = on; }
int GpuContext::device() const { return impl_->device; }
void GpuContext::synchronize() { BDDC_CUDA(cudaStreamSynchronize(impl_->stream)); }
std::int64_t GpuContext::solve_profile(std::int64_t* out, std::int64_t cap) {
    Impl& I = *impl_;
    if (I.fused_trace.p) {  // fused-exchange event ring (BDDC_FUSED_TRACE)
        const std::int64_t n = std::min<std::int64_t>(cap, static_cast<std::int64_t>(I.fused_trace.n));
        BDDC_CUDA(cudaDeviceSynchronize());
        BDDC_CUDA(cudaMemcpy(out, I.fused_trace.p, sizeof(long long) * n, cudaMemcpyDeviceToHost));
        return n;
    }
    if (I.ex_stats.p) {  // exchange diagnostics take precedence (BDDC_EXCH_STATS)
        const std::int64_t n = std::min<std::int64_t>(cap, static_cast<std::int64_t>(I.ex_stats.n));
        BDDC_CUDA(cudaDeviceSynchronize());
        BDDC_CUDA(cudaMemcpy(out, I.ex_stats.p, sizeof(long long) * n, cudaMemcpyDeviceToHost));
        return n;
    }
    if (!I.dbg_buf.p) return 0;
    const std::int64_t n = std::min<std::int64_t>(cap, static_cast<std::int64_t>(I.dbg_buf.n));
    BDDC_CUDA(cudaDeviceSynchronize());
    BDDC_CUDA(cudaMemcpy(out, I.dbg_buf.p, sizeof(long long) * n, cudaMemcpyDeviceToHost));
    return n;
}

// pcg.cpp:111-173 (host; O(iterations))

}  // namespace bddc_b200
