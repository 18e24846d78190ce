// Batched interior solve A_II^{-1} b for every subdomain (replaces reference
// interior_correction, src/preconditioner.cpp:194-213, and the lu_solve it calls,
// src/sparse_lu.cpp:203-237).
//
// One CTA per part (a cluster of P CTAs per subdomain). Each of the 16 warps owns a
// double-buffered shared-memory ring: lane 0 streams the warp's own tile units from HBM
// with cp.async.bulk (TMA bulk copies, mbarrier completion), one unit ahead, so streaming
// never waits for other warps and keeps going across phase barriers. Vectors T/X live in
// shared memory; every output chunk of a phase is owned by one warp (deterministic).
// With P = 2 the two CTAs of a cluster each own one half of the nested-dissection tree
// and exchange the partial sums into the separator chain above the split through
// distributed shared memory.
#include "solve.cuh"

namespace bddc_b200 {
namespace {

constexpr int kThreads = kSolveWarps * 32;
constexpr int kMaxRegEntries = 96;  // per-warp phase / unit tables held in registers (3 per lane)
constexpr int kMaxWarpSlots = 8;    // ring slots per warp (power of two, <= 8)

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, std::uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, std::uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, std::uint32_t bytes, std::uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ double ld_dsmem(const double* local, std::uint32_t rank) {
    std::uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local)), "r"(rank));
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote) : "memory");
    return v;
}

// Per-warp table spread over the lanes' registers: entry i lives in lane i % 32, slot i / 32;
// entries beyond kMaxRegEntries fall back to global memory.
// With more than 16 warps the register budget (64 per thread at 32 warps) does not hold the
// tables: they are read from global memory (L1-resident) instead.
constexpr bool kRegTables = kSolveWarps <= 16;
struct RegTable {
    int v[kRegTables ? kMaxRegEntries / 32 : 1];
    __device__ __forceinline__ int get(int i, const int* fallback, int stride) const {
        if (!kRegTables || i >= kMaxRegEntries) return __ldg(fallback + static_cast<std::int64_t>(i) * stride);
        const int slot = i >> 5;
        const int mine = slot == 0 ? v[0] : (slot == 1 ? v[1] : v[2]);
        return __shfl_sync(0xffffffffu, mine, i & 31);
    }
};

// Checked build (make VARIANT=_checked EXTRA=-DBDDC_CHECKED; compute-sanitizer is closed on
// this pool): every shared-memory access of a tile is bounds-checked against its part's
// vectors and its unit, a violation traps with the step's coordinates.
#ifdef BDDC_CHECKED
#define SOLVE_CHECK(cond, code)                                                                          \
    do {                                                                                                \
        if (!(cond)) {                                                                                  \
            printf("interior solve check %d failed: cta %d warp %d lane %d\n", code, blockIdx.x,          \
                   threadIdx.x >> 5, threadIdx.x & 31);                                                 \
            __trap();                                                                                   \
        }                                                                                               \
    } while (0)
#else
#define SOLVE_CHECK(cond, code) do { } while (0)
#endif
struct TileBounds {
    int ldn_p;   // a part's vector stride: T[0, ldn_p), X[0, ldn_p) (T-relative indices < 2 ldn_p)
    int n_top;   // Q entries
    int room;    // bytes of the unit from the tile data start
};

// One tile GEMV (device_format.hpp): k <= 32 rows, G = 2^lg column groups, lane = r*G + g
// owns row r and columns j = t*G + g; values are stored iteration-major, value(r, t*G + g)
// at [t*S + voff + r*G + g], so every iteration is one contiguous, conflict-free shared-memory
// read per lane. `h` is the lane's own step sub-header (a pair step: lanes 16-31 run tile B,
// sl = lane - 16); it carries every field the lane needs, so decoding is a handful of bit
// extractions. Written for a short issue path (most tiles hold ~5 values per lane): no
// divergent guard around the loop (lanes beyond k*G read in-bounds slack and are masked
// before the reduction), a 4-way body with predicated tails, pointer increments only. The
// G partial sums of a row are reduced with an xor butterfly inside the row's lane group
// (to the step's largest G, uniform over the warp); the row total accumulates into `acc` and
// is flushed by the group's first lane.
template <bool PROF = false>
__device__ __forceinline__ void tile_task(const int4 h, const unsigned char* tile, int sl, double* own, double* other,
                                          double* Q, double& acc, const TileBounds& bnd, long long* tp = nullptr) {
    long long tq = PROF ? clock64() : 0;
#define TILE_T(i) do { if constexpr (PROF) { const long long t_ = clock64(); tp[i] += t_ - tq; tq = t_; } } while (0)
    const unsigned w0 = h.x, w2 = h.z, w3 = h.w;
    const int S = (w0 >> 11) & 63, gmax_lg = (w0 >> 25) & 7;
    const int k = w2 & 63, lg = (w2 >> 6) & 7, flags = (w2 >> 9) & 255, iters = (w2 >> 17) & 511;
    const int G = 1 << lg, kG = k << lg;
    const int g = sl & (G - 1), r = sl >> lg;
    const double* in = (flags & kTaskInOwn) ? own : other;
    const double* M = reinterpret_cast<const double*>(tile) + (w3 & 31) + sl;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    const int full = iters & ~3, rem = iters & 3;
    SOLVE_CHECK(((w0 >> 17) & 255) * 16 <= bnd.room && k >= 1 && k <= 32 && kG <= 32, 1);
    SOLVE_CHECK(sl >= kG || iters == 0 || ((iters - 1) * S + static_cast<int>(w3 & 31) + sl + 1) * 8 <= static_cast<int>((w0 >> 17) & 255) * 16, 2);
    TILE_T(0);
    if (flags & kTaskInIndexed) {
        const std::int32_t* ix = reinterpret_cast<const std::int32_t*>(tile + (((w3 >> 5) & 255) << 4)) + g;
        SOLVE_CHECK(static_cast<int>(((w3 >> 5) & 255) * 16) + iters * G * 4 <= bnd.room, 3);
#ifdef BDDC_CHECKED
        for (int t = 0; t < iters; ++t) SOLVE_CHECK(ix[t * G] >= 0 && ix[t * G] < 2 * bnd.ldn_p, 4);
#endif
#pragma unroll 1
        for (int t = 0; t < full; t += 4) {
            s0 = fma(M[0], in[ix[0]], s0);
            s1 = fma(M[S], in[ix[G]], s1);
            s2 = fma(M[2 * S], in[ix[2 * G]], s2);
            s3 = fma(M[3 * S], in[ix[3 * G]], s3);
            M += 4 * S;
            ix += 4 * G;
        }
        if (rem > 0) s0 = fma(M[0], in[ix[0]], s0);
        if (rem > 1) s1 = fma(M[S], in[ix[G]], s1);
        if (rem > 2) s2 = fma(M[2 * S], in[ix[2 * G]], s2);
    } else {
        const double* v = in + (h.y & 0xffff) + g;
        SOLVE_CHECK(static_cast<int>(h.y & 0xffff) + iters * G <= bnd.ldn_p, 5);
#pragma unroll 1
        for (int t = 0; t < full; t += 4) {
            s0 = fma(M[0], v[0], s0);
            s1 = fma(M[S], v[G], s1);
            s2 = fma(M[2 * S], v[2 * G], s2);
            s3 = fma(M[3 * S], v[3 * G], s3);
            M += 4 * S;
            v += 4 * G;
        }
        if (rem > 0) s0 = fma(M[0], v[0], s0);
        if (rem > 1) s1 = fma(M[S], v[G], s1);
        if (rem > 2) s2 = fma(M[2 * S], v[2 * G], s2);
    }
    TILE_T(1);
    // per-lane partial sums accumulate over the pieces of a chunk (same k, hence same G and
    // lane -> row map); the row's lane group is reduced once, at its last piece (a pair's two
    // halves are in lockstep: both or neither are last)
    acc = ((flags & kTaskFirst) ? 0.0 : acc) + (sl < kG ? (s0 + s1) + (s2 + s3) : 0.0);
    if (!(flags & kTaskLast)) return;
#pragma unroll 1
    for (int off = (1 << gmax_lg) >> 1; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, acc, off);
        if (off < G) acc += o;
    }
    TILE_T(2);
    if (g == 0) {
        if (flags & kTaskPush) {
            if (r < k) {
                const int o = reinterpret_cast<const std::int32_t*>(tile + (((w3 >> 13) & 255) << 4))[r];
                SOLVE_CHECK(static_cast<int>(((w3 >> 13) & 255) * 16) + k * 4 <= bnd.room, 6);
                SOLVE_CHECK(o >= 0 && o < ((flags & kTaskPartial) ? bnd.n_top : bnd.ldn_p), 7);
                if (flags & kTaskPartial) Q[o] += acc;
                else own[o] -= acc;
            }
        } else if (r < static_cast<int>(w2 >> 26)) {
            const int out = (h.y >> 16) + r;
            SOLVE_CHECK(out < bnd.ldn_p, 8);
            if (flags & kTaskDiag) other[out] = acc;
            else own[out] -= acc;
        }
    }
    if constexpr (PROF) __syncwarp();  // (the flush's lanes, timed together)
    TILE_T(3);
#undef TILE_T
}

template <int MODE, int CLUSTER, bool STATS>
__global__ void __launch_bounds__(kThreads, 1) interior_solve_kernel(const SolveParams S) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    pdl_trigger();
    const long long t_entry = STATS ? clock64() : 0;  // CTA 0 prologue / epilogue markers (STATS)
    long long* const mkp = STATS ? S.stats + static_cast<long long>(gridDim.x) * kSolveWarps * 8 + 256 + 2 * 256 * kSolveWarps : nullptr;
    double rz = 0.0;  // MODE 3 with dot_part: this thread's share of r.z
    const PartDesc& pdr = S.parts[blockIdx.x];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const int unit = S.unit_bytes;

    // ---- shared memory carve-up
    std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem_raw);  // [warp][kMaxWarpSlots]
    const int ldn = (S.max_loc + 64 + 1) & ~1;
    double* T = reinterpret_cast<double*>(bars + kSolveWarps * kMaxWarpSlots);
    // X follows this part's T at the part's own stride (device_format.hpp: a merged backward
    // tile addresses both through one index list relative to T)
    const int ldn_p = part_ldn(pdr.n_loc);
    double* X = T + ldn_p;
    double* Q = T + 2 * ldn;
    double* ZG = Q + ((S.max_top + 1) & ~1);
    unsigned char* glut = reinterpret_cast<unsigned char*>(ZG + ((S.max_iface + 1) & ~1));  // spare 1 KB
    // offset arithmetic on smem_raw (not through an integer cast) keeps the shared address
    // space visible to the compiler: tile reads stay LDS instead of generic LD
    unsigned char* ring = smem_raw + ((static_cast<std::size_t>(glut + 33 * 32 - smem_raw) + 127) & ~std::size_t(127));
    const int nsl = 1 << S.slot_shift;  // ring slots per warp
    const int slot_shift = S.slot_shift;
    unsigned char* my_ring = ring + static_cast<std::size_t>(warp) * nsl * unit;
    std::uint64_t* my_bars = bars + warp * kMaxWarpSlots;

    const int n_phases = pdr.n_phases;
    const int ubase = pdr.warp_base[warp];
    const int nunits = pdr.warp_base[warp + 1] - ubase;
    const int* units = S.units + 2 * (pdr.units + ubase);  // {offset16, bytes} pairs
    const std::int32_t* gtable = S.phases + pdr.phases;
    const unsigned char* src = reinterpret_cast<const unsigned char*>(S.stream + pdr.stream);

    if (lane < nsl) mbar_init(&my_bars[lane], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();

    // per-warp registers: unit offsets / bytes, the end unit and kind of each phase
    RegTable uoff, ubytes, uend, pkind;
#pragma unroll
    for (int q = 0; q < (kRegTables ? kMaxRegEntries / 32 : 0); ++q) {
        const int i = q * 32 + lane;
        int2 e = make_int2(0, 0);
        if (i < nunits) e = __ldg(reinterpret_cast<const int2*>(units) + i);
        uoff.v[q] = e.x;
        ubytes.v[q] = e.y;
        uend.v[q] = i < n_phases ? __ldg(gtable + i * kPhaseStride + kSolveWarps + warp) : 0;
        pkind.v[q] = i < n_phases ? __ldg(gtable + i * kPhaseStride + 2 * kSolveWarps) : 0;
    }
    auto issue = [&](int u, int o16, int nb) {  // lane 0 issues unit u into its slot
        if (lane == 0) {
            const int s = u & (nsl - 1);
            mbar_expect_tx(&my_bars[s], static_cast<std::uint32_t>(nb));
            bulk_g2s(my_ring + s * unit, src + static_cast<std::int64_t>(o16) * 16, static_cast<std::uint32_t>(nb),
                     &my_bars[s]);
        }
    };
    auto fetch = [&](int u) {  // whole warp calls (the table lookups are warp shuffles)
        const int o16 = uoff.get(u, units, 2);
        const int nb = ubytes.get(u, units + 1, 2);
        issue(u, o16, nb);
    };
    for (int u = 0; u < nsl && u < nunits; ++u) fetch(u);
    // the table entry of the next refill (unit nsl, then one ahead of each refill): looked up a
    // unit early so the lookup's latency is off the refill's path
    int nx_o16 = 0, nx_nb = 0;
    if (nsl < nunits) {
        nx_o16 = uoff.get(nsl, units, 2);
        nx_nb = ubytes.get(nsl, units + 1, 2);
    }
    // everything above reads only the program (immutable): it overlaps the predecessor's tail
    // under programmatic dependent launch; from here on the inputs are the predecessors'
    pdl_wait();
    if (STATS && blockIdx.x == 0 && tid == 0) mkp[4] = clock64() - t_entry;  // predecessor done
    if (skip_launch(S.skip)) {  // uniform over the cluster: every CTA reads the same flag
        for (int u = 0; u < nsl && u < nunits; ++u) mbar_wait(&my_bars[u], 0);  // drain the prefetch
        return;
    }

    // ---- right-hand side (and, in MODE 1/2, the interface coupling)
    const std::int32_t* gmap = S.gmap + pdr.gmap;
    const int n_loc = pdr.n_loc, n_top = pdr.n_top;
    // rhs gather: four independent index/value loads in flight per thread
    constexpr int kInRows = MODE == 3 ? 4 : 12;  // rows per thread per round (MODE 3: no gather)
    for (int l0 = tid; l0 < ldn_p; l0 += kInRows * kThreads) {
        int gi[kInRows];
#pragma unroll
        for (int q = 0; q < kInRows; ++q) {
            const int l = l0 + q * kThreads;
            gi[q] = MODE != 3 && l < n_loc ? __ldg(gmap + l) : -1;
        }
        double gv[kInRows];
#pragma unroll
        for (int q = 0; q < kInRows; ++q) gv[q] = (MODE != 3 && gi[q] >= 0) ? S.in[gi[q]] : 0.0;
#pragma unroll
        for (int q = 0; q < kInRows; ++q) {
            const int l = l0 + q * kThreads;
            if (l < ldn_p) {
                T[l] = gv[q];
                X[l] = 0.0;  // padded columns of a tile read finite zeros
            }
        }
    }
    for (int l = tid; l < n_top; l += kThreads) Q[l] = 0.0;
    if (MODE == 3 && S.y_in)  // y0 is read at the forward/backward switch: bring it into L2 now
        for (int l = tid * 16; l < n_loc; l += kThreads * 16)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(S.y_in + pdr.gmap + l));
    if (MODE != 0) {
        const SubdomainDesc& sd = S.subs[pdr.sub];
        const int ng = sd.n_iface;
        for (int g = tid; g < ng; g += kThreads) {
            double z;
            if (MODE == 1 || MODE == 3) {
                // z_G = sum over the subdomains sharing the dof of their h, ascending
                // subdomain (reference prolong_add order, preconditioner.cpp:168-169,189-190)
                z = 0.0;
                const bool ll = MODE == 3 && S.ll_h;  // peers' h_i from the LL buffer (multi-GPU, fused)
                const std::uint32_t tag = ll ? ll_tag(S.seq_h) : 0u;
                // the writer's output slot and r entry, loaded alongside the owners' h (independent)
                const int dof = pdr.rank == 0 ? S.iface_writer[sd.iface + g] : -1;  // written dof or -1
                const bool writes = dof >= 0;
                const double rdot = MODE == 3 && writes && S.dot_part && dof < S.n_dot ? S.dot_r[dof] : 0.0;
                // the slot's owners (<= 4): their h slots in one 16-byte load, no owner-list walk
                const int4 o4 = __ldg(reinterpret_cast<const int4*>(S.iface_own4) + sd.iface + g);
                int o0 = 0, o1 = 0;
                if (o4.x <= -2) {  // more than four owners: the owner list of global dof -2 - x
                    o0 = S.gi_own_ptr[-2 - o4.x];
                    o1 = S.gi_own_ptr[-1 - o4.x];
                } else {
                    const int ref[4] = {o4.x, o4.y, o4.z, o4.w};
                    double h[4];
#pragma unroll
                    for (int t = 0; t < 4; ++t)
                        h[t] = ref[t] < 0 ? 0.0
                               : (ll && ref[t] >= S.ll_h_base)
                                   ? ll_get(S.ll_h + 2 * static_cast<std::int64_t>(ref[t] - S.ll_h_base), tag)
                                   : S.hbuf[ref[t]];
#pragma unroll
                    for (int t = 0; t < 4; ++t)
                        if (ref[t] >= 0) z += h[t];
                }
                for (int o = o0; o < o1; o += 4) {  // the owners' loads of a round back to back
                    int ref[4];
                    double h[4];
#pragma unroll
                    for (int t = 0; t < 4; ++t) ref[t] = o + t < o1 ? S.gi_own_ref[o + t] : -1;
#pragma unroll
                    for (int t = 0; t < 4; ++t)
                        h[t] = ref[t] < 0 ? 0.0
                               : (ll && ref[t] >= S.ll_h_base)
                                   ? ll_get(S.ll_h + 2 * static_cast<std::int64_t>(ref[t] - S.ll_h_base), tag)
                                   : S.hbuf[ref[t]];
#pragma unroll
                    for (int t = 0; t < 4; ++t)
                        if (ref[t] >= 0) z += h[t];
                }
                if (writes) {
                    S.out[dof] = z;
                    if (MODE == 3 && S.dot_part && dof < S.n_dot) rz += rdot * z;
                }
            } else {
                z = S.hbuf[sd.hbuf + g];
            }
            ZG[g] = z;
        }
        __syncthreads();
        // coupled rows only ({row, end} pairs); the other rows keep T (MODE 3: zero)
        const int2* cp = reinterpret_cast<const int2*>(S.couple_ptr + pdr.couple_ptr);
        for (int i = tid; i < pdr.n_coupled; i += kThreads) {
            const int2 re = __ldg(cp + i);
            double acc = 0.0;
            for (int e = i ? __ldg(&cp[i - 1].y) : 0; e < re.y; ++e)
                acc += S.couple_val[pdr.couple_ent + e] * ZG[S.couple_gamma[pdr.couple_ent + e]];
            if (MODE == 3) T[re.x] = acc;  // harmonic extension: rhs A_IG z_G
            else T[re.x] -= acc;
        }
    }
    __syncthreads();

    constexpr bool stats = STATS;
    long long t_start = stats ? clock64() : 0, t_wait = 0, t_bar = 0, t_refill = 0, t_tiles = 0, n_tiles = 0;
    if (stats && blockIdx.x == 0 && tid == 0) mkp[5] = t_start - t_entry;  // prologue (incl. the wait for the predecessor)
    long long tprof[4] = {0, 0, 0, 0};  // STATS: decode, loop, reduction, flush cycles
    double acc = 0.0;
    int u = 0;                // this warp's current unit (ring slot u & (nsl - 1))
    int done = 0;             // steps processed (the phase table holds cumulative step counts)
    bool fresh = true;        // unit u not yet waited on
    std::uint32_t cur = 0;    // offset (16 B) of the next step in unit u
    const unsigned char* ubuf = my_ring;
    int4 hdr4 = make_int4(0, 0, 0, 0);  // the lane's sub-header of the next step
    bool split_done = !(MODE == 0 ? S.y_out : (MODE == 3 ? S.y_in : nullptr));
    // phase kind and end step count, looked up a phase ahead
    int nx_kind = pkind.get(0, gtable + 2 * kSolveWarps, kPhaseStride);
    int nx_end = uend.get(0, gtable + kSolveWarps + warp, kPhaseStride);
    for (int ph = 0; ph < n_phases; ++ph) {
        const int kind = nx_kind;
        const int s_end = nx_end;
        if (ph + 1 < n_phases) {
            nx_kind = pkind.get(ph + 1, gtable + 2 * kSolveWarps, kPhaseStride);
            nx_end = uend.get(ph + 1, gtable + kSolveWarps + warp, kPhaseStride);
        }
        if (!split_done && (kind & kPhaseBackward)) {  // forward sweep complete: X = y (block-uniform)
            split_done = true;
            if (MODE == 0) {
                for (int l = tid; l < n_loc; l += kThreads) S.y_out[pdr.gmap + l] = X[l];
            } else {
                // X = y0 - X: eight y0 loads in flight per thread (a dependent chain of global
                // loads here cost ~24k cycles per launch, ~10% of the harmonic solve)
                const double* y0 = S.y_in + pdr.gmap;
                for (int l0 = tid; l0 < n_loc; l0 += 8 * kThreads) {
                    double yv[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int l = l0 + q * kThreads;
                        yv[q] = l < n_loc ? __ldg(y0 + l) : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int l = l0 + q * kThreads;
                        if (l < n_loc) X[l] = yv[q] - X[l];
                    }
                }
                __syncthreads();
            }
            if (stats && blockIdx.x == 0 && tid == 0)
                S.stats[static_cast<long long>(gridDim.x) * kSolveWarps * 8 + 256 + 2 * 256 * kSolveWarps + 3] =
                    clock64() - t_start;
        }
        double* own = (kind & kPhaseBackward) ? X : T;
        double* other = (kind & kPhaseBackward) ? T : X;
        const long long t_ph0 = stats ? clock64() : 0;
        const long long n_tiles0 = n_tiles, t_wait0 = t_wait, t_tiles0 = t_tiles, t_refill0 = t_refill;
        // this phase's steps: the warp's step stream runs on across phases and units (a unit
        // is waited on at its first step and refilled after its last)
        while (done < s_end) {
            if (fresh) {
                const int s = u & (nsl - 1);
                if constexpr (stats) {
                    const long long t0 = clock64();
                    mbar_wait(&my_bars[s], (u >> slot_shift) & 1);
                    t_wait += clock64() - t0;
                } else {
                    mbar_wait(&my_bars[s], (u >> slot_shift) & 1);
                }
                ubuf = my_ring + s * unit;
                cur = 0;
                // the unit's first step: every lane reads sub-header A; in a group step the
                // lanes of the other sub-tiles then read their own
                hdr4 = *reinterpret_cast<const int4*>(ubuf);
                const int nl0 = static_cast<unsigned>(hdr4.x) >> 30;
                if (nl0) hdr4 = *reinterpret_cast<const int4*>(ubuf + 16 * (lane >> (5 - nl0)));
                fresh = false;
            }
            const long long t_tile0 = stats ? clock64() : 0;
            if (stats) ++n_tiles;
            const int4 h = hdr4;
            const unsigned w0 = h.x;
            const int nsub_lg = w0 >> 30;  // sub-tiles: 1, 2 or 4, on 32 >> nsub_lg lanes each
            const int tile_off = static_cast<int>(cur << 4) + (16 << nsub_lg);
            const unsigned char* tile = ubuf + tile_off;
            cur = w0 & 0x1ff;
            if (cur != kNoStep)  // the lane's sub-header of the next step, early
                hdr4 = *reinterpret_cast<const int4*>(ubuf + (cur << 4) + 16 * (lane >> (5 - ((w0 >> 28) & 3))));
            SOLVE_CHECK(tile_off <= unit && (cur == kNoStep || static_cast<int>(cur << 4) < unit), 9);
            long long tp_before[4];
            if constexpr (STATS)
                for (int i = 0; i < 4; ++i) tp_before[i] = tprof[i];
            tile_task<STATS>(h, tile, lane & ((32 >> nsub_lg) - 1), own, other, Q, acc,
                             TileBounds{ldn_p, n_top, unit - tile_off}, tprof);
            if constexpr (STATS) {  // CTA 0, warp 0: its first 512 steps {phase, k|lg|iters, 4 sub-phase cycles}
                if (blockIdx.x == 0 && warp == 0 && lane == 0 && done < 512) {
                    long long* so = S.stats + static_cast<long long>(gridDim.x) * kSolveWarps * 8 + 256 +
                                    5 * 256 * kSolveWarps + 8 + 4 * kSolveWarps + done * 6;
                    so[0] = ph;
                    so[1] = static_cast<long long>(h.z);
                    for (int i = 0; i < 4; ++i) so[2 + i] = tprof[i] - tp_before[i];
                }
            }
            if ((kind & kPhaseChained) && ((h.z >> 9) & kTaskLast))
                __syncwarp();  // a later tile of this warp's job reads what was just written
            ++done;
            if (stats) t_tiles += clock64() - t_tile0;
            if (cur == kNoStep) {
                // unit u consumed: refill its slot with the unit nsl ahead
                const long long t_r0 = stats ? clock64() : 0;
                if (u + nsl < nunits) {
                    // every lane's reads of the slot have completed (their values fed this
                    // unit's flushes), so the bulk copy may overwrite it; a generic-read ->
                    // async-write (WAR) reuse needs no proxy fence (measured: -1.5% per launch)
                    __syncwarp();
                    issue(u + nsl, nx_o16, nx_nb);
                    if (u + nsl + 1 < nunits) {
                        nx_o16 = uoff.get(u + nsl + 1, units, 2);
                        nx_nb = ubytes.get(u + nsl + 1, units + 1, 2);
                    }
                }
                ++u;
                fresh = true;
                if (stats) t_refill += clock64() - t_r0;
            }
        }
        if constexpr (stats) {
            const long long t0 = clock64();
            if (blockIdx.x == 0 && lane == 0 && ph < 256) {  // CTA 0: per (phase, warp) busy cycles and tiles
                long long* pw = S.stats + static_cast<long long>(gridDim.x) * kSolveWarps * 8 + 256;
                pw[ph * kSolveWarps + warp] = t0 - t_ph0;
                pw[256 * kSolveWarps + ph * kSolveWarps + warp] = n_tiles - n_tiles0;
                pw[2 * 256 * kSolveWarps + 8 + ph * kSolveWarps + warp] = t_wait - t_wait0;  // mbarrier waits
                pw[3 * 256 * kSolveWarps + 8 + ph * kSolveWarps + warp] = t_tiles - t_tiles0;  // tile processing
                pw[4 * 256 * kSolveWarps + 8 + ph * kSolveWarps + warp] = t_refill - t_refill0;  // refills
            }
            __syncthreads();
            t_bar += clock64() - t0;
            if (blockIdx.x == 0 && tid == 0)  // phase timeline of CTA 0
                S.stats[static_cast<long long>(gridDim.x) * kSolveWarps * 8 + ph] = clock64() - t_start;
        } else {
            __syncthreads();
        }
        if (CLUSTER > 1 && (kind & kPhaseCombine)) {
            long long* mk = S.stats + static_cast<long long>(gridDim.x) * kSolveWarps * 8 + 256 + 2 * 256 * kSolveWarps;
            if (stats && blockIdx.x == 0 && tid == 0) mk[0] = clock64() - t_start;
            cluster_sync_all();
            if (stats && blockIdx.x == 0 && tid == 0) mk[1] = clock64() - t_start;
            // t_top = ((t - Q_rank0) - Q_rank1) - ... : identical arithmetic in every CTA
            const int cb = __ldg(gtable + ph * kPhaseStride + 2 * kSolveWarps + 1);
            const int ce = __ldg(gtable + ph * kPhaseStride + 2 * kSolveWarps + 2);
            for (int l = cb + tid; l < ce; l += kThreads) {
                const int qi = l - pdr.n_group;
                double q[CLUSTER];
#pragma unroll
                for (int r = 0; r < CLUSTER; ++r) q[r] = pdr.rank == r ? Q[qi] : ld_dsmem(&Q[qi], r);
                double t = T[l];
#pragma unroll
                for (int r = 0; r < CLUSTER; ++r) t -= q[r];
                T[l] = t;
            }
            __syncthreads();
            if (stats && blockIdx.x == 0 && tid == 0) mk[2] = clock64() - t_start;
        }
    }

    if (stats && blockIdx.x == 0 && tid == 0) mkp[6] = clock64() - t_entry;  // phase loop done
    if (stats && lane == 0) {
        long long* o = S.stats + (static_cast<long long>(blockIdx.x) * kSolveWarps + warp) * 8;
        o[0] = clock64() - t_start;
        o[1] = t_wait;
        o[2] = t_bar;
        o[3] = nunits;
        o[4] = t_refill;
        o[5] = t_tiles;
        o[6] = n_tiles;
        if (STATS && blockIdx.x == 0) {  // CTA 0: tile sub-phases (decode, loop, reduction, flush)
            long long* tpo = S.stats + static_cast<long long>(gridDim.x) * kSolveWarps * 8 + 256 + 5 * 256 * kSolveWarps + 8;
            for (int i = 0; i < 4; ++i) tpo[warp * 4 + i] = tprof[i];
        }
    }
    // output: twelve rows per thread per round, all their index loads, then all their r loads,
    // in flight together (two dependent global levels per round; r.z keeps its row order)
    constexpr int kOutRows = 12;
    for (int l0 = tid; l0 < pdr.n_write; l0 += kOutRows * kThreads) {
        int gi[kOutRows];
#pragma unroll
        for (int q = 0; q < kOutRows; ++q) {
            const int l = l0 + q * kThreads;
            gi[q] = l < pdr.n_write ? __ldg(gmap + l) : -1;
        }
        double dr[kOutRows];
#pragma unroll
        for (int q = 0; q < kOutRows; ++q)
            dr[q] = MODE == 3 && S.dot_part && gi[q] >= 0 && gi[q] < S.n_dot ? S.dot_r[gi[q]] : 0.0;
#pragma unroll
        for (int q = 0; q < kOutRows; ++q)
            if (gi[q] >= 0) {
                if (MODE == 3) {
                    // z_I = u0 - extension, or (split apply) the backward sweep's result itself
                    const double z = S.y_in ? T[l0 + q * kThreads] : S.u0[gi[q]] - T[l0 + q * kThreads];
                    S.out[gi[q]] = z;
                    if (S.dot_part && gi[q] < S.n_dot) rz += dr[q] * z;
                } else {
                    S.out[gi[q]] = T[l0 + q * kThreads];
                }
            }
    }
    if (MODE == 3 && S.dot_part) {  // r.z of the entries this CTA wrote (fused PCG dot product)
        __shared__ double red[kSolveWarps];
        rz = block_sum<kThreads>(rz, red);
        if (tid == 0) S.dot_part[blockIdx.x] = rz;
    }
    if (stats && blockIdx.x == 0 && tid == 0) mkp[7] = clock64() - t_entry;  // through the epilogue
    if (CLUSTER > 1) cluster_sync_all();  // keep our Q alive until the partner is done
    if (MODE == 0 || MODE == 3) publish<kThreads>(S.pub);  // after the cluster barrier: non-last CTAs return
}

template <int MODE, int CLUSTER>
void launch_one(const SolveParams& P, const SolveLaunch& L, cudaStream_t stream) {
    auto kern = P.stats ? interior_solve_kernel<MODE, CLUSTER, true> : interior_solve_kernel<MODE, CLUSTER, false>;
    BDDC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(L.n_parts);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = L.smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CLUSTER;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    BDDC_CUDA(cudaLaunchKernelEx(&cfg, kern, P));
}

}  // namespace

std::size_t interior_solve_smem(int max_loc, int max_top, int max_iface, int unit_bytes, int slots_per_warp) {
    return static_cast<std::size_t>(kSolveWarps) * kMaxWarpSlots * 8 +
           8 * (2 * static_cast<std::size_t>((max_loc + 64 + 1) & ~1) + ((max_top + 1) & ~1) +
                ((max_iface + 1) & ~1)) +
           33 * 32 + 128 + static_cast<std::size_t>(kSolveWarps) * slots_per_warp * unit_bytes +
           512;  // slack: lanes beyond a tile's k*G read (and discard) up to 32 values past it
}

int max_solve_smem(int device) {
    int max_smem = 0;
    BDDC_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    return max_smem;
}

void launch_interior_solve(SolveParams P, const SolveLaunch& L, int mode, cudaStream_t stream) {
    if (L.n_parts <= 0) return;
    P.unit_bytes = L.unit_bytes;
    P.slot_shift = L.slot_shift;
    if (L.cluster == 4) {
        if (mode == 0) launch_one<0, 4>(P, L, stream);
        else if (mode == 1) launch_one<1, 4>(P, L, stream);
        else if (mode == 2) launch_one<2, 4>(P, L, stream);
        else launch_one<3, 4>(P, L, stream);
    } else if (L.cluster == 2) {
        if (mode == 0) launch_one<0, 2>(P, L, stream);
        else if (mode == 1) launch_one<1, 2>(P, L, stream);
        else if (mode == 2) launch_one<2, 2>(P, L, stream);
        else launch_one<3, 2>(P, L, stream);
    } else {
        if (mode == 0) launch_one<0, 1>(P, L, stream);
        else if (mode == 1) launch_one<1, 1>(P, L, stream);
        else if (mode == 2) launch_one<2, 1>(P, L, stream);
        else launch_one<3, 1>(P, L, stream);
    }
    BDDC_LAUNCHED();
}

}  // namespace bddc_b200
