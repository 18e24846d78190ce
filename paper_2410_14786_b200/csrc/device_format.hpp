// Layout contract between the host program builder (host/solve_program.cpp,
// host/program.cpp) and the sm_100a kernels (device/*.cu). Plain structs only.
//
// Interior solve "program"
// ------------------------
// A subdomain's supernodal Cholesky factor L of A_II (nested-dissection order) is
// compiled into P "parts" (P = 1, or 2 = a CTA pair in one thread-block cluster:
// each CTA owns one half of the elimination tree; the separator chain above the split
// is processed redundantly by both after one exchange of partial sums through
// distributed shared memory). Each part is
//   * per warp, a sequence of "units" in HBM (<= unit_bytes each, whole tiles with their
//     16-byte headers, filled across phases); every warp prefetches its own units into a
//     private double-buffered shared-memory ring with cp.async.bulk (TMA bulk copies)
//     and its own mbarriers, so streaming never waits on other warps and continues
//     across the phase barriers;
//   * a phase table giving each warp's unit range per phase (phases are separated by
//     CTA barriers).
//
// Every task is one warp-level tile GEMV with a flattened lane mapping: a tile has k
// rows (k <= 32) and ncols columns; lane l = r*G + g < k*G (G = the largest power of two
// with k*G <= 32 column groups) owns row r and columns j = t*G + g for t = 0, 1, ...; the
// tile values are stored iteration-major, value(r, t*G + g) at [t*k*G + r*G + g], so each
// iteration is one contiguous, conflict-free shared-memory read. Partial sums are reduced
// inside each row's group of G lanes with an xor butterfly. Accumulators persist across
// consecutive tasks of the same output (FIRST/LAST flags).
//
// Task kinds (forward: own = T, other = X; backward: own = X, other = T):
//   DIAG : other[out_base + r]  = acc     x_s = L_ss^{-1} t_s     /  y_s = L_ss^{-T} u_s
//   PUSH : own[outidx[r]]      -= acc     t[R_d] -= L_{R_d,d} x_d (forward off-diagonal)
//          Q[outidx[r]]        += acc     (PARTIAL: this CTA's contribution into the top)
//   PULL : own[out_base + r]   -= acc     u_s = x_s - L_{R_s,s}^T y[R_s] (backward)
// A backward chunk is one indexed DIAG tile over [L_ss^{-T} | -BL_s^T]: its index list is
// relative to T (= other) and reaches y_s in X as part_ldn(n_loc) + j.
// Input column j is in[in_ref + j] (contiguous) or in[idx[j]] (IN_INDEXED).
// Pushes of one phase never share a target row (supernodes are coloured per height).
//
// Group steps (pairs and quads): two independent tiles A and B with k <= 16 rows each run side
// by side, A on lanes 0-15 and B on lanes 16-31 (lane - 16 = r*G_B + g), each with its own G
// (k*G <= 16); likewise four tiles of k <= 8 rows on the four 8-lane quarters (k*G <= 8),
// iteration count, input, flags and outputs, so a warp pays one header decode, one loop and
// one butterfly for both. Layout: sub-header A, sub-header B (step header below), values
// iteration-major with stride S = k_A*G_A + k_B*G_B (A's lanes then B's), for
// max(iters_A, iters_B) iterations (the shorter tile's slots are zero and never read), then
// A's and B's index lists (IN_INDEXED: both or neither; 16-byte aligned each), then A's and
// B's output-row lists (those that have one). Chunks of several pieces are paired piece by
// piece (both FIRST/LAST in lockstep).
#pragma once

#include <cstdint>

namespace bddc_b200 {

#ifndef BDDC_SOLVE_WARPS
#define BDDC_SOLVE_WARPS 16
#endif
constexpr int kSolveWarps = BDDC_SOLVE_WARPS;  // consumer warps per interior-solve CTA
constexpr int kMaxSlots = 64;            // max ring slots per CTA (shared slot pool)
constexpr int kPhaseStride = 2 * kSolveWarps + 3;

enum TaskFlags : std::uint8_t {
    kTaskInIndexed = 1,  // input column j at idx[j] (int32 list after the values)
    kTaskFirst = 2,      // start a new accumulator
    kTaskLast = 4,       // flush the accumulator
    kTaskDiag = 8,       // other[out_base + r] = acc
    kTaskPush = 16,      // own[outidx[r]] -= acc (outidx after the values / index list)
    kTaskPartial = 32,   // with PUSH: Q[outidx[r]] += acc
    kTaskInOwn = 64,     // inputs from own (else from other)
    kTaskPair = 128,     // a pair step: two half-warp tiles (layout below)
};

enum PhaseKind : std::int32_t {
    kPhaseNormal = 0,
    kPhaseCombine = 1,
    kPhaseBackward = 2,
    kPhaseChained = 4,  // a warp's later tiles read rows its earlier tiles wrote (subtree jobs)
};

// Builder-side description of one tile (host/solve_program.cpp); on the stream a tile is
// described by a packed step sub-header (below).
struct TileTask {
    std::uint32_t next;     // (builder: unused)
    std::uint32_t in_ref;   // first input local index (contiguous inputs)
    std::uint16_t out_base; // output chunk start (DIAG / PULL)
    std::uint16_t iters;    // ceil(columns / groups): inner-loop trip count
    std::uint8_t nrows;     // k, <= 32
    std::uint8_t groups;    // log2 G; G: the largest power of two with k * G <= 32
    std::uint8_t flags;
    std::uint8_t nvalid;    // rows written on flush
};
static_assert(sizeof(TileTask) == 16, "TileTask must stay 16 bytes");

// On-stream step header: one 16-byte sub-header per tile of the step (a single tile: one; a
// pair step: A, read by lanes 0-15, then B, read by lanes 16-31). Each sub-header holds
// everything its lanes need (the step-wide fields duplicated), and carries the next step's
// offset and pair flag, so a lane prefetches and decodes only its own 16 bytes:
//   w0: [0:9) next step (16-byte units from the unit start; kNoStep ends the unit),
//       [11:17) value stride S (values per iteration: k*G, or the sub-tiles' sum), [17:25)
//       value-section bytes / 16, [25:28) log2 of the step's largest G, [28:30) log2 of the
//       next step's sub-tile count, [30:32) log2 of this step's sub-tile count (1, 2 or 4: the
//       sub-tile of lane l is l / (32 >> that), its 16-byte sub-header at that index)
//   w1: [0:16) in_ref, [16:32) out_base
//   w2: [0:6) k, [6:9) log2 G, [9:17) flags, [17:26) iterations, [26:32) nvalid
//   w3: [0:5) the tile's first value lane within S, [5:13) its index list offset / 16 and
//       [13:21) its output-row list offset / 16, both from the tile data start
constexpr std::uint32_t kNoStep = 0x1ff;
struct StepFields {
    std::uint32_t next = kNoStep, next_nsub_lg = 0, nsub_lg = 0, S = 0, vq = 0, gmax_lg = 0;
    std::uint32_t in_ref = 0, out_base = 0;
    std::uint32_t k = 0, lg = 0, flags = 0, iters = 0, nvalid = 0;
    std::uint32_t voff = 0, ixq = 0, oq = 0;
};
inline void pack_step(const StepFields& f, std::uint32_t w[4]) {
    w[0] = (f.next & 0x1ff) | (f.S & 63) << 11 | (f.vq & 255) << 17 | (f.gmax_lg & 7) << 25 | (f.next_nsub_lg & 3) << 28 |
           (f.nsub_lg & 3) << 30;
    w[1] = (f.in_ref & 0xffff) | (f.out_base & 0xffff) << 16;
    w[2] = (f.k & 63) | (f.lg & 7) << 6 | (f.flags & 255) << 9 | (f.iters & 511) << 17 | (f.nvalid & 63) << 26;
    w[3] = (f.voff & 31) | (f.ixq & 255) << 5 | (f.oq & 255) << 13;
}
inline StepFields unpack_step(const std::uint32_t w[4]) {
    StepFields f;
    f.next = w[0] & 0x1ff;
    f.next_nsub_lg = (w[0] >> 28) & 3;
    f.nsub_lg = (w[0] >> 30) & 3;
    f.S = (w[0] >> 11) & 63;
    f.vq = (w[0] >> 17) & 255;
    f.gmax_lg = (w[0] >> 25) & 7;
    f.in_ref = w[1] & 0xffff;
    f.out_base = w[1] >> 16;
    f.k = w[2] & 63;
    f.lg = (w[2] >> 6) & 7;
    f.flags = (w[2] >> 9) & 255;
    f.iters = (w[2] >> 17) & 511;
    f.nvalid = w[2] >> 26;
    f.voff = w[3] & 31;
    f.ixq = (w[3] >> 5) & 255;
    f.oq = (w[3] >> 13) & 255;
    return f;
}

// Bytes of one tile in the stream (16-byte aligned sections).
inline constexpr int tile_iters(int ncols, int groups) { return (ncols + groups - 1) / groups; }
inline constexpr int tile_value_bytes(int nrows, int ncols, int groups) {
    return tile_iters(ncols, groups) * nrows * groups * 8;
}
inline constexpr int pad16i(int b) { return (b + 15) & ~15; }
// Shared-memory stride of a part's vectors: X = T + part_ldn(n_loc) (64 zero slack entries
// after the local rows), so one index list relative to T reaches both (merged backward tiles).
inline constexpr int part_ldn(int n_loc) { return (n_loc + 64 + 1) & ~1; }

// Phase table entry (kPhaseStride int32):
//   [0 .. W-1]      steps of each warp before this phase (cumulative)
//   [W .. 2W-1]     steps of each warp up to the end of this phase (a warp's steps fill its
//                   units in order across phases: a unit may hold several phases' steps)
//   [2W]            kind (PhaseKind bits)
//   [2W+1, 2W+2]    combine range of local rows [begin, end) (kPhaseCombine, runs after the phase)
// Unit list of a part: for warp w, entries [warp_base[w], warp_base[w+1]) of int2
// {offset in 16-byte units from the part stream start, bytes}. The producer streams the
// part's units in `order` (phase-major, warps interleaved by bytes): int4 entries
// {offset16, bytes, warp | phase << 8, index of the unit within its warp's list}.
struct PartDesc {
    std::int64_t stream;        // offset (doubles) of this part's stream in the pool
    std::int64_t stream_bytes;  // multiple of 16
    std::int64_t units;         // offset (int2 entries) of the part's unit list
    std::int32_t warp_base[kSolveWarps + 1];  // per-warp unit ranges within the part's list
    std::int64_t order;         // offset (int4 entries) of the producer's unit order
    std::int32_t n_units;
    std::int64_t gmap;          // local index -> vector index
    std::int64_t couple_ptr;    // coupled rows only: {local row, end of its entries} int2 pairs
    std::int64_t couple_ent;    // coupling entries (gamma, value)
    std::int32_t phases;        // offset (int32) into the phase pool
    std::int32_t n_phases;
    std::int32_t n_loc;         // local indices: group rows then top rows
    std::int32_t n_group;
    std::int32_t n_top;
    std::int32_t n_write;       // locals written on output (rank 0 also writes the top)
    std::int32_t sub;           // subdomain
    std::int32_t rank;          // 0 .. P-1 within the cluster
    std::int32_t n_coupled;     // local rows with interface coupling (A_IG entries)
};

// Per-subdomain descriptor for the interface steps and stage hooks.
struct SubdomainDesc {
    std::int64_t iface;        // offset: gamma -> vector index / weight / global iface id
    std::int64_t kmat;         // K_i (n_iface x n_iface, row-major)
    std::int64_t phig;         // Phi_G (n_iface x n_primal, row-major)
    std::int64_t phi;          // full Phi (n_local x n_primal, row-major)
    std::int64_t primal;       // primal map
    std::int64_t hbuf;         // h / g scratch (n_iface)
    std::int64_t cbuf;         // coarse contribution (n_primal)
    std::int64_t local_dofs;   // local dof -> vector index
    std::int64_t lrow_ptr;     // local A_GI rows (n_iface + 1) -> (vector index, value)
    std::int32_t n_interior;
    std::int32_t n_iface;
    std::int32_t n_primal;
    std::int32_t n_local;
};

}  // namespace bddc_b200
