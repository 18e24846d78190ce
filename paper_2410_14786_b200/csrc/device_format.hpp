// Layout contract between the host program builder (host/program.cpp) and the
// sm_100a kernels (device/*.cu). Plain structs only: no torch / STL types.
//
// Interior solve "program": each subdomain's supernodal L (nested dissection order)
// is compiled into two streams of column-major FP64 tiles — one for the forward
// sweep L x = b, one for the backward sweep L^T y = x — laid out in consumption
// order, plus per-warp task lists per phase. Every task is the same warp op:
//
//     acc[lane] += sum_j  M[(lane - lane_off) + j*nrows] * in[col(j)]
//
// with lanes mapped to output rows (no shuffles, coalesced tile-column loads), the
// accumulator kept in registers across consecutive tasks of one 32-row output chunk
// (FIRST/LAST flags), and each output chunk owned by exactly one warp per phase
// (deterministic, race-free; host balances chunks across warps).
//
// Phase kinds (two per elimination-tree height):
//   A (gather):  own[out]   -= acc   (forward: t -= L_{s,d} x_d ; backward: u = x - B^T y)
//   B (diag):    other[out]  = acc   (forward: x_s = L_ss^{-1} t_s ; backward: y_s = L_ss^{-T} u_s)
// Forward: own = T, other = X.  Backward: own = X, other = T.  Both in shared memory.
#pragma once

#include <cstdint>

namespace bddc_b200 {

constexpr int kSolveWarps = 16;  // warps per interior-solve CTA (one CTA per subdomain)

enum TaskFlags : std::uint8_t {
    kTaskInIndexed = 1,  // input column j read at position idx[in_ref + j], else in_ref + j
    kTaskFirst = 2,      // start a new accumulator
    kTaskLast = 4,       // flush the accumulator to the output chunk
    kTaskDiag = 8,       // phase-B store (other[out] = acc) instead of own[out] -= acc
};

struct TileTask {
    std::uint32_t m_off;    // tile offset (doubles) within the subdomain's pass stream
    std::uint32_t in_ref;   // contiguous input start position, or offset into the index list
    std::uint16_t out_base; // first row (position) of the 32-row output chunk
    std::uint16_t ncols;    // tile columns (input length)
    std::uint8_t nrows;     // tile rows (leading dimension), <= 32
    std::uint8_t lane_off;  // tile row i is lane i + lane_off
    std::uint8_t flags;
    std::uint8_t nvalid;    // valid lanes of the output chunk on flush
};
static_assert(sizeof(TileTask) == 16, "TileTask must stay 16 bytes");

// Per-subdomain descriptor for the interior solve and the interface steps.
struct SubdomainDesc {
    std::int64_t fwd_stream;   // offset (doubles) of the forward tile stream in the pool
    std::int64_t bwd_stream;   // offset (doubles) of the backward tile stream
    std::int64_t fwd_tasks;    // offset of the forward task list
    std::int64_t bwd_tasks;
    std::int32_t fwd_phases;   // offset into the phase table (kSolveWarps+1 entries per phase)
    std::int32_t bwd_phases;
    std::int32_t n_fwd_phases;
    std::int32_t n_bwd_phases;
    std::int64_t idx_base;     // offset of this subdomain's index lists
    std::int64_t gmap;         // offset: permuted interior position -> vector index
    std::int64_t couple_ptr;   // offset of coupling CSR row pointers (n_interior+1 entries)
    std::int64_t couple_ent;   // offset of coupling entries (gamma index, value)
    std::int64_t iface;        // offset: gamma -> vector index / weight / global iface id
    std::int64_t kmat;         // offset of K_i (n_iface x n_iface, row-major)
    std::int64_t phig;         // offset of Phi_G (n_iface x n_primal, row-major)
    std::int64_t phi;          // offset of the full Phi (n_local x n_primal, row-major)
    std::int64_t primal;       // offset into the primal map pool
    std::int64_t hbuf;         // offset of this subdomain's h / g scratch (n_iface)
    std::int64_t cbuf;         // offset of this subdomain's coarse contribution (n_primal)
    std::int64_t local_dofs;   // offset: local dof -> vector index (stage hooks)
    std::int32_t n_interior;
    std::int32_t n_iface;
    std::int32_t n_primal;
    std::int32_t n_local;
};

}  // namespace bddc_b200
