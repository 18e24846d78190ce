// Compiles one subdomain's supernodal factor into the streamed interior-solve
// program consumed by device/solve.cu (format: device_format.hpp).
#pragma once

#include <cstdint>
#include <vector>

#include "../device_format.hpp"
#include "factor.hpp"

namespace bddc_b200 {

// Template programs (GPU setup): tile values are not known on the host; each stream word
// carries a source code instead (srcmap): kSrcCopy = keep the template word (headers, index
// lists), kSrcZero = 0.0, i >= 0 = +D[i], i <= -3 = -D[-i - 3], D being the subdomain's values
// laid out by a ValueLayout (device/setup.cu fills the streams).
constexpr std::int32_t kSrcCopy = -1;
constexpr std::int32_t kSrcZero = -2;

struct ValueLayout {
    std::vector<std::int64_t> linv_off;  // per supernode: L_ss^{-1} (n_s x n_s row-major) in D
    std::vector<std::int64_t> bl_off;    // per supernode: BL_s = L_{R_s,s} L_ss^{-1} (interior rows x n_s)
    std::int64_t total = 0;
};

struct SolvePools {
    std::vector<double> stream;  // tile values (+ int32 index lists packed in place)
    std::vector<std::int32_t> units;  // per part, per warp: {offset16, bytes} pairs
    std::vector<std::int32_t> order;  // per part: producer order, int4 {offset16, bytes, warp|phase<<8, k}
    std::vector<std::int32_t> phases;
    std::vector<std::int32_t> gmap;
    std::vector<std::int32_t> couple_ptr, couple_gamma;
    std::vector<double> couple_val;
    std::vector<std::int32_t> srcmap;      // template mode: one code per stream word (see kSrcCopy)
    std::vector<std::int32_t> couple_src;  // template mode: local CSR value index of each coupling entry
    std::vector<PartDesc> parts;
    std::int64_t tile_values = 0;   // FP64 values in all tiles (incl. explicit zeros of diag tiles)
    std::int64_t fwd_factor_values = 0;  // factor values the forward sweep reads (all, unless pruned)
    std::int64_t bwd_factor_values = 0;  // factor values the backward sweep reads (all, unless pruned)
    std::int64_t n_tiles = 0;
    std::int32_t max_loc = 0, max_top = 0, max_phases = 0, max_units = 0;
    // GPU setup: the stream is not materialised on the host; stream_words is its length
    // (-1: the host stream is the stream)
    std::int64_t stream_words = -1;
    std::int64_t words() const { return stream_words >= 0 ? stream_words : static_cast<std::int64_t>(stream.size()); }
};

// Appends `src` (built from empty pools) to `dst`, rebasing the parts' offsets.
void append_pools(SolvePools& dst, SolvePools&& src);

// local_to_vec: local dof index (interior first) -> device vector index.
// parts: 1 (one CTA per subdomain) or 2 (CTA pair in a cluster); unit_bytes: size of the
// per-warp TMA units (and of each ring slot).
// prune_forward: the harmonic-extension program (rhs supported on the interior dofs coupled
// to the interface): forward tasks only for supernodes whose subtree holds such a dof.
// prune_backward: the apply's first solve (full forward, y0 kept): the backward sweep only for
// the supernodes that hold an interface-coupled dof or are ancestors of one — the same set —
// so u0 is exact on the dofs A_GI reads and unspecified elsewhere.
void build_solve_program(const InteriorFactor& F, const CsrMatrix& A_local,
                         const std::vector<index_t>& local_to_vec, int sub, int parts, int unit_bytes,
                         SolvePools& pools, bool prune_forward = false, bool prune_backward = false,
                         const ValueLayout* layout = nullptr);

}  // namespace bddc_b200
