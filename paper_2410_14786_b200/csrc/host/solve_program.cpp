#include "solve_program.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <unordered_map>

namespace bddc_b200 {
namespace {

inline std::int64_t pad16(std::int64_t b) { return (b + 15) & ~std::int64_t(15); }

// Subtree jobs per warp in the pruned sweeps (the harmonic program's forward, the head program's
// backward); 0 = level-synchronous like the full sweeps.
constexpr double kPrunedJobsPerWarp = 0.0;

struct Tile {
    TileTask t{};
    int jn = 0;                        // columns of this piece
    std::vector<double> vals;          // numeric mode (empty in template mode: the values are src codes)
    std::vector<std::int32_t> src;     // template mode: value sources (SolvePools::srcmap codes)
    std::vector<std::int32_t> idx;     // input index list (IN_INDEXED)
    std::vector<std::int32_t> outidx;  // output rows (PUSH, last piece)
    std::int64_t nvals() const { return static_cast<std::int64_t>(vals.empty() ? src.size() : vals.size()); }
    std::int64_t bytes() const {
        return pad16(nvals() * 8) + pad16(static_cast<std::int64_t>(idx.size()) * 4) +
               pad16(static_cast<std::int64_t>(outidx.size()) * 4);
    }
};

// One output unit (a 32-row chunk of a supernode, or a row chunk of a push), owned by
// one warp; its pieces accumulate in registers.
struct Chunk {
    std::vector<Tile> tiles;
    std::int64_t cost = 0;
};

struct Phase {
    std::vector<std::vector<Chunk>> jobs;  // each job: ordered chunks owned by one warp
    std::int32_t kind = kPhaseNormal;
    std::int32_t comb_begin = 0, comb_end = 0;
};

// Build the flattened-mapping pieces of one output unit.
// Value of tile entry (r, j) of a chunk: numeric `v` or, building a template, the code `src` of
// where the device fill takes it from (SolvePools::srcmap).
struct TileValue {
    double v;
    std::int32_t src;
};

template <typename Val, typename InIdx>
Chunk make_chunk(int unit_bytes, int k, int ncols, Val val, bool indexed, InIdx in_idx, int in_start, int out_base,
                 int nvalid, std::uint8_t flags, const std::vector<std::int32_t>* outidx, bool tmpl) {
    Chunk ch;
    if (k < 1 || k > 32 || ncols < 1) throw std::logic_error("solve program: bad tile shape");
    int G = 1;
    while (k * G * 2 <= 32) G *= 2;
    // iterations per piece so that header + values + index list + output rows fit a unit
    const int room = unit_bytes - 16 - 128 - 32;
    const int per_iter = 8 * k * G + (indexed ? 4 * G : 0);
    const int per = std::max(1, room / per_iter) * G;  // columns per piece (multiple of G)
    for (int j0 = 0; j0 < ncols; j0 += per) {
        const int jn = std::min(per, ncols - j0);
        const int iters = tile_iters(jn, G);
        Tile T;
        T.jn = jn;
        T.t.in_ref = indexed ? 0u : static_cast<std::uint32_t>(in_start + j0);
        T.t.out_base = static_cast<std::uint16_t>(out_base);
        T.t.iters = static_cast<std::uint16_t>(iters);
        T.t.nrows = static_cast<std::uint8_t>(k);
        T.t.groups = static_cast<std::uint8_t>(__builtin_ctz(static_cast<unsigned>(G)));  // log2 G
        T.t.nvalid = static_cast<std::uint8_t>(nvalid);
        T.t.flags = flags | (indexed ? kTaskInIndexed : 0) | (j0 == 0 ? kTaskFirst : 0) |
                    (j0 + jn >= ncols ? kTaskLast : 0);
        const std::size_t nv = static_cast<std::size_t>(iters) * k * G;
        if (tmpl) T.src.assign(nv, kSrcZero);
        else T.vals.assign(nv, 0.0);
        for (int t = 0; t < iters; ++t)
            for (int g = 0; g < G; ++g) {
                const int j = t * G + g;
                if (j >= jn) continue;
                for (int r = 0; r < k; ++r) {
                    const TileValue tv = val(r, j0 + j);
                    const std::size_t at = static_cast<std::size_t>(t) * k * G + r * G + g;
                    if (!tmpl) T.vals[at] = tv.v;
                    if (tmpl) T.src[at] = tv.src;
                }
            }
        if (indexed) {
            T.idx.resize(static_cast<std::size_t>(iters) * G);
            for (int j = 0; j < iters * G; ++j) T.idx[j] = in_idx(j0 + std::min(j, jn - 1));
        }
        if (outidx && (T.t.flags & kTaskLast)) T.outidx = *outidx;
        // per-tile overhead in iterations (LPT cost model; BDDC_TILE_COST overrides, experiments)
        static const int tile_cost = std::getenv("BDDC_TILE_COST") ? std::atoi(std::getenv("BDDC_TILE_COST")) : 16;
        ch.cost += iters + tile_cost + (indexed ? iters / 2 : 0);
        ch.tiles.push_back(std::move(T));
    }
    return ch;
}

// The tile re-laid out for G2 column groups (same rows, columns and index list; one half of a
// pair step uses k * G2 <= 16 lanes).
Tile regroup(const Tile& T, int G2) {
    const int k = T.t.nrows, G = 1 << T.t.groups, kG = k * G;
    Tile R;
    R.t = T.t;
    R.jn = T.jn;
    R.outidx = T.outidx;
    const int it2 = tile_iters(T.jn, G2);
    R.t.iters = static_cast<std::uint16_t>(it2);
    R.t.groups = static_cast<std::uint8_t>(__builtin_ctz(static_cast<unsigned>(G2)));
    const std::size_t nv = static_cast<std::size_t>(it2) * k * G2;
    if (!T.src.empty()) R.src.assign(nv, kSrcZero);
    if (!T.vals.empty()) R.vals.assign(nv, 0.0);
    for (int j = 0; j < T.jn; ++j)
        for (int r = 0; r < k; ++r) {
            const std::size_t o = static_cast<std::size_t>(j / G) * kG + r * G + j % G;
            const std::size_t n = static_cast<std::size_t>(j / G2) * k * G2 + r * G2 + j % G2;
            if (!T.vals.empty()) R.vals[n] = T.vals[o];
            if (!T.src.empty()) R.src[n] = T.src[o];
        }
    if (!T.idx.empty()) {
        R.idx.resize(static_cast<std::size_t>(it2) * G2);
        for (int j = 0; j < it2 * G2; ++j) R.idx[j] = T.idx[std::min(j, T.jn - 1)];
    }
    return R;
}

// G of a tile of k rows on a sub-tile of `lanes` lanes (k*G <= lanes)
int lane_groups(int k, int lanes) {
    int G = 1;
    while (k * G * 2 <= lanes) G *= 2;
    return G;
}

// Bytes of a pair step (device_format.hpp): two headers, the interleaved values (iteration
// stride kG_A + kG_B, max(iters) iterations), the two index lists, the two output-row lists.
// A tile's shape at G2 column groups (header, index and output-list lengths) without its values:
// the pairing decision is taken on shapes, only paired tiles are re-laid out (regroup).
struct Shape {
    TileTask t;
    std::int64_t nidx, nout;
};
Shape shape_of(const Tile& T, int G2) {
    Shape h{T.t, 0, static_cast<std::int64_t>(T.outidx.size())};
    const int it2 = tile_iters(T.jn, G2);
    h.t.iters = static_cast<std::uint16_t>(it2);
    h.t.groups = static_cast<std::uint8_t>(__builtin_ctz(static_cast<unsigned>(G2)));
    h.nidx = T.idx.empty() ? 0 : static_cast<std::int64_t>(it2) * G2;
    return h;
}

// bytes of a group step (device_format.hpp): the sub-headers, the interleaved values for the
// longest sub-tile's iterations, the index lists, the output-row lists
std::int64_t group_bytes(const std::vector<const Shape*>& g) {
    int im = 0;
    std::int64_t S = 0, lists = 0;
    for (const Shape* h : g) {
        im = std::max<int>(im, h->t.iters);
        S += h->t.nrows << h->t.groups;
        lists += pad16(h->nidx * 4) + pad16(h->nout * 4);
    }
    return 16 * static_cast<std::int64_t>(g.size()) + pad16(im * S * 8) + lists;
}

// A tile's own fields of its step sub-header (the step-wide ones are set at emission); the
// packed ranges are checked here.
StepFields step_fields(const TileTask& t) {
    if (t.iters > 511 || t.nrows > 32 || t.nvalid > 32 || t.in_ref > 0xffff)
        throw std::logic_error("solve program: tile outside the step header ranges");
    StepFields f;
    f.in_ref = t.in_ref;
    f.out_base = t.out_base;
    f.k = t.nrows;
    f.lg = t.groups;
    f.flags = t.flags;
    f.iters = t.iters;
    f.nvalid = t.nvalid;
    return f;
}

}  // namespace

void build_solve_program(const InteriorFactor& F, const CsrMatrix& A, const std::vector<index_t>& l2v, int sub,
                         int P, int unit_bytes, SolvePools& pools, bool prune_forward, bool prune_backward,
                         const ValueLayout* layout) {
    const auto& sn = F.snodes;
    const bool tmpl = layout != nullptr;
    const index_t nsn = static_cast<index_t>(sn.size());
    const index_t nI = F.n_interior;
    // Harmonic-extension program: the forward sweep of A_II^{-1} (A_IG z_G) only reaches the
    // supernodes whose subtree holds an interior dof coupled to the interface (the rhs is zero
    // elsewhere, and so is the forward solution); the backward sweep stays complete.
    std::vector<char> fwd(nsn, 1);
    if (prune_forward || prune_backward) {
        std::fill(fwd.begin(), fwd.end(), 0);
        for (index_t sidx = 0; sidx < nsn; ++sidx) {
            for (index_t c = sn[sidx].col_begin; c < sn[sidx].col_end && !fwd[sidx]; ++c) {
                const index_t v = F.perm[c];
                for (index_t q = A.row_offsets[v]; q < A.row_offsets[v + 1]; ++q)
                    if (A.col_indices[q] >= nI) { fwd[sidx] = 1; break; }
            }
        }
        for (index_t sidx = 0; sidx < nsn; ++sidx)  // postorder: children before parents
            if (fwd[sidx] && sn[sidx].parent >= 0) fwd[sn[sidx].parent] = 1;
    }
    // active = coupled to the interface or an ancestor of such a supernode (the supernodes the
    // pruned sweeps visit; computed for every program, it also steers the part split below)
    std::vector<char> active(nsn, 0);
    for (index_t sidx = 0; sidx < nsn; ++sidx)
        for (index_t c = sn[sidx].col_begin; c < sn[sidx].col_end && !active[sidx]; ++c) {
            const index_t v = F.perm[c];
            for (index_t q = A.row_offsets[v]; q < A.row_offsets[v + 1]; ++q)
                if (A.col_indices[q] >= nI) { active[sidx] = 1; break; }
        }
    for (index_t sidx = 0; sidx < nsn; ++sidx)
        if (active[sidx] && sn[sidx].parent >= 0) active[sn[sidx].parent] = 1;
    std::vector<char> bwdm(nsn, 1);
    if (prune_backward) bwdm = active;
    if (!prune_forward) std::fill(fwd.begin(), fwd.end(), 1);
    for (index_t sidx = 0; sidx < nsn; ++sidx) {
        const std::int64_t ns = sn[sidx].size();
        const std::int64_t v = ns * (ns + 1) / 2 + static_cast<std::int64_t>(sn[sidx].n_interior_rows) * ns;
        if (fwd[sidx]) pools.fwd_factor_values += v;
        if (bwdm[sidx]) pools.bwd_factor_values += v;
    }
    if (P != 1 && P != 2 && P != 4) throw std::invalid_argument("solve program: parts must be 1, 2 or 4");
    // step sub-headers address a unit in 16-byte units with 9-bit step and 8-bit section offsets
    if (unit_bytes < 256 || unit_bytes > 4096 || unit_bytes % 16)
        throw std::invalid_argument("solve program: unit bytes must be a multiple of 16 in [256, 4096]");

    // ---- tree and group assignment (P = 2: halves below the top separator chain)
    std::vector<std::vector<index_t>> children(nsn);
    std::vector<index_t> roots;
    for (index_t s = 0; s < nsn; ++s) {
        if (sn[s].parent >= 0) children[sn[s].parent].push_back(s);
        else roots.push_back(s);
    }
    std::vector<std::int64_t> weight(nsn, 0), aweight(nsn, 0);  // subtree values: all / active only
    for (index_t s = 0; s < nsn; ++s) {
        const std::int64_t ns = sn[s].size();
        const std::int64_t own = ns * (ns + 1) + 2 * ns * sn[s].n_interior_rows;
        weight[s] += own;
        aweight[s] += active[s] ? own : 0;
        if (sn[s].parent >= 0) {
            weight[sn[s].parent] += weight[s];
            aweight[sn[s].parent] += aweight[s];
        }
    }
    // parts: the heaviest subtree of the frontier is expanded into its children (it joins the
    // shared top, solved redundantly by every part after the partial sums are combined) until
    // the frontier holds at least P subtrees; those are dealt to the P parts by weight (LPT)
    std::vector<int> group(nsn, 0);
    if (P > 1) {
        auto expand = [&](int target, std::vector<index_t>& tops) {
            std::vector<index_t> frontier = roots;
            while (static_cast<int>(frontier.size()) < target) {
                auto heavy = std::max_element(frontier.begin(), frontier.end(), [&](index_t a, index_t b) {
                    return weight[a] != weight[b] ? weight[a] < weight[b] : a > b;
                });
                const index_t h = *heavy;
                if (children[h].empty()) break;  // too few subtrees: some parts stay empty
                frontier.erase(heavy);
                tops.push_back(h);
                for (index_t c : children[h]) frontier.push_back(c);
            }
            return frontier;
        };
        std::vector<index_t> tops;
        std::vector<index_t> split_children = expand(P, tops);
        std::sort(split_children.begin(), split_children.end(),
                  [&](index_t a, index_t b) { return weight[a] != weight[b] ? weight[a] > weight[b] : a < b; });
        std::vector<int> gsub(nsn, -2);
        std::vector<int> part_of(split_children.size(), 0);
        {
            std::vector<std::int64_t> load(P, 0);
            for (std::size_t i = 0; i < split_children.size(); ++i) {
                const int g = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
                load[g] += weight[split_children[i]];
                part_of[i] = g;
            }
        }
        // Two parts whose ACTIVE work (what the pruned sweeps visit) is badly unbalanced — a
        // subdomain touching the interface on one or two sides only, e.g. a corner — wait for each
        // other at the combine of every pruned launch. Split one level deeper instead (the two
        // separators above the quarters join the redundant top) and pair the quarters so that
        // both the full and the active work are balanced, when that is clearly better.
        auto imbalance = [&](const std::vector<index_t>& kids, const std::vector<int>& part, int np) {
            std::vector<double> w(np, 0.0), a(np, 0.0);
            for (std::size_t i = 0; i < kids.size(); ++i) {
                w[part[i]] += static_cast<double>(weight[kids[i]]);
                a[part[i]] += static_cast<double>(aweight[kids[i]]);
            }
            const double wt = std::accumulate(w.begin(), w.end(), 0.0), at = std::accumulate(a.begin(), a.end(), 0.0);
            return std::max(wt > 0 ? *std::max_element(w.begin(), w.end()) * np / wt : 1.0,
                            at > 0 ? *std::max_element(a.begin(), a.end()) * np / at : 1.0);
        };
        if (P == 2 && imbalance(split_children, part_of, 2) > 1.25) {
            std::vector<index_t> tops4;
            std::vector<index_t> kids4 = expand(4, tops4);
            if (kids4.size() == 4) {
                std::vector<int> best;
                double best_v = imbalance(split_children, part_of, 2);
                for (int mate = 1; mate < 4; ++mate) {  // quarter 0 with quarter `mate`
                    std::vector<int> pt(4, 1);
                    pt[0] = pt[mate] = 0;
                    const double v = imbalance(kids4, pt, 2);
                    if (v < best_v - 0.1) { best_v = v; best = pt; }
                }
                if (!best.empty()) {
                    split_children = kids4;
                    part_of = best;
                    tops = tops4;
                }
            }
        }
        for (std::size_t i = 0; i < split_children.size(); ++i) gsub[split_children[i]] = part_of[i];
        for (index_t t : tops) gsub[t] = -1;
        for (index_t s = nsn - 1; s >= 0; --s) {
            if (gsub[s] != -2) { group[s] = gsub[s]; continue; }
            const index_t p = sn[s].parent;
            if (p < 0 || group[p] < 0) throw std::logic_error("solve program: supernode without a group");
            group[s] = group[p];
        }
    }
    std::vector<index_t> top;
    for (index_t s = 0; s < nsn; ++s)
        if (group[s] < 0) top.push_back(s);
    std::vector<index_t> owner(nI, -1);
    for (index_t s = 0; s < nsn; ++s)
        for (index_t c = sn[s].col_begin; c < sn[s].col_end; ++c) owner[c] = s;
    // BL_s = L_{R_s,s} L_ss^{-1} (interior rows of R_s): the forward push t[R] -= L_{R,s} x_s
    // becomes t[R] -= BL_s t_s, so it reads the same t_s as the diagonal solve and shares its
    // phase; the backward sweep x_s = L_ss^{-T} y_s - BL_s^T x_R is one chunk with two pieces.
    std::vector<std::vector<double>> BL(nsn);
    for (index_t sidx = 0; sidx < nsn && !tmpl; ++sidx) {
        const Supernode& S = sn[sidx];
        const index_t ns = S.size(), mI = S.n_interior_rows;
        BL[sidx].assign(static_cast<std::size_t>(mI) * ns, 0.0);
        for (index_t a = 0; a < mI; ++a)
            for (index_t j = 0; j < ns; ++j) {
                double acc = 0.0;
                for (index_t k = j; k < ns; ++k)
                    acc += S.B[static_cast<std::size_t>(a) * ns + k] * S.Linv[static_cast<std::size_t>(k) * ns + j];
                BL[sidx][static_cast<std::size_t>(a) * ns + j] = acc;
            }
    }

    // tile values: L_ss^{-1} entries and BL entries (numeric), or their positions in the per-subdomain
    // value array of a ValueLayout (template: the device fills them, device/setup.cu)
    auto linv = [&](index_t s, index_t r, index_t c) -> TileValue {
        const std::int64_t ns = sn[s].size();
        if (tmpl) return {0.0, static_cast<std::int32_t>(layout->linv_off[s] + r * ns + c)};
        return {sn[s].Linv[static_cast<std::size_t>(r * ns + c)], 0};
    };
    auto bl = [&](index_t s, index_t a, index_t j, bool negate) -> TileValue {
        const std::int64_t ns = sn[s].size();
        if (tmpl) {
            const std::int32_t i = static_cast<std::int32_t>(layout->bl_off[s] + a * ns + j);
            return {0.0, negate ? -i - 3 : i};
        }
        const double v = BL[s][static_cast<std::size_t>(a * ns + j)];
        return {negate ? -v : v, 0};
    };
    const TileValue zero{0.0, kSrcZero};

    for (int part = 0; part < P; ++part) {
        // local index space: group positions ascending, then top positions ascending
        std::vector<std::int32_t> loc(nI, -1);
        std::vector<index_t> locpos;
        for (index_t p = 0; p < nI; ++p)
            if (group[owner[p]] == part) { loc[p] = static_cast<std::int32_t>(locpos.size()); locpos.push_back(p); }
        const std::int32_t n_group = static_cast<std::int32_t>(locpos.size());
        for (index_t p = 0; p < nI; ++p)
            if (group[owner[p]] < 0) { loc[p] = static_cast<std::int32_t>(locpos.size()); locpos.push_back(p); }
        const std::int32_t n_loc = static_cast<std::int32_t>(locpos.size());
        const std::int32_t n_top = n_loc - n_group;
        if (n_loc + 64 > 65535) throw std::runtime_error("subdomain interior too large for the solve kernel");

        auto in_group = [&](index_t s) { return group[s] == part; };

        using Chunks = std::vector<Chunk>;
        // output rows per chunk (= per warp job): 32 normally; levels with few chunks use 16
        // or 8 so that their work spreads over more of the 16 warps (set by chunk_rows_for)
        int kr = 32;
        auto diag_fwd = [&](index_t s, Chunks& out) {
            const Supernode& S = sn[s];
            const index_t ns = S.size();
            for (index_t r0 = 0; r0 < ns; r0 += kr) {
                const int nr = static_cast<int>(std::min<index_t>(kr, ns - r0));
                out.push_back(make_chunk(unit_bytes,
                    nr, static_cast<int>(r0 + nr),
                    [&](int r, int j) { return j <= r0 + r ? linv(s, r0 + r, j) : zero; },
                    false, [](int) { return 0; }, loc[S.col_begin], loc[S.col_begin + r0], nr,
                    static_cast<std::uint8_t>(kTaskDiag | kTaskInOwn), nullptr, tmpl));
            }
        };
        // backward chunk of rows q0.. of supernode s: one tile over [L_ss^{-T} y_s | -BL_s^T x_R]
        // (ns - q0 + mI columns), indexed relative to T (= other in the backward sweep): y_s
        // lives in X = T + part_ldn(n_loc), x_R in T; flush T[s rows] = acc
        const std::int32_t xoff = part_ldn(n_loc);
        auto bwd = [&](index_t s, Chunks& out) {
            const Supernode& S = sn[s];
            const index_t ns = S.size(), mI = S.n_interior_rows;
            for (index_t q0 = 0; q0 < ns; q0 += kr) {
                const int nq = static_cast<int>(std::min<index_t>(kr, ns - q0));
                const int na = static_cast<int>(ns - q0);
                out.push_back(make_chunk(unit_bytes,
                    nq, na + static_cast<int>(mI),
                    [&](int r, int j) {
                        if (j < na) return j >= r ? linv(s, q0 + j, q0 + r) : zero;
                        return bl(s, j - na, q0 + r, true);
                    },
                    true,
                    [&](int j) {
                        if (j < na) return xoff + loc[S.col_begin + q0 + j];
                        const std::int32_t l = loc[S.rows[j - na]];
                        if (l < 0) throw std::logic_error("solve program: ancestor row not local");
                        return l;
                    },
                    0, loc[S.col_begin + q0], nq, kTaskDiag, nullptr, tmpl));
            }
        };
        // t[R_d] -= L_{R_d,d} x_d restricted to the target rows accepted by `take`: rows in the
        // own group (or own top) go to own T, rows in the shared top from a group supernode
        // go to Q (partial).
        auto push_fwd = [&](index_t d, Chunks& out, bool from_top, auto take,
                            std::vector<std::vector<index_t>>* tgt = nullptr) {
            const Supernode& D = sn[d];
            const index_t nd = D.size(), mI = D.n_interior_rows;
            for (int pass = 0; pass < 2; ++pass) {
                const bool to_top = pass == 1;
                if (from_top && to_top) continue;
                std::vector<index_t> rows;  // indices a into R_d
                for (index_t a = 0; a < mI; ++a) {
                    if (!take(D.rows[a])) continue;
                    const std::int32_t l = loc[D.rows[a]];
                    if (l < 0) throw std::logic_error("solve program: push target not local");
                    const bool is_top = !from_top && l >= n_group;
                    if (is_top == to_top) rows.push_back(a);
                }
                for (std::size_t c0 = 0; c0 < rows.size(); c0 += static_cast<std::size_t>(kr)) {
                    const int k = static_cast<int>(std::min<std::size_t>(kr, rows.size() - c0));
                    std::vector<std::int32_t> outidx(k);
                    for (int r = 0; r < k; ++r) {
                        const std::int32_t l = loc[D.rows[rows[c0 + r]]];
                        outidx[r] = to_top ? l - n_group : l;
                    }
                    if (tgt) {
                        tgt->emplace_back();
                        for (int r = 0; r < k; ++r) tgt->back().push_back(D.rows[rows[c0 + r]]);
                    }
                    out.push_back(make_chunk(unit_bytes,
                        k, static_cast<int>(nd),
                        [&](int r, int j) { return bl(d, rows[c0 + r], j, false); }, false,
                        [](int) { return 0; }, loc[D.col_begin], 0, k,
                        static_cast<std::uint8_t>(kTaskPush | kTaskInOwn | (to_top ? kTaskPartial : 0)), &outidx,
                        tmpl));
                }
            }
        };
        auto all_rows = [](index_t) { return true; };
        // chunk rows for a level: the largest of 32/16/8 giving at least 2 chunks per warp
        // forward levels: pushes sharing target rows chained into one warp job (up to kMaxChain
        // chunks) instead of coloured into phases; BDDC_MAX_CHAIN=0: colouring only (experiments)
        static const std::size_t kMaxChain = std::getenv("BDDC_MAX_CHAIN") ? std::atoi(std::getenv("BDDC_MAX_CHAIN")) : 8;
        // BDDC_QUAD_TILES=0: no quads (pairs only); BDDC_PAIR_TILES=0: no group steps (experiments)
        static const bool quad_tiles = !std::getenv("BDDC_QUAD_TILES") || std::atoi(std::getenv("BDDC_QUAD_TILES")) != 0;
        // BDDC_PAIR_TILES=0: no pair steps (experiments)
        static const bool pair_tiles = !std::getenv("BDDC_PAIR_TILES") || std::atoi(std::getenv("BDDC_PAIR_TILES")) != 0;
        static const int min_kr = std::getenv("BDDC_MIN_CHUNK_ROWS") ? std::atoi(std::getenv("BDDC_MIN_CHUNK_ROWS")) : 8;
        auto chunk_rows_for = [&](const std::vector<index_t>& rows_per_node) {
            if (min_kr >= 32) return 32;
            for (int k : {32, 16, 8}) {
                if (k == 16 && min_kr >= 16) return 16;
                if (k == 8 && min_kr >= 8) return 8;
                std::int64_t chunks = 0;
                for (index_t r : rows_per_node) chunks += (r + k - 1) / k;
                if (chunks >= 2 * kSolveWarps) return k;
            }
            return 4;
        };
        auto singles = [](Chunks&& cs) {  // level-synchronous phase: every chunk is its own job
            Phase ph;
            for (Chunk& c : cs) {
                ph.jobs.emplace_back();
                ph.jobs.back().push_back(std::move(c));
            }
            return ph;
        };

        // ---- subtree-to-warp mapping: below the cut every warp solves whole subtrees ("jobs")
        // sequentially with no CTA barrier; only the levels above the cut are level-synchronous.
        // The forward and backward sweeps have their own cut: a pruned sweep (few supernodes per
        // level: the boundary band and its ancestors) can trade its level barriers for warp-local
        // chains, a full sweep keeps the levels (measured: the serial chains of full subtrees cost
        // more than the barriers they save)
        struct JobSet {
            std::vector<char> local;
            std::vector<std::vector<index_t>> job_nodes;  // postorder
            std::vector<index_t> job_of, heights;         // heights above the cut
        };
        auto make_jobs = [&](double jpw, bool by_active) {
            JobSet J;
            J.local.assign(nsn, 0);
            const std::vector<std::int64_t>& wt = by_active ? aweight : weight;
            std::vector<index_t> job_roots;
            std::int64_t total = 0;
            for (index_t s = 0; s < nsn; ++s)
                if (in_group(s) && (sn[s].parent < 0 || !in_group(sn[s].parent))) total += wt[s];
            const std::int64_t tau =
                jpw > 0 ? std::max<std::int64_t>(1, static_cast<std::int64_t>(total / (jpw * kSolveWarps))) : 0;
            for (index_t s = nsn - 1; s >= 0; --s) {  // parents before children
                if (!in_group(s)) continue;
                const index_t p = sn[s].parent;
                const bool parent_local = p >= 0 && in_group(p) && J.local[p];
                if (parent_local) { J.local[s] = 1; continue; }
                if (tau > 0 && wt[s] <= tau) { J.local[s] = 1; job_roots.push_back(s); }
            }
            std::sort(job_roots.begin(), job_roots.end());
            J.job_of.assign(nsn, -1);
            J.job_nodes.resize(job_roots.size());
            for (std::size_t j = 0; j < job_roots.size(); ++j) J.job_of[job_roots[j]] = static_cast<index_t>(j);
            for (index_t s = nsn - 1; s >= 0; --s)
                if (J.local[s] && J.job_of[s] < 0) J.job_of[s] = J.job_of[sn[s].parent];
            for (index_t s = 0; s < nsn; ++s)
                if (J.local[s]) J.job_nodes[J.job_of[s]].push_back(s);
            for (index_t s = 0; s < nsn; ++s)
                if (in_group(s) && !J.local[s]) J.heights.push_back(sn[s].height);
            std::sort(J.heights.begin(), J.heights.end());
            J.heights.erase(std::unique(J.heights.begin(), J.heights.end()), J.heights.end());
            return J;
        };
        // BDDC_JOBS_PER_WARP: subtree jobs in every sweep (experiments); BDDC_PRUNED_JOBS: jobs per
        // warp in the pruned sweeps only
        const char* jpw_env = std::getenv("BDDC_JOBS_PER_WARP");
        const char* pj_env = std::getenv("BDDC_PRUNED_JOBS");
        const double jpw_all = jpw_env ? std::atof(jpw_env) : 0.0;
        const double jpw_pruned = pj_env ? std::atof(pj_env) : kPrunedJobsPerWarp;
        const JobSet jf = make_jobs(prune_forward && jpw_all <= 0 ? jpw_pruned : jpw_all, prune_forward && jpw_all <= 0);
        const JobSet jb = make_jobs(prune_backward && jpw_all <= 0 ? jpw_pruned : jpw_all, prune_backward && jpw_all <= 0);

        // greedy colouring of jobs whose target-row sets intersect: each job takes the first
        // colour none of its target rows carries yet (per-row bit mask of used colours; beyond
        // 64 colours the remaining jobs get one colour each)
        std::vector<std::uint64_t> row_colours(nI, 0);
        auto colour = [&](const std::vector<std::vector<index_t>>& targets) {
            std::vector<std::vector<std::size_t>> classes;
            std::vector<index_t> touched;
            for (std::size_t j = 0; j < targets.size(); ++j) {
                if (targets[j].empty()) continue;
                std::uint64_t busy = 0;
                for (index_t r : targets[j]) busy |= row_colours[r];
                std::size_t c;
                if (~busy != 0) {
                    c = static_cast<std::size_t>(__builtin_ctzll(~busy));
                    for (index_t r : targets[j]) {
                        if (!row_colours[r]) touched.push_back(r);
                        row_colours[r] |= std::uint64_t(1) << c;
                    }
                } else {
                    c = std::max<std::size_t>(64, classes.size());
                }
                if (c >= classes.size()) classes.resize(c + 1);
                classes[c].push_back(j);
            }
            for (index_t r : touched) row_colours[r] = 0;
            std::vector<std::vector<std::size_t>> kept;
            for (auto& c : classes)
                if (!c.empty()) kept.push_back(std::move(c));
            return kept;
        };

        std::vector<Phase> phases;
        // ---------------- forward sweep
        {
            // (1) warp-local subtrees: diag + pushes inside the subtree, postorder
            Phase ph;
            ph.kind = kPhaseChained;
            for (std::size_t j = 0; j < jf.job_nodes.size(); ++j) {
                Chunks job;
                for (index_t s : jf.job_nodes[j]) {
                    if (!fwd[s]) continue;
                    diag_fwd(s, job);
                    push_fwd(s, job, false, [&](index_t r) { return jf.local[owner[r]] && jf.job_of[owner[r]] == (index_t)j; });
                }
                ph.jobs.push_back(std::move(job));
            }
            phases.push_back(std::move(ph));
            // (2) pushes leaving each subtree, jobs coloured by target rows
            std::vector<std::vector<index_t>> targets(jf.job_nodes.size());
            std::vector<Chunks> ext(jf.job_nodes.size());
            for (std::size_t j = 0; j < jf.job_nodes.size(); ++j) {
                auto outside = [&](index_t r) { return !(jf.local[owner[r]] && jf.job_of[owner[r]] == (index_t)j); };
                for (index_t s : jf.job_nodes[j]) {
                    if (!fwd[s]) continue;
                    push_fwd(s, ext[j], false, outside);
                    for (index_t a = 0; a < sn[s].n_interior_rows; ++a)
                        if (outside(sn[s].rows[a])) targets[j].push_back(sn[s].rows[a]);
                }
            }
            for (const auto& cls : colour(targets)) {
                Phase pe;
                for (std::size_t j : cls) pe.jobs.push_back(std::move(ext[j]));
                phases.push_back(std::move(pe));
            }
        }
        // (3) levels above the cut, level-synchronous
        for (index_t h : jf.heights) {
            Chunks b;
            std::vector<index_t> nodes, nrows, mrows;
            for (index_t s = 0; s < nsn; ++s)
                if (in_group(s) && !jf.local[s] && sn[s].height == h && fwd[s]) {
                    nodes.push_back(s);
                    nrows.push_back(sn[s].size());
                    mrows.push_back(sn[s].n_interior_rows);
                }
            kr = chunk_rows_for(nrows);
            for (index_t s : nodes) diag_fwd(s, b);
            Phase diag_phase = singles(std::move(b));
            kr = chunk_rows_for(mrows);
            // one job per 32-row output chunk: chunks of one supernode write disjoint rows and
            // spread over the warps; chunks of different supernodes are coloured by target rows
            std::vector<std::vector<index_t>> targets;
            std::vector<Chunks> pushes;
            for (index_t d : nodes) {
                Chunks cs;
                std::vector<std::vector<index_t>> tg;
                push_fwd(d, cs, false, all_rows, &tg);
                for (std::size_t c = 0; c < cs.size(); ++c) {
                    targets.push_back(std::move(tg[c]));
                    pushes.emplace_back();
                    pushes.back().push_back(std::move(cs[c]));
                }
            }
            // Pushes sharing target rows are chained into one warp job (their flushes ordered by
            // the warp) instead of coloured into separate phases, when no chain gets longer than
            // kMaxChain chunks: one phase per level instead of one per colour class (measured:
            // C2 -1% at 8; all levels of the pruned sweeps and most of the full sweeps qualify).
            if (kMaxChain > 0 && !pushes.empty()) {
                std::vector<std::size_t> parent(pushes.size());
                std::iota(parent.begin(), parent.end(), 0);
                auto find = [&](std::size_t x) {
                    while (parent[x] != x) x = parent[x] = parent[parent[x]];
                    return x;
                };
                std::unordered_map<index_t, std::size_t> row_job;
                for (std::size_t j = 0; j < targets.size(); ++j)
                    for (index_t r : targets[j]) {
                        auto [it, fresh] = row_job.emplace(r, j);
                        if (!fresh) parent[find(j)] = find(it->second);
                    }
                std::vector<std::vector<std::size_t>> comps(pushes.size());
                for (std::size_t j = 0; j < pushes.size(); ++j) comps[find(j)].push_back(j);
                std::size_t longest = 0;
                for (const auto& c : comps) longest = std::max(longest, c.size());
                if (longest <= kMaxChain) {
                    Phase pp = std::move(diag_phase);
                    for (const auto& c : comps) {
                        if (c.empty()) continue;
                        pp.jobs.emplace_back();
                        for (std::size_t j : c) pp.jobs.back().push_back(std::move(pushes[j][0]));
                        if (c.size() > 1) pp.kind = kPhaseChained;
                    }
                    phases.push_back(std::move(pp));
                    kr = 32;
                    continue;
                }
                // (a level with a longer chain keeps the colouring: chaining part of it only
                // lengthens the first phase, measured +2%)
            }
            // the diagonal solves read the same final t_s as the pushes (and write X): they
            // share the first colour class's phase
            bool first = true;
            for (const auto& cls : colour(targets)) {
                Phase pp;
                if (first) pp = std::move(diag_phase);
                for (std::size_t j : cls) pp.jobs.push_back(std::move(pushes[j]));
                phases.push_back(std::move(pp));
                first = false;
            }
            if (first) phases.push_back(std::move(diag_phase));
            kr = 32;
        }
        // ---------------- exchange the partial sums into the shared top (P > 1)
        if (P > 1) {
            Phase comb;
            comb.kind = kPhaseCombine;
            comb.comb_begin = n_group;
            comb.comb_end = n_loc;
            phases.push_back(std::move(comb));
        }
        // ---------------- forward sweep: shared top chain (identical in every part)
        for (index_t s : top) {
            if (!fwd[s]) continue;
            Chunks b, ps;
            kr = chunk_rows_for({sn[s].size()});
            diag_fwd(s, b);
            kr = chunk_rows_for({sn[s].n_interior_rows});
            push_fwd(s, ps, true, all_rows);
            kr = 32;
            for (Chunk& c : ps) b.push_back(std::move(c));  // diag and pushes read t_s: one phase
            phases.push_back(singles(std::move(b)));
        }
        // ---------------- backward sweep: top chain, levels above the cut, then subtrees
        for (auto it = top.rbegin(); it != top.rend(); ++it) {
            if (!bwdm[*it]) continue;
            Chunks b;
            kr = chunk_rows_for({sn[*it].size()});
            bwd(*it, b);
            kr = 32;
            Phase pb2 = singles(std::move(b));
            pb2.kind = kPhaseBackward;
            phases.push_back(std::move(pb2));
        }
        for (auto hit = jb.heights.rbegin(); hit != jb.heights.rend(); ++hit) {
            Chunks a, b;
            std::vector<index_t> nrows;
            for (index_t s = 0; s < nsn; ++s)
                if (in_group(s) && !jb.local[s] && sn[s].height == *hit && bwdm[s]) nrows.push_back(sn[s].size());
            kr = chunk_rows_for(nrows);
            for (index_t s = 0; s < nsn; ++s)
                if (in_group(s) && !jb.local[s] && sn[s].height == *hit && bwdm[s]) bwd(s, b);
            kr = 32;
            (void)a;
            Phase pb2 = singles(std::move(b));
            pb2.kind = kPhaseBackward;
            phases.push_back(std::move(pb2));
        }
        {
            Phase ph;
            ph.kind = kPhaseBackward | kPhaseChained;
            for (std::size_t j = 0; j < jb.job_nodes.size(); ++j) {
                Chunks job;
                for (auto it = jb.job_nodes[j].rbegin(); it != jb.job_nodes[j].rend(); ++it)
                    if (bwdm[*it]) bwd(*it, job);
                ph.jobs.push_back(std::move(job));
            }
            phases.push_back(std::move(ph));
        }
        {
            std::vector<Phase> kept;
            for (Phase& ph : phases)
                if (!ph.jobs.empty() || (ph.kind & kPhaseCombine)) kept.push_back(std::move(ph));
            phases.swap(kept);
        }

        // ---------------- emit: LPT warp assignment, then each warp's tiles of a phase are
        // packed into units of <= unit_bytes (whole tiles, headers linked within the unit)
        PartDesc pd{};
        pd.sub = sub;
        pd.rank = part;
        pd.n_loc = n_loc;
        pd.n_group = n_group;
        pd.n_top = n_top;
        pd.n_write = part == 0 ? n_loc : n_group;
        pd.stream = static_cast<std::int64_t>(pools.stream.size());
        pd.phases = static_cast<std::int32_t>(pools.phases.size());
        pd.n_phases = static_cast<std::int32_t>(phases.size());
        std::int64_t pos = 0;
        std::vector<std::int32_t> table(phases.size() * kPhaseStride, 0);
        std::vector<std::vector<std::int32_t>> wunits(kSolveWarps);  // per warp: {offset16, bytes} pairs
        std::vector<std::int32_t> porder;                             // producer order (int4 entries)
        // Each warp's steps fill its units in order ACROSS phases (a unit closes only when the
        // next step does not fit): a warp with one small tile per phase refills once per ~4 KB,
        // not once per phase. The phase table holds cumulative step counts per warp.
        struct Unit {
            std::vector<double> words;
            std::vector<std::int32_t> src;  // template mode: srcmap codes of the words
            std::int64_t used = 0, last_hdr = -1;
            int last_nsub_lg = 0;           // the previous step's sub-headers to link: 1 << this
            int opened = 0;                 // phase in which the unit was opened
        };
        std::vector<Unit> open_unit(kSolveWarps);
        std::vector<std::vector<Unit>> units_of(kSolveWarps);
        std::vector<std::int32_t> steps_of(kSolveWarps, 0);
        for (std::size_t pi = 0; pi < phases.size(); ++pi) {
            Phase& ph = phases[pi];
            std::vector<std::int64_t> jcost(ph.jobs.size(), 0);
            for (std::size_t j = 0; j < ph.jobs.size(); ++j)
                for (const Chunk& c : ph.jobs[j]) jcost[j] += c.cost;
            std::vector<index_t> order(ph.jobs.size());
            std::iota(order.begin(), order.end(), 0);
            std::stable_sort(order.begin(), order.end(), [&](index_t a, index_t b) { return jcost[a] > jcost[b]; });
            std::vector<std::int64_t> load(kSolveWarps, 0);
            std::vector<std::vector<index_t>> per_warp(kSolveWarps);
            for (index_t c : order) {
                const int w = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
                load[w] += jcost[c];
                per_warp[w].push_back(c);
            }
            std::int32_t* row = &table[pi * kPhaseStride];
            for (int w = 0; w < kSolveWarps; ++w) {
                std::sort(per_warp[w].begin(), per_warp[w].end());
                row[w] = steps_of[w];
                // this warp's chunks of the phase; outside chained phases (tiles independent),
                // chunks of <= 16 rows are paired piece by piece into half-warp pair steps
                std::vector<Chunk*> chs;
                std::vector<char> solo;  // the chunk is a job of its own (chained phases: pairable)
                for (index_t c : per_warp[w])
                    for (Chunk& ch : ph.jobs[c]) {
                        chs.push_back(&ch);
                        solo.push_back(ph.jobs[c].size() == 1);
                    }
                // groups: quads of chunks whose tiles have <= 8 rows (8-lane quarters), then pairs
                // of <= 16 rows (half-warps); the members of a group match piece by piece in count,
                // FIRST / LAST / indexed flags, and every group step fits a unit
                std::vector<int> grp(chs.size(), -1);              // group of a chunk
                std::vector<std::vector<int>> groups;              // member chunks
                std::vector<std::vector<std::vector<Shape>>> gshape;  // per group: per member: pieces
                if (pair_tiles) {
                    constexpr std::uint8_t kShape = kTaskInIndexed | kTaskFirst | kTaskLast;
                    for (int lanes : {8, 16}) {
                        if (lanes == 8 && !quad_tiles) continue;
                        const int n = 32 / lanes;
                        std::vector<int> cand;
                        std::vector<std::vector<Shape>> sh(chs.size());
                        for (std::size_t i = 0; i < chs.size(); ++i) {
                            if (grp[i] >= 0) continue;
                            bool ok = !chs[i]->tiles.empty() && (solo[i] || !(ph.kind & kPhaseChained));
                            for (const Tile& t : chs[i]->tiles) ok = ok && t.t.nrows <= lanes;
                            if (!ok) continue;
                            for (const Tile& t : chs[i]->tiles) sh[i].push_back(shape_of(t, lane_groups(t.t.nrows, lanes)));
                            cand.push_back(static_cast<int>(i));
                        }
                        auto same_shape = [&](int a, int b) {
                            if (sh[a].size() != sh[b].size()) return false;
                            for (std::size_t q = 0; q < sh[a].size(); ++q)
                                if ((sh[a][q].t.flags & kShape) != (sh[b][q].t.flags & kShape)) return false;
                            return true;
                        };
                        std::sort(cand.begin(), cand.end(), [&](int a, int b) {
                            if (sh[a].size() != sh[b].size()) return sh[a].size() < sh[b].size();
                            for (std::size_t q = 0; q < sh[a].size(); ++q)
                                if ((sh[a][q].t.flags & kShape) != (sh[b][q].t.flags & kShape))
                                    return (sh[a][q].t.flags & kShape) < (sh[b][q].t.flags & kShape);
                            for (std::size_t q = 0; q < sh[a].size(); ++q)
                                if (sh[a][q].t.iters != sh[b][q].t.iters) return sh[a][q].t.iters < sh[b][q].t.iters;
                            return a < b;
                        });
                        for (std::size_t q = 0; q + n <= cand.size();) {
                            bool ok = true;
                            for (int m = 1; ok && m < n; ++m) ok = same_shape(cand[q], cand[q + m]);
                            for (std::size_t p = 0; ok && p < sh[cand[q]].size(); ++p) {
                                std::vector<const Shape*> g;
                                for (int m = 0; m < n; ++m) g.push_back(&sh[cand[q + m]][p]);
                                ok = group_bytes(g) <= unit_bytes;
                            }
                            if (!ok) { ++q; continue; }
                            groups.emplace_back();
                            gshape.emplace_back();
                            for (int m = 0; m < n; ++m) {
                                grp[cand[q + m]] = static_cast<int>(groups.size()) - 1;
                                groups.back().push_back(cand[q + m]);
                                gshape.back().push_back(sh[cand[q + m]]);
                            }
                            q += n;
                        }
                    }
                }
                // a step of nb bytes in this warp's open unit: {bytes, srcmap codes of its words}
                auto place = [&](std::int64_t nb, int nsub_lg) {
                    if (nb > unit_bytes) throw std::logic_error("solve program: tile larger than a unit");
                    Unit& U = open_unit[w];
                    if (U.used > 0 && U.used + nb > unit_bytes) {
                        units_of[w].push_back(std::move(U));
                        U = Unit{};
                    }
                    if (U.used == 0) U.opened = static_cast<int>(pi);
                    const std::size_t need = static_cast<std::size_t>((U.used + nb + 7) / 8);
                    if (U.words.size() < need) U.words.resize(need, 0.0);
                    if (tmpl && U.src.size() < need) U.src.resize(need, kSrcCopy);
                    char* base = reinterpret_cast<char*>(U.words.data());
                    if (U.last_hdr >= 0)  // link: the previous step's sub-headers name this step
                        for (int h = 0; h < (1 << U.last_nsub_lg); ++h) {
                            std::uint32_t* w0 = reinterpret_cast<std::uint32_t*>(base + U.last_hdr + 16 * h);
                            *w0 = (*w0 & ~(0x1ffu | 3u << 28)) | static_cast<std::uint32_t>(U.used / 16) |
                                  static_cast<std::uint32_t>(nsub_lg) << 28;
                        }
                    U.last_hdr = U.used;
                    U.last_nsub_lg = nsub_lg;
                    char* dst = base + U.used;
                    std::int32_t* src = tmpl ? U.src.data() + U.used / 8 : nullptr;
                    U.used += nb;
                    ++steps_of[w];
                    return std::make_pair(dst, src);
                };
                for (std::size_t i = 0; i < chs.size(); ++i) {
                    if (grp[i] >= 0 && groups[grp[i]][0] != static_cast<int>(i)) continue;  // emitted with its group
                    if (grp[i] < 0) {
                        for (Tile& t : chs[i]->tiles) {
                            auto [dst, srcw] = place(16 + t.bytes(), 0);
                            const std::int64_t vb = pad16(t.nvals() * 8), ib = pad16(static_cast<std::int64_t>(t.idx.size()) * 4);
                            StepFields f = step_fields(t.t);
                            f.S = t.t.nrows << t.t.groups;
                            f.vq = static_cast<std::uint32_t>(vb / 16);
                            f.gmax_lg = t.t.groups;
                            f.ixq = static_cast<std::uint32_t>(vb / 16);
                            f.oq = static_cast<std::uint32_t>((vb + ib) / 16);
                            std::uint32_t hw[4];
                            pack_step(f, hw);
                            std::memcpy(dst, hw, 16);
                            std::memcpy(dst + 16, t.vals.data(), t.vals.size() * 8);
                            if (tmpl) std::copy(t.src.begin(), t.src.end(), srcw + 2);
                            std::int64_t off = 16 + pad16(t.nvals() * 8);
                            if (!t.idx.empty()) std::memcpy(dst + off, t.idx.data(), t.idx.size() * 4);
                            off += pad16(static_cast<std::int64_t>(t.idx.size()) * 4);
                            if (!t.outidx.empty()) std::memcpy(dst + off, t.outidx.data(), t.outidx.size() * 4);
                            pools.tile_values += t.nvals();
                            ++pools.n_tiles;
                        }
                        continue;
                    }
                    // a group step per piece: sub-tiles side by side on 32 / n lanes each
                    const std::vector<int>& members = groups[grp[i]];
                    const int n = static_cast<int>(members.size());
                    const int nsub_lg = n == 4 ? 2 : 1;
                    for (std::size_t p = 0; p < chs[i]->tiles.size(); ++p) {
                        std::vector<Tile> T;
                        std::vector<const Shape*> shp;
                        for (int m = 0; m < n; ++m) {
                            const Tile& src = chs[members[m]]->tiles[p];
                            T.push_back(regroup(src, lane_groups(src.t.nrows, 32 / n)));
                            shp.push_back(&gshape[grp[i]][m][p]);
                        }
                        auto [dst, srcw] = place(group_bytes(shp), nsub_lg);
                        int S = 0, im = 0;
                        std::uint32_t glmax = 0;
                        std::vector<int> kg(n), voff(n);
                        for (int m = 0; m < n; ++m) {
                            kg[m] = T[m].t.nrows << T[m].t.groups;
                            voff[m] = S;
                            S += kg[m];
                            im = std::max<int>(im, T[m].t.iters);
                            glmax = std::max<std::uint32_t>(glmax, T[m].t.groups);
                        }
                        const std::int64_t vb = pad16(static_cast<std::int64_t>(im) * S * 8);
                        std::int64_t off = vb;
                        std::vector<StepFields> f(n);
                        for (int m = 0; m < n; ++m) {  // index lists after the values
                            f[m] = step_fields(T[m].t);
                            f[m].ixq = static_cast<std::uint32_t>(off / 16);
                            off += pad16(static_cast<std::int64_t>(T[m].idx.size()) * 4);
                        }
                        for (int m = 0; m < n; ++m) {  // then the output-row lists
                            f[m].oq = static_cast<std::uint32_t>(off / 16);
                            off += pad16(static_cast<std::int64_t>(T[m].outidx.size()) * 4);
                        }
                        for (int m = 0; m < n; ++m) {
                            f[m].nsub_lg = static_cast<std::uint32_t>(nsub_lg);
                            f[m].S = static_cast<std::uint32_t>(S);
                            f[m].vq = static_cast<std::uint32_t>(vb / 16);
                            f[m].gmax_lg = glmax;
                            f[m].voff = static_cast<std::uint32_t>(voff[m]);
                            std::uint32_t hw[4];
                            pack_step(f[m], hw);
                            std::memcpy(dst + 16 * m, hw, 16);
                        }
                        char* tile = dst + 16 * n;
                        double* V = reinterpret_cast<double*>(tile);
                        const std::size_t w0 = static_cast<std::size_t>(2 * n);  // value words after the sub-headers
                        for (int m = 0; m < n; ++m)
                            for (int t = 0; t < im; ++t)
                                for (int l = 0; l < kg[m]; ++l) {
                                    const std::size_t at = static_cast<std::size_t>(t) * S + voff[m] + l;
                                    const bool in = t < T[m].t.iters;
                                    if (!tmpl) V[at] = in ? T[m].vals[static_cast<std::size_t>(t) * kg[m] + l] : 0.0;
                                    if (tmpl) srcw[w0 + at] = in ? T[m].src[static_cast<std::size_t>(t) * kg[m] + l] : kSrcZero;
                                }
                        for (int m = 0; m < n; ++m) {
                            if (!T[m].idx.empty()) std::memcpy(tile + 16 * f[m].ixq, T[m].idx.data(), T[m].idx.size() * 4);
                            if (!T[m].outidx.empty()) std::memcpy(tile + 16 * f[m].oq, T[m].outidx.data(), T[m].outidx.size() * 4);
                        }
                        pools.tile_values += static_cast<std::int64_t>(im) * S;
                        pools.n_tiles += n;
                    }
                }
                row[kSolveWarps + w] = steps_of[w];
            }
            row[2 * kSolveWarps] = ph.kind;
            row[2 * kSolveWarps + 1] = ph.comb_begin;
            row[2 * kSolveWarps + 2] = ph.comb_end;
        }
        // the units into the part's stream, warp after warp ({offset16, bytes} per unit; the
        // producer-order table lists them with the phase that opened them)
        for (int w = 0; w < kSolveWarps; ++w) {
            if (open_unit[w].used > 0) units_of[w].push_back(std::move(open_unit[w]));
            for (std::size_t k = 0; k < units_of[w].size(); ++k) {
                const Unit& U = units_of[w][k];
                const std::size_t w0 = static_cast<std::size_t>(pd.stream + pos / 8);
                const std::size_t nw = static_cast<std::size_t>(pad16(U.used) / 8);
                pools.stream.resize(w0 + nw, 0.0);
                std::copy(U.words.begin(), U.words.begin() + static_cast<std::ptrdiff_t>(std::min(nw, U.words.size())),
                          pools.stream.begin() + static_cast<std::ptrdiff_t>(w0));
                if (tmpl) {
                    pools.srcmap.resize(w0 + nw, kSrcCopy);
                    std::copy(U.src.begin(), U.src.begin() + static_cast<std::ptrdiff_t>(std::min(nw, U.src.size())),
                              pools.srcmap.begin() + static_cast<std::ptrdiff_t>(w0));
                }
                wunits[w].push_back(static_cast<std::int32_t>(pos / 16));
                wunits[w].push_back(static_cast<std::int32_t>(U.used));
                porder.insert(porder.end(), {static_cast<std::int32_t>(pos / 16), static_cast<std::int32_t>(U.used),
                                             w | (U.opened << 8), static_cast<std::int32_t>(k)});
                pos += pad16(U.used);
            }
        }
        const std::int64_t total = pad16(pos);
        pools.stream.resize(static_cast<std::size_t>(pd.stream + total / 8), 0.0);
        if (tmpl) pools.srcmap.resize(pools.stream.size(), kSrcCopy);
        pd.stream_bytes = total;
        if (total / 16 > (std::int64_t(1) << 31) - 1) throw std::runtime_error("solve program: part stream too large");
        pools.phases.insert(pools.phases.end(), table.begin(), table.end());
        pd.units = static_cast<std::int64_t>(pools.units.size() / 2);
        pd.order = static_cast<std::int64_t>(pools.order.size() / 4);
        pd.n_units = static_cast<std::int32_t>(porder.size() / 4);
        pools.order.insert(pools.order.end(), porder.begin(), porder.end());
        pd.warp_base[0] = 0;
        for (int w = 0; w < kSolveWarps; ++w) {
            pools.units.insert(pools.units.end(), wunits[w].begin(), wunits[w].end());
            pd.warp_base[w + 1] = pd.warp_base[w] + static_cast<std::int32_t>(wunits[w].size() / 2);
            pools.max_units = std::max<std::int32_t>(pools.max_units, static_cast<std::int32_t>(wunits[w].size() / 2));
        }

        pd.gmap = static_cast<std::int64_t>(pools.gmap.size());
        for (index_t l = 0; l < n_loc; ++l) pools.gmap.push_back(l2v[F.perm[locpos[l]]]);
        // interface coupling A_IG, only for the rows that have any (the boundary-adjacent
        // interior dofs): {row, end} pairs so the kernel's threads visit coupled rows only
        if (pools.couple_ptr.size() & 1) pools.couple_ptr.push_back(0);  // int2 alignment
        pd.couple_ptr = static_cast<std::int64_t>(pools.couple_ptr.size());
        pd.couple_ent = static_cast<std::int64_t>(pools.couple_gamma.size());
        pd.n_coupled = 0;
        std::int32_t cnt = 0;
        for (index_t l = 0; l < n_loc; ++l) {
            const index_t v = F.perm[locpos[l]];
            const std::int32_t c0 = cnt;
            for (index_t q = A.row_offsets[v]; q < A.row_offsets[v + 1]; ++q)
                if (A.col_indices[q] >= nI) {
                    pools.couple_gamma.push_back(A.col_indices[q] - nI);
                    pools.couple_val.push_back(tmpl ? 0.0 : A.values[q]);
                    if (tmpl) pools.couple_src.push_back(static_cast<std::int32_t>(q));
                    ++cnt;
                }
            if (cnt > c0) {
                pools.couple_ptr.push_back(static_cast<std::int32_t>(l));
                pools.couple_ptr.push_back(cnt);
                ++pd.n_coupled;
            }
        }
        pools.max_loc = std::max(pools.max_loc, n_loc);
        pools.max_top = std::max(pools.max_top, n_top);
        pools.max_phases = std::max(pools.max_phases, pd.n_phases);
        pools.parts.push_back(pd);
    }
}

void append_pools(SolvePools& dst, SolvePools&& src) {
    if (dst.couple_ptr.size() & 1) dst.couple_ptr.push_back(0);  // int2 alignment of the parts' pairs
    const std::int64_t stream = static_cast<std::int64_t>(dst.stream.size());
    const std::int64_t units = static_cast<std::int64_t>(dst.units.size() / 2);
    const std::int64_t order = static_cast<std::int64_t>(dst.order.size() / 4);
    const std::int32_t phases = static_cast<std::int32_t>(dst.phases.size());
    const std::int64_t gmap = static_cast<std::int64_t>(dst.gmap.size());
    const std::int64_t cptr = static_cast<std::int64_t>(dst.couple_ptr.size());
    const std::int64_t cent = static_cast<std::int64_t>(dst.couple_gamma.size());
    for (PartDesc pd : src.parts) {
        pd.stream += stream;
        pd.units += units;
        pd.order += order;
        pd.phases += phases;
        pd.gmap += gmap;
        pd.couple_ptr += cptr;
        pd.couple_ent += cent;
        dst.parts.push_back(pd);
    }
    auto cat = [](auto& a, auto& b) {
        a.insert(a.end(), b.begin(), b.end());
        b.clear();
        b.shrink_to_fit();
    };
    cat(dst.stream, src.stream);
    cat(dst.units, src.units);
    cat(dst.order, src.order);
    cat(dst.phases, src.phases);
    cat(dst.gmap, src.gmap);
    cat(dst.couple_ptr, src.couple_ptr);
    cat(dst.couple_gamma, src.couple_gamma);
    cat(dst.couple_val, src.couple_val);
    cat(dst.srcmap, src.srcmap);
    cat(dst.couple_src, src.couple_src);
    dst.tile_values += src.tile_values;
    dst.fwd_factor_values += src.fwd_factor_values;
    dst.bwd_factor_values += src.bwd_factor_values;
    dst.n_tiles += src.n_tiles;
    dst.max_loc = std::max(dst.max_loc, src.max_loc);
    dst.max_top = std::max(dst.max_top, src.max_top);
    dst.max_phases = std::max(dst.max_phases, src.max_phases);
    dst.max_units = std::max(dst.max_units, src.max_units);
}

}  // namespace bddc_b200
