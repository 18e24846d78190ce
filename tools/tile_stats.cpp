// Dev tool: histogram of the interior-solve program tiles of one C2 interior subdomain
// (100x100 cells, centre of a 3x3 layout): tiles per (rows, column groups, flags), values,
// phases. Build: make -C tools tile_stats (links the product's host objects).
#include <cstdio>
#include <cstring>
#include <map>
#include <tuple>

#include "../paper_2410_14786_b200/csrc/host/factor.hpp"
#include "../paper_2410_14786_b200/csrc/host/problem.hpp"
#include "../paper_2410_14786_b200/csrc/host/solve_program.hpp"

using namespace bddc_b200;

int main(int argc, char** argv) {
    const int m = argc > 1 ? std::atoi(argv[1]) : 100;
    const int leaf = argc > 2 ? std::atoi(argv[2]) : 24;
    const int mode = argc > 3 ? std::atoi(argv[3]) : 1;  // 0 full, 1 head (pruned bwd), 2 harmonic (pruned fwd)
    PoissonProblem p = assemble_poisson(3 * m, 3 * m, 3, 3);
    const int s = 4;
    const auto& dofs = p.decomposition.subdomain_dofs[s];
    std::vector<index_t> lc(dofs.size() * 2);
    index_t mx = 1 << 30, my = 1 << 30;
    for (index_t g : dofs) { mx = std::min(mx, p.coords[2 * g]); my = std::min(my, p.coords[2 * g + 1]); }
    for (std::size_t l = 0; l < dofs.size(); ++l) {
        lc[2 * l] = p.coords[2 * dofs[l]] - mx;
        lc[2 * l + 1] = p.coords[2 * dofs[l] + 1] - my;
    }
    FactorOptions fo;
    fo.leaf_size = leaf;
    const index_t nI = p.decomposition.interior_counts[s];
    InteriorFactor F = factor_subdomain(p.local_matrices[s], nI, lc.data(), fo);
    SolvePools pools;
    std::vector<index_t> l2v(dofs.begin(), dofs.end());
    build_solve_program(F, p.local_matrices[s], l2v, 0, 2, 4096, pools, mode == 2, mode == 1);
    std::printf("supernodes %zu factor values %lld tiles %lld tile values %lld\n", F.snodes.size(),
                (long long)F.factor_values(), (long long)pools.n_tiles, (long long)pools.tile_values);
    std::map<std::tuple<int, int, int>, std::pair<long long, long long>> hist;  // (k, G, flags) -> tiles, values
    std::map<int, std::pair<long long, long long>> by_iters;
    long long ntile = 0, nval = 0, nsteps = 0, npairs = 0;
    for (const PartDesc& pd : pools.parts) {
        std::printf("part %d: n_loc %d n_top %d phases %d units %d\n", pd.rank, pd.n_loc, pd.n_top, pd.n_phases,
                    pd.n_units);
        const char* base = reinterpret_cast<const char*>(pools.stream.data() + pd.stream);
        for (int w = 0; w < kSolveWarps; ++w)
            for (int u = pd.warp_base[w]; u < pd.warp_base[w + 1]; ++u) {
                const std::int32_t* ue = &pools.units[2 * (pd.units + u)];
                const char* ub = base + std::int64_t(ue[0]) * 16;
                for (std::uint32_t cur = 0; cur != kNoStep;) {
                    std::uint32_t hw[4];
                    std::memcpy(hw, ub + std::int64_t(cur) * 16, 16);
                    const StepFields t = unpack_step(hw);
                    ++nsteps;
                    if (t.nsub_lg) {  // a group step: count its other tiles too
                        ++npairs;
                        for (int q = 1; q < (1 << t.nsub_lg); ++q) {
                            std::memcpy(hw, ub + std::int64_t(cur) * 16 + 16 * q, 16);
                            const StepFields b = unpack_step(hw);
                            ntile++;
                            nval += (long long)b.iters * b.k * (1 << b.lg);
                        }
                    }
                    cur = t.next;
                    const int G = 1 << t.lg;
                    const long long v = (long long)t.iters * t.k * G;
                    auto& h = hist[{(int)t.k, G, (int)(t.flags & (kTaskInIndexed | kTaskDiag | kTaskPush | kTaskPartial))}];
                    h.first++;
                    h.second += v;
                    auto& bi = by_iters[std::min<int>(t.iters, 64)];
                    bi.first++;
                    bi.second += v;
                    ntile++;
                    nval += v;
                }
            }
    }
    std::printf("tiles %lld values %lld (%.1f per tile), warp steps %lld (%lld group steps)\n", ntile, nval,
                double(nval) / ntile, nsteps, npairs);
    std::printf("%4s %3s %5s %8s %10s %8s\n", "k", "G", "flags", "tiles", "values", "v/tile");
    for (auto& [key, c] : hist)
        if (c.first * 200 > ntile)
            std::printf("%4d %3d %5d %8lld %10lld %8.1f\n", std::get<0>(key), std::get<1>(key), std::get<2>(key),
                        c.first, c.second, double(c.second) / c.first);
    std::printf("iters histogram: iters tiles values\n");
    for (auto& [it, c] : by_iters) std::printf("%3d %8lld %10lld\n", it, c.first, c.second);
    return 0;
}
