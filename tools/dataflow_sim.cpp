// Dev tool: predicted makespan of one interior-solve part with CTA barriers between phases vs
// per-warp dependency waits (dataflow), from the program's tile list and a per-tile cost model
// (c0 + c1 * iterations cycles). Host only; links the product's host objects.
#include <algorithm>
#include <array>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <vector>

#include "../paper_2410_14786_b200/csrc/host/factor.hpp"
#include "../paper_2410_14786_b200/csrc/host/problem.hpp"
#include "../paper_2410_14786_b200/csrc/host/solve_program.hpp"

using namespace bddc_b200;

int main(int argc, char** argv) {
    const int m = argc > 1 ? std::atoi(argv[1]) : 100;
    const int mode = argc > 2 ? std::atoi(argv[2]) : 2;  // 0 full, 1 harmonic, 2 head
    const double c0 = argc > 3 ? std::atof(argv[3]) : 600, c1 = argc > 4 ? std::atof(argv[4]) : 40;
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
    fo.leaf_size = 24;
    InteriorFactor F = factor_subdomain(p.local_matrices[s], p.decomposition.interior_counts[s], lc.data(), fo);
    SolvePools sp;
    std::vector<index_t> l2v(dofs.begin(), dofs.end());
    build_solve_program(F, p.local_matrices[s], l2v, 0, 2, 4096, sp, mode == 1, mode == 2);
    const PartDesc& pd = sp.parts[0];
    const int W = kSolveWarps, NP = pd.n_phases, NL = pd.n_loc + 64;
    const char* base = reinterpret_cast<const char*>(sp.stream.data() + pd.stream);
    // per phase per warp: cost and accesses ((vector, row), write?)
    struct Acc { int vec, row; bool w; };
    std::vector<std::vector<double>> cost(NP, std::vector<double>(W, 0.0));
    std::vector<std::vector<std::vector<Acc>>> acc(NP, std::vector<std::vector<Acc>>(W));
    std::vector<int> full(NP, 0);
    bool seen_bwd = false;
    for (int ph = 0; ph < NP; ++ph) {
        const std::int32_t* row = &sp.phases[pd.phases + ph * kPhaseStride];
        const int kind = row[2 * W];
        const bool bwd = kind & kPhaseBackward;
        if (bwd && !seen_bwd) { full[ph] = 1; seen_bwd = true; }
        if (kind & kPhaseCombine) full[ph] = 2;  // combine after the phase
        const int own = bwd ? 1 : 0, other = bwd ? 0 : 1;  // 0 = T, 1 = X, 2 = Q
        for (int w = 0; w < W; ++w) {
            const int ua = ph == 0 ? 0 : sp.phases[pd.phases + (ph - 1) * kPhaseStride + W + w];
            const int ub = row[W + w];
            for (int u = ua; u < ub; ++u) {
                const std::int32_t* ue = &sp.units[2 * (pd.units + pd.warp_base[w] + u)];
                for (std::uint32_t cur = 0; cur != kNoTask;) {
                    TileTask t;
                    std::memcpy(&t, base + std::int64_t(ue[0]) * 16 + std::int64_t(cur) * 16, 16);
                    const char* tile = base + std::int64_t(ue[0]) * 16 + std::int64_t(cur) * 16 + 16;
                    cur = t.next;
                    const int G = 1 << t.groups, k = t.nrows, it = t.iters;
                    cost[ph][w] += c0 + c1 * it;
                    const int vin = (t.flags & kTaskInOwn) ? own : other;
                    const int vbytes = pad16i(it * k * G * 8);
                    if (t.flags & kTaskInIndexed) {
                        const std::int32_t* ix = reinterpret_cast<const std::int32_t*>(tile + vbytes);
                        for (int j = 0; j < it * G; ++j) acc[ph][w].push_back({vin, ix[j], false});
                    } else {
                        for (int j = 0; j < it * G; ++j) acc[ph][w].push_back({vin, int(t.in_ref) + j, false});
                    }
                    if (!(t.flags & kTaskLast)) continue;
                    if (t.flags & kTaskPush) {
                        const int ib = (t.flags & kTaskInIndexed) ? pad16i(it * G * 4) : 0;
                        const std::int32_t* o = reinterpret_cast<const std::int32_t*>(tile + vbytes + ib);
                        for (int r = 0; r < k; ++r) acc[ph][w].push_back({(t.flags & kTaskPartial) ? 2 : own, o[r], true});
                    } else {
                        for (int r = 0; r < t.nvalid; ++r)
                            acc[ph][w].push_back({(t.flags & kTaskDiag) ? other : own, t.out_base + r, true});
                    }
                }
            }
        }
    }
    // barrier model
    double tb = 0;
    for (int ph = 0; ph < NP; ++ph) tb += *std::max_element(cost[ph].begin(), cost[ph].end()) + 200;
    // dataflow model: need[ph][w][v] = latest phase of v that conflicts with w's phase ph
    std::vector<std::array<int, 2>> lastW(3 * NL, {-1, -1});
    std::vector<std::vector<int>> lastR(3 * NL, std::vector<int>(W, -1));
    std::vector<std::vector<double>> fin(NP, std::vector<double>(W, 0.0));
    std::vector<double> wdone(W, 0.0);
    long deps = 0, pairs = 0;
    for (int ph = 0; ph < NP; ++ph) {
        std::vector<std::vector<int>> need(W, std::vector<int>(W, -1));
        for (int w = 0; w < W; ++w)
            for (const Acc& a : acc[ph][w]) {
                const int key = a.vec * NL + a.row;
                if (lastW[key][0] >= 0 && lastW[key][1] != w) need[w][lastW[key][1]] = std::max(need[w][lastW[key][1]], lastW[key][0]);
                if (a.w)
                    for (int v = 0; v < W; ++v)
                        if (v != w) need[w][v] = std::max(need[w][v], lastR[key][v]);
            }
        for (int w = 0; w < W; ++w)
            for (const Acc& a : acc[ph][w]) {
                const int key = a.vec * NL + a.row;
                if (a.w) { lastW[key] = {ph, w}; std::fill(lastR[key].begin(), lastR[key].end(), -1); }
                else lastR[key][w] = ph;
            }
        double all = 0;
        if (full[ph] == 1) for (int v = 0; v < W; ++v) all = std::max(all, wdone[v]);
        for (int w = 0; w < W; ++w) {
            double st = std::max(wdone[w], all);
            for (int v = 0; v < W; ++v) {
                ++pairs;
                if (need[w][v] >= 0) { ++deps; st = std::max(st, fin[need[w][v]][v]); }
            }
            fin[ph][w] = st + cost[ph][w] + 50;
        }
        for (int w = 0; w < W; ++w) wdone[w] = fin[ph][w];
        if (full[ph] == 2) { double mxx = *std::max_element(wdone.begin(), wdone.end()) + 400; std::fill(wdone.begin(), wdone.end(), mxx); for (int w = 0; w < W; ++w) fin[ph][w] = mxx; }
    }
    const double td = *std::max_element(wdone.begin(), wdone.end());
    double work = 0;
    for (auto& c : cost) for (double v : c) work += v;
    std::printf("phases %d, work/warp %.0f, barrier makespan %.0f, dataflow makespan %.0f (%.2fx), dep density %.2f\n",
                NP, work / W, tb, td, tb / td, double(deps) / pairs);
}
