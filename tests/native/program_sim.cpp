// TEST-ONLY: sequential CPU interpreter of the interior-solve program produced by
// build_device_image (device_format.hpp). Lets the CPU test suite validate the
// program builder (phase order, tile layout, cluster split, combine steps) without a
// GPU. It is compiled into tests/native/libbddc_sim.so, never into the product library,
// and executes exactly the task semantics of device/solve.cu.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include <algorithm>
#include <cstdio>

#include "../../paper_2410_14786_b200/csrc/context.hpp"
#include "../../paper_2410_14786_b200/csrc/host/program.hpp"
#include "../../paper_2410_14786_b200/csrc/host/gpu_setup.hpp"

using namespace bddc_b200;

namespace {

struct PartState {
    const PartDesc* pd;
    std::vector<double> T, X, Q;
    int ph = 0;
    bool split_done = false;
    // per warp: step cursor (unit, 16-byte offset in it), steps done; the step stream runs on
    // across phases (device_format.hpp)
    int wu[kSolveWarps] = {}, wdone[kSolveWarps] = {};
    std::uint32_t wcur[kSolveWarps] = {};
};

void run_phase(const SolvePools& sp, PartState& st) {
    const PartDesc& pd = *st.pd;
    const std::int32_t* row = &sp.phases[pd.phases + st.ph * kPhaseStride];
    const int kind = row[2 * kSolveWarps];
    std::vector<double>& own = (kind & kPhaseBackward) ? st.X : st.T;
    std::vector<double>& other = (kind & kPhaseBackward) ? st.T : st.X;
    const char* base = reinterpret_cast<const char*>(sp.stream.data() + pd.stream);
    for (int w = 0; w < kSolveWarps; ++w) {
        double acc[4][32] = {{0}};  // per sub-tile (a group step's 1, 2 or 4), per row
        const int s_end = row[kSolveWarps + w];
        while (st.wdone[w] < s_end) {
            const std::int32_t* ue = &sp.units[2 * (pd.units + pd.warp_base[w] + st.wu[w])];
            const char* ubase = base + std::int64_t(ue[0]) * 16;
            std::uint32_t& cur = st.wcur[w];
            // step sub-headers (device_format.hpp): one per sub-tile (1, 2 or 4); the tile data
            // follows them, every offset is read from the sub-header like the kernel
            StepFields hd[4];
            std::uint32_t hw[4];
            std::memcpy(hw, ubase + std::int64_t(cur) * 16, 16);
            hd[0] = unpack_step(hw);
            const int nsub = 1 << hd[0].nsub_lg;
            for (int q = 1; q < nsub; ++q) {
                std::memcpy(hw, ubase + std::int64_t(cur) * 16 + 16 * q, 16);
                hd[q] = unpack_step(hw);
            }
            const char* tb = ubase + std::int64_t(cur) * 16 + 16 * nsub;
            cur = hd[0].next;
            ++st.wdone[w];
            if (cur == kNoStep) {  // unit consumed
                ++st.wu[w];
                cur = 0;
            }
            for (int q = 0; q < nsub; ++q) {
                const StepFields& task = hd[q];
                const int k = task.k, G = 1 << task.lg, iters = task.iters, S = task.S, voff = task.voff;
                const double* M = reinterpret_cast<const double*>(tb);
                const std::int32_t* ix = reinterpret_cast<const std::int32_t*>(tb + 16 * task.ixq);
                const std::int32_t* ox = reinterpret_cast<const std::int32_t*>(tb + 16 * task.oq);
                if (task.flags & kTaskFirst)
                    for (double& a : acc[q]) a = 0.0;
                const std::vector<double>& in = (task.flags & kTaskInOwn) ? own : other;
                // T-relative indices at or past part_ldn(n_loc) address X (merged backward tiles)
                const int ldn_p = part_ldn(pd.n_loc);
                auto fetch = [&](int idx) -> double {
                    if (&in == &st.T && idx >= ldn_p) return st.X.at(idx - ldn_p);
                    return in.at(idx);
                };
                for (int r = 0; r < k; ++r) {
                    double s = 0.0;
                    for (int it = 0; it < iters; ++it)
                        for (int g = 0; g < G; ++g) {
                            const int j = it * G + g;
                            const double v = (task.flags & kTaskInIndexed) ? fetch(ix[j]) : fetch(static_cast<int>(task.in_ref) + j);
                            s += M[it * S + voff + r * G + g] * v;
                        }
                    acc[q][r] += s;
                }
                if (task.flags & kTaskLast)
                    for (int r = 0; r < static_cast<int>(task.nvalid); ++r) {
                        if (task.flags & kTaskDiag) other.at(static_cast<int>(task.out_base) + r) = acc[q][r];
                        else if (task.flags & kTaskPush) {
                            if (task.flags & kTaskPartial) st.Q.at(ox[r]) += acc[q][r];
                            else own.at(ox[r]) -= acc[q][r];
                        } else own.at(static_cast<int>(task.out_base) + r) -= acc[q][r];
                    }
            }
        }
    }
}

}  // namespace

// harm: 0 full program, 1 harmonic program, 2 head program (y0 -> ybuf, u0 -> out),
// 3 harmonic program with y_in = ybuf (out = L^-T (y0 - L^-1 in)); the split hooks follow
// device/solve.cu (applied at the first backward phase, X = forward result).
static int sim_solve(int cells_x, int cells_y, int kx, int ky, int parts, int leaf_size, int use_coords,
                     int harm, const double* in, double* out, char* err, int errlen, double* ybuf = nullptr) {
    try {
        PoissonProblem pp = assemble_poisson(cells_x, cells_y, kx, ky);
        ProblemData pb;
        pb.constraints = build_constraints(pp.decomposition);
        pb.decomposition = std::move(pp.decomposition);
        pb.global_matrix = std::move(pp.global_matrix);
        pb.local_matrices = std::move(pp.local_matrices);
        if (use_coords) pb.coords = std::move(pp.coords);
        FactorOptions fo;
        fo.leaf_size = leaf_size;
        const BddcSetup setup = bddc_setup(pb.local_matrices, pb.decomposition, pb.constraints,
                                           pb.coords.empty() ? nullptr : pb.coords.data(), 4, fo);
        const DeviceImage img = build_device_image(pb.decomposition, pb.constraints, pb.local_matrices,
                                                   pb.global_matrix, setup, parts, 4096, nullptr, harm != 0);
        const SolvePools& sp = harm == 2 ? img.head : (harm ? img.harm : img.solve);
        for (std::size_t i0 = 0; i0 < sp.parts.size(); i0 += parts) {
            std::vector<PartState> st(parts);
            for (int c = 0; c < parts; ++c) {
                const PartDesc& pd = sp.parts[i0 + c];
                st[c].pd = &pd;
                st[c].T.resize(pd.n_loc);
                st[c].X.assign(pd.n_loc + 64, 0.0);
                st[c].T.resize(pd.n_loc + 64, 0.0);
                st[c].Q.assign(pd.n_top, 0.0);
                for (int l = 0; l < pd.n_loc; ++l) st[c].T[l] = in[sp.gmap[pd.gmap + l]];
            }
            bool progress = true;
            while (progress) {
                progress = false;
                // run every part up to (and including) its next combine phase
                std::vector<int> at_combine(parts, -1);
                for (int c = 0; c < parts; ++c) {
                    PartState& s = st[c];
                    while (s.ph < s.pd->n_phases) {
                        const std::int32_t* row = &sp.phases[s.pd->phases + s.ph * kPhaseStride];
                        if ((harm == 2 || harm == 3) && !s.split_done && (row[2 * kSolveWarps] & kPhaseBackward)) {
                            s.split_done = true;
                            for (int l = 0; l < s.pd->n_loc; ++l) {
                                if (harm == 2) ybuf[s.pd->gmap + l] = s.X[l];
                                else s.X[l] = ybuf[s.pd->gmap + l] - s.X[l];
                            }
                        }
                        run_phase(sp, s);
                        ++s.ph;
                        progress = true;
                        if (parts > 1 && (row[2 * kSolveWarps] & kPhaseCombine)) {
                            at_combine[c] = s.ph - 1;
                            break;
                        }
                    }
                }
                if (parts > 1 && at_combine[0] >= 0) {
                    if (at_combine[1] < 0) throw std::logic_error("parts disagree on combine phases");
                    std::vector<std::vector<double>> Qs = {st[0].Q, st[1].Q};
                    for (int c = 0; c < parts; ++c) {
                        const std::int32_t* row = &sp.phases[st[c].pd->phases + at_combine[c] * kPhaseStride];
                        const int cb = row[2 * kSolveWarps + 1], ce = row[2 * kSolveWarps + 2];
                        for (int l = cb; l < ce; ++l) {
                            const int qi = l - st[c].pd->n_group;
                            st[c].T[l] = (st[c].T[l] - Qs[0][qi]) - Qs[1][qi];
                        }
                    }
                }
            }
            for (int c = 0; c < parts; ++c)
                for (int l = 0; l < st[c].pd->n_write; ++l) out[sp.gmap[st[c].pd->gmap + l]] = st[c].T[l];
        }
        return 0;
    } catch (const std::exception& e) {
        std::snprintf(err, errlen, "%s", e.what());
        return 1;
    }
}

extern "C" int bddc_sim_interior_solve(int cells_x, int cells_y, int kx, int ky, int parts, int leaf_size,
                                       int use_coords, const double* in, double* out, char* err, int errlen) {
    return sim_solve(cells_x, cells_y, kx, ky, parts, leaf_size, use_coords, 0, in, out, err, errlen);
}

// Split apply: head program on r (u0 exact where the interface couples, y0 kept), then the
// harmonic program on c with y_in: z = A_II^-1 (r - c).
extern "C" int bddc_sim_split_solve(int cells_x, int cells_y, int kx, int ky, int parts, int leaf_size,
                                    int use_coords, const double* r, const double* c, double* u0, double* z,
                                    char* err, int errlen) {
    std::vector<double> y(static_cast<std::size_t>(cells_x + 1) * (cells_y + 1) * 2, 0.0);
    if (sim_solve(cells_x, cells_y, kx, ky, parts, leaf_size, use_coords, 2, r, u0, err, errlen, y.data())) return 1;
    return sim_solve(cells_x, cells_y, kx, ky, parts, leaf_size, use_coords, 3, c, z, err, errlen, y.data());
}

// The harmonic-extension program (pruned forward sweep) on an rhs supported on the interior
// dofs coupled to the interface.
extern "C" int bddc_sim_harmonic_solve(int cells_x, int cells_y, int kx, int ky, int parts, int leaf_size,
                                       int use_coords, const double* in, double* out, char* err, int errlen) {
    return sim_solve(cells_x, cells_y, kx, ky, parts, leaf_size, use_coords, 1, in, out, err, errlen);
}

// GPU-setup templates (host/gpu_setup.hpp) against the host-built programs: the class
// templates instantiated per subdomain and filled exactly like device/setup.cu's fill kernel
// (from a value array D = [L_ss^-1 | BL_s] computed from the host factor in the builder's loop
// order) must reproduce every host-built stream word, dof map and coupling entry bit for bit.
// Returns the number of mismatching entries (0 = identical), -1 on error.
extern "C" long bddc_sim_template_check(int cells_x, int cells_y, int kx, int ky, int parts, int leaf_size,
                                        int use_coords, char* err, int errlen) {
    try {
        PoissonProblem pp = assemble_poisson(cells_x, cells_y, kx, ky);
        ProblemData pb;
        pb.constraints = build_constraints(pp.decomposition);
        pb.decomposition = std::move(pp.decomposition);
        pb.global_matrix = std::move(pp.global_matrix);
        pb.local_matrices = std::move(pp.local_matrices);
        if (use_coords) pb.coords = std::move(pp.coords);
        const index_t* coords = pb.coords.empty() ? nullptr : pb.coords.data();
        FactorOptions fo;
        fo.leaf_size = leaf_size;
        const BddcSetup setup = bddc_setup(pb.local_matrices, pb.decomposition, pb.constraints, coords, 4, fo);
        const DeviceImage host = build_device_image(pb.decomposition, pb.constraints, pb.local_matrices,
                                                    pb.global_matrix, setup, parts, 4096, nullptr, true);
        const std::vector<SetupClass> classes = plan_gpu_setup(pb.local_matrices, pb.decomposition, pb.constraints,
                                                               coords, fo, parts, 4096, true, 4);
        BddcSetup meta;
        meta.subs.resize(pb.decomposition.n_subdomains);
        for (index_t i = 0; i < pb.decomposition.n_subdomains; ++i) {
            meta.subs[i].n_local = setup.subs[i].n_local;
            meta.subs[i].n_interior = setup.subs[i].n_interior;
            meta.subs[i].n_iface = setup.subs[i].n_iface;
            meta.subs[i].n_primal = setup.subs[i].n_primal;
        }
        const DeviceImage dev = build_device_image(pb.decomposition, pb.constraints, pb.local_matrices,
                                                   pb.global_matrix, meta, parts, 4096, nullptr, true, &classes);
        long bad = 0;
        auto cmp = [&](const auto& a, const auto& b) {
            if (a.size() != b.size()) return bad += 1000000, void();
            for (std::size_t i = 0; i < a.size(); ++i) bad += std::memcmp(&a[i], &b[i], sizeof(a[i])) != 0;
        };
        for (int k = 0; k < 3; ++k) {
            const SolvePools& H = k == 0 ? host.solve : (k == 1 ? host.harm : host.head);
            const SolvePools& G = k == 0 ? dev.solve : (k == 1 ? dev.harm : dev.head);
            if (G.words() != H.words()) bad += 1000000;
            std::vector<double> filled(static_cast<std::size_t>(G.words()), 0.0);
            for (const auto& f : dev.fills[k]) {
                const SetupClass& C = classes[f.cls];
                const InteriorFactor& F = setup.subs[f.sub].factor;  // host numeric factor of this subdomain
                std::vector<double> D(static_cast<std::size_t>(C.layout.total), 0.0);
                for (std::size_t s = 0; s < F.snodes.size(); ++s) {
                    const Supernode& S = F.snodes[s];
                    const index_t ns = S.size();
                    std::copy(S.Linv.begin(), S.Linv.end(), D.begin() + C.layout.linv_off[s]);
                    for (index_t a = 0; a < S.n_interior_rows; ++a)
                        for (index_t j = 0; j < ns; ++j) {
                            double acc = 0.0;
                            for (index_t q = j; q < ns; ++q) acc += S.B[a * ns + q] * S.Linv[q * ns + j];
                            D[C.layout.bl_off[s] + a * ns + j] = acc;
                        }
                }
                const SolvePools& T = C.prog[k];
                for (std::int64_t w = 0; w < f.words; ++w) {
                    const std::int32_t c = T.srcmap[w];
                    double v = c == kSrcCopy ? T.stream[w] : c == kSrcZero ? 0.0 : c >= 0 ? D[c] : -D[-c - 3];
                    filled[f.dst + w] = v;
                }
            }
            cmp(filled, H.stream);
            cmp(G.gmap, H.gmap);
            cmp(G.couple_val, H.couple_val);
            cmp(G.couple_gamma, H.couple_gamma);
            cmp(G.units, H.units);
            cmp(G.phases, H.phases);
            cmp(G.order, H.order);
            if (G.parts.size() != H.parts.size()) bad += 1000000;
            for (std::size_t p = 0; p < std::min(G.parts.size(), H.parts.size()); ++p)
                bad += std::memcmp(&G.parts[p], &H.parts[p], sizeof(PartDesc)) != 0;
        }
        return bad;
    } catch (const std::exception& e) {
        std::snprintf(err, errlen, "%s", e.what());
        return -1;
    }
}
