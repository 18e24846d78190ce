// ref_driver — TEST INFRASTRUCTURE ONLY (oracle). Never linked into the
// product library. Drives the UNMODIFIED reference library compiled from
// /root/reference/proj/src (see oracle/Makefile) to
//   * dump golden fixtures (maps, matrices, setup blocks, stage vectors, PCG
//     histories) for tests/golden/ via oracle/gen_golden.py, and
//   * time the reference CPU path for bench.py's cpu_baseline / --impl reference.
//
// Reference entry points exercised (file:line into /root/reference/proj):
//   assemble_poisson          src/decomposition.cpp:161-203
//   build_constraints         src/decomposition.cpp:112-159
//   Preconditioner ctor       src/preconditioner.cpp:100-127
//   stage methods + apply     src/preconditioner.cpp:129-249
//   pcg                       src/pcg.cpp:40-109
//   study_rhs                 src/study.cpp:69-75
//   export/ingest bundle      src/bundle.cpp:59-290
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "bddc/bundle.hpp"
#include "bddc/decomposition.hpp"
#include "bddc/pcg.hpp"
#include "bddc/preconditioner.hpp"
#include "bddc/study.hpp"

using namespace bddc;
namespace fs = std::filesystem;

namespace {

// Minimal .npy (v1.0) writer for 1-D little-endian arrays.
template <typename T>
const char* npy_descr();
template <> const char* npy_descr<double>() { return "<f8"; }
template <> const char* npy_descr<std::int32_t>() { return "<i4"; }
template <> const char* npy_descr<std::int64_t>() { return "<i8"; }

template <typename T>
void write_npy(const fs::path& path, const T* data, std::size_t n) {
    std::string header = "{'descr': '" + std::string(npy_descr<T>()) +
                         "', 'fortran_order': False, 'shape': (" + std::to_string(n) + ",), }";
    std::size_t total = 10 + header.size() + 1;
    std::size_t pad = (64 - total % 64) % 64;
    header.append(pad, ' ');
    header.push_back('\n');
    std::ofstream out(path, std::ios::binary);
    if (!out) { std::fprintf(stderr, "cannot write %s\n", path.c_str()); std::exit(2); }
    const char magic[] = "\x93NUMPY";
    out.write(magic, 6);
    const char ver[2] = {1, 0};
    out.write(ver, 2);
    const std::uint16_t hl = static_cast<std::uint16_t>(header.size());
    out.write(reinterpret_cast<const char*>(&hl), 2);
    out.write(header.data(), header.size());
    out.write(reinterpret_cast<const char*>(data), sizeof(T) * n);
}
template <typename T>
void write_npy(const fs::path& p, const std::vector<T>& v) { write_npy(p, v.data(), v.size()); }

void write_csr(const fs::path& dir, const std::string& name, const CsrMatrix& A) {
    std::vector<std::int32_t> shape = {A.nrows, A.ncols};
    write_npy(dir / (name + "_shape.npy"), shape);
    write_npy(dir / (name + "_rowptr.npy"), A.row_offsets);
    write_npy(dir / (name + "_cols.npy"), A.col_indices);
    write_npy(dir / (name + "_vals.npy"), A.values);
}

// Concatenate a list of CSR matrices: shapes [n,2], rowptr concatenated with
// per-matrix offsets [n+1] into it, nnz offsets [n+1].
void write_csr_list(const fs::path& dir, const std::string& name,
                    const std::vector<CsrMatrix>& list) {
    std::vector<std::int32_t> shapes, rowptr, rowptr_off{0}, cols;
    std::vector<std::int64_t> nnz_off{0};
    std::vector<double> vals;
    for (const CsrMatrix& A : list) {
        shapes.push_back(A.nrows);
        shapes.push_back(A.ncols);
        rowptr.insert(rowptr.end(), A.row_offsets.begin(), A.row_offsets.end());
        rowptr_off.push_back(static_cast<std::int32_t>(rowptr.size()));
        cols.insert(cols.end(), A.col_indices.begin(), A.col_indices.end());
        vals.insert(vals.end(), A.values.begin(), A.values.end());
        nnz_off.push_back(static_cast<std::int64_t>(vals.size()));
    }
    write_npy(dir / (name + "_shapes.npy"), shapes);
    write_npy(dir / (name + "_rowptr.npy"), rowptr);
    write_npy(dir / (name + "_rowptr_off.npy"), rowptr_off);
    write_npy(dir / (name + "_cols.npy"), cols);
    write_npy(dir / (name + "_vals.npy"), vals);
    write_npy(dir / (name + "_nnz_off.npy"), nnz_off);
}

template <typename T>
void write_ragged(const fs::path& dir, const std::string& name,
                  const std::vector<std::vector<T>>& lists) {
    std::vector<T> flat;
    std::vector<std::int64_t> off{0};
    for (const auto& l : lists) {
        flat.insert(flat.end(), l.begin(), l.end());
        off.push_back(static_cast<std::int64_t>(flat.size()));
    }
    write_npy(dir / (name + ".npy"), flat);
    write_npy(dir / (name + "_off.npy"), off);
}

SolverOptions outer(double tol) {
    SolverOptions o;
    o.rel_tolerance = tol;
    o.max_iterations = 10000;
    o.record_history = true;
    return o;
}

struct Problem {
    Decomposition decomposition;
    ConstraintSet constraints;
    CsrMatrix global_matrix;
    std::vector<CsrMatrix> local_matrices;
    std::vector<double> rhs;
};

Problem make_square(index_t k, index_t m, std::uint64_t seed) {
    const StructuredGrid grid(k * m);
    PoissonProblem p = assemble_poisson(grid, k);
    Problem out;
    out.constraints = build_constraints(p.decomposition);
    out.decomposition = std::move(p.decomposition);
    out.global_matrix = std::move(p.global_matrix);
    out.local_matrices = std::move(p.local_matrices);
    out.rhs = study_rhs(grid.free_dofs, seed);
    return out;
}

Problem make_bundle(const std::string& manifest) {
    IngestedProblem p = ingest_bundle(manifest);
    Problem out;
    out.decomposition = std::move(p.decomposition);
    out.constraints = std::move(p.constraints);
    out.global_matrix = std::move(p.global_matrix);
    out.local_matrices = std::move(p.local_matrices);
    out.rhs = std::move(p.rhs);
    return out;
}

double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int dump(const Problem& pr, const fs::path& dir, index_t workers, bool stages, bool plain) {
    fs::create_directories(dir);
    const Decomposition& d = pr.decomposition;
    std::vector<std::int32_t> meta = {d.k, d.n_subdomains, d.global_dofs, pr.constraints.n_coarse};
    write_npy(dir / "meta.npy", meta);
    write_ragged(dir, "subdomain_dofs", d.subdomain_dofs);
    write_npy(dir / "interior_counts.npy", d.interior_counts);
    std::vector<std::int32_t> kind, entity;
    for (const DofClass& c : d.classes) {
        kind.push_back(static_cast<std::int32_t>(c.kind));
        entity.push_back(c.entity);
    }
    write_npy(dir / "class_kind.npy", kind);
    write_npy(dir / "class_entity.npy", entity);
    write_npy(dir / "multiplicity.npy", d.multiplicity);
    write_ragged(dir, "weights", d.weights);
    write_ragged(dir, "primal_maps", pr.constraints.primal_maps);
    write_csr_list(dir, "constraints", pr.constraints.constraint_matrices);
    write_csr(dir, "A", pr.global_matrix);
    write_csr_list(dir, "locals", pr.local_matrices);
    write_npy(dir / "rhs.npy", pr.rhs);

    double t0 = now();
    const Preconditioner P(pr.global_matrix, pr.local_matrices, d, pr.constraints, workers);
    const double setup_s = now() - t0;

    std::vector<std::vector<double>> phi, lam, aci;
    for (const SubdomainData& s : P.subdomains()) {
        phi.push_back(s.coarse_basis.values);
        lam.push_back(s.multipliers.values);
        aci.push_back(s.coarse_block.values);
    }
    write_ragged(dir, "phi", phi);
    write_ragged(dir, "lambda", lam);
    write_ragged(dir, "aci", aci);
    write_csr(dir, "Ac", P.coarse().matrix);

    if (stages) {
        const std::vector<double>& r = pr.rhs;
        const std::vector<double> u0 = P.interior_correction(r);
        std::vector<double> cond = spmv(pr.global_matrix, u0);
        for (std::size_t i = 0; i < cond.size(); ++i) cond[i] = r[i] - cond[i];
        const std::vector<double> v1 = P.coarse_correction(cond);
        const std::vector<double> v2 = P.local_correction(cond);
        const std::vector<double> v3 = P.static_condensation_correction(cond, v1, v2);
        const std::vector<double> z = P.apply(r);
        write_npy(dir / "stage_u0.npy", u0);
        write_npy(dir / "stage_condensed.npy", cond);
        write_npy(dir / "stage_v1.npy", v1);
        write_npy(dir / "stage_v2.npy", v2);
        write_npy(dir / "stage_v3.npy", v3);
        write_npy(dir / "apply_rhs.npy", z);
        // stage operators on the raw rhs as well (non-condensed input)
        write_npy(dir / "coarse_of_rhs.npy", P.coarse_correction(r));
        write_npy(dir / "local_of_rhs.npy", P.local_correction(r));
    }

    std::vector<double> x;
    t0 = now();
    const SolveReport rep = pcg(pr.global_matrix, pr.rhs,
                                [&](std::span<const double> r, std::span<double> z) {
                                    const std::vector<double> res = P.apply(r);
                                    std::copy(res.begin(), res.end(), z.begin());
                                },
                                outer(1e-8), x);
    const double solve_s = now() - t0;
    write_npy(dir / "pcg_history.npy", rep.residual_history);
    write_npy(dir / "pcg_x.npy", x);
    std::vector<double> scal = {static_cast<double>(rep.iterations), rep.final_relative_residual,
                                rep.condition_estimate ? *rep.condition_estimate : -1.0,
                                rep.converged ? 1.0 : 0.0, setup_s, solve_s};
    write_npy(dir / "pcg_report.npy", scal);
    if (plain) {
        std::vector<double> xp;
        const SolveReport prep = pcg(pr.global_matrix, pr.rhs, {}, outer(1e-8), xp);
        write_npy(dir / "plain_history.npy", prep.residual_history);
        std::vector<double> ps = {static_cast<double>(prep.iterations), prep.final_relative_residual,
                                  prep.converged ? 1.0 : 0.0};
        write_npy(dir / "plain_report.npy", ps);
    }
    std::printf("{\"iterations\": %d, \"final_relative_residual\": %.17g, \"setup_seconds\": %.6f, "
                "\"solve_seconds\": %.6f}\n",
                rep.iterations, rep.final_relative_residual, setup_s, solve_s);
    return 0;
}

// Timed CPU reference: setup once, then `warmup` + `steps` full PCG solves.
// Prints one JSON line with per-solve seconds.
// plain = true: the reference's plain CG (empty PreconditionerFn, pcg.hpp:33-34; study.cpp
// compare mode :123-135), no preconditioner setup.
int bench(const Problem& pr, index_t workers, int steps, int warmup, bool plain) {
    const Decomposition& d = pr.decomposition;
    double t0 = now();
    std::optional<Preconditioner> P;
    if (!plain) P.emplace(pr.global_matrix, pr.local_matrices, d, pr.constraints, workers);
    const double setup_s = now() - t0;
    std::vector<double> times;
    int iterations = 0;
    double final_rel = 0.0, apply_s = 0.0;
    for (int s = 0; s < warmup + steps; ++s) {
        std::vector<double> x;
        int napply = 0;
        double tapply = 0.0;
        t0 = now();
        PreconditionerFn M;
        if (P)
            M = [&](std::span<const double> r, std::span<double> z) {
                const double ta = now();
                const std::vector<double> res = P->apply(r);
                std::copy(res.begin(), res.end(), z.begin());
                tapply += now() - ta;
                ++napply;
            };
        const SolveReport rep = pcg(pr.global_matrix, pr.rhs, M, outer(1e-8), x);
        const double dt = now() - t0;
        if (s >= warmup) {
            times.push_back(dt);
            apply_s += tapply / std::max(1, napply);
        }
        iterations = rep.iterations;
        final_rel = rep.final_relative_residual;
    }
    double sum = 0.0;
    for (double t : times) sum += t;
    const double mean = times.empty() ? 0.0 : sum / times.size();
    std::printf("{\"global_dofs\": %d, \"n_subdomains\": %d, \"coarse_dim\": %d, \"workers\": %d, "
                "\"setup_seconds\": %.6f, \"solve_seconds_mean\": %.6f, \"apply_seconds_mean\": %.6f, "
                "\"iterations\": %d, \"final_relative_residual\": %.17g, \"steps\": %d}\n",
                d.global_dofs, d.n_subdomains, pr.constraints.n_coarse, workers, setup_s, mean,
                times.empty() ? 0.0 : apply_s / times.size(), iterations, final_rel,
                static_cast<int>(times.size()));
    return 0;
}

void usage() {
    std::fprintf(stderr,
                 "usage:\n"
                 "  ref_driver dump   <k> <m> <seed> <outdir> [workers] [--no-stages] [--plain]\n"
                 "  ref_driver dumpb  <manifest> <outdir> [workers] [--no-stages] [--plain]\n"
                 "  ref_driver bench  <k> <m> <workers> <steps> <warmup> [--plain]\n"
                 "  ref_driver benchb <manifest> <workers> <steps> <warmup> [--plain]\n"
                 "  ref_driver export <k> <m> <seed> <outdir>\n");
}

bool has_flag(int argc, char** argv, const char* f) {
    for (int i = 1; i < argc; ++i)
        if (std::strcmp(argv[i], f) == 0) return true;
    return false;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) { usage(); return 2; }
    const std::string cmd = argv[1];
    try {
        if (cmd == "dump" && argc >= 6) {
            const index_t workers = argc >= 7 && argv[6][0] != '-' ? std::atoi(argv[6]) : 1;
            const Problem pr = make_square(std::atoi(argv[2]), std::atoi(argv[3]),
                                           std::strtoull(argv[4], nullptr, 10));
            return dump(pr, argv[5], workers, !has_flag(argc, argv, "--no-stages"),
                        has_flag(argc, argv, "--plain"));
        }
        if (cmd == "dumpb" && argc >= 4) {
            const index_t workers = argc >= 5 && argv[4][0] != '-' ? std::atoi(argv[4]) : 1;
            const Problem pr = make_bundle(argv[2]);
            return dump(pr, argv[3], workers, !has_flag(argc, argv, "--no-stages"),
                        has_flag(argc, argv, "--plain"));
        }
        if (cmd == "bench" && argc >= 7) {
            const Problem pr = make_square(std::atoi(argv[2]), std::atoi(argv[3]), 1);
            return bench(pr, std::atoi(argv[4]), std::atoi(argv[5]), std::atoi(argv[6]), has_flag(argc, argv, "--plain"));
        }
        if (cmd == "benchb" && argc >= 6) {
            const Problem pr = make_bundle(argv[2]);
            return bench(pr, std::atoi(argv[3]), std::atoi(argv[4]), std::atoi(argv[5]), has_flag(argc, argv, "--plain"));
        }
        if (cmd == "export" && argc >= 6) {
            const index_t k = std::atoi(argv[2]), m = std::atoi(argv[3]);
            const StructuredGrid grid(k * m);
            const PoissonProblem p = assemble_poisson(grid, k);
            const std::vector<double> b = study_rhs(grid.free_dofs, std::strtoull(argv[4], nullptr, 10));
            std::printf("%s\n", export_bundle(p.decomposition, p.local_matrices, b, argv[5]).c_str());
            return 0;
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ref_driver error: %s\n", e.what());
        return 1;
    }
    usage();
    return 2;
}
