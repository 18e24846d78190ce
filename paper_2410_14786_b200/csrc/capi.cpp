// extern "C" boundary (include/bddc_b200.h). Exceptions stop here and become
// status codes; messages are kept verbatim for bddc_last_error().
#include "../../include/bddc_b200.h"

#include <memory>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>

#include "context.hpp"
#include "host/distribute.hpp"
#include "host/problem.hpp"
#include "host/setup.hpp"

using namespace bddc_b200;

struct bddc_problem {
    // filled at creation, read-only afterwards: GPU contexts share it instead of copying it
    std::shared_ptr<ProblemData> shared = std::make_shared<ProblemData>();
    ProblemData& data = *shared;
    std::vector<double> rhs;
    // flattened storage backing bddc_problem_get_view
    std::vector<bddc_csr_view> local_views, constraint_views;
    std::vector<std::int64_t> dof_offsets, primal_offsets;
    std::vector<std::int32_t> dofs, primal;
    std::vector<double> weights;
    std::vector<std::uint8_t> kind;
    std::vector<std::int32_t> entity;

    void flatten() {
        const Decomposition& d = data.decomposition;
        local_views.clear();
        constraint_views.clear();
        for (const auto& A : data.local_matrices)
            local_views.push_back({A.nrows, A.ncols, A.row_offsets.data(), A.col_indices.data(), A.values.data()});
        for (const auto& C : data.constraints.constraint_matrices)
            constraint_views.push_back({C.nrows, C.ncols, C.row_offsets.data(), C.col_indices.data(), C.values.data()});
        dof_offsets.assign(1, 0);
        dofs.clear();
        weights.clear();
        for (index_t i = 0; i < d.n_subdomains; ++i) {
            dofs.insert(dofs.end(), d.subdomain_dofs[i].begin(), d.subdomain_dofs[i].end());
            weights.insert(weights.end(), d.weights[i].begin(), d.weights[i].end());
            dof_offsets.push_back(static_cast<std::int64_t>(dofs.size()));
        }
        primal_offsets.assign(1, 0);
        primal.clear();
        for (const auto& m : data.constraints.primal_maps) {
            primal.insert(primal.end(), m.begin(), m.end());
            primal_offsets.push_back(static_cast<std::int64_t>(primal.size()));
        }
        kind.resize(d.classes.size());
        entity.resize(d.classes.size());
        for (std::size_t g = 0; g < d.classes.size(); ++g) {
            kind[g] = static_cast<std::uint8_t>(d.classes[g].kind);
            entity[g] = d.classes[g].entity;
        }
    }
};

struct bddc_host_setup {
    BddcSetup setup;
    const bddc_problem* problem;
};

struct bddc_rank_plan {
    RankPlan plan;
    bddc_problem local;  // the rank-local problem, viewable like any bddc_problem
    std::vector<std::int32_t> remote_ptr, remote_sub, remote_slot;
};

struct bddc_gpu_ctx {
    std::unique_ptr<GpuContext> ctx;
    std::string last_error;
};

namespace {

thread_local std::string g_last_error;

template <typename Fn>
int guarded(Fn&& fn, bddc_gpu_ctx* ctx = nullptr) {
    try {
        fn();
        return BDDC_OK;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        if (ctx) ctx->last_error = g_last_error;
        return BDDC_ERR_INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        g_last_error = e.what();
        if (ctx) ctx->last_error = g_last_error;
        return BDDC_ERR_OUT_OF_RANGE;
    } catch (const std::runtime_error& e) {
        g_last_error = e.what();
        if (ctx) ctx->last_error = g_last_error;
        const std::string m = e.what();
        if (m.rfind("no CUDA device", 0) == 0) return BDDC_ERR_NO_DEVICE;
        if (m.rfind("CUDA error", 0) == 0) return BDDC_ERR_CUDA;
        return BDDC_ERR_RUNTIME;
    } catch (const std::bad_alloc&) {
        g_last_error = "out of memory";
        if (ctx) ctx->last_error = g_last_error;
        return BDDC_ERR_RUNTIME;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        if (ctx) ctx->last_error = g_last_error;
        return BDDC_ERR_RUNTIME;
    } catch (...) {
        g_last_error = "unknown error";
        if (ctx) ctx->last_error = g_last_error;
        return BDDC_ERR_RUNTIME;
    }
}

CsrMatrix copy_csr(const bddc_csr_view& v) {
    if (v.nrows < 0 || v.ncols < 0 || !v.row_offsets)
        throw std::invalid_argument("csr view: invalid dimensions");
    CsrMatrix A;
    A.nrows = v.nrows;
    A.ncols = v.ncols;
    A.row_offsets.assign(v.row_offsets, v.row_offsets + v.nrows + 1);
    const index_t nnz = A.row_offsets.back();
    A.col_indices.assign(v.col_indices, v.col_indices + nnz);
    A.values.assign(v.values, v.values + nnz);
    A.validate();
    return A;
}

void fill_report(const SolveResult& r, bddc_solve_report* rep, double* history, int32_t cap) {
    if (!rep) return;
    rep->iterations = r.iterations;
    rep->final_relative_residual = r.final_relative_residual;
    rep->converged = r.converged ? 1 : 0;
    rep->has_condition_estimate = r.condition_estimate ? 1 : 0;
    rep->condition_estimate = r.condition_estimate ? *r.condition_estimate : 0.0;
    const int32_t n = static_cast<int32_t>(r.history.size());
    rep->history_length = history ? std::min(n, cap) : 0;
    if (history)
        for (int32_t i = 0; i < rep->history_length; ++i) history[i] = r.history[i];
}

SolverOpts to_opts(const bddc_solver_options* o) {
    SolverOpts s;
    if (o) {
        s.rel_tolerance = o->rel_tolerance;
        s.abs_tolerance = o->abs_tolerance;
        s.max_iterations = o->max_iterations;
        s.record_history = o->record_history != 0;
    }
    return s;
}

GpuOptions to_gpu(const bddc_gpu_options* o) {
    GpuOptions g;
    if (o) {
        g.device = o->device;
        g.workers = o->workers;
        g.coarse_mode = o->coarse_mode;
        g.coarse_rtol = o->coarse_rel_tolerance;
        g.coarse_atol = o->coarse_abs_tolerance;
        g.coarse_max_iterations = o->coarse_max_iterations;
        if (o->leaf_size > 0) g.leaf_size = o->leaf_size;
        if (o->local_blocks > 0) g.local_blocks = o->local_blocks;
        if (o->solve_parts > 0) g.solve_parts = o->solve_parts;
        g.setup_on_device = o->setup_mode != BDDC_SETUP_HOST;
    }
    return g;
}

void copy_blocks(const SubdomainSetup& S, double* phi, double* lambda, double* aci) {
    if (phi) std::memcpy(phi, S.phi.data(), sizeof(double) * S.phi.size());
    if (lambda) std::memcpy(lambda, S.lambda.data(), sizeof(double) * S.lambda.size());
    if (aci) std::memcpy(aci, S.aci.data(), sizeof(double) * S.aci.size());
}

void copy_coarse(const CsrMatrix& A, int32_t* nnz, int32_t* rp, int32_t* ci, double* v) {
    if (nnz) *nnz = A.nnz();
    if (rp) std::memcpy(rp, A.row_offsets.data(), sizeof(int32_t) * A.row_offsets.size());
    if (ci) std::memcpy(ci, A.col_indices.data(), sizeof(int32_t) * A.col_indices.size());
    if (v) std::memcpy(v, A.values.data(), sizeof(double) * A.values.size());
}

}  // namespace

extern "C" {

const char* bddc_last_error(void) { return g_last_error.c_str(); }
int32_t bddc_abi_version(void) { return 3; }
const char* bddc_switch_name(int32_t i) { return env_switch_name(i); }

int64_t bddc_kernel_launches(void) { return g_kernel_launches.load(); }

void bddc_default_gpu_options(bddc_gpu_options* o) {
    if (!o) return;
    o->device = 0;
    o->workers = 0;
    o->coarse_mode = BDDC_COARSE_DIRECT;
    o->coarse_rel_tolerance = 1e-12;
    o->coarse_abs_tolerance = 0.0;
    o->coarse_max_iterations = 500;
    o->leaf_size = 24;
    o->local_blocks = 8;
    o->setup_mode = BDDC_SETUP_DEVICE;
    o->solve_parts = 0;
}

void bddc_default_solver_options(bddc_solver_options* o) {
    if (!o) return;
    o->rel_tolerance = 1e-8;
    o->abs_tolerance = 0.0;
    o->max_iterations = 1000;
    o->record_history = 0;
}

int bddc_problem_poisson(int32_t cells_x, int32_t cells_y, int32_t kx, int32_t ky, double kappa_decades,
                         uint64_t kappa_seed, uint64_t rhs_seed, bddc_problem** out) {
    return guarded([&] {
        if (!out) throw std::invalid_argument("bddc_problem_poisson: null output");
        auto p = std::make_unique<bddc_problem>();
        std::vector<double> kappa;
        if (kappa_decades != 0.0) kappa = log_uniform_kappa(cells_x, cells_y, kappa_decades, kappa_seed);
        PoissonProblem pb = assemble_poisson(cells_x, cells_y, kx, ky, kappa.empty() ? nullptr : kappa.data());
        p->data.constraints = build_constraints(pb.decomposition);
        p->data.decomposition = std::move(pb.decomposition);
        p->data.global_matrix = std::move(pb.global_matrix);
        p->data.local_matrices = std::move(pb.local_matrices);
        p->data.coords = std::move(pb.coords);
        p->rhs = study_rhs(p->data.decomposition.global_dofs, rhs_seed);
        p->flatten();
        *out = p.release();
    });
}

int bddc_problem_from_view(const bddc_problem_view* v, bddc_problem** out) {
    return guarded([&] {
        if (!v || !out) throw std::invalid_argument("bddc_problem_from_view: null argument");
        if (v->n_subdomains < 1 || v->global_dofs < 0) throw std::invalid_argument("bddc_problem_from_view: bad sizes");
        auto p = std::make_unique<bddc_problem>();
        ProblemData& pd = p->data;
        Decomposition& d = pd.decomposition;
        d.n_subdomains = v->n_subdomains;
        d.global_dofs = v->global_dofs;
        d.subdomain_dofs.resize(d.n_subdomains);
        d.weights.resize(d.n_subdomains);
        d.interior_counts.assign(v->interior_counts, v->interior_counts + d.n_subdomains);
        for (index_t i = 0; i < d.n_subdomains; ++i) {
            const std::int64_t b = v->dof_offsets[i], e = v->dof_offsets[i + 1];
            d.subdomain_dofs[i].assign(v->subdomain_dofs + b, v->subdomain_dofs + e);
            d.weights[i].assign(v->weights + b, v->weights + e);
            for (index_t g : d.subdomain_dofs[i])
                if (g < 0 || g >= d.global_dofs) throw std::invalid_argument("subdomain map: dof out of range");
        }
        d.classes.resize(d.global_dofs);
        d.multiplicity.assign(d.global_dofs, 0);
        for (index_t g = 0; g < d.global_dofs; ++g) {
            d.classes[g].kind = v->class_kind ? static_cast<DofKind>(v->class_kind[g]) : DofKind::interior;
            d.classes[g].entity = v->class_entity ? v->class_entity[g] : -1;
        }
        if (v->multiplicity) d.multiplicity.assign(v->multiplicity, v->multiplicity + d.global_dofs);
        else
            for (const auto& dofs : d.subdomain_dofs)
                for (index_t g : dofs) d.multiplicity[g]++;
        if (!v->class_kind)
            for (index_t g = 0; g < d.global_dofs; ++g)
                d.classes[g].kind = d.multiplicity[g] > 1 ? DofKind::edge : DofKind::interior;
        pd.global_matrix = copy_csr(v->global_matrix);
        for (index_t i = 0; i < d.n_subdomains; ++i) {
            pd.local_matrices.push_back(copy_csr(v->local_matrices[i]));
            pd.constraints.constraint_matrices.push_back(copy_csr(v->constraint_matrices[i]));
            pd.constraints.primal_maps.emplace_back(v->primal_maps + v->primal_offsets[i],
                                                    v->primal_maps + v->primal_offsets[i + 1]);
        }
        pd.constraints.n_coarse = v->n_coarse;
        if (v->coords) pd.coords.assign(v->coords, v->coords + 2 * static_cast<std::size_t>(d.global_dofs));
        if (v->rhs) p->rhs.assign(v->rhs, v->rhs + d.global_dofs);
        p->flatten();
        *out = p.release();
    });
}

int bddc_problem_get_view(const bddc_problem* p, bddc_problem_view* v) {
    return guarded([&] {
        if (!p || !v) throw std::invalid_argument("bddc_problem_get_view: null argument");
        const ProblemData& pd = p->data;
        const Decomposition& d = pd.decomposition;
        std::memset(v, 0, sizeof *v);
        v->n_subdomains = d.n_subdomains;
        v->global_dofs = d.global_dofs;
        v->n_coarse = pd.constraints.n_coarse;
        const CsrMatrix& A = pd.global_matrix;
        v->global_matrix = {A.nrows, A.ncols, A.row_offsets.data(), A.col_indices.data(), A.values.data()};
        v->local_matrices = p->local_views.data();
        v->constraint_matrices = p->constraint_views.data();
        v->dof_offsets = p->dof_offsets.data();
        v->subdomain_dofs = p->dofs.data();
        v->weights = p->weights.data();
        v->interior_counts = d.interior_counts.data();
        v->primal_offsets = p->primal_offsets.data();
        v->primal_maps = p->primal.data();
        v->class_kind = p->kind.data();
        v->class_entity = p->entity.data();
        v->multiplicity = d.multiplicity.data();
        v->coords = pd.coords.empty() ? nullptr : pd.coords.data();
        v->rhs = p->rhs.empty() ? nullptr : p->rhs.data();
    });
}

int bddc_problem_export_bundle(const bddc_problem* p, const char* directory) {
    return guarded([&] {
        if (!p || !directory) throw std::invalid_argument("bddc_problem_export_bundle: null argument");
        export_bundle(p->data.decomposition, p->data.local_matrices, p->rhs, directory);
    });
}

int bddc_problem_ingest_bundle(const char* manifest_path, bddc_problem** out) {
    return guarded([&] {
        if (!manifest_path || !out) throw std::invalid_argument("bddc_problem_ingest_bundle: null argument");
        IngestedProblem ing = ingest_bundle(manifest_path);
        auto p = std::make_unique<bddc_problem>();
        p->data.decomposition = std::move(ing.decomposition);
        p->data.local_matrices = std::move(ing.local_matrices);
        p->data.constraints = std::move(ing.constraints);
        p->data.global_matrix = std::move(ing.global_matrix);
        p->rhs = std::move(ing.rhs);
        p->flatten();
        *out = p.release();
    });
}

void bddc_problem_destroy(bddc_problem* p) { delete p; }

int bddc_host_setup_create(const bddc_problem* p, const bddc_gpu_options* opt, bddc_host_setup** out) {
    return guarded([&] {
        if (!p || !out) throw std::invalid_argument("bddc_host_setup_create: null argument");
        const GpuOptions g = to_gpu(opt);
        FactorOptions fo;
        fo.leaf_size = g.leaf_size;
        auto s = std::make_unique<bddc_host_setup>();
        s->problem = p;
        const int workers = g.workers > 0 ? g.workers : 8;
        s->setup = bddc_setup(p->data.local_matrices, p->data.decomposition, p->data.constraints,
                              p->data.coords.empty() ? nullptr : p->data.coords.data(), workers, fo);
        *out = s.release();
    });
}

int bddc_host_setup_blocks(const bddc_host_setup* s, int32_t i, double* phi, double* lambda, double* aci) {
    return guarded([&] {
        if (!s) throw std::invalid_argument("null setup");
        if (i < 0 || i >= static_cast<int32_t>(s->setup.subs.size())) throw std::out_of_range("subdomain index");
        copy_blocks(s->setup.subs[i], phi, lambda, aci);
    });
}

int bddc_host_setup_coarse(const bddc_host_setup* s, int32_t* nnz, int32_t* rp, int32_t* ci, double* v) {
    return guarded([&] {
        if (!s) throw std::invalid_argument("null setup");
        copy_coarse(s->setup.coarse_matrix, nnz, rp, ci, v);
    });
}

int bddc_host_setup_interior_solve(const bddc_host_setup* s, int32_t i, double* x) {
    return guarded([&] {
        if (!s || !x) throw std::invalid_argument("null argument");
        if (i < 0 || i >= static_cast<int32_t>(s->setup.subs.size())) throw std::out_of_range("subdomain index");
        factor_solve(s->setup.subs[i].factor, x, 1);
    });
}

int bddc_host_setup_stats(const bddc_host_setup* s, bddc_stats* st) {
    return guarded([&] {
        if (!s || !st) throw std::invalid_argument("null argument");
        std::memset(st, 0, sizeof *st);
        st->setup_seconds = s->setup.seconds;
        for (const auto& sub : s->setup.subs) {
            st->factor_values += sub.factor.factor_values();
            st->interior_dofs += sub.n_interior;
            st->max_interior = std::max(st->max_interior, sub.n_interior);
            st->max_interface = std::max(st->max_interface, sub.n_iface);
        }
        st->n_subdomains = static_cast<int32_t>(s->setup.subs.size());
        st->global_dofs = s->problem->data.decomposition.global_dofs;
        st->n_coarse = s->setup.coarse_matrix.nrows;
        st->unique_subdomains = s->setup.unique_subdomains;
    });
}

void bddc_host_setup_destroy(bddc_host_setup* s) { delete s; }

int bddc_gpu_create(const bddc_problem* p, const bddc_gpu_options* opt, bddc_gpu_ctx** out) {
    return guarded([&] {
        if (!p || !out) throw std::invalid_argument("bddc_gpu_create: null argument");
        auto c = std::make_unique<bddc_gpu_ctx>();
        c->ctx = std::make_unique<GpuContext>(std::shared_ptr<const ProblemData>(p->shared), to_gpu(opt));
        *out = c.release();
    });
}

int bddc_dist_unique_id(uint8_t* id) {
    return guarded([&] {
        if (!id) throw std::invalid_argument("bddc_dist_unique_id: null argument");
        char buf[128];
        dist_nccl_id(buf);
        std::memcpy(id, buf, 128);
    });
}

int bddc_gpu_create_dist(const bddc_problem* p, const bddc_gpu_options* opt, const bddc_dist_options* dist,
                         bddc_gpu_ctx** out) {
    return guarded([&] {
        if (!p || !dist || !out) throw std::invalid_argument("bddc_gpu_create_dist: null argument");
        if (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world)
            throw std::invalid_argument("bddc_gpu_create_dist: bad rank / world");
        DistSpec spec;
        spec.rank = dist->rank;
        spec.world = dist->world;
        std::memcpy(spec.nccl_id, dist->nccl_id, 128);
        if (dist->subdomain_rank)
            spec.sub_rank.assign(dist->subdomain_rank, dist->subdomain_rank + p->data.decomposition.n_subdomains);
        auto c = std::make_unique<bddc_gpu_ctx>();
        c->ctx = std::make_unique<GpuContext>(std::shared_ptr<const ProblemData>(p->shared), to_gpu(opt), &spec);
        *out = c.release();
    });
}

int bddc_gpu_layout(const bddc_gpu_ctx* c, int32_t* n_local, int32_t* n_rows, int32_t* n_owned,
                    int32_t* local_to_global) {
    return guarded([&] {
        if (!c) throw std::invalid_argument("bddc_gpu_layout: null context");
        const GpuContext& g = *c->ctx;
        if (n_local) *n_local = g.n();
        if (n_rows) *n_rows = g.n_rows();
        if (n_owned) *n_owned = g.n_owned();
        if (local_to_global) {
            const auto& l2g = g.local_to_global();
            if (l2g.empty())
                for (index_t l = 0; l < g.n(); ++l) local_to_global[l] = l;
            else
                std::memcpy(local_to_global, l2g.data(), sizeof(int32_t) * l2g.size());
        }
    });
}

int bddc_rank_plan_create(const bddc_problem* p, int32_t rank, int32_t world, const int32_t* subdomain_rank,
                          bddc_rank_plan** out) {
    return guarded([&] {
        if (!p || !out) throw std::invalid_argument("bddc_rank_plan_create: null argument");
        auto r = std::make_unique<bddc_rank_plan>();
        r->plan = make_rank_plan(p->data, rank, world, subdomain_rank);
        r->local.data = std::move(r->plan.local);
        r->plan.local = ProblemData{};
        r->local.rhs.resize(r->local.data.decomposition.global_dofs);
        if (!p->rhs.empty())
            for (index_t l = 0; l < r->plan.n_local; ++l) r->local.rhs[l] = p->rhs[r->plan.local_to_global[l]];
        r->local.flatten();
        r->remote_ptr.assign(1, 0);
        for (const auto& lst : r->plan.remote_owners) {
            for (const auto& [gsub, k] : lst) {
                r->remote_sub.push_back(gsub);
                r->remote_slot.push_back(k);
            }
            r->remote_ptr.push_back(static_cast<std::int32_t>(r->remote_sub.size()));
        }
        *out = r.release();
    });
}

int bddc_rank_plan_get_view(const bddc_rank_plan* r, bddc_rank_plan_view* v) {
    return guarded([&] {
        if (!r || !v) throw std::invalid_argument("bddc_rank_plan_get_view: null argument");
        const RankPlan& P = r->plan;
        std::memset(v, 0, sizeof *v);
        v->rank = P.rank;
        v->world = P.world;
        v->n_local = P.n_local;
        v->n_rows = P.n_rows;
        v->n_owned = P.n_owned;
        v->n_subdomains_global = static_cast<int32_t>(P.sub_rank.size());
        v->local_to_global = P.local_to_global.data();
        v->subdomain_rank = P.sub_rank.data();
        v->n_local_subdomains = static_cast<int32_t>(P.subdomains.size());
        v->subdomains = P.subdomains.data();
        v->n_halo_peers = static_cast<int32_t>(P.halo_peers.size());
        v->halo_peers = P.halo_peers.data();
        v->halo_send_off = P.halo_send_off.data();
        v->halo_send_idx = P.halo_send_idx.data();
        v->halo_recv_off = P.halo_recv_off.data();
        v->n_iface_peers = static_cast<int32_t>(P.iface_peers.size());
        v->iface_peers = P.iface_peers.data();
        v->iface_send_off = P.iface_send_off.data();
        v->iface_send_slot = P.iface_send_slot.data();
        v->iface_recv_off = P.iface_recv_off.data();
        v->n_local_slots = P.n_local_slots;
        v->n_remote_slots = P.n_remote_slots;
        v->remote_ptr = r->remote_ptr.data();
        v->remote_subdomain = r->remote_sub.data();
        v->remote_slot = r->remote_slot.data();
        v->cbuf_pad = P.cbuf_pad;
        v->cbuf_offset = P.cbuf_offset.data();
        v->local_problem = &r->local;
    });
}

void bddc_rank_plan_destroy(bddc_rank_plan* r) { delete r; }

int bddc_gpu_apply(bddc_gpu_ctx* c, const double* r, double* z) {
    return guarded([&] {
        if (!c || !r || !z) throw std::invalid_argument("bddc_gpu_apply: null argument");
        c->ctx->apply_host(r, z);
    }, c);
}

int bddc_gpu_apply_device(bddc_gpu_ctx* c, const double* r, double* z, void* stream) {
    return guarded([&] {
        if (!c || !r || !z) throw std::invalid_argument("bddc_gpu_apply_device: null argument");
        c->ctx->apply_device(r, z, stream);
    }, c);
}

int bddc_gpu_stage(bddc_gpu_ctx* c, int32_t stage, const double* in0, const double* in1,
                   const double* in2, double* out) {
    return guarded([&] {
        if (!c || !in0 || !out) throw std::invalid_argument("bddc_gpu_stage: null argument");
        if (stage < 0 || stage > 3) throw std::invalid_argument("bddc_gpu_stage: unknown stage");
        if (stage == BDDC_STAGE_STATIC_CONDENSATION && (!in1 || !in2))
            throw std::invalid_argument("bddc_gpu_stage: static condensation needs r, v1, v2");
        c->ctx->stage_host(static_cast<Stage>(stage), in0, in1, in2, out);
    }, c);
}

int bddc_gpu_pcg(bddc_gpu_ctx* c, const double* b, const bddc_solver_options* opt, int32_t precondition,
                 double* x, bddc_solve_report* rep, double* history, int32_t cap) {
    return guarded([&] {
        if (!c || !b || !x) throw std::invalid_argument("bddc_gpu_pcg: null argument");
        const SolveResult r = c->ctx->pcg_host(b, to_opts(opt), x, precondition != 0);
        fill_report(r, rep, history, cap);
    }, c);
}

int bddc_gpu_pcg_device(bddc_gpu_ctx* c, const double* b, const bddc_solver_options* opt,
                        int32_t precondition, double* x, bddc_solve_report* rep, double* history,
                        int32_t cap, void* stream) {
    return guarded([&] {
        if (!c || !b || !x) throw std::invalid_argument("bddc_gpu_pcg_device: null argument");
        const SolveResult r = c->ctx->pcg_device(b, to_opts(opt), x, precondition != 0, stream);
        fill_report(r, rep, history, cap);
    }, c);
}

int bddc_gpu_subdomain_blocks(const bddc_gpu_ctx* c, int32_t i, double* phi, double* lambda, double* aci) {
    return guarded([&] {
        if (!c) throw std::invalid_argument("null context");
        const auto& subs = c->ctx->setup().subs;
        if (i < 0 || i >= static_cast<int32_t>(subs.size())) throw std::out_of_range("subdomain index");
        c->ctx->subdomain_blocks(i, phi, lambda, aci);
    });
}

int bddc_gpu_coarse_matrix(const bddc_gpu_ctx* c, int32_t* nnz, int32_t* rp, int32_t* ci, double* v) {
    return guarded([&] {
        if (!c) throw std::invalid_argument("null context");
        copy_coarse(c->ctx->setup().coarse_matrix, nnz, rp, ci, v);
    });
}

int bddc_gpu_get_stats(const bddc_gpu_ctx* c, bddc_stats* st) {
    return guarded([&] {
        if (!c || !st) throw std::invalid_argument("null argument");
        std::memset(st, 0, sizeof *st);
        const GpuContext& g = *c->ctx;
        st->setup_seconds = g.setup_seconds();
        st->factor_values = g.factor_values();
        st->interior_solve_bytes = g.interior_pass_bytes();
        st->apply_bytes = g.apply_bytes();
        st->interior_apply_bytes = g.interior_apply_bytes();
        st->n_subdomains = g.problem().decomposition.n_subdomains;
        st->global_dofs = g.problem().decomposition.global_dofs;
        st->n_coarse = g.problem().constraints.n_coarse;
        st->unique_subdomains = g.setup().unique_subdomains;
        st->graph_captures = g.graph_captures();
        st->coarse_mode = g.coarse_mode();
        st->switches = g.switches();
        st->setup_device_seconds = g.setup_device_seconds();
        for (const auto& sub : g.setup().subs) {
            st->interior_dofs += sub.n_interior;
            st->max_interior = std::max(st->max_interior, sub.n_interior);
            st->max_interface = std::max(st->max_interface, sub.n_iface);
        }
    });
}

int bddc_gpu_set_profile(bddc_gpu_ctx* c, int32_t on) {
    return guarded([&] {
        if (!c) throw std::invalid_argument("null context");
        c->ctx->set_profile(on != 0);
    }, c);
}

int bddc_gpu_kernel_times(const bddc_gpu_ctx* c, bddc_kernel_times* t, int32_t reset) {
    return guarded([&] {
        if (!c || !t) throw std::invalid_argument("null argument");
        GpuContext& g = const_cast<GpuContext&>(*c->ctx);
        const KernelTimes k = g.kernel_times();
        t->interior_ms = k.interior_ms;
        t->interior_launches = k.interior_launches;
        t->iface_ms = k.iface_ms;
        t->apply_ms = k.apply_ms;
        t->applies = k.applies;
        if (reset) g.reset_kernel_times();
    });
}

int bddc_gpu_synchronize(bddc_gpu_ctx* c) {
    return guarded([&] {
        if (!c) throw std::invalid_argument("null context");
        c->ctx->synchronize();
    }, c);
}

int64_t bddc_gpu_solve_profile(bddc_gpu_ctx* c, int64_t* out, int64_t cap) {
    std::int64_t n = 0;
    const int rc = guarded([&] {
        if (!c || !out) throw std::invalid_argument("null argument");
        n = c->ctx->solve_profile(out, cap);
    }, c);
    return rc == BDDC_OK ? n : -1;
}

const char* bddc_gpu_last_error(const bddc_gpu_ctx* c) { return c ? c->last_error.c_str() : g_last_error.c_str(); }

void bddc_gpu_destroy(bddc_gpu_ctx* c) { delete c; }

}  // extern "C"
