"""Python mirror of the reference solver/preconditioner API over the C-ABI.

Names and argument meaning follow the reference C++ API (/root/reference/proj):
  Problem.poisson      -> assemble_poisson + build_constraints + study_rhs
                          (src/decomposition.cpp:161-203, :112-159; src/study.cpp:69-75)
  Preconditioner       -> bddc::Preconditioner (include/bddc/preconditioner.hpp:62-104)
  Preconditioner.apply / coarse_correction / local_correction / interior_correction /
  static_condensation_correction  -> src/preconditioner.cpp:129-249
  pcg                  -> bddc::pcg (include/bddc/pcg.hpp:43-45)
  SolverOptions / SolveReport -> include/bddc/pcg.hpp:17-30
Errors map back to the reference's exception types: InvalidArgument (ValueError) for
std::invalid_argument, OutOfRange (IndexError) for std::out_of_range, BddcError for
std::runtime_error, messages verbatim.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


@dataclass
class SolverOptions:
    rel_tolerance: float = 1e-8
    abs_tolerance: float = 0.0
    max_iterations: int = 1000
    record_history: bool = False

    def c(self) -> L.SolverOptions:
        return L.SolverOptions(self.rel_tolerance, self.abs_tolerance, self.max_iterations,
                               1 if self.record_history else 0)


@dataclass
class SolveReport:
    iterations: int = 0
    final_relative_residual: float = 0.0
    residual_history: list = field(default_factory=list)
    condition_estimate: float | None = None
    converged: bool = False


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _csr(view: L.CsrView):
    n = view.nrows
    rp = np.ctypeslib.as_array(view.row_offsets, shape=(n + 1,)).copy()
    nnz = int(rp[-1])
    cols = np.ctypeslib.as_array(view.col_indices, shape=(max(nnz, 1),))[:nnz].copy() if nnz else np.zeros(0, np.int32)
    vals = np.ctypeslib.as_array(view.values, shape=(max(nnz, 1),))[:nnz].copy() if nnz else np.zeros(0)
    return (int(view.nrows), int(view.ncols), rp, cols, vals)


class Problem:
    """A decomposed problem owned by the native library (bddc_problem*)."""

    def __init__(self, handle: int, owner=None):
        self._h = C.c_void_p(handle)
        self._owner = owner  # borrowed handle (e.g. a RankPlan's local problem): never destroyed here
        self._view = L.ProblemView()
        L.check(L.lib().bddc_problem_get_view(self._h, C.byref(self._view)))

    @classmethod
    def poisson(cls, cells_x: int, kx: int, cells_y: int | None = None, ky: int | None = None,
                kappa_decades: float = 0.0, kappa_seed: int = 0x5EED, rhs_seed: int = 1) -> "Problem":
        h = C.c_void_p()
        L.check(L.lib().bddc_problem_poisson(cells_x, cells_y or cells_x, kx, ky or kx, kappa_decades,
                                             kappa_seed, rhs_seed, C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_bundle(cls, manifest_path: str) -> "Problem":
        """Reference bundle ingestion (src/bundle.cpp:113-290, `ingest_bundle`): the local
        matrices, maps, classes and rhs of an external (e.g. openCARP-exported) problem."""
        h = C.c_void_p()
        L.check(L.lib().bddc_problem_ingest_bundle(manifest_path.encode(), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_arrays(cls, global_matrix, local_matrices, subdomain_dofs, interior_counts, weights,
                    constraint_matrices, primal_maps, n_coarse, class_kind=None, class_entity=None,
                    multiplicity=None, rhs=None, coords=None) -> "Problem":
        """Drop-in path for externally decomposed problems (the reference's in-memory
        Decomposition + ConstraintSet + matrices). CSR arguments are (nrows, ncols, rowptr,
        cols, vals) tuples; everything is deep-copied by the library."""
        keep = []

        def arr(a, dt):
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a

        def csr(m):
            nr, nc, rp, ci, va = m
            rp, ci, va = arr(rp, np.int32), arr(ci, np.int32), arr(va, np.float64)
            return L.CsrView(int(nr), int(nc), rp.ctypes.data_as(C.POINTER(C.c_int32)),
                             ci.ctypes.data_as(C.POINTER(C.c_int32)), va.ctypes.data_as(C.POINTER(C.c_double)))

        ns = len(local_matrices)
        v = L.ProblemView()
        v.n_subdomains, v.global_dofs, v.n_coarse = ns, int(global_matrix[0]), int(n_coarse)
        v.global_matrix = csr(global_matrix)
        locs = (L.CsrView * ns)(*[csr(m) for m in local_matrices])
        cons = (L.CsrView * ns)(*[csr(m) for m in constraint_matrices])
        keep += [locs, cons]
        v.local_matrices, v.constraint_matrices = locs, cons
        doff = arr(np.concatenate([[0], np.cumsum([len(d) for d in subdomain_dofs])]), np.int64)
        poff = arr(np.concatenate([[0], np.cumsum([len(p) for p in primal_maps])]), np.int64)
        ptr = lambda a, t: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
        v.dof_offsets = ptr(doff, C.c_int64)
        v.subdomain_dofs = ptr(arr(np.concatenate(subdomain_dofs), np.int32), C.c_int32)
        v.weights = ptr(arr(np.concatenate(weights), np.float64), C.c_double)
        v.interior_counts = ptr(arr(interior_counts, np.int32), C.c_int32)
        v.primal_offsets = ptr(poff, C.c_int64)
        v.primal_maps = ptr(arr(np.concatenate(primal_maps), np.int32), C.c_int32)
        if class_kind is not None:
            v.class_kind = ptr(arr(class_kind, np.uint8), C.c_uint8)
        if class_entity is not None:
            v.class_entity = ptr(arr(class_entity, np.int32), C.c_int32)
        if multiplicity is not None:
            v.multiplicity = ptr(arr(multiplicity, np.int32), C.c_int32)
        if rhs is not None:
            v.rhs = ptr(arr(rhs, np.float64), C.c_double)
        if coords is not None:
            v.coords = ptr(arr(coords, np.int32), C.c_int32)
        h = C.c_void_p()
        L.check(L.lib().bddc_problem_from_view(C.byref(v), C.byref(h)))
        return cls(h.value)

    def coords(self):
        v = self._view
        return self._arr(v.coords, 2 * v.global_dofs) if v.coords else None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value and getattr(self, "_owner", None) is None:
            try:
                L.lib().bddc_problem_destroy(h)
            except TypeError:  # interpreter shutdown: the module globals are already gone
                return
            self._h = C.c_void_p()

    @property
    def handle(self):
        return self._h

    @property
    def global_dofs(self) -> int:
        return int(self._view.global_dofs)

    @property
    def n_subdomains(self) -> int:
        return int(self._view.n_subdomains)

    @property
    def n_coarse(self) -> int:
        return int(self._view.n_coarse)

    def _arr(self, ptr, n, dtype=None):
        if n == 0:
            return np.zeros(0, dtype=dtype or np.float64)
        return np.ctypeslib.as_array(ptr, shape=(n,)).copy()

    def rhs(self) -> np.ndarray:
        v = self._view
        return self._arr(v.rhs, v.global_dofs) if v.rhs else np.zeros(v.global_dofs)

    def dof_offsets(self) -> np.ndarray:
        return self._arr(self._view.dof_offsets, self.n_subdomains + 1)

    def subdomain_dofs(self) -> list:
        off = self.dof_offsets()
        flat = self._arr(self._view.subdomain_dofs, int(off[-1]))
        return [flat[off[i]:off[i + 1]] for i in range(self.n_subdomains)]

    def weights(self) -> list:
        off = self.dof_offsets()
        flat = self._arr(self._view.weights, int(off[-1]))
        return [flat[off[i]:off[i + 1]] for i in range(self.n_subdomains)]

    def interior_counts(self) -> np.ndarray:
        return self._arr(self._view.interior_counts, self.n_subdomains)

    def primal_maps(self) -> list:
        off = self._arr(self._view.primal_offsets, self.n_subdomains + 1)
        flat = self._arr(self._view.primal_maps, int(off[-1]))
        return [flat[off[i]:off[i + 1]] for i in range(self.n_subdomains)]

    def classes(self):
        n = self.global_dofs
        return self._arr(self._view.class_kind, n), self._arr(self._view.class_entity, n)

    def multiplicity(self) -> np.ndarray:
        return self._arr(self._view.multiplicity, self.global_dofs)

    def global_matrix(self):
        return _csr(self._view.global_matrix)

    def local_matrix(self, i: int):
        return _csr(self._view.local_matrices[i])

    def constraint_matrix(self, i: int):
        return _csr(self._view.constraint_matrices[i])

    def export_bundle(self, directory: str) -> str:
        L.check(L.lib().bddc_problem_export_bundle(self._h, directory.encode()))
        return directory.rstrip("/") + "/manifest.txt"


def gpu_options(device=0, workers=0, coarse_mode="direct", coarse_options: SolverOptions | None = None,
                leaf_size=24, local_blocks=8, solve_parts=0, setup="device") -> L.GpuOptions:
    o = L.GpuOptions()
    L.lib().bddc_default_gpu_options(C.byref(o))
    o.device, o.workers = device, workers
    o.coarse_mode = L.COARSE_CG if coarse_mode == "cg" else L.COARSE_DIRECT
    if coarse_options is not None:
        o.coarse_rel_tolerance = coarse_options.rel_tolerance
        o.coarse_abs_tolerance = coarse_options.abs_tolerance
        o.coarse_max_iterations = coarse_options.max_iterations
    o.leaf_size, o.local_blocks, o.solve_parts = leaf_size, local_blocks, solve_parts
    if setup not in ("device", "host"):
        raise ValueError("setup must be 'device' or 'host'")
    o.setup_mode = 1 if setup == "host" else 0
    return o


class HostSetup:
    """Host-side setup only (no GPU): factors, Phi/Lambda/A_ci, A_c. Test tooling."""

    def __init__(self, problem: Problem, **kw):
        self.problem = problem
        h = C.c_void_p()
        L.check(L.lib().bddc_host_setup_create(problem.handle, C.byref(gpu_options(**kw)), C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            L.lib().bddc_host_setup_destroy(self._h)
            self._h = C.c_void_p()

    def blocks(self, i: int):
        nl = len(self.problem.subdomain_dofs()[i])
        npr = len(self.problem.primal_maps()[i])
        phi, lam, aci = np.zeros(nl * npr), np.zeros(npr * npr), np.zeros(npr * npr)
        L.check(L.lib().bddc_host_setup_blocks(self._h, i, _dptr(phi), _dptr(lam), _dptr(aci)))
        return phi.reshape(nl, npr), lam.reshape(npr, npr), aci.reshape(npr, npr)

    def coarse_matrix(self):
        nnz = C.c_int32()
        L.check(L.lib().bddc_host_setup_coarse(self._h, C.byref(nnz), None, None, None))
        n = self.problem.n_coarse
        rp, ci, v = np.zeros(n + 1, np.int32), np.zeros(nnz.value, np.int32), np.zeros(nnz.value)
        L.check(L.lib().bddc_host_setup_coarse(self._h, None, rp.ctypes.data_as(C.POINTER(C.c_int32)),
                                               ci.ctypes.data_as(C.POINTER(C.c_int32)), _dptr(v)))
        return rp, ci, v

    def interior_solve(self, i: int, b: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(b, dtype=np.float64).copy()
        L.check(L.lib().bddc_host_setup_interior_solve(self._h, i, _dptr(x)))
        return x

    def stats(self) -> dict:
        s = L.Stats()
        L.check(L.lib().bddc_host_setup_stats(self._h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in L.Stats._fields_}


def _i32(ptr, n) -> np.ndarray:
    if n <= 0:
        return np.zeros(0, dtype=np.int32)
    return np.ctypeslib.as_array(ptr, shape=(n,)).copy()


class RankPlan:
    """Host-only view of one rank's partition of a problem (bddc_rank_plan_*): the rank-local
    vector layout, halo / interface exchange lists and the gathered coarse layout."""

    def __init__(self, problem: Problem, rank: int, world: int, subdomain_rank=None):
        self.problem = problem
        h = C.c_void_p()
        sr = None
        if subdomain_rank is not None:
            self._sr = np.ascontiguousarray(subdomain_rank, dtype=np.int32)
            sr = self._sr.ctypes.data_as(C.POINTER(C.c_int32))
        L.check(L.lib().bddc_rank_plan_create(problem.handle, rank, world, sr, C.byref(h)))
        self._h = h
        v = L.RankPlanView()
        L.check(L.lib().bddc_rank_plan_get_view(h, C.byref(v)))
        self.rank, self.world = v.rank, v.world
        self.n_local, self.n_rows, self.n_owned = v.n_local, v.n_rows, v.n_owned
        self.local_to_global = _i32(v.local_to_global, v.n_local)
        self.subdomain_rank = _i32(v.subdomain_rank, v.n_subdomains_global)
        self.subdomains = _i32(v.subdomains, v.n_local_subdomains)
        self.halo_peers = _i32(v.halo_peers, v.n_halo_peers)
        self.halo_send_off = _i32(v.halo_send_off, v.n_halo_peers + 1)
        self.halo_send_idx = _i32(v.halo_send_idx, int(self.halo_send_off[-1]))
        self.halo_recv_off = _i32(v.halo_recv_off, v.n_halo_peers + 1)
        self.iface_peers = _i32(v.iface_peers, v.n_iface_peers)
        self.iface_send_off = _i32(v.iface_send_off, v.n_iface_peers + 1)
        self.iface_send_slot = _i32(v.iface_send_slot, int(self.iface_send_off[-1]))
        self.iface_recv_off = _i32(v.iface_recv_off, v.n_iface_peers + 1)
        self.n_local_slots, self.n_remote_slots = v.n_local_slots, v.n_remote_slots
        self.remote_ptr = _i32(v.remote_ptr, v.n_rows + 1)
        self.remote_subdomain = _i32(v.remote_subdomain, int(self.remote_ptr[-1]))
        self.remote_slot = _i32(v.remote_slot, int(self.remote_ptr[-1]))
        self.cbuf_pad = v.cbuf_pad
        self.cbuf_offset = _i32(v.cbuf_offset, v.n_subdomains_global)
        self.local_problem = Problem(v.local_problem, owner=self)

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            L.lib().bddc_rank_plan_destroy(self._h)
            self._h = C.c_void_p()


def dist_unique_id() -> bytes:
    """A fresh 128-byte NCCL unique id (rank 0 creates it; broadcast it to the other ranks)."""
    buf = (C.c_uint8 * 128)()
    L.check(L.lib().bddc_dist_unique_id(buf))
    return bytes(buf)


class Preconditioner:
    """B200 BDDC preconditioner (reference bddc::Preconditioner semantics).

    dist=(rank, world, nccl_id[, subdomain_rank]) builds one rank of a multi-GPU
    preconditioner from the GLOBAL problem (every rank passes the same problem); host-vector
    calls then take global vectors and fill the entries of the rank's subdomains."""

    def __init__(self, problem: Problem, device: int = 0, workers: int = 0, coarse_mode: str = "direct",
                 coarse_options: SolverOptions | None = None, leaf_size: int = 24, local_blocks: int = 8,
                 solve_parts: int = 0, dist=None, setup: str = "device"):
        self.problem = problem
        self.n = problem.global_dofs
        h = C.c_void_p()
        opts = gpu_options(device, workers, coarse_mode, coarse_options, leaf_size, local_blocks, solve_parts, setup)
        if dist is None:
            L.check(L.lib().bddc_gpu_create(problem.handle, C.byref(opts), C.byref(h)))
        else:
            d = L.DistOptions()
            d.rank, d.world = int(dist[0]), int(dist[1])
            C.memmove(d.nccl_id, bytes(dist[2]), 128)
            if len(dist) > 3 and dist[3] is not None:
                self._sr = np.ascontiguousarray(dist[3], dtype=np.int32)
                d.subdomain_rank = self._sr.ctypes.data_as(C.POINTER(C.c_int32))
            L.check(L.lib().bddc_gpu_create_dist(problem.handle, C.byref(opts), C.byref(d), C.byref(h)))
        self._h = h

    def layout(self):
        """(n_local, n_rows, n_owned, local_to_global) of the device vectors."""
        nl, nr, no = C.c_int32(), C.c_int32(), C.c_int32()
        L.check(L.lib().bddc_gpu_layout(self._h, C.byref(nl), C.byref(nr), C.byref(no), None), self._h)
        l2g = np.zeros(max(nl.value, 1), dtype=np.int32)
        L.check(L.lib().bddc_gpu_layout(self._h, None, None, None, l2g.ctypes.data_as(C.POINTER(C.c_int32))),
                self._h)
        return nl.value, nr.value, no.value, l2g[:nl.value]

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            try:
                L.lib().bddc_gpu_destroy(self._h)
            except TypeError:  # interpreter shutdown: the module globals are already gone
                return
            self._h = C.c_void_p()

    def _vec(self, r) -> np.ndarray:
        r = np.ascontiguousarray(r, dtype=np.float64)
        if r.size != self.n:
            raise L.InvalidArgument(L.ERR_INVALID_ARGUMENT, "bddc apply: residual size mismatch")
        return r

    def apply(self, r) -> np.ndarray:
        r = self._vec(r)
        z = np.empty(self.n)
        L.check(L.lib().bddc_gpu_apply(self._h, _dptr(r), _dptr(z)), self._h)
        return z

    def apply_device(self, r_ptr: int, z_ptr: int, stream: int = 0) -> None:
        L.check(L.lib().bddc_gpu_apply_device(self._h, C.c_void_p(r_ptr), C.c_void_p(z_ptr),
                                              C.c_void_p(stream)), self._h)

    def _stage(self, stage: int, r, v1=None, v2=None) -> np.ndarray:
        r = self._vec(r)
        a = self._vec(v1) if v1 is not None else None
        b = self._vec(v2) if v2 is not None else None
        out = np.empty(self.n)
        L.check(L.lib().bddc_gpu_stage(self._h, stage, _dptr(r), _dptr(a) if a is not None else None,
                                       _dptr(b) if b is not None else None, _dptr(out)), self._h)
        return out

    def interior_correction(self, r):
        return self._stage(L.STAGE_INTERIOR, r)

    def coarse_correction(self, r):
        return self._stage(L.STAGE_COARSE, r)

    def local_correction(self, r):
        return self._stage(L.STAGE_LOCAL, r)

    def static_condensation_correction(self, r, v1, v2):
        return self._stage(L.STAGE_STATIC_CONDENSATION, r, v1, v2)

    def subdomain_blocks(self, i: int):
        nl = len(self.problem.subdomain_dofs()[i])
        npr = len(self.problem.primal_maps()[i])
        phi, lam, aci = np.zeros(nl * npr), np.zeros(npr * npr), np.zeros(npr * npr)
        L.check(L.lib().bddc_gpu_subdomain_blocks(self._h, i, _dptr(phi), _dptr(lam), _dptr(aci)))
        return phi.reshape(nl, npr), lam.reshape(npr, npr), aci.reshape(npr, npr)

    def coarse_matrix(self):
        """A_c (CSR rowptr, cols, values) as assembled by this context (reference CoarseProblem)."""
        nnz = C.c_int32()
        L.check(L.lib().bddc_gpu_coarse_matrix(self._h, C.byref(nnz), None, None, None))
        n = self.problem.n_coarse
        rp, ci, v = np.zeros(n + 1, np.int32), np.zeros(nnz.value, np.int32), np.zeros(nnz.value)
        L.check(L.lib().bddc_gpu_coarse_matrix(self._h, None, rp.ctypes.data_as(C.POINTER(C.c_int32)),
                                               ci.ctypes.data_as(C.POINTER(C.c_int32)), _dptr(v)))
        return rp, ci, v

    def stats(self) -> dict:
        s = L.Stats()
        L.check(L.lib().bddc_gpu_get_stats(self._h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in L.Stats._fields_}

    def set_profile(self, on: bool) -> None:
        L.check(L.lib().bddc_gpu_set_profile(self._h, 1 if on else 0), self._h)

    def kernel_times(self, reset: bool = False) -> dict:
        t = L.KernelTimes()
        L.check(L.lib().bddc_gpu_kernel_times(self._h, C.byref(t), 1 if reset else 0))
        return {k: getattr(t, k) for k, _ in L.KernelTimes._fields_}

    def solve_profile(self) -> np.ndarray:
        """Per-CTA, per-warp cycle accounting {total, mbarrier wait, barrier wait, units} of the last
        interior solve, followed by the phase timeline of CTA 0 (diagnostics; BDDC_SOLVE_STATS=1)."""
        cap = 1 << 20
        out = np.zeros(cap, dtype=np.int64)
        n = L.lib().bddc_gpu_solve_profile(self._h, out.ctypes.data_as(C.POINTER(C.c_int64)), cap)
        return out[:max(n, 0)]

    def synchronize(self) -> None:
        L.check(L.lib().bddc_gpu_synchronize(self._h), self._h)

    def pcg(self, b, options: SolverOptions | None = None, precondition: bool = True, out=None):
        """Device-resident PCG with M = self.apply (reference pcg + study.cpp:113-119).
        `out` (optional, float64, length n; e.g. pinned) receives the solution."""
        options = options or SolverOptions()
        b = self._vec(b)
        if out is None:
            x = np.empty(self.n)
        else:
            x = out
            if x.dtype != np.float64 or x.size != self.n or not x.flags.c_contiguous:
                raise L.InvalidArgument(L.ERR_INVALID_ARGUMENT, "pcg: out must be a contiguous float64 vector of size n")
        rep = L.SolveReport()
        cap = options.max_iterations + 1
        hist = np.zeros(cap)
        L.check(L.lib().bddc_gpu_pcg(self._h, _dptr(b), C.byref(options.c()), 1 if precondition else 0,
                                     _dptr(x), C.byref(rep), _dptr(hist), cap), self._h)
        return x, _report(rep, hist)

    def pcg_device(self, b_ptr: int, x_ptr: int, options: SolverOptions | None = None,
                   precondition: bool = True, stream: int = 0):
        options = options or SolverOptions()
        rep = L.SolveReport()
        cap = options.max_iterations + 1
        hist = np.zeros(cap)
        L.check(L.lib().bddc_gpu_pcg_device(self._h, C.c_void_p(b_ptr), C.byref(options.c()),
                                            1 if precondition else 0, C.c_void_p(x_ptr), C.byref(rep),
                                            _dptr(hist), cap, C.c_void_p(stream)), self._h)
        return _report(rep, hist)


def _report(rep: L.SolveReport, hist: np.ndarray) -> SolveReport:
    return SolveReport(rep.iterations, rep.final_relative_residual, hist[:rep.history_length].tolist(),
                       rep.condition_estimate if rep.has_condition_estimate else None, bool(rep.converged))


def pcg(preconditioner: Preconditioner, b, options: SolverOptions | None = None, precondition: bool = True):
    """bddc::pcg(A, b, M, opts, x) with A = the problem's global matrix and M = BDDC apply
    (precondition=False is the reference's empty PreconditionerFn, i.e. plain CG)."""
    return preconditioner.pcg(b, options, precondition)
