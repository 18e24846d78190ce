"""ctypes binding of the C-ABI in include/bddc_b200.h.

Loads the in-tree paper_2410_14786_b200/lib/libbddc_b200.so and fails loudly when it
is missing: there is no Python or CPU fallback for the hot path.
"""
from __future__ import annotations

import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libbddc_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "bddc_b200.h")

OK = 0
ERR_INVALID_ARGUMENT = 1
ERR_RUNTIME = 2
ERR_OUT_OF_RANGE = 3
ERR_CUDA = 4
ERR_NO_DEVICE = 5

STAGE_INTERIOR, STAGE_COARSE, STAGE_LOCAL, STAGE_STATIC_CONDENSATION = 0, 1, 2, 3
COARSE_DIRECT, COARSE_CG = 0, 1

i32, i64, u8, u64, f64 = C.c_int32, C.c_int64, C.c_uint8, C.c_uint64, C.c_double
P = C.POINTER


class CsrView(C.Structure):
    _fields_ = [("nrows", i32), ("ncols", i32), ("row_offsets", P(i32)), ("col_indices", P(i32)),
                ("values", P(f64))]


class ProblemView(C.Structure):
    _fields_ = [
        ("n_subdomains", i32), ("global_dofs", i32), ("n_coarse", i32),
        ("global_matrix", CsrView),
        ("local_matrices", P(CsrView)), ("constraint_matrices", P(CsrView)),
        ("dof_offsets", P(i64)), ("subdomain_dofs", P(i32)), ("weights", P(f64)),
        ("interior_counts", P(i32)), ("primal_offsets", P(i64)), ("primal_maps", P(i32)),
        ("class_kind", P(u8)), ("class_entity", P(i32)), ("multiplicity", P(i32)),
        ("coords", P(i32)), ("rhs", P(f64)),
    ]


class GpuOptions(C.Structure):
    _fields_ = [("device", i32), ("workers", i32), ("coarse_mode", i32),
                ("coarse_rel_tolerance", f64), ("coarse_abs_tolerance", f64),
                ("coarse_max_iterations", i32), ("leaf_size", i32), ("local_blocks", i32),
                ("solve_parts", i32), ("setup_mode", i32)]


class DistOptions(C.Structure):
    _fields_ = [("rank", i32), ("world", i32), ("nccl_id", C.c_uint8 * 128), ("subdomain_rank", P(i32))]


class RankPlanView(C.Structure):
    _fields_ = [("rank", i32), ("world", i32), ("n_local", i32), ("n_rows", i32), ("n_owned", i32),
                ("n_subdomains_global", i32), ("local_to_global", P(i32)), ("subdomain_rank", P(i32)),
                ("n_local_subdomains", i32), ("subdomains", P(i32)),
                ("n_halo_peers", i32), ("halo_peers", P(i32)), ("halo_send_off", P(i32)),
                ("halo_send_idx", P(i32)), ("halo_recv_off", P(i32)),
                ("n_iface_peers", i32), ("iface_peers", P(i32)), ("iface_send_off", P(i32)),
                ("iface_send_slot", P(i32)), ("iface_recv_off", P(i32)),
                ("n_local_slots", i32), ("n_remote_slots", i32), ("remote_ptr", P(i32)),
                ("remote_subdomain", P(i32)), ("remote_slot", P(i32)),
                ("cbuf_pad", i32), ("cbuf_offset", P(i32)), ("local_problem", C.c_void_p)]


class SolverOptions(C.Structure):
    _fields_ = [("rel_tolerance", f64), ("abs_tolerance", f64), ("max_iterations", i32),
                ("record_history", i32)]


class SolveReport(C.Structure):
    _fields_ = [("iterations", i32), ("final_relative_residual", f64), ("history_length", i32),
                ("has_condition_estimate", i32), ("condition_estimate", f64), ("converged", i32)]


class Stats(C.Structure):
    _fields_ = [("setup_seconds", f64), ("factor_values", i64), ("interior_solve_bytes", i64),
                ("apply_bytes", i64), ("n_subdomains", i32), ("global_dofs", i32), ("n_coarse", i32),
                ("unique_subdomains", i32), ("max_interior", i32), ("max_interface", i32), ("interior_dofs", i64),
                ("interior_apply_bytes", i64), ("graph_captures", i64), ("coarse_mode", i32), ("switches", i32),
                ("setup_device_seconds", f64)]


class KernelTimes(C.Structure):
    _fields_ = [("interior_ms", f64), ("interior_launches", i64), ("iface_ms", f64), ("apply_ms", f64), ("applies", i64)]


vp = C.c_void_p
pd = P(f64)
SIGNATURES = {
    "bddc_last_error": (C.c_char_p, []),
    "bddc_abi_version": (i32, []),
    "bddc_switch_name": (C.c_char_p, [i32]),
    "bddc_kernel_launches": (i64, []),
    "bddc_default_gpu_options": (None, [P(GpuOptions)]),
    "bddc_default_solver_options": (None, [P(SolverOptions)]),
    "bddc_problem_poisson": (C.c_int, [i32, i32, i32, i32, f64, u64, u64, P(vp)]),
    "bddc_problem_from_view": (C.c_int, [P(ProblemView), P(vp)]),
    "bddc_problem_get_view": (C.c_int, [vp, P(ProblemView)]),
    "bddc_problem_export_bundle": (C.c_int, [vp, C.c_char_p]),
    "bddc_problem_ingest_bundle": (C.c_int, [C.c_char_p, P(vp)]),
    "bddc_problem_destroy": (None, [vp]),
    "bddc_host_setup_create": (C.c_int, [vp, P(GpuOptions), P(vp)]),
    "bddc_host_setup_blocks": (C.c_int, [vp, i32, pd, pd, pd]),
    "bddc_host_setup_coarse": (C.c_int, [vp, P(i32), P(i32), P(i32), pd]),
    "bddc_host_setup_interior_solve": (C.c_int, [vp, i32, pd]),
    "bddc_host_setup_stats": (C.c_int, [vp, P(Stats)]),
    "bddc_host_setup_destroy": (None, [vp]),
    "bddc_gpu_create": (C.c_int, [vp, P(GpuOptions), P(vp)]),
    "bddc_dist_unique_id": (C.c_int, [P(C.c_uint8)]),
    "bddc_gpu_create_dist": (C.c_int, [vp, P(GpuOptions), P(DistOptions), P(vp)]),
    "bddc_gpu_layout": (C.c_int, [vp, P(i32), P(i32), P(i32), P(i32)]),
    "bddc_rank_plan_create": (C.c_int, [vp, i32, i32, P(i32), P(vp)]),
    "bddc_rank_plan_get_view": (C.c_int, [vp, P(RankPlanView)]),
    "bddc_rank_plan_destroy": (None, [vp]),
    "bddc_gpu_apply": (C.c_int, [vp, pd, pd]),
    "bddc_gpu_apply_device": (C.c_int, [vp, vp, vp, vp]),
    "bddc_gpu_stage": (C.c_int, [vp, i32, pd, pd, pd, pd]),
    "bddc_gpu_pcg": (C.c_int, [vp, pd, P(SolverOptions), i32, pd, P(SolveReport), pd, i32]),
    "bddc_gpu_pcg_device": (C.c_int, [vp, vp, P(SolverOptions), i32, vp, P(SolveReport), pd, i32, vp]),
    "bddc_gpu_subdomain_blocks": (C.c_int, [vp, i32, pd, pd, pd]),
    "bddc_gpu_coarse_matrix": (C.c_int, [vp, P(i32), P(i32), P(i32), pd]),
    "bddc_gpu_get_stats": (C.c_int, [vp, P(Stats)]),
    "bddc_gpu_set_profile": (C.c_int, [vp, i32]),
    "bddc_gpu_kernel_times": (C.c_int, [vp, P(KernelTimes), i32]),
    "bddc_gpu_synchronize": (C.c_int, [vp]),
    "bddc_gpu_solve_profile": (i64, [vp, P(i64), i64]),
    "bddc_gpu_last_error": (C.c_char_p, [vp]),
    "bddc_gpu_destroy": (None, [vp]),
}


class BddcError(RuntimeError):
    """Raised for a non-OK status; .code is the C status, .kind the reference exception type."""

    KINDS = {ERR_INVALID_ARGUMENT: "invalid_argument", ERR_RUNTIME: "runtime_error",
             ERR_OUT_OF_RANGE: "out_of_range", ERR_CUDA: "cuda_error", ERR_NO_DEVICE: "no_device"}

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code
        self.kind = self.KINDS.get(code, "error")


class InvalidArgument(BddcError, ValueError):
    pass


class OutOfRange(BddcError, IndexError):
    pass


_lib = None


def header_symbols() -> list[str]:
    """Every function the public header declares (for the export check)."""
    text = re.sub(r"/\*.*?\*/", "", open(HEADER_PATH).read(), flags=re.S)
    return sorted(set(re.findall(r"\b(bddc_[a-z_0-9]+)\s*\(", text)))


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                              "g.build()'` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(code: int, ctx=None) -> None:
    if code == OK:
        return
    L = lib()
    msg = (L.bddc_gpu_last_error(ctx) if ctx else L.bddc_last_error()) or b""
    msg = msg.decode()
    if code == ERR_INVALID_ARGUMENT:
        raise InvalidArgument(code, msg)
    if code == ERR_OUT_OF_RANGE:
        raise OutOfRange(code, msg)
    raise BddcError(code, msg)
