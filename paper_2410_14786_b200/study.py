"""Study harness on the GPU path: the reference's experiment runner and CSV schema.

Mirrors include/bddc/study.hpp and src/study.cpp:40-217 (names, modes, row semantics, CSV
format) so paper-style sweeps run as one call and their CSV diffs cleanly against the
reference's own output:

  run_study(config)                weak / strong / compare / single over config.k_list
                                   (study.cpp:77-143): Poisson on k x k subdomains, study_rhs,
                                   setup timed around the Preconditioner, solve timed around
                                   pcg (outer rtol config.tolerance, 10,000 iterations max);
                                   compare mode adds a plain-CG row per k; build or solve
                                   failures land in the row's error column.
  run_bundle_study(manifest, cfg)  one BDDC-CG row on an ingested bundle with its own rhs
                                   (study.cpp:145-179).
  write_csv / write_csv_file       kCsvHeader and the row format of study.cpp:181-217.

The timings are host wall clock like the reference's (steady_clock around the same spans);
the setup includes the host factorisation and the device upload.
"""
from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

from .solver import Preconditioner, Problem, SolverOptions

MODES = ("weak", "strong", "compare", "single")
KCSV_HEADER = ("mode,k,n_subdomains,global_dofs,coarse_dim,setup_seconds,solve_seconds,"
               "iterations,final_relative_residual,condition_estimate,error")


def parse_study_mode(name: str) -> str:
    if name not in MODES:
        raise ValueError("unknown study mode: " + name)
    return name


def study_mode_name(mode: str) -> str:
    return mode if mode in MODES else "?"


@dataclass
class ExperimentConfig:
    mode: str = "compare"
    k_list: list = field(default_factory=list)
    cells: int = 32  # cells per subdomain side (weak/compare/single); global cells (strong)
    tolerance: float = 1e-8
    worker_count: int = 1  # host threads of the setup (the GPU path ignores it for the solve)
    seed: int = 1
    output_path: str = ""

    def validate(self) -> None:  # study.cpp:59-66
        if not self.k_list:
            raise ValueError("config: k list is empty")
        if any(k < 2 for k in self.k_list):
            raise ValueError("config: every k must be at least 2")
        if self.worker_count < 1:
            raise ValueError("config: worker_count must be at least 1")
        if not self.tolerance > 0.0:
            raise ValueError("config: tolerance must be positive")
        if self.cells < 2:
            raise ValueError("config: cells must be at least 2")


@dataclass
class StudyRow:
    mode: str = ""
    k: int = 0
    n_subdomains: int = 0
    global_dofs: int = 0
    coarse_dim: int = 0
    setup_seconds: float = 0.0
    solve_seconds: float = 0.0
    iterations: int = 0
    final_relative_residual: float = 0.0
    condition_estimate: float | None = None
    error: str = ""
    converged: bool = False


def _outer(tol: float) -> SolverOptions:
    return SolverOptions(tol, 0.0, 10000, False)


def _fill(row: StudyRow, rep) -> None:  # study.cpp:31-37
    row.iterations = rep.iterations
    row.final_relative_residual = rep.final_relative_residual
    row.condition_estimate = rep.condition_estimate
    row.converged = rep.converged
    if not rep.converged:
        row.error = "not converged"


def _solve_rows(row: StudyRow, problem: Problem, b, config: ExperimentConfig, device: int, compare: bool):
    t0 = time.perf_counter()
    pre = Preconditioner(problem, device=device, workers=config.worker_count)
    row.setup_seconds = time.perf_counter() - t0
    row.coarse_dim = problem.n_coarse
    t0 = time.perf_counter()
    _, rep = pre.pcg(b, _outer(config.tolerance))
    row.solve_seconds = time.perf_counter() - t0
    _fill(row, rep)
    rows = [row]
    if compare:  # plain CG on the same system (empty PreconditionerFn), study.cpp:120-131
        plain = StudyRow(**{**row.__dict__})
        plain.coarse_dim, plain.setup_seconds = 0, 0.0
        t0 = time.perf_counter()
        _, prep = pre.pcg(b, _outer(config.tolerance), precondition=False)
        plain.solve_seconds = time.perf_counter() - t0
        _fill(plain, prep)
        plain.error = "" if prep.converged else "not converged"
        rows.append(plain)
    return rows


def _message(e: Exception) -> str:
    msg = e.args[-1] if e.args else str(e)  # BddcError(code, message) or a plain exception
    return msg.decode() if isinstance(msg, bytes) else str(msg)


def run_study(config: ExperimentConfig, device: int = 0) -> list:
    config.validate()
    ks = list(config.k_list)[:1] if config.mode == "single" else list(config.k_list)
    rows = []
    for k in ks:
        row = StudyRow(mode=config.mode, k=k, n_subdomains=k * k)
        try:
            cells = config.cells if config.mode == "strong" else k * config.cells
            if config.mode == "strong" and cells % k != 0:
                raise ValueError(f"strong mode: global cells {cells} not divisible by k = {k}")
            problem = Problem.poisson(cells, k, rhs_seed=config.seed)
            row.global_dofs = problem.global_dofs
            rows += _solve_rows(row, problem, problem.rhs(), config, device, config.mode == "compare")
        except Exception as e:  # noqa: BLE001 - reference: failures populate the error column
            row.error = _message(e)
            row.converged = False
            rows.append(row)
    return rows


def run_bundle_study(manifest_path: str, config: ExperimentConfig, device: int = 0) -> list:
    row = StudyRow(mode="single")
    try:
        problem = Problem.from_bundle(manifest_path)
        ns = problem.n_subdomains
        side = int(ns ** 0.5 + 0.5)
        row.k = side if side * side == ns else 0
        row.n_subdomains = ns
        row.global_dofs = problem.global_dofs
        return _solve_rows(row, problem, problem.rhs(), config, device, False)
    except Exception as e:  # noqa: BLE001
        row.error = _message(e)
        row.converged = False
        return [row]


_libc = ctypes.CDLL(None)


def _g17(v: float) -> str:
    """C printf("%.17g") (the reference's CSV digits; Python's % formatting differs)."""
    buf = ctypes.create_string_buffer(64)
    _libc.snprintf(buf, 64, b"%.17g", ctypes.c_double(v))
    return buf.value.decode()


def write_csv(rows, out) -> None:  # study.cpp:185-210
    out.write(KCSV_HEADER + "\n")
    for r in rows:
        cond = _g17(r.condition_estimate) if r.condition_estimate is not None else ""
        err = r.error.replace(",", ";").replace("\n", ";")
        out.write(f"{r.mode},{r.k},{r.n_subdomains},{r.global_dofs},{r.coarse_dim},"
                  f"{r.setup_seconds:.6f},{r.solve_seconds:.6f},{r.iterations},"
                  f"{_g17(r.final_relative_residual)},{cond},{err}\n")


def write_csv_file(path: str, rows) -> None:
    try:
        with open(path, "w") as f:
            write_csv(rows, f)
    except OSError as e:
        raise RuntimeError("cannot open output file: " + path) from e
