"""The non-default device paths stay correct (GPU): every switch of the apply / PCG loop
(csrc/device/context.cu) against the reference's golden PCG run and apply.

Each case runs in a fresh process because the switches are read once per process.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/tests")
from conftest import golden, history_err
from paper_2410_14786_b200 import Preconditioner, Problem, SolverOptions
out = {}
for name in ("k4m8", "c1"):
    g = golden(name)
    k, m, seed = (int(v) for v in g["config"])
    p = Problem.poisson(k * m, k, rhs_seed=seed)
    pre = Preconditioner(p)
    x, rep = pre.pcg(p.rhs(), SolverOptions(1e-8, 0.0, 10000, True))
    xr = g["pcg_x"] if "pcg_x" in g else None
    xe = float(np.abs(x - xr).max() / np.abs(xr).max()) if xr is not None else 0.0
    ae = float(np.abs(pre.apply(p.rhs()) - g["apply_rhs"]).max() / np.abs(g["apply_rhs"]).max()) if "apply_rhs" in g else 0.0
    out[name] = [rep.iterations, int(g["pcg_report"][0]), history_err(rep.residual_history, g["pcg_history"]), xe, ae]
print(json.dumps(out))
""".replace("ROOT", repr(ROOT))

CASES = [
    {"BDDC_SPLIT": "0"},            # full solve + u0 - extension
    {"BDDC_HARMONIC": "0"},         # unpruned second solve (MODE 1)
    {"BDDC_GRAPH": "0"},            # eager launches instead of the per-iteration graph
    {"BDDC_COOP_COARSE": "1"},      # r_c once per GPU in a cooperative K_i grid
    {"BDDC_DIR_SPMV": "1"},         # p = z + beta p fused into the SpMV
    {"BDDC_PDL": "1"},              # programmatic dependent launch
    {"BDDC_PROFILE_STRIDE": "1"},   # (profiling off here; the stride must not change results)
    {"BDDC_STEP": "1"},             # xpay / SpMV / update as one cooperative launch
    {"BDDC_K_FULL": "1"},           # row-major K_i, local_blocks CTAs per subdomain
    {"BDDC_PAIR_TILES": "0"},       # no pair steps in the interior-solve programs
    {"BDDC_MAX_CHAIN": "0"},        # forward levels coloured into phases only
    {"BDDC_QUAD_TILES": "0"},       # pairs only (no 8-lane quads)
    {"BDDC_SETUP_SCRATCH_CACHE": "0"},  # setup scratch freed after every setup
    {"BDDC_ELL16": "0"},            # 32-bit ELL columns instead of 16-bit row offsets
]


@pytest.mark.parametrize("env", CASES, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_switch_keeps_parity(gpu, env):
    r = subprocess.run([sys.executable, "-c", SCRIPT], env={**os.environ, **env}, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for name, (it, it_ref, herr, xerr, aerr) in res.items():
        assert it == it_ref, (name, it, it_ref)
        assert herr <= 1e-10, (name, herr)
        assert xerr <= 1e-10, (name, xerr)
        assert aerr <= 1e-11, (name, aerr)


def test_switches_reported_and_no_exchange_guarded(gpu):
    # the active BDDC_* switches are reported in the stats, and the wrong-results
    # timing switch BDDC_NO_EXCHANGE=1 is refused unless BDDC_EXPERIMENTS=1 is also set
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2410_14786_b200 import Preconditioner, Problem, lib\n"
            "p = Problem.poisson(16, 2)\n"
            "try:\n    pre = Preconditioner(p)\nexcept Exception as e:\n    print('ERR', e); raise SystemExit(0)\n"
            "st = pre.stats(); names = [lib().bddc_switch_name(i).decode() for i in range(32) "
            "if st['switches'] >> i & 1]\nprint('OK', ','.join(names))\n") % ROOT
    env = {k: v for k, v in os.environ.items() if not k.startswith("BDDC_")}
    r = subprocess.run([sys.executable, "-c", code], env={**env, "BDDC_NO_EXCHANGE": "1"}, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "ERR" in r.stdout and "BDDC_EXPERIMENTS" in r.stdout
    r = subprocess.run([sys.executable, "-c", code], env={**env, "BDDC_PDL": "1"}, capture_output=True, text=True,
                       timeout=300)
    assert r.stdout.strip().splitlines()[-1] == "OK BDDC_PDL"
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.stdout.strip().splitlines()[-1] == "OK"


def test_repeated_solve_reuses_graphs(gpu):
    # the cached PCG graphs are keyed by the kernels' parameter block (padding
    # cleared); an identical second solve must not re-capture
    sys.path.insert(0, ROOT)
    from paper_2410_14786_b200 import Preconditioner, Problem, SolverOptions

    p = Problem.poisson(128, 4)
    pre = Preconditioner(p)
    opts = SolverOptions(1e-8, 0.0, 10000, True)
    pre.pcg(p.rhs(), opts)
    n1 = pre.stats()["graph_captures"]
    for _ in range(3):
        pre.pcg(p.rhs(), opts)
    assert n1 >= 1 and pre.stats()["graph_captures"] == n1


PLAIN_SCRIPT = r"""
import hashlib, json, sys
import numpy as np
sys.path.insert(0, ROOT)
from paper_2410_14786_b200 import Preconditioner, Problem, SolverOptions
out = {}
cases = {"c2": Problem.poisson(800, 8), "kappa": Problem.poisson(240, 4, kappa_decades=4.0, kappa_seed=7)}
for name, p in cases.items():
    pre = Preconditioner(p)
    for cap in (10000, 7):
        x, rep = pre.pcg(p.rhs(), SolverOptions(1e-8, 0.0, cap, True), precondition=False)
        out[f"{name}/{cap}"] = [rep.iterations, bool(rep.converged), [float(h).hex() for h in rep.residual_history],
                                hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest(),
                                None if rep.condition_estimate is None else float(rep.condition_estimate).hex()]
# symmetric, not SPD (the negated Laplacian): pcg.cpp:75-78 at the first iteration
p = Problem.poisson(32, 2)
nr, nc, rp, ci, va = p.global_matrix()
neg = Problem.from_arrays((nr, nc, rp, ci, -va), [p.local_matrix(i) for i in range(p.n_subdomains)],
                          p.subdomain_dofs(), p.interior_counts(), p.weights(),
                          [p.constraint_matrix(i) for i in range(p.n_subdomains)], p.primal_maps(), p.n_coarse,
                          rhs=p.rhs())
try:
    Preconditioner(neg).pcg(neg.rhs(), SolverOptions(1e-8, 0.0, 100, True), precondition=False)
    out["neg"] = "no error"
except Exception as e:
    out["neg"] = str(e)
print(json.dumps(out))
""".replace("ROOT", repr(ROOT))


def test_plain_cg_one_launch_matches_kernel_loop(gpu):
    # plain CG on one GPU runs as one cooperative launch (pcg.cu plain_cg_kernel); its phases are
    # the per-kernel loop's (BDDC_PLAIN_LOOP=0), so histories, x and the Lanczos estimate are
    # bitwise identical, at convergence and at the iteration cap, and "not SPD" is raised alike
    env = {k: v for k, v in os.environ.items() if not k.startswith("BDDC_")}
    res = []
    # (and 16-bit ELL column offsets give the 32-bit columns' iterates bit for bit)
    for extra in ({}, {"BDDC_PLAIN_LOOP": "0"}, {"BDDC_ELL16": "0"}):
        r = subprocess.run([sys.executable, "-c", PLAIN_SCRIPT], env={**env, **extra}, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res.append(json.loads(r.stdout.strip().splitlines()[-1]))
    one, loop, col32 = res
    assert one == loop
    assert one == col32
    assert one["c2/10000"][0] == 1649 and one["c2/10000"][1]
    assert one["c2/7"][0] == 7 and not one["c2/7"][1] and len(one["c2/7"][2]) == 8
    assert "matrix not SPD" in one["neg"]


STEP_SCRIPT = r"""
import hashlib, json, sys
import numpy as np
sys.path.insert(0, ROOT)
from paper_2410_14786_b200 import Preconditioner, Problem, SolverOptions
out = {}
for name, args in (("c2", (800, 8)), ("k4m8", (32, 4))):
    p = Problem.poisson(*args, rhs_seed=1)
    pre = Preconditioner(p)
    for cap in (10000, 5):
        x, rep = pre.pcg(p.rhs(), SolverOptions(1e-8, 0.0, cap, True))
        out[f"{name}/{cap}"] = [rep.iterations, rep.converged, [float(h).hex() for h in rep.residual_history],
                                hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest(),
                                None if rep.condition_estimate is None else float(rep.condition_estimate).hex()]
print(json.dumps(out))
""".replace("ROOT", repr(ROOT))


def test_pcg_step_one_launch_matches_kernel_loop(gpu):
    # BDDC_STEP=1: xpay + SpMV + update (+ check) of each BDDC-PCG iteration run as one cooperative
    # launch (pcg.cu pcg_step_kernel); its phases are the per-kernel loop's, so histories, x and
    # the Lanczos estimate are bitwise identical, at convergence and at the cap
    env = {k: v for k, v in os.environ.items() if not k.startswith("BDDC_")}
    res = []
    for extra in ({"BDDC_STEP": "1"}, {}):
        r = subprocess.run([sys.executable, "-c", STEP_SCRIPT], env={**env, **extra}, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res.append(json.loads(r.stdout.strip().splitlines()[-1]))
    one, loop = res
    assert one == loop
    assert one["c2/10000"][0] == 11 and one["c2/10000"][1]
    assert one["c2/5"][0] == 5 and not one["c2/5"][1]
