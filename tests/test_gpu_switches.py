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
