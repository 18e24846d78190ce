"""GPU setup (reference setup_subdomain / assemble_coarse,
src/preconditioner.cpp:34-98, lu_factor src/sparse_lu.cpp:80-195): the device factorisation,
Schur complements, saddle reduction, coarse basis, coarse blocks and coarse matrix against the
reference's own setup products (tests/golden), mirroring tests/test_host_setup.py, plus the
device-set-up preconditioner against the host-set-up one."""
import numpy as np
import pytest

import bddc_oracle as o
from conftest import golden, history_err
from paper_2410_14786_b200 import BddcError, Preconditioner, Problem, SolverOptions

pytestmark = pytest.mark.gpu
OPTS = SolverOptions(1e-8, 0.0, 10000, True)


def _problem(g):
    cfg = [int(v) for v in g["config"]]
    if len(cfg) == 3:
        k, m, seed = cfg
        return Problem.poisson(k * m, k, rhs_seed=seed)
    cx, cy, kx, ky, dm, ks, seed = cfg
    return Problem.poisson(cx, kx, cy, ky, kappa_decades=dm / 1000.0, kappa_seed=ks, rhs_seed=seed)


@pytest.mark.parametrize("name", ["k2m4", "k3m4", "k3m6", "k4m8", "r4x2m8", "h4m8"])
def test_device_blocks_match_reference(gpu, name):
    g = golden(name)
    p = _problem(g)
    pre = Preconditioner(p)  # setup on the device (default)
    st = pre.stats()
    assert st["setup_device_seconds"] > 0.0
    blocks = [pre.subdomain_blocks(i) for i in range(p.n_subdomains)]
    phi = np.concatenate([b[0].ravel() for b in blocks])
    lam = np.concatenate([b[1].ravel() for b in blocks])
    aci = np.concatenate([b[2].ravel() for b in blocks])
    scale = max(1.0, np.abs(g["aci"]).max())
    assert np.abs(phi - g["phi"]).max() < 1e-11
    assert np.abs(lam - g["lambda"]).max() < 1e-11 * scale
    assert np.abs(aci - g["aci"]).max() < 1e-11 * scale
    rp, ci, v = pre.coarse_matrix()
    assert np.array_equal(rp, g["Ac_rowptr"]) and np.array_equal(ci, g["Ac_cols"])
    assert np.abs(v - g["Ac_vals"]).max() < 1e-11 * scale


def test_device_saddle_identities(gpu):
    # test_bddc.cpp:56-91 on the device products: C Phi = I, A Phi + C^T Lambda = 0, A_ci symmetric
    p = Problem.poisson(12, 3)
    pre = Preconditioner(p)
    for i in range(p.n_subdomains):
        phi, lam, aci = pre.subdomain_blocks(i)
        A = o.Csr(*p.local_matrix(i)).dense()
        Cm = o.Csr(*p.constraint_matrix(i)).dense()
        assert np.abs(Cm @ phi - np.eye(Cm.shape[0])).max() <= 1e-10
        assert np.abs(A @ phi + Cm.T @ lam).max() <= 1e-10 * np.abs(A).sum(1).max()
        assert np.abs(aci - aci.T).max() <= 1e-12 * max(1.0, np.abs(aci).max())


@pytest.mark.parametrize("setup_args", [(128, 4, None), (352, 8, 2.0)], ids=["c1ish", "c5"])
def test_device_setup_matches_host_setup(gpu, setup_args):
    cells, k, dec = setup_args
    kw = dict(kappa_decades=dec, kappa_seed=0x5EED) if dec else {}
    p = Problem.poisson(cells, k, **kw)
    dev, host = Preconditioner(p), Preconditioner(p, setup="host")
    r = p.rhs()
    zd, zh = dev.apply(r), host.apply(r)
    assert np.abs(zd - zh).max() <= 1e-12 * np.abs(zh).max()
    xd, rd = dev.pcg(r, OPTS)
    xh, rh = host.pcg(r, OPTS)
    assert rd.iterations == rh.iterations
    assert history_err(rd.residual_history, rh.residual_history) <= 1e-10


def test_device_setup_c2_and_c5_against_reference(gpu):
    # the BASELINE configs solved after a device setup: C2 (64 subdomains, 9 setup classes) and C5
    # (heterogeneous: no two subdomains share values) to the reference's iteration counts / histories
    for name, p in (("c2", Problem.poisson(800, 8)),
                    ("c5", Problem.poisson(352, 8, kappa_decades=2.0, kappa_seed=0x5EED))):
        g = golden(name)
        pre = Preconditioner(p)
        x, rep = pre.pcg(p.rhs(), OPTS)
        assert rep.iterations == int(g["pcg_report"][0]), name
        assert history_err(rep.residual_history, g["pcg_history"]) <= 1e-10, name
        stride = int(g["pcg_x_sample_stride"][0])
        assert np.abs(x[::stride] - g["pcg_x_sample"]).max() <= 1e-10 * np.abs(g["pcg_x_sample"]).max()


def test_device_setup_error_names_subdomain(gpu):
    # test_bddc.cpp:371-402 on the device path: duplicated constraint rows -> singular saddle
    p = Problem.poisson(8, 2)
    cons = [p.constraint_matrix(i) for i in range(p.n_subdomains)]
    nr, nc, rp, ci, va = cons[0]
    row0 = slice(rp[0], rp[1])
    dup = (2, nc, np.array([0, rp[1] - rp[0], 2 * (rp[1] - rp[0])]), np.concatenate([ci[row0], ci[row0]]),
           np.concatenate([va[row0], va[row0]]))
    pm = p.primal_maps()
    pm[0] = np.array([0, 1])
    broken = Problem.from_arrays(p.global_matrix(), [p.local_matrix(i) for i in range(p.n_subdomains)],
                                 p.subdomain_dofs(), p.interior_counts(), p.weights(), [dup] + cons[1:], pm,
                                 p.n_coarse, *p.classes(), p.multiplicity(), p.rhs())
    with pytest.raises(BddcError, match="bddc setup: subdomain 0"):
        Preconditioner(broken)


SADDLE_SCRIPT = r"""
import hashlib, json, sys
import numpy as np
sys.path.insert(0, ROOT)
from paper_2410_14786_b200 import Preconditioner, Problem
out = {}
for name, p in (("c2", Problem.poisson(800, 8)), ("kappa", Problem.poisson(240, 4, 180, 3, kappa_decades=3.0))):
    pre = Preconditioner(p)
    h = hashlib.sha256()
    for i in range(p.n_subdomains):
        for blk in pre.subdomain_blocks(i):
            h.update(np.ascontiguousarray(blk).tobytes())
    h.update(np.ascontiguousarray(pre.apply(p.rhs())).tobytes())  # K_i enters the apply
    out[name] = h.hexdigest()
print(json.dumps(out))
""".replace("ROOT", repr(__import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))))


def test_cluster_saddle_inverse_is_bitwise_the_global_one(gpu):
    # the saddle Gauss-Jordan with the matrix in a CTA cluster's shared memory (setup.cu
    # saddle_gj_cluster_kernel) and the global-memory one (BDDC_SADDLE_GLOBAL=1) make the same
    # pivot choices and updates: Phi, Lambda, A_ci and the apply (K_i) are bitwise identical
    import json
    import os
    import subprocess
    import sys

    env = {k: v for k, v in os.environ.items() if not k.startswith("BDDC_")}
    res = []
    for extra in ({}, {"BDDC_SADDLE_GLOBAL": "1"}):
        r = subprocess.run([sys.executable, "-c", SADDLE_SCRIPT], env={**env, **extra}, capture_output=True,
                           text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
        res.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert res[0] == res[1]


def test_repeated_setups_share_scratch_and_problem(gpu):
    """Constructions of different sizes in one process (the cached setup scratch block grows and
    is reused; every context shares its problem's data): each preconditioner's blocks and apply
    are bitwise those of the first construction of the same problem, also after the problem
    handle that built an earlier context is gone."""
    small = Problem.poisson(128, 4, rhs_seed=3)
    big = Problem.poisson(352, 8, kappa_decades=2.0, kappa_seed=0x5EED, rhs_seed=5)
    r_small = np.random.default_rng(1).standard_normal(small.global_dofs)
    first = Preconditioner(small)
    z0 = first.apply(r_small)
    b0 = [first.subdomain_blocks(i)[2] for i in range(small.n_subdomains)]
    second = Preconditioner(big)  # larger scratch: the cached block is replaced
    r_big = np.random.default_rng(2).standard_normal(big.global_dofs)
    zb = second.apply(r_big)
    del first
    third = Preconditioner(small)  # the larger cached block is reused
    assert np.array_equal(third.apply(r_small), z0)
    assert all(np.array_equal(third.subdomain_blocks(i)[2], b0[i]) for i in range(small.n_subdomains))
    # a context outlives the Python problem object that built it (shared problem data)
    tmp = Problem.poisson(352, 8, kappa_decades=2.0, kappa_seed=0x5EED, rhs_seed=5)
    fourth = Preconditioner(tmp)
    fourth.problem = None
    del tmp
    assert np.array_equal(fourth.apply(r_big), zb)
    del second
    assert np.array_equal(fourth.apply(r_big), zb)
