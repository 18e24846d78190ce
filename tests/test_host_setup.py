"""Host setup (C++; no GPU): coarse bases, multipliers, coarse blocks and the coarse
matrix against the reference (tests/golden), plus the reference's setup identities
(test_bddc.cpp:56-125, 371-402) and the device-program builder via its CPU simulator."""
import ctypes as C
import json
import os
import sys

import numpy as np
import pytest

import bddc_oracle as o
from conftest import ROOT, golden
from paper_2410_14786_b200 import BddcError, HostSetup, InvalidArgument, Problem
from paper_2410_14786_b200 import _lib


@pytest.mark.parametrize("name", ["k2m4", "k3m4", "k3m6", "k4m8", "r4x2m8", "h4m8"])
def test_blocks_match_reference(name):
    g = golden(name)
    cfg = [int(v) for v in g["config"]]
    if len(cfg) == 3:
        k, m, seed = cfg
        p = Problem.poisson(k * m, k, rhs_seed=seed)
    else:
        cx, cy, kx, ky, dm, ks, seed = cfg
        p = Problem.poisson(cx, kx, cy, ky, kappa_decades=dm / 1000.0, kappa_seed=ks, rhs_seed=seed)
    s = HostSetup(p, workers=4)
    phi = np.concatenate([s.blocks(i)[0].ravel() for i in range(p.n_subdomains)])
    lam = np.concatenate([s.blocks(i)[1].ravel() for i in range(p.n_subdomains)])
    aci = np.concatenate([s.blocks(i)[2].ravel() for i in range(p.n_subdomains)])
    scale = max(1.0, np.abs(g["aci"]).max())
    assert np.abs(phi - g["phi"]).max() < 1e-11
    assert np.abs(lam - g["lambda"]).max() < 1e-11 * scale
    assert np.abs(aci - g["aci"]).max() < 1e-11 * scale
    rp, ci, v = s.coarse_matrix()
    assert np.array_equal(rp, g["Ac_rowptr"]) and np.array_equal(ci, g["Ac_cols"])
    assert np.abs(v - g["Ac_vals"]).max() < 1e-11 * scale


def test_saddle_identities():
    # test_bddc.cpp:56-91: C Phi = I, A Phi + C^T Lambda = 0, A_ci symmetric
    p = Problem.poisson(12, 3)
    s = HostSetup(p)
    for i in range(p.n_subdomains):
        phi, lam, aci = s.blocks(i)
        A = o.Csr(*p.local_matrix(i)).dense()
        Cm = o.Csr(*p.constraint_matrix(i)).dense()
        assert np.abs(Cm @ phi - np.eye(Cm.shape[0])).max() <= 1e-10
        assert np.abs(A @ phi + Cm.T @ lam).max() <= 1e-10 * np.abs(A).sum(1).max()
        assert np.abs(aci - aci.T).max() <= 1e-12


def test_floating_subdomain_coarse_block():
    # test_bddc.cpp:93-107: centre subdomain block is PSD with constants in its null space
    p = Problem.poisson(12, 3)
    s = HostSetup(p)
    aci = s.blocks(4)[2]
    assert aci.shape == (8, 8)
    eig = np.linalg.eigvalsh(aci)
    assert abs(eig[0]) <= 1e-10 and eig[1] > 1e-6
    assert np.abs(aci @ np.ones(8)).max() <= 1e-10
    assert np.linalg.eigvalsh(s.blocks(0)[2])[0] > 1e-8


def test_interior_factor_solves():
    p = Problem.poisson(24, 3)
    s = HostSetup(p, leaf_size=8)
    for i in (0, 4):
        ni = int(p.interior_counts()[i])
        A = o.Csr(*p.local_matrix(i)).dense()[:ni, :ni]
        b = np.random.default_rng(i).standard_normal(ni)
        x = s.interior_solve(i, b)
        assert np.abs(A @ x - b).max() <= 1e-12 * np.abs(b).max() * 10


def test_setup_error_names_subdomain():
    # test_bddc.cpp:371-402: duplicated constraint rows make subdomain 0 singular
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
        HostSetup(broken)


def test_from_arrays_round_trip():
    p = Problem.poisson(16, 2)
    q = Problem.from_arrays(p.global_matrix(), [p.local_matrix(i) for i in range(4)], p.subdomain_dofs(),
                            p.interior_counts(), p.weights(), [p.constraint_matrix(i) for i in range(4)],
                            p.primal_maps(), p.n_coarse, *p.classes(), p.multiplicity(), p.rhs())
    a, b = HostSetup(p), HostSetup(q)  # q has no coords: graph nested dissection
    for i in range(4):
        assert np.abs(a.blocks(i)[0] - b.blocks(i)[0]).max() < 1e-12
    with pytest.raises(InvalidArgument):
        bad = [p.local_matrix(i) for i in range(4)]
        nr, nc, rp, ci, va = bad[0]
        bad[0] = (nr, nc, rp, ci[::-1].copy(), va)  # unsorted columns
        Problem.from_arrays(p.global_matrix(), bad, p.subdomain_dofs(), p.interior_counts(), p.weights(),
                            [p.constraint_matrix(i) for i in range(4)], p.primal_maps(), p.n_coarse)


# ---- device-program builder, executed by the test-only CPU interpreter (tests/native)
SIM = os.path.join(ROOT, "tests", "native", "libbddc_sim.so")


@pytest.fixture(scope="module")
def sim():
    import subprocess

    _lib.lib()
    subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "native"), "-s"], check=True)
    return C.CDLL(SIM)


@pytest.mark.parametrize("k,m,parts,leaf,coords", [(2, 4, 1, 16, 1), (3, 6, 2, 16, 1), (4, 8, 2, 4, 1),
                                                   (4, 16, 2, 16, 1), (4, 16, 2, 8, 0), (3, 32, 1, 16, 0),
                                                   (3, 32, 2, 16, 1)])
def test_device_program_reproduces_interior_solve(sim, k, m, parts, leaf, coords):
    prob, cs, b = o.poisson_setup(k, m)
    P = o.Preconditioner(prob.global_matrix, prob.local_matrices, prob.decomposition, cs)
    ref = P.interior_correction(b)
    out = np.zeros_like(b)
    err = C.create_string_buffer(512)
    dp = C.POINTER(C.c_double)
    rc = sim.bddc_sim_interior_solve(k * m, k * m, k, k, parts, leaf, coords, b.ctypes.data_as(dp),
                                     out.ctypes.data_as(dp), err, 512)
    assert rc == 0, err.value
    assert np.abs(out - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("k,m,parts,leaf,coords", [(3, 6, 2, 16, 1), (4, 16, 2, 8, 0), (3, 32, 2, 24, 1),
                                                   (3, 32, 1, 24, 1)])
def test_harmonic_program_matches_full_solve(sim, k, m, parts, leaf, coords):
    # second interior solve of the apply: A_II^{-1} (A_IG z_G) with a pruned forward sweep must
    # equal the full solve of the same (interface-coupled) right-hand side
    prob, cs, _ = o.poisson_setup(k, m)
    A = prob.global_matrix.scipy()
    kinds = prob.decomposition.kind == o.INTERIOR
    rng = np.random.default_rng(5)
    n = A.shape[0]
    v = np.where(~kinds, rng.standard_normal(n), 0.0)   # values on interface dofs
    c = np.where(kinds, A @ v, 0.0)                     # A_IG v on interior dofs
    P = o.Preconditioner(prob.global_matrix, prob.local_matrices, prob.decomposition, cs)
    ref = P.interior_correction(c)
    out = np.zeros_like(c)
    err = C.create_string_buffer(512)
    dp = C.POINTER(C.c_double)
    rc = sim.bddc_sim_harmonic_solve(k * m, k * m, k, k, parts, leaf, coords, c.ctypes.data_as(dp),
                                     out.ctypes.data_as(dp), err, 512)
    assert rc == 0, err.value
    assert np.abs(out - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("k,m,parts,leaf,coords", [(3, 6, 2, 16, 1), (4, 16, 2, 8, 0), (3, 32, 2, 24, 1),
                                                   (3, 32, 1, 24, 1)])
def test_split_apply_programs(sim, k, m, parts, leaf, coords):
    # split apply: the head program (full forward, pruned backward) gives u0 = A_II^-1 r exactly
    # on the interior dofs coupled to the interface and keeps y0 = L^-1 r; the harmonic program
    # with y_in then returns z_I = A_II^-1 (r - A_IG v) from one backward sweep
    prob, cs, _ = o.poisson_setup(k, m)
    A = prob.global_matrix.scipy()
    kinds = prob.decomposition.kind == o.INTERIOR
    rng = np.random.default_rng(11)
    n = A.shape[0]
    r = np.where(kinds, rng.standard_normal(n), 0.0)
    v = np.where(~kinds, rng.standard_normal(n), 0.0)
    c = np.where(kinds, A @ v, 0.0)
    P = o.Preconditioner(prob.global_matrix, prob.local_matrices, prob.decomposition, cs)
    ref_u0 = P.interior_correction(r)
    ref_z = P.interior_correction(r - c)
    coupled = kinds & (np.abs(A[:, np.flatnonzero(~kinds)]).sum(axis=1).A1 > 0)
    u0, z = np.zeros(n), np.zeros(n)
    err = C.create_string_buffer(512)
    dp = C.POINTER(C.c_double)
    rc = sim.bddc_sim_split_solve(k * m, k * m, k, k, parts, leaf, coords, r.ctypes.data_as(dp),
                                  c.ctypes.data_as(dp), u0.ctypes.data_as(dp), z.ctypes.data_as(dp), err, 512)
    assert rc == 0, err.value
    assert coupled.sum() > 0
    assert np.abs(u0[coupled] - ref_u0[coupled]).max() <= 1e-12 * np.abs(ref_u0).max()
    assert np.abs(z[kinds] - ref_z[kinds]).max() <= 1e-12 * np.abs(ref_z).max()


@pytest.mark.parametrize("cx,cy,kx,ky,parts,leaf,coords", [(32, 32, 4, 4, 2, 24, 1), (32, 32, 4, 4, 1, 24, 1),
                                                           (64, 32, 4, 2, 2, 16, 1), (32, 32, 4, 4, 2, 24, 0),
                                                           (300, 300, 3, 3, 2, 24, 1)])
def test_gpu_setup_templates_reproduce_host_programs(sim, cx, cy, kx, ky, parts, leaf, coords):
    # the GPU setup instantiates one program template per setup class and fills
    # its values on the device from D = [L_ss^-1 | BL_s] (host/gpu_setup.cpp, device/setup.cu).
    # Emulating that fill with the host factor's values must give back the host-built programs
    # word for word (streams, dof maps, coupling entries, tables, part descriptors).
    sim.bddc_sim_template_check.restype = C.c_long
    err = C.create_string_buffer(512)
    bad = sim.bddc_sim_template_check(cx, cy, kx, ky, parts, leaf, coords, err, 512)
    assert bad == 0, err.value


VARIANT_SCRIPT = r"""
import ctypes as C, json, os, sys
import numpy as np
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/oracle")
import bddc_oracle as o
sim = C.CDLL(os.path.join(ROOT, "tests", "native", "libbddc_sim.so"))
dp = C.POINTER(C.c_double)
out = {}
for k, m, parts, leaf in ((3, 32, 2, 24), (4, 16, 2, 8), (3, 32, 1, 16)):
    prob, cs, b = o.poisson_setup(k, m)
    P = o.Preconditioner(prob.global_matrix, prob.local_matrices, prob.decomposition, cs)
    ref = P.interior_correction(b)
    z = np.zeros_like(b)
    err = C.create_string_buffer(512)
    rc = sim.bddc_sim_interior_solve(k * m, k * m, k, k, parts, leaf, 1, b.ctypes.data_as(dp), z.ctypes.data_as(dp), err, 512)
    out[f"{k}/{m}/{parts}/{leaf}"] = [rc, err.value.decode(), float(np.abs(z - ref).max() / np.abs(ref).max())]
print(json.dumps(out))
""".replace("ROOT", repr(ROOT))


@pytest.mark.parametrize("env", [{"BDDC_PAIR_TILES": "0"}, {"BDDC_QUAD_TILES": "0"}, {"BDDC_MAX_CHAIN": "0"},
                                 {"BDDC_MAX_CHAIN": "100"}, {"BDDC_MIN_CHUNK_ROWS": "4"}],
                         ids=lambda e: ",".join(f"{a}={b}" for a, b in e.items()))
def test_program_shape_switches_keep_the_solve(sim, env):
    # the builder's shape switches (group steps, chained levels, chunk rows; read once per
    # process) change the program, never the solve: the CPU interpreter reproduces the oracle
    import subprocess
    r = subprocess.run([sys.executable, "-c", VARIANT_SCRIPT], env={**os.environ, **env}, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for case, (rc, msg, e) in res.items():
        assert rc == 0, (case, msg)
        assert e <= 1e-12, (case, e)
