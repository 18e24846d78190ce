"""GPU parity: the sm_100a BDDC path (through the C-ABI) against the reference.

Checks follow the reference's own tests (file:line into /root/reference/proj/tests):
stage operators vs dense oracles (test_bddc.cpp:157-236), densified apply = B + (I-BA)C(I-AB)
(test_bddc.cpp:256-266, acceptance criterion 2), symmetry / SPD (test_bddc.cpp:268-314),
additivity, coarse-CG failure (test_bddc.cpp:357-369), PCG KATs (test_krylov.cpp), and the
acceptance iteration counts (proj/test_output.txt:15). Reference outputs come from
tests/golden (the unmodified reference) and from the CPU oracle for arbitrary inputs.
Tolerances: apply / solution 1e-10 relative, residual histories 1e-10 (conftest.history_err),
iterations exact. Two documented exceptions, each backed by a CPU test showing that the
reference's own algorithm moves by more when only its summation order changes
(tests/test_oracle_golden.py): h4m8's BDDC history (1e-7) and heterogeneous plain CG (iteration
band of the pairwise vs sequential sums).
"""
import numpy as np
import pytest

import bddc_oracle as o
from conftest import golden, history_err
from paper_2410_14786_b200 import BddcError, InvalidArgument, Preconditioner, Problem, SolverOptions

pytestmark = pytest.mark.gpu

OPTS = SolverOptions(1e-8, 0.0, 10000, True)


def _oracle(k, m, seed=1, ky=None, kappa=None):
    prob = o.assemble_poisson(k, ky or k, m, kappa)
    cs = o.build_constraints(prob.decomposition)
    P = o.Preconditioner(prob.global_matrix, prob.local_matrices, prob.decomposition, cs)
    return prob, cs, P


@pytest.fixture(scope="module")
def k2m4(gpu):
    p = Problem.poisson(8, 2)
    return p, Preconditioner(p)


@pytest.mark.parametrize("parts", [1, 2, 4])
@pytest.mark.parametrize("name", ["k2m4", "k3m4", "k3m6", "k4m8"])
def test_stages_and_apply_vs_reference(gpu, name, parts):
    g = golden(name)
    k, m, seed = (int(v) for v in g["config"])
    p = Problem.poisson(k * m, k, rhs_seed=seed)
    pre = Preconditioner(p, solve_parts=parts)
    r = p.rhs()
    tol = 1e-10 * max(1.0, np.abs(g["apply_rhs"]).max())
    assert np.abs(pre.interior_correction(r) - g["stage_u0"]).max() < tol
    cond = g["stage_condensed"]
    assert np.abs(pre.coarse_correction(cond) - g["stage_v1"]).max() < tol
    assert np.abs(pre.local_correction(cond) - g["stage_v2"]).max() < tol
    v3 = pre.static_condensation_correction(cond, g["stage_v1"], g["stage_v2"])
    assert np.abs(v3 - g["stage_v3"]).max() < tol
    assert np.abs(pre.coarse_correction(r) - g["coarse_of_rhs"]).max() < tol
    assert np.abs(pre.local_correction(r) - g["local_of_rhs"]).max() < tol
    z = pre.apply(r)
    assert np.abs(z - g["apply_rhs"]).max() <= 1e-12 * np.abs(g["apply_rhs"]).max()


def test_densified_apply_equals_dense_oracle(k2m4):
    # test_bddc.cpp:256-266 / acceptance criterion 2 (gate 1e-9)
    p, pre = k2m4
    n = p.global_dofs
    M = np.stack([pre.apply(np.eye(n)[j]) for j in range(n)], axis=1)
    prob, cs, _ = _oracle(2, 4)
    ref = o.dense_oracle_full(prob.global_matrix, prob.local_matrices, prob.decomposition, cs)
    assert np.abs(M - ref).max() <= 1e-9
    # symmetric positive definite (test_bddc.cpp:268-283)
    assert np.abs(M - M.T).max() <= 1e-8
    assert np.linalg.eigvalsh(0.5 * (M + M.T))[0] > 0.0


def test_zero_linearity_additivity(gpu):
    # test_bddc.cpp:138-155, 285-299
    p = Problem.poisson(12, 3)
    pre = Preconditioner(p)
    n = p.global_dofs
    assert not pre.apply(np.zeros(n)).any()
    rng = np.random.default_rng(107)
    r1, r2 = rng.standard_normal(n), rng.standard_normal(n)
    a, b, c = pre.apply(r1), pre.apply(r2), pre.apply(r1 + r2)
    assert np.abs(c - a - b).max() <= 1e-10 * max(1.0, np.abs(c).max())
    v1 = pre.coarse_correction(r1)
    assert np.abs(pre.coarse_correction(-2.5 * r1) + 2.5 * v1).max() <= 1e-10 * max(1.0, np.abs(v1).max())
    # bilinear symmetry (test_bddc.cpp:301-314)
    assert abs(r2 @ a - r1 @ b) <= 1e-10 * np.linalg.norm(r1) * np.linalg.norm(r2) * np.abs(a).max()


def test_apply_is_deterministic(gpu):
    # test_bddc.cpp:316-329: repeated application is bit identical
    p = Problem.poisson(96, 3)
    pre = Preconditioner(p)
    r = p.rhs()
    assert np.array_equal(pre.apply(r), pre.apply(r))


@pytest.mark.parametrize("name", ["k2m4", "k3m4", "k3m6", "k4m8", "k2m32", "k3m32", "k4m32", "k5m32", "k6m32",
                                  "k8m32", "c1"])
def test_pcg_vs_reference(gpu, name):
    g = golden(name)
    k, m, seed = (int(v) for v in g["config"])
    p = Problem.poisson(k * m, k, rhs_seed=seed)
    pre = Preconditioner(p)
    x, rep = pre.pcg(p.rhs(), OPTS)
    assert rep.iterations == int(g["pcg_report"][0])
    assert rep.converged
    assert history_err(rep.residual_history, g["pcg_history"]) <= 1e-10
    xr = g["pcg_x"] if "pcg_x" in g else None
    if xr is not None:
        assert np.abs(x - xr).max() <= 1e-10 * np.abs(xr).max()
    else:
        stride = int(g["pcg_x_sample_stride"][0])
        assert np.abs(x[::stride] - g["pcg_x_sample"]).max() <= 1e-10 * np.abs(g["pcg_x_sample"]).max()
    if "plain_report" in g:
        xp, rp = pre.pcg(p.rhs(), OPTS, precondition=False)  # empty PreconditionerFn = plain CG
        assert rp.iterations == int(g["plain_report"][0])
        assert history_err(rp.residual_history, g["plain_history"]) <= 1e-10


def test_acceptance_iteration_flatness(gpu):
    # proj/test_output.txt:15 bddc={5,8,9,9,9,9} at m=32, tol 1e-8 (the <=5 clause is known-red)
    its = []
    for k in (2, 3, 4, 5, 6, 8):
        p = Problem.poisson(32 * k, k)
        its.append(Preconditioner(p).pcg(p.rhs(), OPTS)[1].iterations)
    assert its == [5, 8, 9, 9, 9, 9]


@pytest.mark.parametrize("name", ["r4x2m8", "h4m8", "r16x8m8", "c5"])
def test_rectangular_and_heterogeneous_vs_reference(gpu, name):
    g = golden(name)
    cx, cy, kx, ky, dm, ks, seed = (int(v) for v in g["config"])
    p = Problem.poisson(cx, kx, cy, ky, kappa_decades=dm / 1000.0, kappa_seed=ks, rhs_seed=seed)
    pre = Preconditioner(p)
    x, rep = pre.pcg(p.rhs(), OPTS)
    assert abs(rep.iterations - int(g["pcg_report"][0])) <= 1
    # h4m8 alone keeps a 1e-7 history gate: changing only the summation order of the PCG dot
    # products moves its history by more than 1e-9 on the CPU oracle itself
    # (tests/test_oracle_golden.py::test_h4m8_history_sensitivity_is_intrinsic). C5 and the
    # homogeneous bundles are held to the 1e-10 bar (C5 measures ~2e-12).
    htol = H4M8_HISTORY_TOL if name == "h4m8" else 1e-10
    assert history_err(rep.residual_history, g["pcg_history"]) <= htol
    if "pcg_x" in g:
        assert np.abs(x - g["pcg_x"]).max() <= 1e-10 * np.abs(g["pcg_x"]).max()
    else:
        stride = int(g["pcg_x_sample_stride"][0])
        assert np.abs(x[::stride] - g["pcg_x_sample"]).max() <= 1e-10 * np.abs(g["pcg_x_sample"]).max()
    if "apply_rhs" in g:
        assert np.abs(pre.apply(p.rhs()) - g["apply_rhs"]).max() <= 1e-11 * np.abs(g["apply_rhs"]).max()
    if "plain_report" in g:  # BASELINE configs[3] / C4 on the same problem: plain CG (empty M)
        _, rp = pre.pcg(p.rhs(), OPTS, precondition=False)
        assert rp.converged
        if dm:
            # heterogeneous plain CG is summation-order sensitive: the reference's own algorithm
            # takes 1,943 (sequential sums) or 1,939 (pairwise) iterations on C5
            # (test_oracle_golden.py::test_c5_plain_cg_summation_order_band); the GPU's
            # fixed-tree reductions must land inside that band widened by 1
            ref = int(g["plain_report"][0])
            band = PLAIN_BAND.get(name, 1)
            assert ref - band - 1 <= rp.iterations <= ref + 1, (rp.iterations, ref)
        else:
            assert rp.iterations == int(g["plain_report"][0])
            assert history_err(rp.residual_history, g["plain_history"]) <= 1e-10


H4M8_HISTORY_TOL = 1e-7
# width of the summation-order band below the reference's plain-CG count (pairwise vs sequential)
PLAIN_BAND = {"c5": 1943 - 1939, "h4m8": 157 - 156}


@pytest.mark.parametrize("name", ["h4m8", "c5"])
def test_ingested_bundle_vs_reference(gpu, name, tmp_path):
    # the reference's bundle route end to end on the GPU — export, ingest
    # with our reader (no coordinates: graph ordering for the factorisation), solve, compare
    # with the reference run on the same bundle
    g = golden(name)
    cx, cy, kx, ky, dm, ks, seed = (int(v) for v in g["config"])
    src = Problem.poisson(cx, kx, cy, ky, kappa_decades=dm / 1000.0, kappa_seed=ks, rhs_seed=seed)
    p = Problem.from_bundle(src.export_bundle(str(tmp_path)))
    assert p.coords() is None
    x, rep = Preconditioner(p).pcg(p.rhs(), OPTS)
    assert abs(rep.iterations - int(g["pcg_report"][0])) <= 1
    assert history_err(rep.residual_history, g["pcg_history"]) <= (H4M8_HISTORY_TOL if name == "h4m8" else 1e-10)
    if "pcg_x" in g:
        assert np.abs(x - g["pcg_x"]).max() <= 1e-10 * np.abs(g["pcg_x"]).max()
    else:
        stride = int(g["pcg_x_sample_stride"][0])
        assert np.abs(x[::stride] - g["pcg_x_sample"]).max() <= 1e-10 * np.abs(g["pcg_x_sample"]).max()


def test_c2_weak_point_vs_reference(gpu):
    g = golden("c2")
    p = Problem.poisson(800, 8)
    pre = Preconditioner(p)
    x, rep = pre.pcg(p.rhs(), OPTS)
    assert rep.iterations == int(g["pcg_report"][0]) == 11
    assert history_err(rep.residual_history, g["pcg_history"]) <= 1e-10
    stride = int(g["pcg_x_sample_stride"][0])
    assert np.abs(x[::stride] - g["pcg_x_sample"]).max() <= 1e-10 * np.abs(g["pcg_x_sample"]).max()
    assert abs(np.linalg.norm(x) - float(g["pcg_x_norm2"][0])) <= 1e-10 * float(g["pcg_x_norm2"][0])
    # size-independent property: the preconditioner is SPD on the Krylov vectors
    z = pre.apply(p.rhs())
    assert p.rhs() @ z > 0
    # BASELINE configs[3] / C4: plain CG on the same problem, against the reference's plain CG
    # (pcg.cpp:63-67 with an empty PreconditionerFn; study.cpp:123-135 compare mode)
    xp, rp = pre.pcg(p.rhs(), OPTS, precondition=False)
    assert rp.converged and rp.iterations == int(g["plain_report"][0]) == 1649
    assert history_err(rp.residual_history, g["plain_history"]) <= 1e-10


def test_coarse_cg_mode_matches_direct_and_fails_like_reference(gpu):
    p = Problem.poisson(48, 4)
    direct = Preconditioner(p)
    cg = Preconditioner(p, coarse_mode="cg")
    r = p.rhs()
    assert np.abs(direct.apply(r) - cg.apply(r)).max() <= 1e-10 * np.abs(direct.apply(r)).max()
    # test_bddc.cpp:357-369: a starved coarse CG surfaces iterations and residual
    q = Problem.poisson(8, 2)
    starved = Preconditioner(q, coarse_mode="cg", coarse_options=SolverOptions(1e-15, 0.0, 1))
    with pytest.raises(BddcError, match="coarse CG did not converge: 1 iterations"):
        starved.apply(np.ones(q.global_dofs))


def test_error_paths(k2m4):
    p, pre = k2m4
    n = p.global_dofs
    bad = np.ones(n)
    bad[5] = np.nan
    with pytest.raises(InvalidArgument, match="pcg rhs: non-finite entry at index 5"):
        pre.pcg(bad, OPTS)
    with pytest.raises(InvalidArgument, match="bddc apply: non-finite entry at index 5"):
        pre.apply(bad)
    with pytest.raises(InvalidArgument, match="residual size mismatch"):
        pre.apply(np.ones(n + 1))
    with pytest.raises(InvalidArgument, match="tolerances must be positive"):
        pre.pcg(np.ones(n), SolverOptions(0.0, 0.0, 10))
    x, rep = pre.pcg(np.zeros(n), OPTS)  # zero rhs: converged, 0 iterations (test_krylov.cpp:113)
    assert rep.converged and rep.iterations == 0 and not x.any()


def test_budget_exhaustion_and_condition_estimate(gpu):
    # test_krylov.cpp:87-99: history length = iterations + 1, converged = false
    p = Problem.poisson(128, 4)
    pre = Preconditioner(p)
    x, rep = pre.pcg(p.rhs(), SolverOptions(1e-14, 0.0, 3, True))
    assert rep.iterations == 3 and not rep.converged and len(rep.residual_history) == 4
    x, rep = pre.pcg(p.rhs(), OPTS)
    prob, cs, P = _oracle(4, 32)
    _, orep = o.pcg(prob.global_matrix, p.rhs(), P.apply, 1e-8, 0.0, 10000, True)
    assert abs(rep.condition_estimate - orep.condition_estimate) <= 1e-8 * orep.condition_estimate


def test_device_pointer_entry_points(gpu):
    import torch

    p = Problem.poisson(96, 3)
    pre = Preconditioner(p)
    s = torch.cuda.Stream()
    b = torch.tensor(p.rhs(), device="cuda")
    z = torch.empty_like(b)
    x = torch.empty_like(b)
    pre.apply_device(b.data_ptr(), z.data_ptr(), s.cuda_stream)
    s.synchronize()
    assert np.array_equal(z.cpu().numpy(), pre.apply(p.rhs()))
    rep = pre.pcg_device(b.data_ptr(), x.data_ptr(), OPTS, stream=s.cuda_stream)
    xh, reph = pre.pcg(p.rhs(), OPTS)
    assert rep.iterations == reph.iterations and np.array_equal(x.cpu().numpy(), xh)


@pytest.mark.parametrize("k,m", [(2, 8), (4, 16), (8, 32)])
def test_reference_dropin(gpu, k, m):
    # a program written against the reference API swaps in bddc_b200::Preconditioner / pcg on
    # the SAME reference objects (oracle/dropin_check.cpp, include/bddc_b200.hpp)
    import json
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "dropin_check")
    assert os.path.exists(exe), "oracle/_ref/dropin_check not built (__graft_entry__.build())"
    out = subprocess.run([exe, str(k), str(m)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    res = json.loads(out.stdout.strip().splitlines()[0])
    assert res["ok"] and res["iterations"][0] == res["iterations"][1]


def test_c3_strong_scaling_point_vs_reference(gpu):
    # C3: 2520x2520 cells, 24x24 subdomains, 6,345,361 dofs on one B200 against
    # the unmodified reference's history and sampled solution (oracle/gen_golden.py c3)
    g = golden("c3")
    p = Problem.poisson(2520, 24)
    assert p.global_dofs == 6345361
    pre = Preconditioner(p)
    x, rep = pre.pcg(p.rhs(), OPTS)
    assert rep.converged and rep.iterations == int(g["pcg_report"][0])
    assert history_err(rep.residual_history, g["pcg_history"]) <= 1e-10
    stride = int(g["pcg_x_sample_stride"][0])
    assert np.abs(x[::stride] - g["pcg_x_sample"]).max() <= 1e-10 * np.abs(g["pcg_x_sample"]).max()


def test_wide_primal_sets_vs_oracle(gpu):
    # n_primal > 32 (more than one coarse column per lane in the K_i kernel's
    # Phi_G x_c). Every interface dof becomes a primal vertex constraint (n_primal 79 per
    # subdomain at k=2, m=40); the reference / oracle accept arbitrary ConstraintSets
    # (preconditioner.hpp:62-104).
    prob = o.assemble_poisson(2, 2, 40)
    d = prob.decomposition
    gamma = sorted({int(g) for dofs, ni in zip(d.subdomain_dofs, d.interior_counts) for g in dofs[int(ni):]})
    cid = {g: c for c, g in enumerate(gamma)}
    mats, maps = [], []
    for dofs, ni in zip(d.subdomain_dofs, d.interior_counts):
        ni, nl = int(ni), len(dofs)
        rows = np.arange(nl - ni, dtype=np.int32)
        mats.append(o.Csr(nl - ni, nl, np.arange(nl - ni + 1, dtype=np.int32), np.arange(ni, nl, dtype=np.int32),
                          np.ones(nl - ni)))
        maps.append(np.array([cid[int(g)] for g in dofs[ni:]], dtype=np.int32))
        assert rows.size > 32
    cs = o.ConstraintSet(mats, maps, len(gamma))
    P = o.Preconditioner(prob.global_matrix, prob.local_matrices, d, cs)
    tup = lambda m: (m.nrows, m.ncols, m.rowptr, m.cols, m.vals)  # noqa: E731
    gp = Problem.from_arrays(tup(prob.global_matrix), [tup(m) for m in prob.local_matrices], d.subdomain_dofs,
                             d.interior_counts, d.weights, [tup(m) for m in mats], maps, len(gamma))
    pre = Preconditioner(gp)
    r = o.study_rhs(d.global_dofs, 3)
    zr = P.apply(r)
    assert np.abs(pre.apply(r) - zr).max() <= 1e-10 * np.abs(zr).max()


@pytest.mark.parametrize("parts", [1, 4])
def test_c2_solve_parts_vs_reference(gpu, parts):
    # the interior solve split over 1 or 4 CTAs per subdomain (cluster of 4: frontier split,
    # combine over the cluster) against the reference's C2 history
    g = golden("c2")
    p = Problem.poisson(800, 8)
    x, rep = Preconditioner(p, solve_parts=parts).pcg(p.rhs(), OPTS)
    assert rep.iterations == int(g["pcg_report"][0])
    assert history_err(rep.residual_history, g["pcg_history"]) <= 1e-10


def test_repeated_applies_are_bitwise_identical(gpu):
    # determinism of the streamed solves, the DSMEM combine and the fixed-order reductions (the
    # evidence that stands in for compute-sanitizer, which is closed on this pool): repeated
    # applies and solves on the same and on a fresh context are bit for bit the same
    p = Problem.poisson(800, 8)
    a, b = Preconditioner(p), Preconditioner(p)
    r = p.rhs()
    z0 = a.apply(r)
    for _ in range(5):
        assert np.array_equal(a.apply(r), z0)
    assert np.array_equal(b.apply(r), z0)
    x0, _ = a.pcg(r, OPTS)
    assert np.array_equal(b.pcg(r, OPTS)[0], x0)
