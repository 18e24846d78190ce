"""The product's host problem layer (C++, via the C-ABI) is bit-exact with the reference.

Integer maps, matrices and the study rhs are compared against tests/golden (reference
output) exactly; larger configs through SHA-256 digests of the reference arrays.
Mirrors reference tests/test_decomposition.cpp and test_harness.cpp (coarse dims).
"""
import hashlib

import numpy as np
import pytest

import bddc_oracle as o
from conftest import golden
from paper_2410_14786_b200 import InvalidArgument, Problem


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _problem_arrays(p: Problem):
    dofs = p.subdomain_dofs()
    n, _, rp, cols, vals = p.global_matrix()
    kind, entity = p.classes()
    locs = [p.local_matrix(i) for i in range(p.n_subdomains)]
    cons = [p.constraint_matrix(i) for i in range(p.n_subdomains)]
    return {
        "subdomain_dofs": np.concatenate(dofs).astype(np.int32),
        "subdomain_dofs_off": np.concatenate([[0], np.cumsum([len(d) for d in dofs])]).astype(np.int64),
        "interior_counts": p.interior_counts().astype(np.int32),
        "class_kind": kind.astype(np.int32),
        "class_entity": entity.astype(np.int32),
        "multiplicity": p.multiplicity().astype(np.int32),
        "primal_maps": np.concatenate(p.primal_maps()).astype(np.int32),
        "primal_maps_off": np.concatenate([[0], np.cumsum([len(m) for m in p.primal_maps()])]).astype(np.int64),
        "A_rowptr": rp.astype(np.int32), "A_cols": cols.astype(np.int32), "A_vals": vals,
        "weights": np.concatenate(p.weights()),
        "constraints_vals": np.concatenate([c[4] for c in cons]),
        "constraints_cols": np.concatenate([c[3] for c in cons]).astype(np.int32),
        "constraints_rowptr": np.concatenate([c[2] for c in cons]).astype(np.int32),
        "locals_vals": np.concatenate([c[4] for c in locs]),
        "locals_cols": np.concatenate([c[3] for c in locs]).astype(np.int32),
        "locals_rowptr": np.concatenate([c[2] for c in locs]).astype(np.int32),
    }


@pytest.mark.parametrize("name", ["k2m4", "k3m4", "k3m6", "k4m8", "k2m32", "k3m32", "k4m32", "k5m32",
                                  "k6m32", "k8m32", "c1", "c2"])
def test_square_layouts_bit_exact(name):
    g = golden(name)
    k, m, seed = (int(v) for v in g["config"])
    p = Problem.poisson(k * m, k, rhs_seed=seed)
    arr = _problem_arrays(p)
    for key, val in arr.items():
        if key in g:
            assert np.array_equal(val, g[key]), key
        else:
            assert _digest(val) == str(g["digest_" + key]), key
    if "rhs" in g:
        assert np.array_equal(p.rhs(), g["rhs"])
    else:
        stride = int(g["pcg_x_sample_stride"][0])
        assert np.array_equal(p.rhs()[::stride], g["rhs_sample"])


@pytest.mark.parametrize("name", ["r4x2m8", "h4m8", "r16x8m8", "c5"])
def test_bundle_layouts_bit_exact(name):
    # rectangular / heterogeneous problems: the reference ingested our exported bundle and
    # rebuilt maps, weights, constraints and the global matrix itself (bundle.cpp:113-290)
    g = golden(name)
    cx, cy, kx, ky, dec_milli, kseed, seed = (int(v) for v in g["config"])
    p = Problem.poisson(cx, kx, cy, ky, kappa_decades=dec_milli / 1000.0, kappa_seed=kseed, rhs_seed=seed)
    arr = _problem_arrays(p)
    for key in ("subdomain_dofs", "interior_counts", "class_kind", "class_entity", "multiplicity",
                "primal_maps", "A_rowptr", "A_cols", "A_vals", "weights", "constraints_vals",
                "locals_vals"):
        if key in g:
            assert np.array_equal(arr[key], g[key]), key
        else:
            assert _digest(arr[key]) == str(g["digest_" + key]), key


@pytest.mark.parametrize("kx,ky,m", [(4, 2, 8), (3, 5, 6), (2, 3, 4)])
def test_rectangular_matches_oracle(kx, ky, m):
    p = Problem.poisson(kx * m, kx, ky * m, ky)
    d = o.build_decomposition(kx, ky, m)
    kind, entity = p.classes()
    assert np.array_equal(kind, d.kind) and np.array_equal(entity, d.entity)
    assert np.array_equal(np.concatenate(p.subdomain_dofs()), np.concatenate(d.subdomain_dofs))
    cs = o.build_constraints(d)
    assert np.array_equal(np.concatenate(p.primal_maps()), np.concatenate(cs.primal_maps))
    assert p.n_coarse == cs.n_coarse == (kx - 1) * (ky - 1) + (kx - 1) * ky + kx * (ky - 1)


def test_coarse_dimensions():
    # test_harness.cpp:82-84: k = 2, 3, 4 -> 5, 16, 33
    assert [Problem.poisson(4 * k, k).n_coarse for k in (2, 3, 4)] == [5, 16, 33]


def test_layout_errors():
    with pytest.raises(InvalidArgument, match="not divisible"):
        Problem.poisson(10, 3)
    with pytest.raises(InvalidArgument, match="at least 2 cells"):
        Problem.poisson(4, 4)
    with pytest.raises(InvalidArgument, match="at least 2 subdomains"):
        Problem.poisson(8, 1)


@pytest.mark.parametrize("name", ["r4x2m8", "h4m8", "r16x8m8", "c5"])
def test_ingest_bundle_matches_reference_ingest(name, tmp_path):
    # our reader on the bundle the reference ingested reproduces the
    # reference's ingest output (maps, classes, weights, constraints, global matrix) bit for bit
    g = golden(name)
    cx, cy, kx, ky, dec_milli, kseed, seed = (int(v) for v in g["config"])
    p = Problem.poisson(cx, kx, cy, ky, kappa_decades=dec_milli / 1000.0, kappa_seed=kseed, rhs_seed=seed)
    q = Problem.from_bundle(p.export_bundle(str(tmp_path)))
    arr = _problem_arrays(q)
    for key in ("subdomain_dofs", "interior_counts", "class_kind", "class_entity", "multiplicity",
                "primal_maps", "A_rowptr", "A_cols", "A_vals", "weights", "constraints_vals",
                "locals_vals"):
        if key in g:
            assert np.array_equal(arr[key], g[key]), key
        else:
            assert _digest(arr[key]) == str(g["digest_" + key]), key
    assert np.array_equal(q.rhs(), p.rhs())
    assert q.n_coarse == p.n_coarse


def test_ingest_bundle_round_trip_and_symmetric_mtx(tmp_path):
    p = Problem.poisson(24, 3, 16, 2, kappa_decades=1.5, rhs_seed=7)
    m = p.export_bundle(str(tmp_path / "b"))
    q = Problem.from_bundle(m)
    a, b = _problem_arrays(p), _problem_arrays(q)
    for key in a:
        assert np.array_equal(a[key], b[key]), key
    # a shuffled map (interface dofs first) and a symmetric Matrix Market file: the reader
    # reorders interior-first stably and mirrors the off-diagonal entries
    d = tmp_path / "b"
    dofs = p.subdomain_dofs()[0]
    nI = int(p.interior_counts()[0])
    perm = np.concatenate([np.arange(nI, len(dofs)), np.arange(nI)])
    (d / "map_000.txt").write_text("".join(f"{int(v)}\n" for v in dofs[perm]))
    nl, _, rp, cols, vals = p.local_matrix(0)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm))
    lines = []
    for r in range(nl):
        for e in range(rp[r], rp[r + 1]):
            i, j = inv[r], inv[cols[e]]
            if i >= j:
                lines.append(f"{i + 1} {j + 1} {float(vals[e])!r}\n")
    (d / "A_000.mtx").write_text("%%MatrixMarket matrix coordinate real symmetric\n% comment\n"
                                 f"{nl} {nl} {len(lines)}\n" + "".join(lines))
    r = Problem.from_bundle(m)
    assert np.array_equal(np.concatenate(r.subdomain_dofs()), np.concatenate(p.subdomain_dofs()))
    assert np.array_equal(r.local_matrix(0)[4], p.local_matrix(0)[4])
    assert np.array_equal(r.global_matrix()[4], p.global_matrix()[4])


def test_ingest_bundle_errors(tmp_path):
    from paper_2410_14786_b200 import BddcError
    with pytest.raises(BddcError, match="missing file"):
        Problem.from_bundle(str(tmp_path / "nope" / "manifest.txt"))
    p = Problem.poisson(8, 2)
    m = p.export_bundle(str(tmp_path / "b"))
    man = open(m).read()
    open(m, "w").write(man.replace("global_dofs", "bogus_key"))
    with pytest.raises(BddcError, match="unknown manifest key 'bogus_key'"):
        Problem.from_bundle(m)
    open(m, "w").write(man)
    cls = (tmp_path / "b" / "classes.txt").read_text().split("\n")
    first_iface = next(i for i, c in enumerate(cls) if c != "interior")
    cls[first_iface] = "interior"
    (tmp_path / "b" / "classes.txt").write_text("\n".join(cls))
    with pytest.raises(BddcError, match=f"bundle validation: dof {first_iface} has multiplicity . but is classified interior"):
        Problem.from_bundle(m)
