"""CPU oracle for the BDDC-PCG hot path — TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference algorithm (arXiv 2410.14786 reference,
/root/reference/proj). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg may import this module, and only as the checker. The product
path (paper_2410_14786_b200) never imports it and has no CPU fallback.

Pinned against the unmodified reference: tests/test_oracle_golden.py checks every
function here against tests/golden/*.npz, which oracle/gen_golden.py produced by
running the reference library compiled from its own sources (oracle/Makefile).

Restated functions (file:line into /root/reference/proj):
  q1_element_matrix       src/grid.cpp:19-39
  classify_dofs           src/decomposition.cpp:30-59   (generalised to kx x ky)
  build_weights           src/decomposition.cpp:61-71
  build_decomposition     src/decomposition.cpp:73-110
  build_constraints       src/decomposition.cpp:112-159
  assemble_poisson        src/decomposition.cpp:161-203
  global_from_locals      src/decomposition.cpp:205-222
  csr_from_triplets       src/csr_matrix.cpp:52-88
  spmv                    src/csr_matrix.cpp:90-102
  study_rhs               src/study.cpp:69-75  (libstdc++ mt19937_64 + normal_distribution)
  pcg                     src/pcg.cpp:40-109
  condition_estimate      src/pcg.cpp:111-173
  Preconditioner          src/preconditioner.cpp:12-249 (saddle LU -> scipy SuperLU)
  DenseOracle.full        tests/bddc_dense_oracle.hpp:21-130
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

INTERIOR, EDGE, CORNER = 0, 1, 2


# --------------------------------------------------------------------------- CSR
@dataclass
class Csr:
    nrows: int
    ncols: int
    rowptr: np.ndarray
    cols: np.ndarray
    vals: np.ndarray

    def scipy(self) -> sp.csr_matrix:
        return sp.csr_matrix((self.vals, self.cols, self.rowptr), shape=(self.nrows, self.ncols))

    def dense(self) -> np.ndarray:
        d = np.zeros((self.nrows, self.ncols))
        for i in range(self.nrows):
            for p in range(self.rowptr[i], self.rowptr[i + 1]):
                d[i, self.cols[p]] += self.vals[p]
        return d


def csr_from_triplets(nrows: int, ncols: int, rows, cols, vals) -> Csr:
    """csr_matrix.cpp:52-88: stable sort by (row, col); duplicates summed in input order."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    if rows.size and (rows.min() < 0 or rows.max() >= nrows or cols.min() < 0 or cols.max() >= ncols):
        raise ValueError("from_triplets: entry out of range")
    order = np.lexsort((cols, rows))  # stable
    r, c, v = rows[order], cols[order], vals[order]
    if r.size == 0:
        return Csr(nrows, ncols, np.zeros(nrows + 1, np.int32), np.zeros(0, np.int32), np.zeros(0))
    key = r * ncols + c
    new = np.ones(r.size, dtype=bool)
    new[1:] = key[1:] != key[:-1]
    gid = np.cumsum(new) - 1
    out = np.zeros(int(gid[-1]) + 1)
    np.add.at(out, gid, v)  # sequential, in sorted (== input) order, from 0.0
    ur, uc = r[new], c[new]
    rowptr = np.zeros(nrows + 1, dtype=np.int64)
    np.add.at(rowptr, ur + 1, 1)
    rowptr = np.cumsum(rowptr)
    return Csr(nrows, ncols, rowptr.astype(np.int32), uc.astype(np.int32), out)


def spmv(A: Csr, x: np.ndarray) -> np.ndarray:
    return A.scipy() @ x


# -------------------------------------------------------------------------- grid
def q1_element_matrix() -> np.ndarray:
    """grid.cpp:19-39 — same operation order, so bit-identical."""
    g0 = 0.5 - 0.5 / math.sqrt(3.0)
    g1 = 0.5 + 0.5 / math.sqrt(3.0)
    K = [[0.0] * 4 for _ in range(4)]
    for x, y in ((g0, g0), (g1, g0), (g1, g1), (g0, g1)):
        dN = ((-(1 - y), -(1 - x)), (1 - y, -x), (y, x), (-y, 1 - x))
        for a in range(4):
            for b in range(4):
                K[a][b] += 0.25 * (dN[a][0] * dN[b][0] + dN[a][1] * dN[b][1])
    return np.array(K)


@dataclass
class Decomposition:
    kx: int
    ky: int
    m: int
    global_dofs: int
    subdomain_dofs: list
    interior_counts: np.ndarray
    kind: np.ndarray
    entity: np.ndarray
    multiplicity: np.ndarray
    weights: list

    @property
    def n_subdomains(self) -> int:
        return len(self.subdomain_dofs)


def classify_dofs(kx: int, ky: int, m: int):
    """decomposition.cpp:30-59, entity numbering generalised to kx x ky (reduces to
    the reference formulas when kx == ky; SURVEY Appendix A probe4)."""
    nfx, nfy = kx * m - 1, ky * m - 1
    ix = np.tile(np.arange(1, nfx + 1), nfy)
    iy = np.repeat(np.arange(1, nfy + 1), nfx)
    on_x = ix % m == 0
    on_y = iy % m == 0
    kind = np.zeros(nfx * nfy, np.int32)
    entity = np.full(nfx * nfy, -1, np.int32)
    c = on_x & on_y
    kind[c] = CORNER
    entity[c] = (iy[c] // m - 1) * (kx - 1) + (ix[c] // m - 1)
    v = on_x & ~on_y
    kind[v] = EDGE
    entity[v] = (iy[v] // m) * (kx - 1) + (ix[v] // m - 1)
    h = on_y & ~on_x
    kind[h] = EDGE
    entity[h] = (kx - 1) * ky + (iy[h] // m - 1) * kx + ix[h] // m
    return kind, entity


def build_decomposition(kx: int, ky: int, m: int) -> Decomposition:
    """decomposition.cpp:73-110: interior-first ascending, then interface ascending."""
    if min(kx, ky) < 1 or kx * ky < 2 or m < 2:
        raise ValueError("decomposition: bad layout")
    nfx, nfy = kx * m - 1, ky * m - 1
    kind, entity = classify_dofs(kx, ky, m)
    mult = np.zeros(nfx * nfy, np.int32)
    dofs_list, counts = [], []
    for sy in range(ky):
        for sx in range(kx):
            iys = np.arange(sy * m, (sy + 1) * m + 1)
            ixs = np.arange(sx * m, (sx + 1) * m + 1)
            IY, IX = np.meshgrid(iys, ixs, indexing="ij")
            IX, IY = IX.ravel(), IY.ravel()
            ok = (IX >= 1) & (IX <= nfx) & (IY >= 1) & (IY <= nfy)
            dof = ((IY - 1) * nfx + (IX - 1))[ok]
            mult[dof] += 1
            interior = dof[kind[dof] == INTERIOR]
            interface = dof[kind[dof] != INTERIOR]
            counts.append(interior.size)
            dofs_list.append(np.concatenate([interior, interface]).astype(np.int32))
    weights = [1.0 / mult[d].astype(np.float64) for d in dofs_list]
    return Decomposition(kx, ky, m, nfx * nfy, dofs_list, np.array(counts, np.int32), kind, entity,
                         mult, weights)


@dataclass
class ConstraintSet:
    constraint_matrices: list
    primal_maps: list
    n_coarse: int


def build_constraints(d: Decomposition) -> ConstraintSet:
    """decomposition.cpp:112-159: corners first then edges, ascending entity ids."""
    corners = sorted(set(d.entity[d.kind == CORNER].tolist()))
    edges = sorted(set(d.entity[d.kind == EDGE].tolist()))
    cid = {e: i for i, e in enumerate(corners)}
    eid = {e: i + len(corners) for i, e in enumerate(edges)}
    mats, maps = [], []
    for i, dofs in enumerate(d.subdomain_dofs):
        rows: dict[int, list[int]] = {}
        for l, g in enumerate(dofs):
            k = d.kind[g]
            if k == CORNER:
                rows.setdefault(cid[int(d.entity[g])], []).append(l)
            elif k == EDGE:
                rows.setdefault(eid[int(d.entity[g])], []).append(l)
        if not rows:
            raise RuntimeError(f"constraints: subdomain {i} has no interface constraints; "
                               "the saddle system would be singular")
        tr, tc, tv, pm = [], [], [], []
        for row, primal in enumerate(sorted(rows)):
            pm.append(primal)
            locs = rows[primal]
            value = 1.0 / float(len(locs))
            tr += [row] * len(locs)
            tc += locs
            tv += [value] * len(locs)
        mats.append(csr_from_triplets(len(pm), len(dofs), tr, tc, tv))
        maps.append(np.array(pm, np.int32))
    return ConstraintSet(mats, maps, len(corners) + len(edges))


@dataclass
class PoissonProblem:
    decomposition: Decomposition
    global_matrix: Csr
    local_matrices: list


def assemble_poisson(kx: int, ky: int, m: int, kappa=None) -> PoissonProblem:
    """decomposition.cpp:161-203 (kappa: optional per-element coefficient, row-major
    over the kx*m x ky*m cells; None = the reference's unit Laplacian)."""
    d = build_decomposition(kx, ky, m)
    K = q1_element_matrix()
    nfx, nfy = kx * m - 1, ky * m - 1
    ncx = kx * m

    def gdof(ix, iy):
        ok = (ix >= 1) & (ix <= nfx) & (iy >= 1) & (iy <= nfy)
        return np.where(ok, (iy - 1) * nfx + (ix - 1), -1)

    locals_ = []
    g2l = np.full(d.global_dofs, -1, np.int64)
    for si, dofs in enumerate(d.subdomain_dofs):
        g2l[dofs] = np.arange(dofs.size)
        sx, sy = si % kx, si // kx
        cy, cx = np.meshgrid(np.arange(sy * m, (sy + 1) * m), np.arange(sx * m, (sx + 1) * m),
                             indexing="ij")
        cx, cy = cx.ravel(), cy.ravel()
        vids = np.stack([gdof(cx, cy), gdof(cx + 1, cy), gdof(cx + 1, cy + 1), gdof(cx, cy + 1)], 1)
        scale = None if kappa is None else np.asarray(kappa)[cy * ncx + cx]
        tr, tc, tv = [], [], []
        # element-major, then a, then b: identical triplet order to the reference
        A_idx = np.repeat(np.arange(4), 4)
        B_idx = np.tile(np.arange(4), 4)
        va, vb = vids[:, A_idx], vids[:, B_idx]
        kv = np.broadcast_to(K[A_idx, B_idx], va.shape)
        if scale is not None:
            kv = scale[:, None] * kv
        ok = (va >= 0) & (vb >= 0)
        tr = g2l[va[ok]]
        tc = g2l[vb[ok]]
        tv = kv[ok]
        locals_.append(csr_from_triplets(dofs.size, dofs.size, tr, tc, tv))
        g2l[dofs] = -1
    A = global_from_locals(d, locals_)
    return PoissonProblem(d, A, locals_)


def global_from_locals(d: Decomposition, locals_: list) -> Csr:
    """decomposition.cpp:205-222."""
    rr, cc, vv = [], [], []
    for dofs, Ai in zip(d.subdomain_dofs, locals_):
        rows = np.repeat(np.arange(Ai.nrows), np.diff(Ai.rowptr))
        rr.append(dofs[rows])
        cc.append(dofs[Ai.cols])
        vv.append(Ai.vals)
    return csr_from_triplets(d.global_dofs, d.global_dofs, np.concatenate(rr), np.concatenate(cc),
                             np.concatenate(vv))


# --------------------------------------------------------------------- study_rhs
_MT_N, _MT_M = 312, 156
_MATRIX_A = np.uint64(0xB5026F5AA96619E9)
_UPPER = np.uint64(0xFFFFFFFF80000000)
_LOWER = np.uint64(0x7FFFFFFF)


def _mt19937_64(seed: int, count: int) -> np.ndarray:
    """std::mt19937_64 output stream (vectorised twist)."""
    mt = np.zeros(_MT_N, dtype=np.uint64)
    mt[0] = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        for i in range(1, _MT_N):
            prev = int(mt[i - 1])
            mt[i] = np.uint64((6364136223846793005 * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF)
    out = np.empty(count + _MT_N, dtype=np.uint64)
    produced = 0
    one = np.uint64(1)
    while produced < count:
        # twist: element i depends on i+1 and i+M (both possibly updated earlier)
        new = mt.copy()
        for lo, hi in ((0, _MT_N - _MT_M), (_MT_N - _MT_M, _MT_N - 1)):
            x = (new[lo:hi] & _UPPER) | (new[lo + 1:hi + 1] & _LOWER)
            xa = (x >> one) ^ np.where((x & one) == one, _MATRIX_A, np.uint64(0))
            src = (np.arange(lo, hi) + _MT_M) % _MT_N
            new[lo:hi] = new[src] ^ xa
        x = (new[_MT_N - 1] & _UPPER) | (new[0] & _LOWER)
        xa = (x >> one) ^ (_MATRIX_A if (x & one) == one else np.uint64(0))
        new[_MT_N - 1] = new[_MT_M - 1] ^ xa
        mt = new
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        out[produced:produced + _MT_N] = y
        produced += _MT_N
    return out[:count]


def study_rhs(n: int, seed: int) -> np.ndarray:
    """study.cpp:69-75: libstdc++ normal_distribution (Marsaglia polar; returns y*mult
    first and caches x*mult) over generate_canonical<double,53>(mt19937_64)."""
    need = int(1.3 * n) + 64
    while True:
        draws = _mt19937_64(seed, 2 * ((need + 1) // 2))
        u = draws.astype(np.float64) / 18446744073709551616.0
        u[u >= 1.0] = np.nextafter(1.0, 0.0)
        x = 2.0 * u[0::2] - 1.0
        y = 2.0 * u[1::2] - 1.0
        r2 = x * x + y * y
        idx = np.nonzero(~((r2 > 1.0) | (r2 == 0.0)))[0]
        if 2 * idx.size >= n:
            break
        need = int(need * 1.5)
    idx = idx[:(n + 1) // 2]
    mult = np.array([math.sqrt(-2.0 * math.log(v) / v) for v in r2[idx].tolist()])
    vals = np.empty(2 * idx.size)
    vals[0::2] = y[idx] * mult
    vals[1::2] = x[idx] * mult
    return vals[:n].copy()


# --------------------------------------------------------------------------- PCG
@dataclass
class SolveReport:
    iterations: int = 0
    final_relative_residual: float = 0.0
    residual_history: list = field(default_factory=list)
    condition_estimate: float | None = None
    converged: bool = False


def sequential_dot(a: np.ndarray, b: np.ndarray) -> float:
    """dot exactly as vector_ops.hpp:15-22: one left-to-right running sum (np.cumsum is sequential;
    no fused multiply-add, like the reference's -O3 x86-64 build)."""
    return float(np.cumsum(a * b)[-1]) if a.size else 0.0


def pcg(A, b, M=None, rel_tolerance=1e-8, abs_tolerance=0.0, max_iterations=1000,
        record_history=False, dot=np.dot):
    """pcg.cpp:40-109 (zero initial guess, recurrence residual). `dot` = np.dot (pairwise sums)
    by default; `sequential_dot` reproduces the reference's summation order bit for bit."""
    if not rel_tolerance > 0.0 or abs_tolerance < 0.0:
        raise ValueError("pcg: tolerances must be positive")
    if max_iterations < 1:
        raise ValueError("pcg: max_iterations must be at least 1")
    As = A.scipy() if isinstance(A, Csr) else A
    b = np.asarray(b, dtype=np.float64)
    if not np.all(np.isfinite(b)):
        raise ValueError("pcg rhs: non-finite entry at index %d" % int(np.argmin(np.isfinite(b))))
    rep = SolveReport()
    x = np.zeros_like(b)
    norm_b = math.sqrt(float(dot(b, b)))
    if record_history:
        rep.residual_history.append(1.0)
    if norm_b == 0.0:
        rep.converged = True
        return x, rep
    r = b.copy()
    z = M(r) if M is not None else r.copy()
    p = z.copy()
    rho = float(dot(r, z))
    alphas, betas = [], []
    rel = 1.0
    for it in range(1, max_iterations + 1):
        q = As @ p
        curv = float(dot(p, q))
        if curv <= 0.0:
            raise RuntimeError("matrix not SPD")
        alpha = rho / curv
        alphas.append(alpha)
        x += alpha * p
        r -= alpha * q
        rel = math.sqrt(float(dot(r, r))) / norm_b
        if record_history:
            rep.residual_history.append(rel)
        rep.iterations = it
        if rel <= rel_tolerance or (abs_tolerance > 0.0 and rel * norm_b <= abs_tolerance):
            rep.converged = True
            break
        if it == max_iterations:
            break
        z = M(r) if M is not None else r.copy()
        rho_next = float(dot(r, z))
        beta = rho_next / rho
        betas.append(beta)
        rho = rho_next
        p = z + beta * p
    rep.final_relative_residual = rel
    rep.condition_estimate = condition_estimate(alphas, betas)
    return x, rep


def condition_estimate(alphas, betas):
    """pcg.cpp:111-125 + Sturm bisection pcg.cpp:127-173."""
    k = len(alphas)
    if k < 2 or len(betas) + 1 < k:
        return None
    diag = [0.0] * k
    off = [0.0] * (k - 1)
    for i in range(k):
        diag[i] = 1.0 / alphas[i]
        if i > 0:
            diag[i] += betas[i - 1] / alphas[i - 1]
        if i + 1 < k:
            off[i] = math.sqrt(betas[i]) / alphas[i]
    lo, hi = _tridiag_extremes(diag, off)
    if not lo > 0.0:
        return None
    return hi / lo


def _tridiag_extremes(diag, off):
    n = len(diag)
    if n == 1:
        return diag[0], diag[0]
    lo = hi = diag[0]
    for i in range(n):
        rad = (abs(off[i - 1]) if i > 0 else 0.0) + (abs(off[i]) if i + 1 < n else 0.0)
        lo = min(lo, diag[i] - rad)
        hi = max(hi, diag[i] + rad)

    def below(x):
        cnt, q = 0, 1.0
        for i in range(n):
            o2 = off[i - 1] * off[i - 1] if i > 0 else 0.0
            q = diag[i] - x - o2 / q
            if q == 0.0:
                q = 1e-300
            if q < 0.0:
                cnt += 1
        return cnt

    def bisect(target):
        a, b = lo, hi
        step = 0
        while step < 200 and b - a > 1e-15 * max(1.0, abs(b)):
            mid = 0.5 * (a + b)
            if below(mid) >= target:
                b = mid
            else:
                a = mid
            step += 1
        return 0.5 * (a + b)

    return bisect(1), bisect(n)


# ---------------------------------------------------------------- preconditioner
class Preconditioner:
    """preconditioner.cpp:100-249. Local saddle and interior systems are solved with
    scipy's SuperLU instead of the reference's own threshold LU (same linear algebra)."""

    def __init__(self, A: Csr, locals_: list, d: Decomposition, cs: ConstraintSet,
                 coarse_rtol=1e-12, coarse_max_iterations=500, exact_coarse=False):
        self.A, self.d, self.cs = A, d, cs
        self.As = A.scipy()
        self.locals = locals_
        self.saddle_lu, self.interior_lu, self.phi, self.lam, self.aci = [], [], [], [], []
        for i, (Ai, Ci) in enumerate(zip(locals_, cs.constraint_matrices)):
            try:
                As_ = Ai.scipy()
                Cs = Ci.scipy()
                S = sp.bmat([[As_, Cs.T], [Cs, None]], format="csc")
                lu = spla.splu(S)
                nl, npr = Ai.nrows, Ci.nrows
                rhs = np.zeros((nl + npr, npr))
                rhs[nl:, :] = np.eye(npr)
                sol = lu.solve(rhs)
                if not np.all(np.isfinite(sol)):
                    raise RuntimeError("singular saddle system")
                self.saddle_lu.append(lu)
                self.phi.append(sol[:nl])
                self.lam.append(sol[nl:])
                self.aci.append(sol[:nl].T @ (As_ @ sol[:nl]))
                ni = int(d.interior_counts[i])
                self.interior_lu.append(spla.splu(As_[:ni, :ni].tocsc()) if ni else None)
            except Exception as e:  # preconditioner.cpp:119-121
                raise RuntimeError(f"bddc setup: subdomain {i}: {e}") from e
        tr, tc, tv = [], [], []
        for blk, mp in zip(self.aci, cs.primal_maps):
            for r in range(blk.shape[0]):
                for c in range(blk.shape[1]):
                    if blk[r, c] != 0.0:
                        tr.append(mp[r]); tc.append(mp[c]); tv.append(blk[r, c])
        self.Ac = csr_from_triplets(cs.n_coarse, cs.n_coarse, tr, tc, tv)
        self.coarse_rtol, self.coarse_max = coarse_rtol, coarse_max_iterations
        self.exact_coarse = exact_coarse

    # preconditioner.cpp:129-171
    def coarse_correction(self, r):
        d = self.d
        rc = np.zeros(self.cs.n_coarse)
        for i, dofs in enumerate(d.subdomain_dofs):
            c = self.phi[i].T @ (d.weights[i] * r[dofs])
            for j, q in enumerate(self.cs.primal_maps[i]):
                rc[q] += c[j]
        if self.exact_coarse:
            xc = np.linalg.solve(self.Ac.dense(), rc)
        else:
            xc, rep = pcg(self.Ac, rc, None, self.coarse_rtol, 0.0, self.coarse_max)
            if not rep.converged:
                raise RuntimeError("coarse CG did not converge: %d iterations, relative residual %f"
                                   % (rep.iterations, rep.final_relative_residual))
        v1 = np.zeros(d.global_dofs)
        for i, dofs in enumerate(d.subdomain_dofs):
            loc = d.weights[i] * (self.phi[i] @ xc[self.cs.primal_maps[i]])
            np.add.at(v1, dofs, loc)
        return v1

    # preconditioner.cpp:173-192
    def local_correction(self, r):
        d = self.d
        v2 = np.zeros(d.global_dofs)
        for i, dofs in enumerate(d.subdomain_dofs):
            w = d.weights[i]
            npr = self.cs.constraint_matrices[i].nrows
            rhs = np.concatenate([w * r[dofs], np.zeros(npr)])
            sol = self.saddle_lu[i].solve(rhs)
            np.add.at(v2, dofs, w * sol[:dofs.size])
        return v2

    # preconditioner.cpp:194-213
    def interior_correction(self, r):
        d = self.d
        u = np.zeros(d.global_dofs)
        for i, dofs in enumerate(d.subdomain_dofs):
            ni = int(d.interior_counts[i])
            if ni:
                u[dofs[:ni]] += self.interior_lu[i].solve(r[dofs[:ni]])
        return u

    # preconditioner.cpp:215-223
    def static_condensation_correction(self, r, v1, v2):
        return self.interior_correction(r - self.As @ (v1 + v2))

    # preconditioner.cpp:225-249
    def apply(self, r):
        r = np.asarray(r, dtype=np.float64)
        if r.size != self.d.global_dofs:
            raise ValueError("bddc apply: residual size mismatch")
        if not np.all(np.isfinite(r)):
            raise ValueError("bddc apply: non-finite entry at index %d" % int(np.argmin(np.isfinite(r))))
        u0 = self.interior_correction(r)
        cond = r - self.As @ u0
        v1 = self.coarse_correction(cond)
        v2 = self.local_correction(cond)
        v3 = self.static_condensation_correction(cond, v1, v2)
        return u0 + v1 + v2 + v3


def dense_oracle_full(A: Csr, locals_: list, d: Decomposition, cs: ConstraintSet) -> np.ndarray:
    """tests/bddc_dense_oracle.hpp:21-130: B + (I - B A) C (I - A B)."""
    n = d.global_dofs
    Ad = A.dense()
    E = np.zeros((n, cs.n_coarse))
    iface = np.zeros((n, n))
    Acd = np.zeros((cs.n_coarse, cs.n_coarse))
    for i, dofs in enumerate(d.subdomain_dofs):
        Ai, Ci = locals_[i].dense(), cs.constraint_matrices[i].dense()
        nl, nc = Ai.shape[0], Ci.shape[0]
        S = np.zeros((nl + nc, nl + nc))
        S[:nl, :nl] = Ai
        S[nl:, :nl] = Ci
        S[:nl, nl:] = Ci.T
        inv = np.linalg.inv(S)
        Z, phi = inv[:nl, :nl], inv[:nl, nl:]
        mp = cs.primal_maps[i]
        Acd[np.ix_(mp, mp)] += phi.T @ Ai @ phi
        w = d.weights[i]
        E[np.ix_(dofs, mp)] += w[:, None] * phi
        iface[np.ix_(dofs, dofs)] += w[:, None] * Z * w[None, :]
    iface += E @ np.linalg.inv(Acd) @ E.T
    B = np.zeros((n, n))
    for i, dofs in enumerate(d.subdomain_dofs):
        ni = int(d.interior_counts[i])
        Ai = locals_[i].dense()
        B[np.ix_(dofs[:ni], dofs[:ni])] += np.linalg.inv(Ai[:ni, :ni])
    left = np.eye(n) - B @ Ad
    return left @ iface @ left.T + B


def poisson_setup(k: int, m: int, ky: int | None = None, seed: int = 1, kappa=None):
    """Convenience: problem, constraints and study rhs as study.cpp:90-101 builds them."""
    ky = k if ky is None else ky
    prob = assemble_poisson(k, ky, m, kappa)
    cs = build_constraints(prob.decomposition)
    b = study_rhs(prob.decomposition.global_dofs, seed)
    return prob, cs, b
