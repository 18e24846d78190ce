"""Generate tests/golden/*.npz from the UNMODIFIED reference (TEST INFRASTRUCTURE).

Runs oracle/_ref/ref_driver (built by `make -C oracle` from /root/reference/proj/src)
and packs its .npy dumps into compressed fixtures. Run in the build container
(where /root/reference exists); the fixtures are committed and travel to the GPU box.

    python oracle/gen_golden.py            # all fixtures
    python oracle/gen_golden.py k2m4 c1    # selected ones

Fixture kinds
  full   : every dump array (small problems; maps, matrices, Phi/Lambda/A_ci, stages, PCG)
  solve  : PCG report/history/solution + rhs-apply + integer-map digests (mid-size)
  history: PCG report/history, plain-CG report, map digests, sampled solution (large)
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
DRIVER = os.path.join(HERE, "_ref", "ref_driver")
GOLDEN = os.path.join(REPO, "tests", "golden")

# name -> (k, m, seed, kind, extra flags)
CONFIGS = {
    "k2m4": (2, 4, 1, "full", ["--plain"]),
    "k3m4": (3, 4, 1, "full", ["--plain"]),
    "k3m6": (3, 6, 7, "full", ["--plain"]),
    "k4m8": (4, 8, 1, "full", ["--plain"]),
    "k2m32": (2, 32, 1, "solve", ["--plain"]),
    "k3m32": (3, 32, 1, "solve", ["--plain"]),
    "k4m32": (4, 32, 1, "solve", ["--plain"]),
    "k5m32": (5, 32, 1, "solve", ["--plain"]),
    "k6m32": (6, 32, 1, "solve", ["--plain"]),
    "k8m32": (8, 32, 1, "history", ["--plain"]),
    "c1": (4, 64, 1, "solve", ["--plain"]),
    "c2": (8, 100, 1, "history", ["--no-stages", "--plain"]),  # C2 + C4 (plain CG, 1,649 its)
    "c2g4": (16, 100, 1, "history", ["--no-stages"]),   # C2 weak-scaling layout at 4 GPUs
    "c3": (24, 105, 1, "history", ["--no-stages"]),     # C3 strong scaling, 6,345,361 dofs
}

# Problems the reference cannot assemble itself (rectangular layouts, heterogeneous
# coefficients) reach it through its own bundle ingestion (src/bundle.cpp:113-290): the
# bundle is written by this repo's exporter, solved by the unmodified reference.
# name -> (cells_x, cells_y, kx, ky, kappa_decades, kappa_seed, rhs_seed, kind)
BUNDLES = {
    "r4x2m8": (32, 16, 4, 2, 0.0, 0, 1, "full"),
    "h4m8": (32, 32, 4, 4, 2.0, 0x5EED, 1, "full"),
    "r16x8m8": (128, 64, 16, 8, 0.0, 0, 1, "solve"),
    "c5": (352, 352, 8, 8, 2.0, 0x5EED, 1, "history"),
    "c2g2": (1600, 800, 16, 8, 0.0, 0, 1, "history"),  # C2 weak-scaling layout at 2 GPUs
    "c2g8": (3200, 1600, 32, 16, 0.0, 0, 1, "history"),  # C2 weak-scaling layout at 8 GPUs (n_c 1,441)
}

NO_PLAIN = {"c2g8"}  # plain CG at 5.1M dofs is ~5 min of reference time and adds nothing

MAP_ARRAYS = ("subdomain_dofs", "subdomain_dofs_off", "interior_counts", "class_kind",
              "class_entity", "multiplicity", "primal_maps", "primal_maps_off",
              "A_rowptr", "A_cols", "A_vals", "weights", "constraints_vals",
              "constraints_cols", "constraints_rowptr", "locals_vals", "locals_cols",
              "locals_rowptr")


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run(name: str) -> None:
    workers = str(min(8, os.cpu_count() or 1))
    if name in BUNDLES:
        cx, cy, kx, ky, dec, kseed, seed, kind = BUNDLES[name]
        flags = [] if name in NO_PLAIN else ["--plain"]
        sys.path.insert(0, REPO)
        from paper_2410_14786_b200 import Problem

        with tempfile.TemporaryDirectory() as bdir, tempfile.TemporaryDirectory() as tmp:
            prob = Problem.poisson(cx, kx, cy, ky, kappa_decades=dec, kappa_seed=kseed, rhs_seed=seed)
            manifest = prob.export_bundle(bdir)
            cmd = [DRIVER, "dumpb", manifest, tmp, workers] + flags
            out = subprocess.run(cmd, check=True, capture_output=True, text=True).stdout
            arrays = {f[:-4]: np.load(os.path.join(tmp, f)) for f in os.listdir(tmp) if f.endswith(".npy")}
        config = np.array([cx, cy, kx, ky, int(dec * 1000), kseed, seed], dtype=np.int64)
    else:
        k, m, seed, kind, flags = CONFIGS[name]
        with tempfile.TemporaryDirectory() as tmp:
            cmd = [DRIVER, "dump", str(k), str(m), str(seed), tmp, workers] + flags
            out = subprocess.run(cmd, check=True, capture_output=True, text=True).stdout
            arrays = {f[:-4]: np.load(os.path.join(tmp, f)) for f in os.listdir(tmp) if f.endswith(".npy")}
        config = np.array([k, m, seed], dtype=np.int64)
    keep: dict[str, np.ndarray] = {"config": config}
    if kind == "full":
        keep.update(arrays)
    else:
        for key in ("meta", "pcg_report", "pcg_history", "plain_report", "plain_history", "Ac_vals",
                    "Ac_cols", "Ac_rowptr", "Ac_shape", "aci", "aci_off", "interior_counts"):
            if key in arrays:
                keep[key] = arrays[key]
        if kind == "solve":
            for key in ("pcg_x", "rhs", "apply_rhs"):
                if key in arrays:
                    keep[key] = arrays[key]
        else:
            stride = 97
            keep["pcg_x_sample_stride"] = np.array([stride])
            keep["pcg_x_sample"] = arrays["pcg_x"][::stride].copy()
            keep["pcg_x_norm2"] = np.array([np.linalg.norm(arrays["pcg_x"])])
            keep["rhs_sample"] = arrays["rhs"][::stride].copy()
        for key in MAP_ARRAYS:
            keep["digest_" + key] = np.array(digest(arrays[key]))
    os.makedirs(GOLDEN, exist_ok=True)
    path = os.path.join(GOLDEN, name + ".npz")
    np.savez_compressed(path, **keep)
    print(f"{name}: {os.path.getsize(path)/1024:.1f} KiB  {out.strip()}")


def main(argv: list[str]) -> None:
    if not os.path.exists(DRIVER):
        subprocess.run(["make", "-C", HERE, "-j8"], check=True)
    names = argv or (list(CONFIGS) + list(BUNDLES))
    for n in names:
        run(n)


if __name__ == "__main__":
    main(sys.argv[1:])
