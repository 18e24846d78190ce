"""Multi-GPU parity driver, run under torchrun (one rank per GPU) by tests/test_gpu_distributed.py.

Every rank builds the same global problem, a distributed preconditioner (its block of
subdomains) and, as the parity reference, a single-GPU preconditioner of the whole problem on
its own device. Checks (BASELINE.json parity bar):
  * the distributed apply equals the single-GPU apply BIT FOR BIT on the rank's dofs (same
    factors, same owner-ordered interface sums, r_c summed over all subdomains in ascending order);
  * distributed PCG: identical iteration count, residual history within 1e-10 and solution
    within 1e-10 of the single-GPU solve and of the reference's golden fixtures (bundle route,
    tests/golden/r4x2m8, r16x8m8);
  * the C-ABI host entry points fill exactly the rank's rows.
Prints one JSON line per config on rank 0 and exits non-zero on any failure.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch
    import torch.distributed as dist

    from conftest import golden, history_err
    from paper_2410_14786_b200 import Preconditioner, Problem, SolverOptions
    from paper_2410_14786_b200.distributed import fresh_nccl_id, init

    rank, world, local_rank, nid = init()
    opts = SolverOptions(1e-8, 0.0, 10000, True)
    # (golden fixture, (cells_x, cells_y, kx, ky[, kappa_decades, kappa_seed]))
    cfgs = [("r4x2m8", (32, 16, 4, 2)), ("k4m8", (32, 32, 4, 4)), ("r16x8m8", (128, 64, 16, 8)),
            ("h4m8", (32, 32, 4, 4, 2.0, 0x5EED)), ("c5", (352, 352, 8, 8, 2.0, 0x5EED)),
            ("c2g2", (1600, 800, 16, 8))]
    if world >= 4:
        cfgs.append(("c2g4", (1600, 1600, 16, 16)))
        # the N=8 weak-scaling layout (32x16 subdomains, n_c = 1,441: the cooperative coarse grid)
        # at 128 subdomains per GPU on the 4 GPUs reachable here
        cfgs.append(("c2g8", (3200, 1600, 32, 16)))
    # C3 strong scaling (6.35M dofs, 24x24 subdomains) split over the ranks (DIST_CHECK_C3=0 skips)
    if os.environ.get("DIST_CHECK_C3", "1") != "0":
        cfgs.append(("c3", (2520, 2520, 24, 24)))
    failures = []
    for name, cfg in cfgs:
        cx, cy, kx, ky = cfg[:4]
        kappa = cfg[4:] if len(cfg) > 4 else (0.0, 0x5EED)
        if kx * ky < world:
            continue
        prob = Problem.poisson(cx, kx, cy, ky, kappa_decades=kappa[0], kappa_seed=kappa[1], rhs_seed=1)
        b = prob.rhs()
        single = Preconditioner(prob, device=local_rank, solve_parts=2)  # same program split as the ranks
        pre = Preconditioner(prob, device=local_rank, dist=(rank, world, nid), solve_parts=2)
        nid = fresh_nccl_id()  # the next communicator needs its own id
        n_local, n_rows, n_owned, l2g = pre.layout()
        rows = l2g[:n_rows]
        res = {"config": name, "rank": rank, "world": world, "n_rows": n_rows, "n_owned": n_owned}
        z1 = single.apply(b)
        zd = np.full(prob.global_dofs, np.nan)
        zd = _apply(pre, b, zd)
        res["apply_bitwise"] = bool(np.array_equal(zd[rows], z1[rows]))
        res["apply_untouched_elsewhere"] = bool(np.isnan(np.delete(zd, rows)).all())
        x1, r1 = single.pcg(b, opts)
        xd, rd = pre.pcg(b, opts)
        res["iterations"] = [rd.iterations, r1.iterations]
        res["history_err_vs_single"] = history_err(rd.residual_history, r1.residual_history)
        res["x_err_vs_single"] = float(np.abs(xd[rows] - x1[rows]).max() / np.abs(x1).max())
        try:
            g = golden(name)
            res["history_err_vs_reference"] = history_err(rd.residual_history, g["pcg_history"])
            res["iterations_reference"] = int(g["pcg_report"][0])
            if "pcg_x" in g:
                res["x_err_vs_reference"] = float(np.abs(xd[rows] - g["pcg_x"][rows]).max() / np.abs(g["pcg_x"]).max())
            elif "pcg_x_sample" in g:  # large problems: every stride-th entry of the reference solution
                stride = int(g["pcg_x_sample_stride"][0])
                idx = np.intersect1d(rows, np.arange(0, prob.global_dofs, stride))
                xs = g["pcg_x_sample"]
                res["x_err_vs_reference"] = float(np.abs(xd[idx] - xs[idx // stride]).max() / np.abs(xs).max())
        except FileNotFoundError:
            pass
        # device entry point on the rank-local layout
        dev = f"cuda:{local_rank}"
        bl = torch.from_numpy(np.ascontiguousarray(b[l2g])).to(dev)
        xl = torch.empty_like(bl)
        rep = pre.pcg_device(bl.data_ptr(), xl.data_ptr(), opts)
        res["device_matches_host"] = bool(np.array_equal(xl.cpu().numpy()[:n_rows], xd[rows])) and \
            rep.iterations == rd.iterations
        # pinned (device-mapped) host buffers: zero-copy gather / scatter, same rows, same bits
        b_pin = torch.from_numpy(b).pin_memory().numpy()
        x_pin = torch.full((prob.global_dofs,), float("nan"), dtype=torch.float64).pin_memory().numpy()
        xp, rp = pre.pcg(b_pin, opts, out=x_pin)
        z_pin = _apply(pre, b_pin, torch.full((prob.global_dofs,), float("nan"),
                                              dtype=torch.float64).pin_memory().numpy())
        res["pinned_matches_pageable"] = bool(np.array_equal(xp[rows], xd[rows])) and \
            bool(np.isnan(np.delete(xp, rows)).all()) and rp.iterations == rd.iterations and \
            bool(np.array_equal(z_pin[rows], zd[rows])) and bool(np.isnan(np.delete(z_pin, rows)).all())
        if name == "k4m8":  # a non-finite rhs: every rank rejects it with the smallest global index
            from paper_2410_14786_b200 import InvalidArgument
            bad = b.copy()
            j = prob.global_dofs // 2 + 3
            bad[j], bad[prob.global_dofs - 1] = np.nan, np.inf
            try:
                pre.pcg(bad, opts)
                res["nonfinite_rejected"] = False
            except InvalidArgument as e:
                res["nonfinite_rejected"] = f"non-finite entry at index {j}" in str(e)
            res["usable_after_error"] = pre.pcg(b, opts)[1].iterations == rd.iterations
        # h4m8 alone is summation-order sensitive beyond 1e-10 (the CPU oracle moves by more than
        # 1e-9 when only its dot-product order changes: test_oracle_golden.py::
        # test_h4m8_history_sensitivity_is_intrinsic); C5 and the rest are held to 1e-10
        htol = 1e-7 if name == "h4m8" else 1e-10
        ok = (res["apply_bitwise"] and res["apply_untouched_elsewhere"] and rd.iterations == r1.iterations
              and res["history_err_vs_single"] <= htol and res["x_err_vs_single"] <= 1e-10
              and res["device_matches_host"] and res["pinned_matches_pageable"] and rd.converged and res.get("nonfinite_rejected", True)
              and res.get("usable_after_error", True))
        if "history_err_vs_reference" in res:
            ok = ok and res["history_err_vs_reference"] <= htol and abs(rd.iterations - res["iterations_reference"]) <= (
                1 if name == "h4m8" else 0)
        if "x_err_vs_reference" in res:
            ok = ok and res["x_err_vs_reference"] <= 1e-10
        res["ok"] = bool(ok)
        allres = [None] * world
        dist.all_gather_object(allres, res)
        if rank == 0:
            for rr in allres:
                print(json.dumps(rr), flush=True)
        failures += [rr for rr in allres if not rr["ok"]]
        del pre, single
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(1 if failures else 0)


def _apply(pre, b, out):
    import ctypes as C

    from paper_2410_14786_b200 import _lib as L

    bb = np.ascontiguousarray(b, dtype=np.float64)
    L.check(L.lib().bddc_gpu_apply(pre._h, bb.ctypes.data_as(C.POINTER(C.c_double)),
                                   out.ctypes.data_as(C.POINTER(C.c_double))), pre._h)
    return out


if __name__ == "__main__":
    main()
