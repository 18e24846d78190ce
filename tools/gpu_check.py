"""Quick GPU sanity/perf probe (development tool, not a test): parity vs golden fixtures
and timings of apply / PCG at C1 and C2."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_14786_b200 import Preconditioner, Problem, SolverOptions  # noqa: E402


def run(name, k, m, reps=20, leaf=16):
    g = np.load(os.path.join(ROOT, "tests", "golden", name + ".npz"))
    t = time.time()
    p = Problem.poisson(k * m, k, rhs_seed=1)
    t_prob = time.time() - t
    t = time.time()
    pre = Preconditioner(p, leaf_size=leaf)
    t_setup = time.time() - t
    st = pre.stats()
    b = p.rhs()
    out = {"name": name, "problem_s": round(t_prob, 3), "setup_s": round(t_setup, 3), "stats": st}
    if "apply_rhs" in g:
        z = pre.apply(b)
        out["apply_rel_err"] = float(np.abs(z - g["apply_rhs"]).max() / np.abs(g["apply_rhs"]).max())
    import torch

    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    rd = torch.tensor(b, device="cuda")
    zd = torch.empty_like(rd)
    s = stream.cuda_stream
    for _ in range(3):
        pre.apply_device(rd.data_ptr(), zd.data_ptr(), s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        pre.apply_device(rd.data_ptr(), zd.data_ptr(), s)
    e1.record()
    torch.cuda.synchronize()
    out["apply_ms"] = e0.elapsed_time(e1) / reps
    out["apply_GBps"] = st["apply_bytes"] / (out["apply_ms"] * 1e-3) / 1e9
    za = zd.cpu().numpy()
    if "apply_rhs" in g:
        out["apply_dev_rel_err"] = float(np.abs(za - g["apply_rhs"]).max() / np.abs(g["apply_rhs"]).max())
    pre.set_profile(True)
    for _ in range(reps):
        pre.apply_device(rd.data_ptr(), zd.data_ptr(), s)
    out["kernel_times"] = pre.kernel_times(reset=True)
    pre.set_profile(False)
    x, rep = pre.pcg(b, SolverOptions(1e-8, 0.0, 10000, True))
    t = time.time()
    x, rep = pre.pcg(b, SolverOptions(1e-8, 0.0, 10000, True))
    out["pcg_s"] = time.time() - t
    out["iterations"] = rep.iterations
    out["golden_iterations"] = int(g["pcg_report"][0])
    gh = g["pcg_history"]
    n = min(len(gh), len(rep.residual_history))
    out["hist_rel_err"] = float(np.max(np.abs(np.array(rep.residual_history[:n]) - gh[:n]) / gh[:n]))
    if "pcg_x" in g:
        out["x_rel_err"] = float(np.abs(x - g["pcg_x"]).max() / np.abs(g["pcg_x"]).max())
    else:
        stride = int(g["pcg_x_sample_stride"][0])
        xs = g["pcg_x_sample"]
        out["x_rel_err"] = float(np.abs(x[::stride] - xs).max() / np.abs(xs).max())
    print(out, flush=True)


if __name__ == "__main__":
    leaf = int(os.environ.get("LEAF", "24"))
    cfgs = {"k4m8": (4, 8), "c1": (4, 64), "c2": (8, 100)}
    names = sys.argv[1:] or list(cfgs)
    for nm in names:
        run(nm, *cfgs[nm], leaf=leaf)
