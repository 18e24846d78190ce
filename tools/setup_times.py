import sys, time; sys.path.insert(0, '/root/repo')
from paper_2410_14786_b200 import Problem, Preconditioner
for name, args, kw in [("c2", (800, 8), {}), ("c5", (352, 8), dict(kappa_decades=2.0, kappa_seed=0x5EED)), ("c3", (2520, 24), {})]:
    p = Problem.poisson(*args, **kw)
    for setup in ("device", "host"):
        t = time.time(); pre = Preconditioner(p, setup=setup); dt = time.time() - t
        print(name, setup, "ctor", round(dt, 3), "stats", {k: pre.stats()[k] for k in ("setup_seconds", "setup_device_seconds", "unique_subdomains")}, flush=True)
        del pre
