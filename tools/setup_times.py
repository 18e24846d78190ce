"""Dev probe: wall time of Preconditioner construction (device vs host setup) at C2 / C5 / C3,
best of three constructions per configuration (BDDC_SETUP_TIMES=1 adds the phase breakdown)."""
import sys
import time

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2410_14786_b200 import Preconditioner, Problem  # noqa: E402

for name, args, kw in [("c2", (800, 8), {}), ("c5", (352, 8), dict(kappa_decades=2.0, kappa_seed=0x5EED)),
                       ("c3", (2520, 24), {})]:
    p = Problem.poisson(*args, **kw)
    for setup in ("device", "host"):
        best = None
        for _ in range(3 if setup == "device" else 1):
            t = time.time()
            pre = Preconditioner(p, setup=setup)
            dt = time.time() - t
            st = pre.stats()
            print("  ", name, setup, "ctor %.3f s" % dt, flush=True)
            if best is None or st["setup_seconds"] < best[1]["setup_seconds"]:
                best = (dt, st)
            del pre
        print(name, setup, "ctor %.3f s" % best[0], "setup_seconds %.3f" % best[1]["setup_seconds"],
              "device %.3f" % best[1]["setup_device_seconds"], "classes", best[1]["unique_subdomains"], flush=True)
