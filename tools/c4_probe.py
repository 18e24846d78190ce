import sys, time; sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2410_14786_b200 import Problem, Preconditioner, SolverOptions
p = Problem.poisson(800, 8)
o = SolverOptions(1e-8, 0.0, 10000, True)
for setup in ("device", "host"):
    pre = Preconditioner(p, setup=setup)
    b = torch.tensor(p.rhs(), device="cuda"); x = torch.empty_like(b); s = torch.cuda.Stream()
    for _ in range(2): pre.pcg_device(b.data_ptr(), x.data_ptr(), o, precondition=False, stream=s.cuda_stream)
    torch.cuda.synchronize(); g0 = pre.stats()["graph_captures"]
    t = time.time()
    for _ in range(5): r = pre.pcg_device(b.data_ptr(), x.data_ptr(), o, precondition=False, stream=s.cuda_stream)
    torch.cuda.synchronize(); dt = (time.time() - t) / 5
    print(setup, "plain ms", dt * 1e3, "its", r.iterations, "captures", g0, pre.stats()["graph_captures"], flush=True)
    t = time.time()
    for _ in range(5): r = pre.pcg_device(b.data_ptr(), x.data_ptr(), o, stream=s.cuda_stream)
    torch.cuda.synchronize(); print(setup, "bddc ms", (time.time() - t) / 5 * 1e3, r.iterations, flush=True)
    del pre
