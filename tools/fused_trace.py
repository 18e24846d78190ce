"""Timeline of the fused peer-memory exchanges at N > 1 (dev tool; BDDC_FUSED_TRACE=1, torchrun).

Events per kernel id (0 solve0, 1 restrict, 2 K_i, 3 harmonic solve, 4 xpay/init_rho, 5 spmv_dot,
6 update, 7 check): 0 = CTA 0 enters its wait, 1 = CTA 0 done waiting, 2 = the last CTA finished
its outputs, 3 = the last CTA released the flags. Prints the mean gap between consecutive events
(in time order) over the steady-state iterations of the last solve."""
import collections
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_14786_b200 import Problem, Preconditioner, SolverOptions  # noqa: E402
from paper_2410_14786_b200.distributed import init  # noqa: E402

rank, world, lr, nid = init()
lay = tuple(int(v) for v in os.environ["LAYOUT"].split("x")) if os.environ.get("LAYOUT") else {2: (16, 8), 4: (16, 16)}[world]
p = Problem.poisson(lay[0] * 100, lay[0], lay[1] * 100, lay[1])
pre = Preconditioner(p, device=lr, dist=(rank, world, nid))
nl, nr, no, l2g = pre.layout()
b = torch.tensor(p.rhs()[l2g], device=f"cuda:{lr}")
x = torch.empty_like(b)
opts = SolverOptions(1e-8, 0.0, 10000, True)
for _ in range(3):
    pre.pcg_device(b.data_ptr(), x.data_ptr(), opts)
torch.cuda.synchronize()
n0 = int(pre.solve_profile()[0])
pre.pcg_device(b.data_ptr(), x.data_ptr(), opts)
torch.cuda.synchronize()
tr = pre.solve_profile()
n1 = int(tr[0])
ev = tr[1:1 + 2 * n1].reshape(-1, 2)[n0:]
ev = ev[np.argsort(ev[:, 1], kind="stable")]
names = ["solve0", "restrict", "K_i", "harm", "xpay", "spmv", "update", "check"]
what = ["wait>", "wait<", "done", "rel"]
lab = [f"{names[i // 4]}.{what[i % 4]}" for i in ev[:, 0]]
t = ev[:, 1].astype(np.int64)
gaps = collections.defaultdict(list)
for i in range(1, len(lab)):
    gaps[(lab[i - 1], lab[i])].append(t[i] - t[i - 1])
order = []
for i in range(1, len(lab)):
    k = (lab[i - 1], lab[i])
    if k not in order:
        order.append(k)
lines = [f"rank {rank}: {len(lab)} events, span {(t[-1] - t[0]) / 1e3:.1f} us"]
for k in order:
    g = np.array(gaps[k])
    lines.append(f"rank {rank} {k[0]:>15s} -> {k[1]:<15s} n {len(g):4d} mean {g.mean() / 1e3:7.2f} us  median {np.median(g) / 1e3:7.2f}")
print("\n".join(lines), flush=True)
torch.distributed.barrier()
