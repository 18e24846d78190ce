"""Dev probe: C2 BDDC-PCG device time vs the nested-dissection leaf size (and solve parts)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_14786_b200 import Preconditioner, Problem, SolverOptions  # noqa: E402

p = Problem.poisson(800, 8, rhs_seed=1)
opts = SolverOptions(1e-8, 0.0, 10000, True)
for leaf in [int(v) for v in os.environ.get("LEAVES", "16 24 32 40 48").split()]:
    pre = Preconditioner(p, leaf_size=leaf)
    s = torch.cuda.Stream()
    b = torch.tensor(p.rhs(), device="cuda")
    x = torch.empty_like(b)
    for _ in range(3):
        pre.pcg_device(b.data_ptr(), x.data_ptr(), opts, stream=s.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(20):
        rep = pre.pcg_device(b.data_ptr(), x.data_ptr(), opts, stream=s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    st = pre.stats()
    print(f"leaf {leaf}: {e0.elapsed_time(e1) / 20:.4f} ms/solve, iterations {rep.iterations}, "
          f"factor values {st.get('factor_values', '?')}", flush=True)
    del pre
