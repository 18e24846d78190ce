"""Dev probe: C2 apply only (no PCG), mean interior-solve launch and apply time (profiled)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_14786_b200 import Preconditioner, Problem  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
p = Problem.poisson(800, 8) if cfg == "c2" else Problem.poisson(2520, 24)
pre = Preconditioner(p)
s = torch.cuda.Stream()
r = torch.tensor(p.rhs(), device="cuda")
z = torch.empty_like(r)
for _ in range(5):
    pre.apply_device(r.data_ptr(), z.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
pre.kernel_times(reset=True)
pre.set_profile(True)
for _ in range(50):
    pre.apply_device(r.data_ptr(), z.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
kt = pre.kernel_times(reset=True)
print(os.environ.get("TAG", ""), cfg, "interior launch us %.1f" % (1e3 * kt["interior_ms"] / max(1, kt["interior_launches"])),
      "apply us %.1f" % (1e3 * kt["apply_ms"] / max(1, kt["applies"])), {k: v for k, v in kt.items()}, flush=True)
