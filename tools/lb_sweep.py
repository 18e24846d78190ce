"""Apply time vs CTAs per subdomain of the K_i GEMV (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_14786_b200 import Preconditioner, Problem  # noqa: E402

p = Problem.poisson(800, 8)
for lb in (4, 6, 8, 12, 16):
    pre = Preconditioner(p, local_blocks=lb)
    st = torch.cuda.Stream()
    r = torch.tensor(p.rhs(), device="cuda")
    z = torch.empty_like(r)
    for _ in range(3):
        pre.apply_device(r.data_ptr(), z.data_ptr(), st.cuda_stream)
    torch.cuda.synchronize()
    pre.set_profile(True)
    for _ in range(50):
        pre.apply_device(r.data_ptr(), z.data_ptr(), st.cuda_stream)
    kt = pre.kernel_times(reset=True)
    pre.set_profile(False)
    print("local_blocks", lb, "iface_ms", round(kt["iface_ms"] / kt["applies"], 4), "apply_ms",
          round(kt["apply_ms"] / kt["applies"], 4), flush=True)
    del pre
