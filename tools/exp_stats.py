"""Per-warp cycle accounting of the interior solve (dev tool; run with BDDC_SOLVE_STATS=1).
Prints mean/max of {total, mbarrier wait, CTA-barrier wait} over all warps and the phase
timeline of CTA 0 (cycles per phase) of the last launch (the second interior solve)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_14786_b200 import Preconditioner, Problem  # noqa: E402
import torch  # noqa: E402

k, m = int(os.environ.get("K", 8)), int(os.environ.get("M", 100))
p = Problem.poisson(k * m, k)
pre = Preconditioner(p, leaf_size=int(os.environ.get("LEAF", 24)), solve_parts=int(os.environ.get("PARTS", 0)))
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
r = torch.tensor(p.rhs(), device="cuda")
z = torch.empty_like(r)
for _ in range(3):
    pre.apply_device(r.data_ptr(), z.data_ptr(), st.cuda_stream)
torch.cuda.synchronize()
raw = pre.solve_profile()
n_parts = 2 * k * k if int(os.environ.get("PARTS", 0)) != 1 else k * k
W = int(os.environ.get("WARPS", 16))
w = raw.reshape(-1)[:n_parts * W * 8].reshape(-1, 8)
tl = raw.reshape(-1)[n_parts * W * 8:]
tot, wait, bar = w[:, 0].astype(float), w[:, 1].astype(float), w[:, 2].astype(float)
print(f"warps {len(w)}: total mean {tot.mean():.0f} max {tot.max():.0f} cycles")
print(f"  mbarrier wait {wait.mean():.0f} ({100 * wait.mean() / tot.mean():.0f}%), CTA barrier {bar.mean():.0f} "
      f"({100 * bar.mean() / tot.mean():.0f}%), work {np.mean(tot - wait - bar):.0f} "
      f"({100 * np.mean(tot - wait - bar) / tot.mean():.0f}%)")
refill, tiles, ntiles = w[:, 4].astype(float), w[:, 5].astype(float), w[:, 6].astype(float)
print(f"  refill (fence + TMA issue) {refill.mean():.0f} ({100 * refill.mean() / tot.mean():.0f}%), tile processing "
      f"{tiles.mean():.0f} ({100 * tiles.mean() / tot.mean():.0f}%), tiles per warp {ntiles.mean():.0f} -> "
      f"{tiles.sum() / max(1, ntiles.sum()):.0f} cycles per tile")
tl = tl[tl > 0]
d = np.diff(np.concatenate([[0], tl]))
print("CTA 0 phase durations (cycles):", " ".join(str(int(x)) for x in d))
