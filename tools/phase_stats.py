"""Per-phase accounting of the interior solve (dev tool; BDDC_SOLVE_STATS=1): for CTA 0 of the
apply's last interior-solve launch (the harmonic program), each phase's duration, the busiest and
mean warp busy cycles and tiles, so the barrier waits split into imbalance vs critical path."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_14786_b200 import Preconditioner, Problem  # noqa: E402

W = int(os.environ.get("WARPS", 16))
p = Problem.poisson(800, 8)
pre = Preconditioner(p)
s = torch.cuda.Stream()
r = torch.tensor(p.rhs(), device="cuda")
z = torch.empty_like(r)
for _ in range(3):
    pre.apply_device(r.data_ptr(), z.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
raw = pre.solve_profile()
nparts = 128
tl = raw[nparts * W * 8: nparts * W * 8 + 256]
pw = raw[nparts * W * 8 + 256: nparts * W * 8 + 256 + 256 * W].reshape(256, W)
nt = raw[nparts * W * 8 + 256 + 256 * W: nparts * W * 8 + 256 + 2 * 256 * W].reshape(256, W)
wt = raw[nparts * W * 8 + 256 + 2 * 256 * W + 8: nparts * W * 8 + 256 + 3 * 256 * W + 8].reshape(256, W)
tt = raw[nparts * W * 8 + 256 + 3 * 256 * W + 8: nparts * W * 8 + 256 + 4 * 256 * W + 8].reshape(256, W)
rf = raw[nparts * W * 8 + 256 + 4 * 256 * W + 8: nparts * W * 8 + 256 + 5 * 256 * W + 8].reshape(256, W)
nph = int((tl > 0).sum())
prev = 0
tot_dur = tot_max = tot_mean = 0
print(" ph   dur   busy_max  busy_mean  tiles_max tiles_mean  wait_max wait_mean  tile@max refill@max")
for ph in range(nph):
    dur = int(tl[ph] - prev) if tl[ph] > prev else 0
    prev = max(prev, int(tl[ph]))
    bm, bmean = int(pw[ph].max()), float(pw[ph].mean())
    tot_dur += dur
    tot_max += bm
    tot_mean += bmean
    print(f"{ph:3d} {dur:6d} {bm:9d} {bmean:10.0f} {int(nt[ph].max()):9d} {nt[ph].mean():10.1f} "
          f"{int(wt[ph].max()):9d} {wt[ph].mean():9.0f} {int(tt[ph][pw[ph].argmax()]):9d} {int(rf[ph][pw[ph].argmax()]):9d}")
mk = raw[nparts * W * 8 + 256 + 2 * 256 * W: nparts * W * 8 + 256 + 2 * 256 * W + 8]
print("CTA 0 since kernel entry: predecessor done", mk[4], "prologue done", mk[5], "phase loop done", mk[6],
      "epilogue done", mk[7])
print("markers (cycles since start): before cluster sync", mk[0], "after", mk[1], "after combine", mk[2],
      "after split switch", mk[3], "| timeline at the combine phase end", [int(t) for t in tl[:nph] if 0 < t <= mk[0]][-1:])
print(f"sum: duration {tot_dur}, sum of busiest warps {tot_max}, sum of mean busy {tot_mean:.0f}")
# per-CTA totals (cycles from start to the end of the phase loop, busiest warp), slowest first
w = raw[:nparts * W * 8].reshape(nparts, W, 8)
tot = w[:, :, 0].max(axis=1)
order = np.argsort(-tot)
print("slowest CTAs (subdomain, rank, cycles):", [(int(c) // 2, int(c) % 2, int(tot[c])) for c in order[:8]])
print("fastest CTAs:", [(int(c) // 2, int(c) % 2, int(tot[c])) for c in order[-4:]], "median", int(np.median(tot)))
tp = raw[nparts * W * 8 + 256 + 5 * 256 * W + 8: nparts * W * 8 + 256 + 5 * 256 * W + 8 + 4 * W].reshape(W, 4)
print("CTA 0 tile sub-phase cycles per warp (decode, loop, reduction, flush):")
for w_ in range(W):
    print("  warp", w_, [int(v) for v in tp[w_]])
so = raw[nparts * W * 8 + 256 + 5 * 256 * W + 8 + 4 * W: nparts * W * 8 + 256 + 5 * 256 * W + 8 + 4 * W + 512 * 6].reshape(512, 6)
print("CTA 0 warp 0 steps: phase k lg iters | decode loop reduction flush cycles")
for st in so:
    if st[1] == 0 and st[0] == 0 and st[2] == 0:
        continue
    z = int(st[1]) & 0xffffffff
    print(f"  ph {int(st[0]):3d} k {z & 63:2d} lg {(z >> 6) & 7} it {(z >> 17) & 511:3d} flags {(z >> 9) & 255:3d} | "
          f"{int(st[2]):5d} {int(st[3]):5d} {int(st[4]):5d} {int(st[5]):5d}")
