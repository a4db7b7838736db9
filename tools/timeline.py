"""Kernel timeline of one sng_dbscan_device call (torch.profiler / CUPTI sees the
kernels libsngb.so launches): per-kernel start, duration and the idle gap
before it.  Not part of the product.

    python tools/timeline.py --config 2 [--reps 3] > gpurun_out/timeline_cfg2.txt
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2006_06743_b200 as sng  # noqa: E402
from paper_2006_06743_b200 import synthetic  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=2)
p.add_argument("--reps", type=int, default=3)
a = p.parse_args()
w = synthetic.CONFIGS[a.config]
x = torch.from_numpy(synthetic.generate(a.config)).cuda()
for _ in range(3):
    sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(a.reps):
        sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev_end = t0
busy = 0.0
tot_gap = 0.0
for e in evs:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    gap = max(0.0, s - prev_end)
    tot_gap += gap
    busy += d
    print(f"{(s - t0):10.1f} us  {d:9.1f} us  gap {gap:7.1f}  {e.name[:90]}")
    prev_end = max(prev_end, e.time_range.end)
span = prev_end - t0
print(f"# {a.reps} calls: span {span:.1f} us, kernel busy {busy:.1f} us, idle gaps {tot_gap:.1f} us "
      f"({tot_gap / span * 100:.1f} %), per call span {span / a.reps:.1f} us")
