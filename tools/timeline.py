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
p.add_argument("--host", action="store_true", help="the host C-ABI call from pinned memory (bench e2e)")
a = p.parse_args()
w = synthetic.CONFIGS[a.config]
pts = synthetic.generate(a.config)
if a.host:
    import ctypes as C
    from paper_2006_06743_b200 import _lib
    host = torch.from_numpy(pts).pin_memory()
    n, d = pts.shape
    labels_h = torch.empty(n, dtype=torch.int32).pin_memory()
    roles_h = torch.empty(n, dtype=torch.uint8).pin_memory()
    L = _lib.lib()
    o = _lib.SngbOpts(0, 0, None, 0, 0)

    def call():
        sng._check(L.sngb_dbscan_f32(C.cast(host.data_ptr(), C.POINTER(C.c_float)), n, d, w.eps,
                                     w.min_pts, w.rate, w.seed, C.byref(o),
                                     C.cast(labels_h.data_ptr(), C.POINTER(C.c_int32)),
                                     C.cast(roles_h.data_ptr(), C.POINTER(C.c_uint8)), None))
else:
    x = torch.from_numpy(pts).cuda()

    def call():
        sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed)
for _ in range(3):
    call()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(a.reps):
        call()
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
