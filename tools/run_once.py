"""Run sng_dbscan_device once (after one warm-up) on a BASELINE config -- the
command profiled by ncu (profiles/).  Not part of the product.

    python tools/run_once.py --config 2 [--n N] [--reps R]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2006_06743_b200 as sng  # noqa: E402
from paper_2006_06743_b200 import synthetic  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=2)
p.add_argument("--n", type=int, default=None)
p.add_argument("--reps", type=int, default=1)
a = p.parse_args()
w = synthetic.CONFIGS[a.config]
pts = synthetic.generate(a.config, n=a.n)
rate = w.rate if a.n is None else min(1.0, w.draws / a.n)
x = torch.from_numpy(pts).cuda()
for _ in range(1 + a.reps):
    labels, roles, gi = sng.sng_dbscan_device(x, w.eps, w.min_pts, rate, w.seed, timing=True)
torch.cuda.synchronize()
print({k: v for k, v in gi.as_dict().items() if k.startswith("ms_") or k in
       ("edges", "cluster_count", "collisions", "kernel_launches", "gather_bytes",
                                                    "gather_pairs", "filter_bits", "band_rechecks")})
