"""Gather time vs row width (d) on random data: A/B helper for the wide-row
kernel.  Not part of the product.

    SNGB_LIBRARY=... python tools/dsweep.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2006_06743_b200 as sng  # noqa: E402

n, draws = int(os.environ.get("DSWEEP_N", 70000)), 700
for d in (100, 200, 380, 500, 620, 740, 784, 900, 1000, 1024):
    rng = np.random.default_rng(d)
    x = torch.from_numpy(rng.random((n, d), dtype=np.float32)).cuda()
    eps = float(np.sqrt(d / 6.0) * 0.9)  # ~ a few percent accepted
    best = None
    for _ in range(4):
        keys, gi = sng.sampled_edges_device(x, eps, draws / n, 7, 0, n, timing=True)
        best = gi.ms_gather if best is None else min(best, gi.ms_gather)
    print(f"d={d} edges={keys.numel()} gather_ms={best:.3f} "
          f"TB/s={n * draws * 4 * d / best / 1e9:.2f}", flush=True)
