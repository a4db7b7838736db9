"""Time one config under several scheduling settings (env knobs read per call
by the library).  A/B helper, not part of the product.

    python tools/sched_sweep.py --config 5 [--reps 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2006_06743_b200 as sng  # noqa: E402
from paper_2006_06743_b200 import synthetic  # noqa: E402

SETTINGS = {
    "default": {},
    "sequential": {"SNGB_OVERLAP": "0"},
    "static_persistent": {"SNGB_GATHER_DYN": "0"},
    "nonpersistent_rpb128": {"SNGB_GATHER_RPB": "128"},
    "overlap_rpb128": {"SNGB_OVERLAP": "1"},
}
KNOBS = ("SNGB_OVERLAP", "SNGB_GATHER_RPB", "SNGB_SAMPLER_RPB", "SNGB_PRIO", "SNGB_GATHER_DYN")

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=5)
p.add_argument("--reps", type=int, default=2)
p.add_argument("--only", default="")
a = p.parse_args()
w = synthetic.CONFIGS[a.config]
x = torch.from_numpy(synthetic.generate(a.config)).cuda()
ref_edges = None
for name, env in SETTINGS.items():
    if a.only and name not in a.only.split(","):
        continue
    for k in KNOBS:
        os.environ.pop(k, None)
    os.environ.update(env)
    best = None
    for _ in range(1 + a.reps):
        _, _, gi = sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True)
        torch.cuda.synchronize()
        if best is None or gi.ms_total < best.ms_total:
            best = gi
    ref_edges = ref_edges or best.edges
    assert best.edges == ref_edges, (name, best.edges, ref_edges)
    print(f"cfg{a.config} {name:28s} total={best.ms_total:9.2f} gather={best.ms_gather:9.2f} "
          f"sample={best.ms_sample:9.2f} extras={best.ms_extras:8.2f}", flush=True)
