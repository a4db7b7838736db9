import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2006_06743_b200 as sng
from paper_2006_06743_b200 import synthetic
w = synthetic.CONFIGS[2]
pts = synthetic.generate(2)
import torch
host = torch.from_numpy(pts).pin_memory().numpy()
ds = sng.Dataset(host)
for rep in range(4):
    info = sng.ClusterRunInfo()
    t0 = time.perf_counter()
    c = sng.sng_dbscan(ds, sng.SngParams(eps=w.eps, min_pts=w.min_pts, rate=w.rate, seed=w.seed), info, timing=True)
    t1 = time.perf_counter()
g = info.gpu
print(os.environ.get("SNGB_GATHER_PHASES", "-"), "wall %.2f ms" % ((t1 - t0) * 1e3), {k: round(v, 3) for k, v in g.items() if k.startswith("ms_")}, "filter", g["filter_bits"], "edges", g["edges"])
