"""Per-stage device times of one sng_dbscan_device call (timing flag):
python tools/stage_times.py CONFIG.  Not part of the product."""
import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2006_06743_b200 as sng
from paper_2006_06743_b200 import synthetic
cfg = int(sys.argv[1])
w = synthetic.CONFIGS[cfg]
pts = torch.from_numpy(synthetic.generate(cfg)).cuda()
for rep in range(4):
    lab, rol, info = sng.sng_dbscan_device(pts, w.eps, w.min_pts, w.rate, w.seed, timing=True)
g = info.as_dict()
print(os.environ.get("SNGB_SORTED_DEDUP", "0"), {k: round(v, 3) for k, v in g.items() if k.startswith("ms_")}, g.get("edges"), g.get("directed_accepts"))
