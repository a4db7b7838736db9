"""Default stream scheduling vs SNGB_OVERLAP=0 on the small shapes (not part of the product)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_06743_b200 as sng
from paper_2006_06743_b200 import synthetic
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for cfg in (1, 2, 3):
    w = synthetic.CONFIGS[cfg]
    x = torch.from_numpy(synthetic.generate(cfg)).cuda()
    for name, env in (("default", {}), ("overlap0", {"SNGB_OVERLAP": "0"}), ("overlap1", {"SNGB_OVERLAP": "1"}),
                      ("overlap0_rpb0", {"SNGB_OVERLAP": "0", "SNGB_SAMPLER_RPB": "0"}),
                      ("default_rpb64", {"SNGB_SAMPLER_RPB": "64"}), ("default_rpb8", {"SNGB_SAMPLER_RPB": "8"})):
        for k in ("SNGB_OVERLAP", "SNGB_SAMPLER_RPB"):
            os.environ.pop(k, None)
        os.environ.update(env)
        for _ in range(3):
            sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True)
        ts = []
        for _ in range(15):
            flush.zero_()
            _, _, gi = sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True)
            ts.append((gi.ms_total, gi.ms_sample, gi.ms_gather))
        print(json.dumps({"cfg": cfg, "variant": name, "ms_total": round(statistics.median(t[0] for t in ts), 4),
                          "ms_sample": round(statistics.median(t[1] for t in ts), 4),
                          "ms_gather": round(statistics.median(t[2] for t in ts), 4)}), flush=True)
    del x
