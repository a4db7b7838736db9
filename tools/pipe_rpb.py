"""k_floyd_pipe: rows per sampler block sweep on cfg5 (not part of the product)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_06743_b200 as sng
from paper_2006_06743_b200 import synthetic
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
w = synthetic.CONFIGS[cfg]
x = torch.from_numpy(synthetic.generate(cfg)).cuda()
os.environ["SNGB_FLOYD_PIPE"] = "1"
for ov in (None, "0"):
    for rpb in ("8", "16", "32", "64", "128", "0"):
        os.environ["SNGB_SAMPLER_RPB"] = rpb
        if ov is None: os.environ.pop("SNGB_OVERLAP", None)
        else: os.environ["SNGB_OVERLAP"] = ov
        sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True)
        runs = [sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True) for _ in range(3)]
        print(json.dumps({"cfg": cfg, "overlap": ov or "auto", "rpb": rpb,
                          "ms_total": statistics.median(r[2].ms_total for r in runs),
                          "ms_sample": statistics.median(r[2].ms_sample for r in runs),
                          "ms_gather": statistics.median(r[2].ms_gather for r in runs)}), flush=True)
