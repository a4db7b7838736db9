"""k_floyd_pipe vs k_floyd_lean by draws per vertex (the pipe_wanted crossover; not part
of the product): cfg5-shaped data at n = 4 M, sampler alone (SNGB_OVERLAP=0)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_06743_b200 as sng
from paper_2006_06743_b200 import synthetic
n = 4_000_000
w = synthetic.CONFIGS[5]
x = torch.from_numpy(synthetic.generate(5, n=n)).cuda()
os.environ["SNGB_OVERLAP"] = "0"
for D in (1100, 1500, 2048, 2100, 2600, 3000, 3400, 3800, 4096):
    rec = {"n": n, "draws": D}
    for pipe in ("0", "1"):
        os.environ["SNGB_FLOYD_PIPE"] = pipe
        for rpb in ("8", "64"):
            os.environ["SNGB_SAMPLER_RPB"] = rpb
            sng.sng_dbscan_device(x, w.eps, w.min_pts, D / n, w.seed, timing=True)
            runs = [sng.sng_dbscan_device(x, w.eps, w.min_pts, D / n, w.seed, timing=True) for _ in range(3)]
            rec[("pipe" if pipe == "1" else "lean") + "_rpb" + rpb] = round(statistics.median(r[2].ms_sample for r in runs), 3)
    print(json.dumps(rec), flush=True)
