"""Floyd kernel A/B (not part of the product): ms_sample of k_floyd_bloom and
k_floyd_warp on full-size configs, sequential with the gather (SNGB_OVERLAP=0).

    SNGB_LIBRARY=tools/ab/libsngb_fwr16.so python tools/floyd_ab.py 4 5
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2006_06743_b200 as sng  # noqa: E402
from paper_2006_06743_b200 import synthetic  # noqa: E402

lib = os.path.basename(os.environ.get("SNGB_LIBRARY", "libsngb.so"))
os.environ["SNGB_OVERLAP"] = "0"
os.environ["SNGB_FUSED"] = "0"
for cfg in [int(c) for c in sys.argv[1:]] or [5]:
    w = synthetic.CONFIGS[cfg]
    x = torch.from_numpy(synthetic.generate(cfg)).cuda()
    for fw in ("0", "1"):
        os.environ["SNGB_FLOYD_WARP"] = fw
        sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True)
        ms = [sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True)[2].ms_sample
              for _ in range(3)]
        print(json.dumps({"cfg": cfg, "lib": lib, "kernel": "k_floyd_warp" if fw == "1" else "k_floyd_bloom",
                          "ms_sample": statistics.median(ms)}), flush=True)
    del x
    torch.cuda.empty_cache()
