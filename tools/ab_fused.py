"""A/B timing of the fused Floyd + head gather (sngb_fused.cu) against the two
kernels, on full-size BASELINE configs.  Not part of the product.

    SNGB_LIBRARY=... python tools/ab_fused.py [cfg ...]

Prints one JSON line per (cfg, variant): median step ms over 5 timed calls (CUDA
events, 256 MB L2 flush before each), the library's stage times, and a digest
of the labels (variants must agree).
"""
import hashlib
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2006_06743_b200 as sng  # noqa: E402
from paper_2006_06743_b200 import synthetic  # noqa: E402

cfgs = [int(a) for a in sys.argv[1:]] or [3, 4, 5]
variants = [("fused", {"SNGB_FUSED": "1"}), ("two_kernels", {"SNGB_FUSED": "0"}),
            ("two_kernels_bloom", {"SNGB_FUSED": "0", "SNGB_FLOYD_BLOOM": "1"})]
if os.environ.get("AB_VARIANTS"):
    variants = [v for v in variants if v[0] in os.environ["AB_VARIANTS"].split(",")]
lib = os.path.basename(os.environ.get("SNGB_LIBRARY", "libsngb.so"))
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for cfg in cfgs:
    w = synthetic.CONFIGS[cfg]
    x = torch.from_numpy(synthetic.generate(cfg)).cuda()
    for name, env in variants:
        for k in ("SNGB_FUSED", "SNGB_FLOYD_BLOOM"):
            os.environ.pop(k, None)
        os.environ.update(env)
        for _ in range(2):
            sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True)
        ms, infos = [], []
        for _ in range(5):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            lab, rol, gi = sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True)
            b.record()
            b.synchronize()
            ms.append(a.elapsed_time(b))
            infos.append(gi.as_dict())
        g = infos[-1]
        print(json.dumps({"cfg": cfg, "variant": name, "lib": lib, "step_ms": statistics.median(ms),
                          "ms_sample": g["ms_sample"], "ms_gather": g["ms_gather"],
                          "ms_extras": g["ms_extras"], "ms_sort": g["ms_sort"],
                          "ms_cluster": g["ms_cluster"], "edges": g["edges"],
                          "collisions": g["collisions"],
                          "labels": hashlib.sha256(lab.cpu().numpy().tobytes()).hexdigest()[:16]}),
              flush=True)
    del x
    torch.cuda.empty_cache()
