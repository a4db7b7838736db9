"""cfg5 (or --config k): the Floyd kernel beside the head gather under several
co-scheduling settings (env knobs read per call by the library).  A/B helper,
not part of the product.

    python tools/overlap_sweep.py --config 5
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2006_06743_b200 as sng  # noqa: E402
from paper_2006_06743_b200 import synthetic  # noqa: E402

KNOBS = ("SNGB_OVERLAP", "SNGB_SAMPLER_RPB", "SNGB_SAMPLER_BPSM", "SNGB_GATHER_BPSM",
         "SNGB_FLOYD_WARP", "SNGB_FUSED", "SNGB_GATHER_RPB")
if os.environ.get("SWEEP") == "rpb":
    SETTINGS = [("sequential_bloom", {"SNGB_OVERLAP": "0"})]
    for gb in (os.environ.get("SWEEP_G", "4,3,2,1").split(",")):
        for srpb in (os.environ.get("SWEEP_RPB", "32,8").split(",")):
            SETTINGS.append((f"overlap_bloom_rpb{srpb}_g{gb}",
                             {"SNGB_OVERLAP": "1", "SNGB_SAMPLER_RPB": srpb, "SNGB_GATHER_BPSM": gb}))
    SETTINGS.append(("overlap_bloom_rpb32_gather_rpb128",
                     {"SNGB_OVERLAP": "1", "SNGB_SAMPLER_RPB": "32", "SNGB_GATHER_RPB": "128"}))
else:
  SETTINGS = [("sequential_bloom", {"SNGB_OVERLAP": "0"}),
            ("sequential_warp", {"SNGB_OVERLAP": "0", "SNGB_FLOYD_WARP": "1"})]
for fw in (("0", "1") if os.environ.get("SWEEP") != "rpb" else ()):
    for sb, gb in (("1", "3"), ("2", "3"), ("4", "3"), ("2", "2"), ("4", "2"), ("8", "2")):
        if fw == "0" and sb in ("4", "8"):
            continue  # the bloom kernel's blocks are 9 warps
        SETTINGS.append((f"overlap_{'warp' if fw == '1' else 'bloom'}_s{sb}_g{gb}",
                         {"SNGB_OVERLAP": "1", "SNGB_SAMPLER_RPB": "0", "SNGB_SAMPLER_BPSM": sb,
                          "SNGB_GATHER_BPSM": gb, "SNGB_FLOYD_WARP": fw}))
    SETTINGS.append((f"overlap_{'warp' if fw == '1' else 'bloom'}_rpb32",
                     {"SNGB_OVERLAP": "1", "SNGB_FLOYD_WARP": fw}))

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=5)
p.add_argument("--reps", type=int, default=3)
a = p.parse_args()
w = synthetic.CONFIGS[a.config]
x = torch.from_numpy(synthetic.generate(a.config)).cuda()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
ref = None
for name, env in SETTINGS:
    for k in KNOBS:
        os.environ.pop(k, None)
    os.environ["SNGB_FUSED"] = "0"
    os.environ.update(env)
    sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed)
    ms = []
    for _ in range(a.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lab, _, gi = sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed)
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    h = hash(lab.cpu().numpy().tobytes())
    ref = ref if ref is not None else h
    print(json.dumps({"cfg": a.config, "setting": name, "step_ms": statistics.median(ms),
                      "same_labels": h == ref}), flush=True)
