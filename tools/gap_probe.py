"""Outer CUDA-event time of a call minus the library's own E_START..E_END (diagnostic)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_06743_b200 as sng
from paper_2006_06743_b200 import synthetic
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = synthetic.CONFIGS[cfg]
x = torch.from_numpy(synthetic.generate(cfg)).cuda()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()
for name, env in (("default", {}), ("rpb8", {"SNGB_SAMPLER_RPB": "8"}), ("rpb0", {"SNGB_SAMPLER_RPB": "0"}), ("noflush", {}), ("overlap0", {"SNGB_OVERLAP": "0"})):
    for k in ("SNGB_SAMPLER_RPB", "SNGB_OVERLAP"):
        os.environ.pop(k, None)
    os.environ.update(env)
    for _ in range(2):
        sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True)
    outer, inner = [], []
    for _ in range(6):
        if name != "noflush":
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        _, _, gi = sng.sng_dbscan_device(x, w.eps, w.min_pts, w.rate, w.seed, timing=True)
        b.record(st)
        torch.cuda.synchronize()
        outer.append(a.elapsed_time(b)); inner.append(gi.ms_total)
    print(json.dumps({"cfg": cfg, "variant": name, "outer_ms": round(statistics.median(outer), 3),
                      "ms_total": round(statistics.median(inner), 3),
                      "ms_sample": round(gi.ms_sample, 3), "ms_gather": round(gi.ms_gather, 3)}), flush=True)
