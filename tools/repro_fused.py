import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
os.environ.update({"SNGB_HEAD": "2", "SNGB_HEAD_KIND": "0", "SNGB_FLOYD_NO_BITMAP": "1", "SNGB_FUSED": "1", "SNGB_Q8": "0"})
import paper_2006_06743_b200 as sng
rng = np.random.default_rng(31)
pts = rng.random((3000, 3), dtype=np.float32)
info = sng.ClusterRunInfo()
c = sng.sng_dbscan(sng.Dataset(pts), sng.SngParams(eps=0.05, min_pts=3, rate=0.05, seed=31), info)
print("ok", c.cluster_count, info.edges)
