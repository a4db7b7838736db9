"""Wall time of many small sng_dbscan calls: separate vs sngb_dbscan_batch_f32.
Not part of the product.  python tools/batch_timing.py [count] [n]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2006_06743_b200 as sng  # noqa: E402
from paper_2006_06743_b200 import synthetic  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 64
n = int(sys.argv[2]) if len(sys.argv) > 2 else 5000
w = synthetic.CONFIGS[1]
probs = [(sng.Dataset(synthetic.generate(1, n=n)),
          sng.SngParams(eps=w.eps, min_pts=w.min_pts, rate=min(1.0, 200 / n), seed=s))
         for s in range(count)]
for rep in range(3):
    t0 = time.perf_counter()
    a = [sng.sng_dbscan(ds, p) for ds, p in probs]
    t1 = time.perf_counter()
    b = sng.sng_dbscan_batch(probs)
    t2 = time.perf_counter()
assert all((x.assignment == y.assignment).all() for x, y in zip(a, b))
print(f"{count} problems of n={n}: separate {1e3 * (t1 - t0):.1f} ms, batch {1e3 * (t2 - t1):.1f} ms "
      f"({(t1 - t0) / (t2 - t1):.2f}x)")
