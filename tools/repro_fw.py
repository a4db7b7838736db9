"""Debug repro (not part of the product): k_floyd_warp on the failing shape
with the bounds-checking test build tools/ab/libsngb_fwdbg.so."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_06743_b200 import _lib
os.environ["SNGB_FLOYD_NO_BITMAP"] = "1"
L = _lib.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "ab", "libsngb_fwdbg.so"))
_lib._lib = L
import paper_2006_06743_b200 as sng
from oracle import Oracle
for n, d, eps, rate, seed, force in [(3000, 2, 0.05, 0.3, 1, None), (3000, 2, 0.05, 0.3, 1, "7"),
                                     (20000, 16, 1.0, 0.02, 3, "7"), (6000, 3, 0.1, 0.8, 4, "7")]:
    if force: os.environ["SNGB_TEST_FORCE_IRREGULAR"] = force
    else: os.environ.pop("SNGB_TEST_FORCE_IRREGULAR", None)
    rng = np.random.default_rng(seed)
    pts = rng.random((n, d), dtype=np.float32)
    keys, _ = Oracle().sampled_edges(pts, eps, rate, seed)
    g = sng.build_sampled_graph(sng.Dataset(pts), eps, rate, seed=seed)
    print(n, d, rate, force, "equal" if np.array_equal(g.keys, keys) else "DIFFERENT", flush=True)
