"""sngdbscan -- the Python module the reference planned (proj/CMakeLists.txt:11,
pybind11; proj/python/CMakeLists.txt:1 is a placeholder), over libsngb.so.

    import sngdbscan
    labels, roles, info = sngdbscan.sng_dbscan(points, eps=0.03, min_pts=10, rate=0.1, seed=1,
                                               num_gpus=None)

``points``: float32 / float64 [n, d].  ``num_gpus``: None or 1 = one GPU, N = shard
the rows over N GPUs of this process, -1 = all.  The extension is built in-tree
by ``python -m paper_2006_06743_b200.build`` (sngdbscan/_sngdbscan*.so); there
is no CPU fallback.
"""
from ._sngdbscan import (ABI_VERSION, BORDER, CORE, NOISE, dbscan_exact,  # noqa: F401
                         device_count, sng_dbscan)

__all__ = ["sng_dbscan", "dbscan_exact", "device_count", "NOISE", "CORE", "BORDER",
           "ABI_VERSION"]
