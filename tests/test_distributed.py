"""Multi-GPU sharding/merge logic of paper_2006_06743_b200.distributed, run on
CPU with gloo at world_size 2 (and 3).  The per-rank edge builder is the
oracle and the device merge steps are numpy stand-ins with the contract of
include/sngb.h (test-only injection; production uses the CUDA entry points,
whose GPU parity is in tests/test_gpu_merge.py).  Both merges -- the
fixed-point union-find merge (key routing, SUM/MIN all-reduces, rounds until
no rank changes) and the all-gather merge -- must reproduce the
single-process reference result exactly on every rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2006_06743_b200.distributed import (INT32_MAX, MergeOps, all_gather_varlen,
                                               shard_bounds)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def numpy_merge_ops() -> MergeOps:
    """CPU stand-ins for the sngb_*_device merge steps (same contracts)."""

    def ends(keys):
        k = keys.numpy().view(np.uint64)
        return (k >> np.uint64(32)).astype(np.int64), (k & np.uint64(0xFFFFFFFF)).astype(np.int64)

    def unique_keys(keys, n):
        return torch.from_numpy(np.unique(keys.numpy()))

    def degrees(keys, n, degree):
        a, b = ends(keys)
        d = degree.numpy()
        np.add.at(d, a, 1)
        np.add.at(d, b, 1)
        return degree

    def components(keys, n, degree, min_pts, parent):
        p = parent.numpy()
        before = p.copy()
        core = degree.numpy() >= min_pts

        def find(x):
            while p[x] != x:
                p[x] = p[p[x]]
                x = p[x]
            return x

        for a, b in zip(*ends(keys)):
            if core[a] and core[b]:
                ra, rb = find(a), find(b)
                if ra != rb:
                    p[max(ra, rb)] = min(ra, rb)
        for v in np.flatnonzero(core):
            p[v] = find(v)
        return int((p != before).sum())

    def border(keys, n, degree, min_pts, parent, border):
        a, b = ends(keys)
        core, p, br = degree.numpy() >= min_pts, parent.numpy(), border.numpy()
        m = core[a] & ~core[b]
        np.minimum.at(br, b[m], p[a[m]])
        m = core[b] & ~core[a]
        np.minimum.at(br, a[m], p[b[m]])

    def relabel(n, degree, min_pts, parent, border):
        core, p, br = degree.numpy() >= min_pts, parent.numpy(), border.numpy()
        root = np.where(core, p, br)
        first = {}
        for v in range(n):
            if root[v] != INT32_MAX:
                first.setdefault(int(root[v]), v)
        order = {r: i for i, r in enumerate(sorted(first, key=first.get))}
        labels = np.array([order[int(r)] if r != INT32_MAX else -1 for r in root], np.int32)
        roles = np.where(core, 0, np.where(root != INT32_MAX, 1, 2)).astype(np.uint8)
        return torch.from_numpy(labels), torch.from_numpy(roles), {"clusters": len(order)}

    return MergeOps(unique_keys, degrees, components, border, relabel)


def _worker(rank, world, port, case, merge, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import Oracle
    from paper_2006_06743_b200.distributed import sng_dbscan_sharded
    from paper_2006_06743_b200 import synthetic
    orc = Oracle()
    cfg, n, eps, mp_, rate, seed = case
    pts = synthetic.generate(cfg, n=n)

    def edge_fn(points, eps, rate, seed, rb, re):
        keys, evals = orc.sampled_edges_rows(points.numpy(), eps, rate, seed, rb, re, threads=1)
        return torch.from_numpy(keys.view(np.int64)), {"evals": evals}

    def cluster_fn(keys, n, min_pts):
        k = np.unique(keys.numpy().view(np.uint64))  # dedup like sngb_cluster_edges_device
        labels, roles, cnt = orc.cluster_edges(k, n, min_pts)
        return torch.from_numpy(labels), torch.from_numpy(roles), {"edges": len(k), "clusters": cnt}

    labels, roles, st = sng_dbscan_sharded(torch.from_numpy(pts), eps, mp_, rate, seed,
                                           edge_fn=edge_fn, cluster_fn=cluster_fn, merge=merge,
                                           merge_ops=numpy_merge_ops())
    edges = st["edges"] if merge == "fixed_point" else st["cluster_info"]["edges"]
    np.save(os.path.join(out_dir, f"labels{rank}.npy"), labels.numpy())
    np.save(os.path.join(out_dir, f"roles{rank}.npy"), roles.numpy())
    with open(os.path.join(out_dir, f"edges{rank}.txt"), "w") as f:
        f.write(f"{edges} {st['shard_edges']} {st['edge_info']['evals']}")
    dist.destroy_process_group()


@pytest.mark.parametrize("merge", ["fixed_point", "allgather"])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", [(1, 6000, 0.03, 10, 0.1, 1), (4, 20000, 0.1, 4, 0.05, 4),
                                  (5, 8000, 1.2, 5, 0.2, 5)])
def test_sharded_matches_single_process(tmp_path, oracle, world, case, merge):
    cfg, n, eps, mp_, rate, seed = case
    mp.start_processes(_worker, args=(world, _free_port(), case, merge, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    from paper_2006_06743_b200 import synthetic
    pts = synthetic.generate(cfg, n=n)
    labels, roles, info, keys = oracle.sng_dbscan(pts, eps, mp_, rate, seed)
    total_evals = 0
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"labels{r}.npy"), labels)
        np.testing.assert_array_equal(np.load(tmp_path / f"roles{r}.npy"), roles)
        e, _, ev = (int(x) for x in open(tmp_path / f"edges{r}.txt").read().split())
        assert e == info["edges"]
        total_evals += ev
    assert total_evals == info["distance_evals"]


def test_shard_bounds_cover_rows():
    for n in (1, 2, 7, 100, 1001):
        for w in (1, 2, 3, 8):
            spans = [shard_bounds(n, w, r) for r in range(w)]
            covered = [i for b, e in spans for i in range(b, e)]
            assert covered == list(range(n))


def _gather_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = torch.arange(rank * 10, rank * 10 + rank + 1, dtype=torch.int64)  # lengths 1, 2, 3
    g = all_gather_varlen(t)
    np.save(os.path.join(out_dir, f"g{rank}.npy"), g.numpy())
    dist.destroy_process_group()


def test_all_gather_varlen(tmp_path):
    mp.start_processes(_gather_worker, args=(3, _free_port(), str(tmp_path)), nprocs=3,
                       join=True, start_method="spawn")
    want = [0, 10, 11, 20, 21, 22]
    for r in range(3):
        assert np.load(tmp_path / f"g{r}.npy").tolist() == want
