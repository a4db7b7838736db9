"""Multi-GPU sharding/merge logic of paper_2006_06743_b200.distributed, run on
CPU with gloo at world_size 2 (and 3).  The per-rank edge builder and the
clusterer are the oracle (test-only injection; production uses the CUDA
entry points): the union of the shards' edges, all-gathered and clustered on
every rank, must reproduce the single-process reference result exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2006_06743_b200.distributed import all_gather_varlen, shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, out_dir):
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
                                           edge_fn=edge_fn, cluster_fn=cluster_fn)
    np.save(os.path.join(out_dir, f"labels{rank}.npy"), labels.numpy())
    np.save(os.path.join(out_dir, f"roles{rank}.npy"), roles.numpy())
    with open(os.path.join(out_dir, f"edges{rank}.txt"), "w") as f:
        f.write(f"{st['cluster_info']['edges']} {st['shard_edges']} {st['edge_info']['evals']}")
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", [(1, 6000, 0.03, 10, 0.1, 1), (4, 20000, 0.1, 4, 0.05, 4),
                                  (5, 8000, 1.2, 5, 0.2, 5)])
def test_sharded_matches_single_process(tmp_path, oracle, world, case):
    cfg, n, eps, mp_, rate, seed = case
    mp.start_processes(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
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
