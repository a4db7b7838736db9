"""Multi-GPU SNG-DBSCAN: query rows sharded across ranks, points replicated.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Every
rank holds the full fp32 point replica (broadcast from rank 0, or each rank
uploads the same host array), and rank r samples and eps-tests the query rows
[r*n/W, (r+1)*n/W): the per-vertex work of graph.cpp:146-177 is independent,
so that step -- the hot path -- has no communication at all.

The edges then have to be clustered as one graph.  Two merges are provided:

``merge="fixed_point"`` (default, the north star's scheme)
  1. route: each shard's canonical keys (a<<32|b, a<b, sorted, unique) go to
     the owner of the smaller endpoint a -- one all-to-all.  A mutual draw (u
     drew v on one rank, v drew u on another) is the only cross-shard
     duplicate; after routing both copies sit on one rank, which dedups them
     (graph.cpp:34-40);
  2. degrees: every owner counts its keys on both endpoints, SUM all-reduce of
     int32[n] -> the sampled degree and the core mask on every rank
     (graph.hpp:28, clusterer.cpp:12-13);
  3. local union-find over the owned core-core keys (graph.cpp:222-235),
     hooking larger roots under smaller ones, so roots are minimum indices;
  4. fixed point: MIN all-reduce of the parent array, local re-union from the
     reduced forest, repeat until no rank changed an entry.  Each round moves
     every component's minimum across all ranks' edges, so it ends in a few
     rounds; at the fixed point every rank holds the same forest whose roots
     are the components' smallest core vertices;
  5. border roots by MIN all-reduce (clusterer.cpp:26-37) and the relabel
     (clusterer.cpp:41-51), computed identically on every rank.
  Traffic: 8 B per accepted edge once, then 4 B x n per all-reduce round.

``merge="allgather"``
  All-gather the shard keys; every rank clusters the whole edge set
  (sngb_cluster_edges_device).  8 B per edge to every rank, no rounds.

The edge builder and the merge steps are injectable so the host-side logic is
testable on CPU with gloo (tests/test_distributed.py); the production defaults
are the CUDA entry points of include/sngb.h and there is no CPU fallback.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch
import torch.distributed as dist

INT32_MAX = 0x7FFFFFFF


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous query-row shard of `rank` (graph.cpp:52-56 chunking, by rank)."""
    chunk = (n + world - 1) // world
    b = min(n, rank * chunk)
    return b, min(n, b + chunk)


def all_gather_varlen(t: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather 1-D tensors of different lengths (pad to the max, then trim)."""
    world = dist.get_world_size(group)
    if world == 1:
        return t
    cnt = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    sizes = [int(c.item()) for c in cnts]
    m = max(sizes)
    pad = torch.zeros(max(m, 1), dtype=t.dtype, device=t.device)
    pad[: t.numel()] = t
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return torch.cat([o[:s] for o, s in zip(outs, sizes)])


def route_keys_to_owners(keys: torch.Tensor, n: int, group=None) -> torch.Tensor:
    """All-to-all of canonical keys to the rank owning the smaller endpoint.

    `keys` must be sorted (as the edge builder returns them), so the keys for
    each destination are one contiguous run found by a binary search on the
    shard starts."""
    world = dist.get_world_size(group)
    if world == 1:
        return keys
    starts = torch.tensor([shard_bounds(n, world, r)[0] for r in range(world)] + [n],
                          dtype=torch.int64, device=keys.device) << 32
    cuts = torch.searchsorted(keys, starts)
    send = (cuts[1:] - cuts[:-1]).to(torch.int64)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    send_l, recv_l = send.tolist(), recv.tolist()
    out = torch.empty(sum(recv_l), dtype=keys.dtype, device=keys.device)
    dist.all_to_all_single(out, keys, recv_l, send_l, group=group)
    return out


@dataclass
class MergeOps:
    """The device steps of the fixed-point merge (include/sngb.h)."""
    unique_keys: Callable
    degrees: Callable
    components: Callable
    border: Callable
    relabel: Callable


def cuda_merge_ops() -> MergeOps:
    from . import (border_device, components_device, degrees_device, relabel_device,
                   unique_keys_device)
    return MergeOps(unique_keys_device, degrees_device, components_device, border_device,
                    relabel_device)


def _default_edge_fn(points, eps, rate, seed, row_begin, row_end):
    from . import sampled_edges_device
    keys, gi = sampled_edges_device(points, eps, rate, seed, row_begin, row_end, timing=True)
    return keys, gi


def _default_cluster_fn(keys, n, min_pts):
    from . import cluster_edges_device
    return cluster_edges_device(keys, n, min_pts)


def fixed_point_merge(keys: torch.Tensor, n: int, min_pts: int, group=None,
                      ops: MergeOps | None = None, max_rounds: int = 64):
    """Steps 1-5 of the module docstring for this rank's (sorted unique) keys.

    Returns (labels, roles, relabel info, stats) -- identical on every rank."""
    ops = ops or cuda_merge_ops()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    routed = route_keys_to_owners(keys, n, group) if world > 1 else keys
    owned = ops.unique_keys(routed, n)
    degree = ops.degrees(owned, n, torch.zeros(n, dtype=torch.int32, device=keys.device))
    if world > 1:
        dist.all_reduce(degree, op=dist.ReduceOp.SUM, group=group)
    parent = torch.arange(n, dtype=torch.int32, device=keys.device)
    ops.components(owned, n, degree, min_pts, parent)
    rounds = 0
    if world > 1:
        while True:
            dist.all_reduce(parent, op=dist.ReduceOp.MIN, group=group)
            changed = ops.components(owned, n, degree, min_pts, parent)
            rounds += 1
            flag = torch.tensor([changed], dtype=torch.int64, device=keys.device)
            dist.all_reduce(flag, op=dist.ReduceOp.SUM, group=group)
            if int(flag.item()) == 0:
                break
            if rounds >= max_rounds:
                raise RuntimeError(f"union-find merge did not converge in {max_rounds} rounds")
    border = torch.full((n,), INT32_MAX, dtype=torch.int32, device=keys.device)
    ops.border(owned, n, degree, min_pts, parent, border)
    if world > 1:
        dist.all_reduce(border, op=dist.ReduceOp.MIN, group=group)
    labels, roles, info = ops.relabel(n, degree, min_pts, parent, border)
    edges = torch.tensor([owned.numel()], dtype=torch.int64, device=keys.device)
    if world > 1:
        dist.all_reduce(edges, op=dist.ReduceOp.SUM, group=group)
    return labels, roles, info, {"routed_keys": int(routed.numel()),
                                 "owned_edges": int(owned.numel()), "edges": int(edges.item()),
                                 "merge_rounds": rounds}


def sng_dbscan_sharded(points: torch.Tensor, eps: float, min_pts: int, rate: float, seed: int,
                       group=None, edge_fn: Callable | None = None,
                       cluster_fn: Callable | None = None, merge: str = "fixed_point",
                       merge_ops: MergeOps | None = None):
    """sng::sng_dbscan over all ranks of `group`; every rank returns the labels.

    points: the full [n, d] fp32 replica on this rank's device.
    Returns (labels, roles, stats dict) -- labels/roles on points.device.
    """
    edge_fn = edge_fn or _default_edge_fn
    if not (eps > 0.0):
        from . import InvalidArgument
        raise InvalidArgument("eps must be > 0")
    if min_pts < 1:
        from . import InvalidArgument
        raise InvalidArgument("min_pts must be >= 1")
    if merge not in ("fixed_point", "allgather"):
        raise ValueError(f"unknown merge {merge!r}")
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = points.shape[0]
    rb, re = shard_bounds(n, world, rank)
    keys, ginfo = edge_fn(points, eps, rate, seed, rb, re)
    stats = {"shard": (rb, re), "shard_edges": int(keys.numel()), "edge_info": ginfo,
             "merge": merge}
    if merge == "fixed_point":
        labels, roles, cinfo, mst = fixed_point_merge(keys, n, min_pts, group, merge_ops)
        stats.update(mst)
    else:
        cluster_fn = cluster_fn or _default_cluster_fn
        all_keys = all_gather_varlen(keys, group) if world > 1 else keys
        labels, roles, cinfo = cluster_fn(all_keys, n, min_pts)
        stats["gathered_keys"] = int(all_keys.numel())
    stats["cluster_info"] = cinfo
    return labels, roles, stats
