"""GPU parity of the multi-GPU merge steps (include/sngb.h: unique_keys,
degrees, components, border, relabel) through the C ABI.

This run has one GPU, so W ranks are emulated one after another in a single
process: rank r builds the edges of its row shard with
sngb_sampled_edges_f32_device, the keys are routed to the owner of the
smaller endpoint, and the NCCL SUM / MIN all-reduces of
distributed.fixed_point_merge are done here with torch reductions over the
per-rank arrays (no rank ever waits on another).  The labels must equal the
single-GPU call and the oracle, bit for bit.  The host loop itself (routing,
all-reduces, termination) runs under gloo in tests/test_distributed.py.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2006_06743_b200 as sng  # noqa: E402
from paper_2006_06743_b200 import synthetic  # noqa: E402
from paper_2006_06743_b200.distributed import INT32_MAX, shard_bounds  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if sng.device_count() < 1:
        pytest.fail("no CUDA device: the GPU path has no CPU fallback")


def emulate_ranks(x, eps, min_pts, rate, seed, world):
    n = x.shape[0]
    shards = []
    for r in range(world):
        rb, re = shard_bounds(n, world, r)
        keys, _ = sng.sampled_edges_device(x, eps, rate, seed, rb, re)
        shards.append(keys)
    # route to the owner of the smaller endpoint (all-to-all)
    owned = []
    for r in range(world):
        rb, re = shard_bounds(n, world, r)
        parts = [k[((k >> 32) >= rb) & ((k >> 32) < re)] for k in shards]
        owned.append(sng.unique_keys_device(torch.cat(parts), n))
    deg = sum(sng.degrees_device(k, n) for k in owned)  # SUM all-reduce
    parents = []
    for k in owned:
        p = torch.arange(n, dtype=torch.int32, device=x.device)
        sng.components_device(k, n, deg, min_pts, p)
        parents.append(p)
    rounds = 0
    while True:
        g = torch.stack(parents).amin(0)  # MIN all-reduce
        parents = [g.clone() for _ in range(world)]
        changed = sum(sng.components_device(k, n, deg, min_pts, p)
                      for k, p in zip(owned, parents))
        rounds += 1
        if changed == 0:
            break
        assert rounds < 64
    for p in parents[1:]:
        assert torch.equal(p, parents[0])
    borders = []
    for k, p in zip(owned, parents):
        b = torch.full((n,), INT32_MAX, dtype=torch.int32, device=x.device)
        sng.border_device(k, n, deg, min_pts, p, b)
        borders.append(b)
    border = torch.stack(borders).amin(0)
    labels, roles, gi = sng.relabel_device(n, deg, min_pts, parents[0], border)
    return labels, roles, gi, sum(k.numel() for k in owned), rounds


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("cfg,n", [(1, 20000), (2, 6000), (3, 50000), (5, 60000)])
def test_emulated_ranks_match_single_gpu_and_oracle(oracle, cfg, n, world):
    w = synthetic.CONFIGS[cfg]
    pts = synthetic.generate(cfg, n=n)
    rate = min(1.0, w.draws / n)
    x = torch.from_numpy(pts).cuda()
    labels, roles, gi, edges, rounds = emulate_ranks(x, w.eps, w.min_pts, rate, w.seed, world)
    l1, r1, g1 = sng.sng_dbscan_device(x, w.eps, w.min_pts, rate, w.seed)
    assert torch.equal(labels, l1)
    assert torch.equal(roles, r1)
    assert edges == g1.edges
    assert gi.cluster_count == g1.cluster_count
    assert (gi.core_count, gi.border_count, gi.noise_count) == \
        (g1.core_count, g1.border_count, g1.noise_count)
    ol, orl, oinfo, _ = oracle.sng_dbscan(pts, w.eps, w.min_pts, rate, w.seed)
    np.testing.assert_array_equal(labels.cpu().numpy(), ol)
    np.testing.assert_array_equal(roles.cpu().numpy(), orl)
    assert edges == oinfo["edges"]


def test_unique_keys_matches_numpy():
    g = torch.Generator().manual_seed(3)
    n = 1000
    a = torch.randint(0, n - 1, (50000,), generator=g)
    b = a + 1 + torch.randint(0, 10, (50000,), generator=g)
    b = torch.minimum(b, torch.full_like(b, n - 1))
    a = torch.where(a == b, a - 1, a).clamp(min=0)
    keys = (a << 32) | b
    keys = keys[a < b]
    out = sng.unique_keys_device(keys.cuda(), n)
    np.testing.assert_array_equal(out.cpu().numpy(), np.unique(keys.numpy()))
    assert sng.unique_keys_device(torch.empty(0, dtype=torch.int64, device="cuda"), n).numel() == 0


def test_components_chain_and_changed_count():
    # path 0-1-2-...-9, all core (min_pts=1): one set rooted at 0
    n = 10
    keys = torch.tensor([(i << 32) | (i + 1) for i in range(n - 1)], dtype=torch.int64).cuda()
    deg = sng.degrees_device(keys, n)
    assert deg.tolist() == [1] + [2] * (n - 2) + [1]
    p = torch.arange(n, dtype=torch.int32, device="cuda")
    assert sng.components_device(keys, n, deg, 1, p) == n - 1
    assert p.tolist() == [0] * n
    assert sng.components_device(keys, n, deg, 1, p) == 0  # fixed point
    # min_pts=2: the ends are border points of the one cluster
    p = torch.arange(n, dtype=torch.int32, device="cuda")
    sng.components_device(keys, n, deg, 2, p)
    b = torch.full((n,), INT32_MAX, dtype=torch.int32, device="cuda")
    sng.border_device(keys, n, deg, 2, p, b)
    labels, roles, gi = sng.relabel_device(n, deg, 2, p, b)
    assert labels.tolist() == [0] * n
    assert roles.tolist() == [1] + [0] * (n - 2) + [1]
    assert (gi.cluster_count, gi.core_count, gi.border_count, gi.noise_count) == (1, 8, 2, 0)


def test_merge_steps_reject_bad_keys():
    n = 10
    deg = torch.zeros(n, dtype=torch.int32, device="cuda")
    for bad in ((3 << 32) | 3, (5 << 32) | 2, (1 << 32) | 10):
        keys = torch.tensor([bad], dtype=torch.int64, device="cuda")
        with pytest.raises(sng.InvalidArgument):
            sng.degrees_device(keys, n, deg)
        with pytest.raises(sng.InvalidArgument):
            sng.components_device(keys, n, deg, 1, torch.arange(n, dtype=torch.int32,
                                                               device="cuda"))
        if bad != (5 << 32) | 2:  # unique_keys canonicalises swapped pairs
            with pytest.raises(sng.InvalidArgument):
                sng.unique_keys_device(keys, n)
    assert deg.sum().item() == 0  # nothing written by the failed calls
    with pytest.raises(sng.InvalidArgument):  # int32 vertex arrays: n < 2^31
        sng.degrees_device(torch.empty(0, dtype=torch.int64, device="cuda"), 1 << 31, deg)
