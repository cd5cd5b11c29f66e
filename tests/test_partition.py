"""Multi-GPU subtree partition (SURVEY §8(e) mechanism 2; include/ttn_cbc.h ttn_ctx_set_comm).

CPU (host logic, no device): the partition plan covers the tree with whole subtrees under a
connected replicated top, and two gloo ranks agree on the plan, on the NCCL-id transport and
on a disjoint, complete split of the subtree work.  GPU: the partitioned schedule (1-rank
NCCL communicator, 2 and 4 subtree groups) reproduces the plain apply.
"""
import os
import socket

import numpy as np
import pytest

import workloads as W

TREES = {
    "cfg4_t3ns": W.make_config(4).parent,
    "binary31": W.complete_binary(31),
    "binary63": W.complete_binary(63),
    "star3x2": W.star_of_chains_literal(3, 2),
    "chain9": W.chain(9),
}


def _plan(parent, parts):
    import paper_2601_19650_b200 as P
    return P.ttn_partition_plan(parent, parts)


@pytest.mark.parametrize("name", sorted(TREES))
@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_plan_is_whole_subtrees_under_connected_top(name, parts):
    parent = TREES[name]
    g = _plan(parent, parts)
    n = len(parent)
    root = parent.index(-1)
    assert g[root] == -1
    for i in range(n):
        p = parent[i]
        if p < 0:
            continue
        if g[i] == -1:
            assert g[p] == -1, "the top must be connected to the root"
        elif g[p] != -1:
            assert g[p] == g[i], "a subtree lies in one group"
    assert all(-1 <= x < max(parts, 1) for x in g)
    if parts == 1:
        assert all(x == -1 for x in g)


def test_plan_config4_uses_the_chains():
    parent = TREES["cfg4_t3ns"]
    g2, g4 = _plan(parent, 2), _plan(parent, 4)
    assert g2.count(-1) == 1 and sorted(g2.count(k) for k in range(2)) == [33, 33]   # junction subtrees
    assert g4.count(-1) == 3 and [g4.count(k) for k in range(4)] == [16, 16, 16, 16]  # the 4 chains (B:10)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2601_19650_b200 as P
        fake_id = bytes(np.random.default_rng(1234).integers(0, 256, 128, dtype=np.uint8)) if rank == 0 else None
        uid = P.share_bytes(fake_id, 128)
        parent = TREES["cfg4_t3ns"]
        plan = P.ttn_partition_plan(parent, 4)
        mine = [i for i, x in enumerate(plan) if x >= 0 and x % world == rank]
        out[rank] = (uid, plan, mine)
    finally:
        dist.destroy_process_group()


def test_two_gloo_ranks_agree_on_id_plan_and_split():
    import torch.multiprocessing as mp
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gloo_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    (u0, p0, m0), (u1, p1, m1) = out[0], out[1]
    assert u0 == u1 and len(u0) == 128
    assert p0 == p1
    assert not set(m0) & set(m1)
    assert sorted(m0 + m1) == [i for i, x in enumerate(p0) if x >= 0]
    assert len(m0) == len(m1) == 32


# ------------------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("tree,chi,D,mb", [("binary31", 4, 3, 6), ("star3x2", 3, 2, 4), ("binary63", 3, 2, 4)])
@pytest.mark.parametrize("parts", [2, 4])
@pytest.mark.parametrize("slices", [None, 3])
def test_partitioned_schedule_matches_plain_apply(tree, chi, D, mb, parts, slices, monkeypatch):
    """slices=3: the top's G-route compresses are row-split into 3 virtual slices (the
    multi-GPU path of cbc.cpp split_rows with every slice on this rank), so sum_s X_s^H X_s
    must reproduce the plain Gram X^H X."""
    import torch
    if slices is not None:
        monkeypatch.setenv("TTN_PARTITION_SLICES", str(slices))
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_19650_b200 as P
    from ._helpers import gpu_pair, to_oracle, distances
    from oracle import norm
    parent = TREES[tree]
    inst = W.configs.random_instance(parent, [2] * len(parent), chi, D, mb, seed=5)
    ctx = P.Context(0)
    try:
        op, st = gpu_pair(P, ctx, inst)
        ref, rep0 = P.cbc_apply(ctx, op, st, mb)
        P.ttn_ctx_set_comm(ctx, P.ttn_comm_unique_id(), 0, 1, parts)
        got, rep1 = P.cbc_apply(ctx, op, st, mb)
        P.ttn_ctx_set_comm(ctx, None)
        a, b = to_oracle(P, got, parent), to_oracle(P, ref, parent)
        assert a.bonds() == b.bonds()
        d_cos, d_rel = distances(a, b)
        # partition phases batch fewer Grams per launch, so the eigensolver may take its
        # cluster kernel where the plain apply takes the per-CTA one: agreement to rounding
        # (1 - cos is quadratic in the distance; the overlap-based d_rel floors near 1e-8, A18)
        assert d_cos <= 1e-14, (d_cos, d_rel)
        assert abs(rep1["discarded_weight_sum"] - rep0["discarded_weight_sum"]) <= 1e-12 * max(1.0, rep0["discarded_weight_sum"])
        assert abs(rep1["norm"] - rep0["norm"]) <= 1e-12 * rep0["norm"]
        assert rep0["split_compresses"] == 0
        assert (rep1["split_compresses"] > 0) == (slices is not None)
    finally:
        ctx.close()


@pytest.mark.gpu
@pytest.mark.parametrize("slices", [None, 4])
def test_partitioned_config4_matches_golden(slices, monkeypatch):
    import json
    if slices is not None:
        monkeypatch.setenv("TTN_PARTITION_SLICES", str(slices))
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_19650_b200 as P
    from ._helpers import gpu_pair, to_oracle
    from oracle import norm
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cfg4_seed0.json")))
    inst = W.make_config(4, seed=0)
    ctx = P.Context(0)
    try:
        op, st = gpu_pair(P, ctx, inst)
        P.ttn_ctx_set_comm(ctx, P.ttn_comm_unique_id(), 0, 1, 4)
        out, rep = P.cbc_apply(ctx, op, st, inst.max_bond)
        P.ttn_ctx_set_comm(ctx, None)
        phi = to_oracle(P, out, inst.parent)
        assert phi.bonds() == gold["bonds"]
        assert abs(norm(phi) ** 2 - gold["phi_norm2"]) <= 1e-10 * gold["phi_norm2"]
        assert (rep["split_compresses"] > 0) == (slices is not None)
    finally:
        ctx.close()


def _bench_worker(rank, world, port, out):
    import sys
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import bench
        seeds = bench.shard_seeds(rank, 64, False)
        ms = 100.0 + 10.0 * rank          # rank 1 is the slower one
        weak = bench.aggregate(ms, 1e12, 64, world, False, "cpu")
        strong = bench.aggregate(ms, 5e12, 1, world, True, "cpu")
        out[rank] = (seeds, weak, strong, bench.shard_seeds(rank, 1, True))
    finally:
        dist.destroy_process_group()


def test_two_gloo_ranks_bench_sharding_and_max_over_ranks():
    """bench.py's N > 1 logic on CPU: disjoint seed shards (weak scaling), max-over-ranks time,
    summed work; a partitioned apply counts its replicated applies once."""
    import torch.multiprocessing as mp
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_bench_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    (s0, w0, p0, r0), (s1, w1, p1, r1) = out[0], out[1]
    assert sorted(s0 + s1) == list(range(128)) and not set(s0) & set(s1)
    assert w0 == w1 == (110.0, 2e12, 128.0)
    assert p0 == p1 == (110.0, 5e12, 1.0)
    assert r0 == r1 == [0]
