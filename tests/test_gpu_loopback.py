"""The partitioned multi-rank schedule (include/ttn_cbc.h) actually executed with
world = 2 and 3 ranks on ONE GPU through the in-process loopback communicator: every rank is a
context on its own stream driven by its own host thread, so the non-owner branches (receive
a broadcast factor, owner-rooted output broadcasts, cross-rank split-row all-reduces) run.
Every rank must return the plain apply's result; config 4 also against the oracle golden."""
import json
import os
import threading

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_19650_b200 as P
    return P


def _ranks(P, inst, world, parts, mb):
    import torch
    from ._helpers import gpu_pair
    grp = P.LoopbackGroup(world)
    streams = [torch.cuda.Stream(0) for _ in range(world)]
    ctxs = [P.Context(0, s.cuda_stream) for s in streams]
    try:
        for r, c in enumerate(ctxs):
            P.ttn_ctx_set_comm_loopback(c, grp, r, parts)
        pairs = [gpu_pair(P, c, inst) for c in ctxs]
        res, err = [None] * world, [None] * world

        def work(r):
            try:
                res[r] = P.cbc_apply(ctxs[r], pairs[r][0], pairs[r][1], mb)
            except Exception as e:   # surfaced below
                err[r] = e
        th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=600)
        assert not any(t.is_alive() for t in th), "loopback ranks did not finish"
        for e in err:
            if e is not None:
                raise e
        return [([h.get(i) for i in range(h.n_nodes)], rep) for h, rep in res]
    finally:
        for c in ctxs:
            c.close()
        grp.close()


def _plain(P, inst, mb):
    from ._helpers import gpu_pair
    ctx = P.Context(0)
    try:
        op, st = gpu_pair(P, ctx, inst)
        out, rep = P.cbc_apply(ctx, op, st, mb)
        return [out.get(i) for i in range(out.n_nodes)], rep
    finally:
        ctx.close()


@pytest.mark.parametrize("world,parts", [(2, 2), (2, 4), (3, 4)])
@pytest.mark.parametrize("tree,chi,D,mb", [("binary31", 4, 3, 6), ("binary63", 3, 2, 4)])
def test_loopback_ranks_match_plain_apply(P, world, parts, tree, chi, D, mb):
    from oracle import TTN
    from ._helpers import distances
    parent = W.complete_binary(31 if tree == "binary31" else 63)
    inst = W.configs.random_instance(parent, [2] * len(parent), chi, D, mb, seed=6)
    ref, rep0 = _plain(P, inst, mb)
    outs = _ranks(P, inst, world, parts, mb)
    b = TTN(parent, ref, "state")
    for r, (tens, rep) in enumerate(outs):
        a = TTN(parent, tens, "state")
        assert a.bonds() == b.bonds(), r
        assert distances(a, b)[0] <= 1e-14, r
        assert abs(rep["norm"] - rep0["norm"]) <= 1e-12 * rep0["norm"]
        assert abs(rep["discarded_weight_sum"] - rep0["discarded_weight_sum"]) <= 1e-12 * max(1.0, rep0["discarded_weight_sum"])
    for tens, _ in outs[1:]:   # every rank holds the same result
        assert all(np.array_equal(x, y) for x, y in zip(tens, outs[0][0]))


@pytest.mark.parametrize("parts", [2, 4])
def test_loopback_config4_two_ranks(P, parts):
    """BASELINE config 4 partitioned over 2 ranks (parts = 2: one junction subtree per rank;
    parts = 4: one chain pair per rank and the junction top's 16384 x 2048 Grams row-split
    across the ranks with a cross-rank all-reduce)."""
    from oracle import TTN, norm
    from ._helpers import distances
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cfg4_seed0.json")))
    inst = W.make_config(4, seed=0)
    outs = _ranks(P, inst, 2, parts, inst.max_bond)
    ref, rep0 = _plain(P, inst, inst.max_bond)
    b = TTN(inst.parent, ref, "state")
    for tens, rep in outs:
        a = TTN(inst.parent, tens, "state")
        assert a.bonds() == gold["bonds"]
        assert abs(norm(a) ** 2 - gold["phi_norm2"]) <= 1e-10 * gold["phi_norm2"]
        assert distances(a, b)[0] <= 1e-12
        assert (rep["split_compresses"] > 0) == (parts == 4)


@pytest.mark.parametrize("world,slices", [(2, 4), (3, 3)])
def test_loopback_row_splits_match_plain_apply(P, world, slices, monkeypatch):
    """TTN_PARTITION_SLICES forces the row splits on small trees: the replicated top's Grams
    (split_rows) and its final sweep (final_split: CholeskyQR2 and R from all-reduced partial
    sums, the new tensors scattered and all-reduced) over `world` ranks, several slices each."""
    from oracle import TTN
    from ._helpers import distances
    monkeypatch.setenv("TTN_PARTITION_SLICES", str(slices))
    parent = W.complete_binary(63)
    inst = W.configs.random_instance(parent, [2] * 63, 3, 2, 4, seed=8)
    ref, rep0 = _plain(P, inst, 4)
    outs = _ranks(P, inst, world, 4, 4)
    b = TTN(parent, ref, "state")
    for tens, rep in outs:
        a = TTN(parent, tens, "state")
        assert a.bonds() == b.bonds()
        assert distances(a, b)[0] <= 1e-14
        assert rep["split_compresses"] > 0
        assert abs(rep["norm"] - rep0["norm"]) <= 1e-12 * rep0["norm"]
