"""Speculative ranks and CUDA-graph replay (include/ttn_cbc.h
ttn_ctx_set_schedule): the speculative schedule and its graph replays give the same result as
the per-level synchronised schedule, bit for bit, and the oracle's within the parity bounds;
rank-deficient data falls back to the synchronised schedule with the right answer."""
import numpy as np
import pytest

import workloads as W
from oracle import TTN, cbc_apply as oracle_cbc

from ._helpers import distances, gpu_pair, oracle_pair, to_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_19650_b200 as P
    return P


def _tensors(P, h):
    return [h.get(i) for i in range(h.n_nodes)]


@pytest.mark.parametrize("cfg,mb", [(1, 6), (1, 12), (2, None), (3, None)])
def test_speculative_and_graph_equal_synchronised(P, cfg, mb):
    inst = W.make_config(cfg, seed=3)
    mb = mb or inst.max_bond
    ctx = P.Context(0)
    try:
        op_g, st_g = gpu_pair(P, ctx, inst)
        P.ttn_ctx_set_schedule(ctx, False, False)
        ref, rref = P.cbc_apply(ctx, op_g, st_g, mb)
        assert rref["host_syncs"] > 1
        P.ttn_ctx_set_schedule(ctx, True, True)
        # speculative, speculative + capture, replay, replay
        runs = [P.cbc_apply(ctx, op_g, st_g, mb) for _ in range(4)]
        want = _tensors(P, ref)
        for out, rep in runs:
            assert rep["host_syncs"] == 1, rep
            got = _tensors(P, out)
            assert all(np.array_equal(a, b) for a, b in zip(got, want))
            assert rep["norm"] == rref["norm"]
            assert abs(rep["discarded_weight_sum"] - rref["discarded_weight_sum"]) <= 1e-13 * max(1.0, rref["discarded_weight_sum"])
            assert rep["max_bond"] == rref["max_bond"] and rep["exact_factors"] == rref["exact_factors"]
        op_o, psi_o = oracle_pair(inst)
        phi_o = oracle_cbc(op_o, psi_o, mb)
        assert distances(to_oracle(P, runs[-1][0], inst.parent), phi_o)[0] <= 1e-10
    finally:
        ctx.close()


def test_graph_replay_tracks_new_inputs_and_batches(P):
    """Different handles (new addresses) get their own speculative run / capture; a batch is
    one graph; results match the synchronised schedule."""
    ctx = P.Context(0)
    try:
        insts = [W.make_config(3, seed=s) for s in (10, 11, 12)]
        pairs = [gpu_pair(P, ctx, i) for i in insts]
        for _ in range(3):
            outs, reps = P.cbc_apply_batch(ctx, [p[0] for p in pairs], [p[1] for p in pairs], 32)
        P.ttn_ctx_set_schedule(ctx, False, False)
        refs, _ = P.cbc_apply_batch(ctx, [p[0] for p in pairs], [p[1] for p in pairs], 32)
        for a, b in zip(outs, refs):
            assert all(np.array_equal(x, y) for x, y in zip(_tensors(P, a), _tensors(P, b)))
    finally:
        ctx.close()


def test_graph_keyed_on_shapes_replays_fresh_inputs(P):
    """The graph is keyed on shapes only: applies on fresh handles with new data (the
    end-to-end path) replay it after copying their inputs into the graph's buffers; every
    result equals the synchronised schedule's on the same input, bit for bit."""
    ctx = P.Context(0)
    try:
        insts = [W.make_config(3, seed=s) for s in (20, 21, 22, 20, 23)]
        got = []
        for inst in insts:   # speculative, speculative + capture, replay x3 (fresh handles each)
            op, st = gpu_pair(P, ctx, inst)
            out, rep = P.cbc_apply(ctx, op, st, inst.max_bond)
            assert rep["host_syncs"] == 1, rep
            got.append(_tensors(P, out))
        P.ttn_ctx_set_schedule(ctx, False, False)
        for inst, g in zip(insts, got):
            op, st = gpu_pair(P, ctx, inst)
            ref, _ = P.cbc_apply(ctx, op, st, inst.max_bond)
            assert all(np.array_equal(x, y) for x, y in zip(g, _tensors(P, ref)))
        assert all(np.array_equal(x, y) for x, y in zip(got[0], got[3]))   # same data, same result
    finally:
        ctx.close()


def test_rank_deficient_falls_back(P):
    """Circuit layers are rank deficient (exact zeros in the Gram spectra): the device check
    fails, the apply re-runs synchronised, and the result equals the oracle's."""
    ctx = P.Context(0)
    try:
        inst = W.make_config(5, seed=2)
        parent = inst.parent
        cur = P.ttn_create(ctx, P.TTN_STATE, parent, inst.phys, inst.state_bond, inst.state)
        ref = TTN(parent, [t.copy() for t in inst.state])
        for layer in range(4):
            o, ob, _ = W.circuit_layer_operator(parent, 2, layer)
            oh = P.ttn_create(ctx, P.TTN_OPERATOR, parent, [2] * 63, ob, o)
            cur, rep = P.cbc_apply(ctx, oh, cur, 256)
            ref = oracle_cbc(TTN(parent, o, "operator"), ref, 256)
            assert abs(rep["norm"] - 1.0) <= 1e-12
        g = to_oracle(P, cur, parent)
        assert g.bonds() == ref.bonds()
        assert distances(g, ref)[0] <= 1e-10
    finally:
        ctx.close()


def test_tolerance_uses_synchronised_ranks(P):
    inst = W.make_config(1, max_bond=12)
    ctx = P.Context(0)
    try:
        op_g, st_g = gpu_pair(P, ctx, inst)
        out, rep = P.cbc_apply(ctx, op_g, st_g, 12, 0.05)
        assert rep["host_syncs"] > 1
        op_o, psi_o = oracle_pair(inst)
        phi_o = oracle_cbc(op_o, psi_o, 12, 0.05)
        g = to_oracle(P, out, inst.parent)
        assert g.bonds() == phi_o.bonds() and distances(g, phi_o)[0] <= 1e-10
    finally:
        ctx.close()
