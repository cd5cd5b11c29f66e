"""GPU edge cases of the CBC path vs the CPU oracle (same seeded inputs): single-node and
two-node trees, max_bond = 1, ragged per-edge bonds, a root that is not node 0, physical
dimension 1, and a batch whose instances have different bonds (cbc_apply_batch allows it)."""
import numpy as np
import pytest

import workloads as W
from oracle import TTN, cbc_apply as oracle_cbc, exact_apply, norm, to_dense_operator, to_dense_state
from workloads.configs import Instance
from workloads.generators import operator_shapes, random_tree_tensors, state_shapes

from ._helpers import distances, gpu_pair, oracle_pair, to_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_19650_b200 as P
    return P


@pytest.fixture(scope="module")
def ctx(P):
    c = P.Context(0)
    yield c
    c.close()


def ragged_instance(parent, phys, sbond, obond, max_bond, seed):
    rng = np.random.default_rng(seed)
    st = random_tree_tensors(rng, state_shapes(parent, phys, sbond))
    op = random_tree_tensors(rng, operator_shapes(parent, phys, obond))
    return Instance("ragged", list(parent), list(phys), list(sbond), list(obond), st, op, max_bond)


def run_and_check(P, ctx, inst, exact=False):
    op_g, st_g = gpu_pair(P, ctx, inst)
    out, rep = P.cbc_apply(ctx, op_g, st_g, inst.max_bond)
    phi_g = to_oracle(P, out, inst.parent)
    op_o, psi_o = oracle_pair(inst)
    phi_o = oracle_cbc(op_o, psi_o, inst.max_bond)
    assert phi_g.bonds() == phi_o.bonds()
    d_cos, d_rel = distances(phi_g, phi_o)
    assert d_cos <= 1e-10, (d_cos, d_rel)
    on2 = norm(exact_apply(op_o, psi_o)) ** 2
    assert abs(norm(phi_g) ** 2 - norm(phi_o) ** 2) <= 1e-10 * on2
    if exact:
        ex = to_dense_operator(op_o) @ to_dense_state(psi_o)
        assert np.linalg.norm(to_dense_state(phi_g) - ex) <= 1e-12 * np.linalg.norm(ex)
    return phi_g, rep


def test_single_node_tree(P, ctx):
    inst = ragged_instance([-1], [5], [1], [1], 4, seed=1)
    phi, rep = run_and_check(P, ctx, inst, exact=True)   # no bond to compress: phi = O psi
    assert phi.bonds() == [1]


def test_two_node_tree(P, ctx):
    for mb in (1, 2, 64):
        inst = ragged_instance([-1, 0], [3, 4], [1, 5], [1, 3], mb, seed=2)
        run_and_check(P, ctx, inst, exact=(mb == 64))


def test_max_bond_one(P, ctx):
    inst = W.configs.random_instance(W.complete_binary(7), [2] * 7, 3, 2, 1, seed=3)
    phi, rep = run_and_check(P, ctx, inst)
    assert phi.bonds() == [1] * 7


def test_ragged_bonds_and_root_in_the_middle(P, ctx):
    # chain 0-1-2-3-4-5 rooted at node 3 (parent array is not heap-ordered)
    parent = [1, 2, 3, -1, 3, 4]
    sb = [3, 5, 7, 1, 6, 2]
    ob = [2, 3, 2, 1, 4, 3]
    for mb in (64, 5):
        inst = ragged_instance(parent, [2, 3, 2, 2, 3, 2], sb, ob, mb, seed=4)
        run_and_check(P, ctx, inst, exact=(mb == 64))


def test_physical_dim_one_nodes(P, ctx):
    parent = W.complete_binary(7)
    inst = ragged_instance(parent, [1, 2, 1, 2, 2, 2, 2], [1, 4, 3, 2, 2, 3, 3], [1, 2, 3, 2, 2, 2, 2], 3, seed=5)
    run_and_check(P, ctx, inst)


def test_batch_with_different_bonds(P, ctx):
    parent = W.complete_binary(15)
    insts = [W.configs.random_instance(parent, [2] * 15, chi, D, 6, seed=10 + chi) for chi, D in ((3, 2), (5, 3), (4, 4))]
    pairs = [gpu_pair(P, ctx, i) for i in insts]
    outs, reps = P.cbc_apply_batch(ctx, [p[0] for p in pairs], [p[1] for p in pairs], 6)
    for inst, out, rep in zip(insts, outs, reps):
        phi_g = to_oracle(P, out, parent)
        op_o, psi_o = oracle_pair(inst)
        phi_o = oracle_cbc(op_o, psi_o, 6)
        assert phi_g.bonds() == phi_o.bonds()
        assert distances(phi_g, phi_o)[0] <= 1e-10
        assert abs(rep["norm"] - norm(phi_o)) <= 1e-10 * norm(phi_o)


def test_worker_subbatches_match_single_stream(P, ctx):
    """ttn_ctx_set_workers: concurrent sub-batches on internal streams give the same results."""
    parent = W.complete_binary(15)
    insts = [W.configs.random_instance(parent, [2] * 15, 4, 3, 6, seed=40 + s) for s in range(9)]
    pairs = [gpu_pair(P, ctx, i) for i in insts]
    ref, rref = P.cbc_apply_batch(ctx, [p[0] for p in pairs], [p[1] for p in pairs], 6)
    P.ttn_ctx_set_workers(ctx, 4)
    try:
        got, rgot = P.cbc_apply_batch(ctx, [p[0] for p in pairs], [p[1] for p in pairs], 6)
    finally:
        P.ttn_ctx_set_workers(ctx, 1)
    for a, b, ra, rb in zip(got, ref, rgot, rref):
        x, y = to_oracle(P, a, parent), to_oracle(P, b, parent)
        assert x.bonds() == y.bonds()
        # same arithmetic per instance: the tensors agree to rounding (the overlap-based
        # distance floors near 1e-8, reading A18, so compare entries)
        for tx, ty in zip(x.tensors, y.tensors):
            assert np.allclose(tx, ty, rtol=0, atol=1e-12 * max(1.0, np.abs(ty).max()))
        assert abs(ra["norm"] - rb["norm"]) <= 1e-12 * rb["norm"]


def test_get_data_batch_matches_per_tensor_reads(P, ctx):
    """ttn_get_data_batch (one synchronisation) returns what ttn_get_tensor returns node by
    node, and refuses a buffer that is too small."""
    parent = W.complete_binary(7)
    insts = [W.configs.random_instance(parent, [2] * 7, 3, 2, 4, seed=70 + s) for s in range(3)]
    outs = []
    for i in insts:
        op_g, st_g = gpu_pair(P, ctx, i)
        outs.append(P.cbc_apply(ctx, op_g, st_g, i.max_bond)[0])
    sizes = [sum(int(np.prod(o.shape(q))) for q in range(o.n_nodes)) for o in outs]
    bufs = [np.empty(sz, dtype=np.complex128) for sz in sizes]
    P.ttn_get_data_batch(ctx, outs, bufs)
    for o, b in zip(outs, bufs):
        ref = np.concatenate([P.ttn_get_tensor(ctx, o, q).ravel() for q in range(o.n_nodes)])
        assert np.array_equal(b, ref)
    with pytest.raises(P.TTNError):
        P.ttn_get_data_batch(ctx, outs, [np.empty(sizes[0] - 1, dtype=np.complex128)] + bufs[1:])


@pytest.mark.parametrize("chi,D,mb", [(25, 6, 32), (40, 5, 32), (33, 7, 32)])
def test_gram_orders_between_kernel_variants(P, ctx, chi, D, mb):
    """G-route Gram orders n = chi * D of 150, 200 and 231 at the depth-1 nodes of a 31-node
    binary tree (m = 2 * 32 * 32 rows): between and beyond the 128 / 192 / 256 instantiations
    of the tridiagonalisation, ragged against its row groups and its shared-memory tail;
    truncated, GPU vs oracle."""
    parent = W.complete_binary(31)
    inst = W.configs.random_instance(parent, [2] * 31, chi, D, mb, seed=11)
    run_and_check(P, ctx, inst)


def test_torch_caching_allocator_hook(P):
    """ttn_allocator wired to PyTorch's caching allocator (SURVEY §8(b) PyTorch interop): the
    library's workspaces and TTN handles come out of torch's pool (torch's allocated bytes grow
    while handles live and return when they are destroyed), and the results are unchanged."""
    import torch
    base = torch.cuda.memory_allocated(0)
    ctx = P.Context(0, allocator="torch")
    try:
        inst = W.make_config(3, seed=4)
        op_g, st_g = gpu_pair(P, ctx, inst)
        held = torch.cuda.memory_allocated(0) - base
        n_in = sum(t.size for t in inst.state) + sum(t.size for t in inst.op)
        assert held >= 16 * n_in
        out, rep = P.cbc_apply(ctx, op_g, st_g, inst.max_bond)
        phi_g = to_oracle(P, out, inst.parent)
        op_o, psi_o = oracle_pair(inst)
        phi_o = oracle_cbc(op_o, psi_o, inst.max_bond)
        assert distances(phi_g, phi_o)[0] <= 1e-10
        assert phi_g.bonds() == phi_o.bonds()
        for h in (out, op_g, st_g):
            h.destroy()
    finally:
        ctx.close()
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated(0) == base


def test_exact_factor_shortcut_and_its_fallback(P, ctx):
    """untruncated compresses (tol = 0, max_bond >= min(m, n)) of Grams too
    large for the one-launch Jacobi solver (order > 32) whose Gram is certified full rank take
    the Cholesky factor instead of the eigensolver (report exact_factors), and the result is
    still exact (dense O psi).  Leaf 1 has two equal bond columns, so its up-Gram (order 40)
    is singular: the certificate fails and that compress goes through the eigensolver (its
    factor rank drops to the numerical rank 39); leaf 2's up-Gram and both down-Grams (orders
    40 and 36) are certified."""
    parent = [-1, 0, 0]
    rng = np.random.default_rng(41)
    st = [W.complex_gaussian(rng, (4, 1, 40, 36)), W.complex_gaussian(rng, (64, 40)), W.complex_gaussian(rng, (48, 36))]
    st[1][:, 1] = st[1][:, 0]                         # rank-deficient up-Gram of leaf 1
    ops = [W.complex_gaussian(rng, (4, 4, 1, 1, 1)), W.complex_gaussian(rng, (64, 64, 1)),
           W.complex_gaussian(rng, (48, 48, 1))]
    inst = Instance("rankdef", parent, [4, 64, 48], [1, 40, 36], [1, 1, 1], st, ops, 64)
    phi_g, phi_o, rep, op_o, psi_o = _run_plain(P, ctx, inst)
    assert phi_g.bonds() == phi_o.bonds()
    ex = to_dense_operator(op_o) @ to_dense_state(psi_o)
    assert np.linalg.norm(to_dense_state(phi_g) - ex) <= 1e-12 * np.linalg.norm(ex)
    assert rep["exact_factors"] == 3, rep


def _run_plain(P, ctx, inst):
    op_g, st_g = gpu_pair(P, ctx, inst)
    out, rep = P.cbc_apply(ctx, op_g, st_g, inst.max_bond)
    op_o, psi_o = oracle_pair(inst)
    return to_oracle(P, out, inst.parent), oracle_cbc(op_o, psi_o, inst.max_bond), rep, op_o, psi_o
