"""SURVEY §8(f) rows on the same GPU path:
 f1  the paper's circuit experiment structure: apply layers of 2-qubit gates and
     then their adjoints in reverse order; untruncated, the state must return to |0...0>
     (oracle-free: Err = ||psi_0 - U^dagger U psi_0|| -> 0), truncated Err > 0 and it matches
     the oracle run on the same layers;
 f4  the paper's positive-bias entry distribution U[-0.5, 1] vs the oracle.
"""
import numpy as np
import pytest

import workloads as W
from oracle import TTN, cbc_apply as oracle_cbc, norm, overlap
from workloads.configs import Instance
from workloads.generators import operator_shapes, product_zero_state, state_shapes

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


def adjoint_layer(ops):
    """O^dagger of a TTNO: conjugate every tensor and swap its (sigma', sigma) legs."""
    return [np.ascontiguousarray(np.conj(np.swapaxes(t, 0, 1))) for t in ops]


def run_layers(P, ctx, parent, layers, max_bond):
    n = len(parent)
    phys = [2] * n
    st = P.ttn_create(ctx, P.TTN_STATE, parent, phys, [1] * n, product_zero_state(parent, phys))
    for ops, bond in layers:
        op = P.ttn_create(ctx, P.TTN_OPERATOR, parent, phys, bond, ops)
        nxt, rep = P.cbc_apply(ctx, op, st, max_bond)
        st.destroy()
        op.destroy()
        st = nxt
    return to_oracle(P, st, parent)


def oracle_layers(parent, layers, max_bond):
    n = len(parent)
    psi = TTN(list(parent), product_zero_state(parent, [2] * n))
    for ops, bond in layers:
        psi = oracle_cbc(TTN(list(parent), ops, "operator"), psi, max_bond)
    return psi


@pytest.mark.parametrize("nq,nl", [(15, 4), (31, 3)])
def test_f1_circuit_then_inverse_returns_to_zero_state(P, ctx, nq, nl):
    parent = W.complete_binary(nq)
    fwd = []
    for layer in range(nl):
        ops, bond, _ = W.circuit_layer_operator(parent, 7, layer)
        fwd.append((ops, bond))
    layers = fwd + [(adjoint_layer(o), b) for o, b in reversed(fwd)]
    phi = run_layers(P, ctx, parent, layers, 256)
    psi0 = TTN(list(parent), product_zero_state(parent, [2] * nq))
    err = np.sqrt(max(norm(phi) ** 2 + 1.0 - 2.0 * overlap(psi0, phi).real, 0.0))
    assert abs(overlap(psi0, phi) - 1.0) <= 1e-12, overlap(psi0, phi)
    assert err <= 2e-7   # overlap-based distance floor (reading A18)


def test_f1_truncated_error_matches_oracle(P, ctx):
    parent = W.complete_binary(15)
    fwd = []
    for layer in range(4):
        ops, bond, _ = W.circuit_layer_operator(parent, 11, layer)
        fwd.append((ops, bond))
    layers = fwd + [(adjoint_layer(o), b) for o, b in reversed(fwd)]
    phi_g = run_layers(P, ctx, parent, layers, 4)
    phi_o = oracle_layers(parent, layers, 4)
    assert phi_g.bonds() == phi_o.bonds()
    assert distances(phi_g, phi_o)[0] <= 1e-10
    psi0 = TTN(list(parent), product_zero_state(parent, [2] * 15))
    err_g = 1.0 - overlap(psi0, phi_g).real
    err_o = 1.0 - overlap(psi0, phi_o).real
    assert err_g > 1e-6 and abs(err_g - err_o) <= 1e-10


def positive_bias_instance(parent, chi, D, max_bond, seed):
    rng = np.random.default_rng(seed)
    n = len(parent)
    phys = [2] * n
    sb = [1 if parent[i] < 0 else chi for i in range(n)]
    ob = [1 if parent[i] < 0 else D for i in range(n)]
    u = lambda shp: rng.uniform(-0.5, 1.0, size=shp) + 1j * rng.uniform(-0.5, 1.0, size=shp)  # noqa: E731
    st = [u(s) for s in state_shapes(parent, phys, sb)]
    op = [u(s) for s in operator_shapes(parent, phys, ob)]
    return Instance("posbias", list(parent), phys, sb, ob, st, op, max_bond)


@pytest.mark.parametrize("mb", [3, 8])
def test_f4_positive_bias_entries(P, ctx, mb):
    inst = positive_bias_instance(W.complete_binary(15), 4, 3, mb, seed=21)
    op_g, st_g = gpu_pair(P, ctx, inst)
    out, rep = P.cbc_apply(ctx, op_g, st_g, mb)
    phi_g = to_oracle(P, out, inst.parent)
    op_o, psi_o = oracle_pair(inst)
    phi_o = oracle_cbc(op_o, psi_o, mb)
    assert phi_g.bonds() == phi_o.bonds()
    assert distances(phi_g, phi_o)[0] <= 1e-10
    assert abs(norm(phi_g) - norm(phi_o)) <= 1e-10 * norm(phi_o)


@pytest.mark.parametrize("kind,mb", [("mps", 6), ("ttree", 4), ("binary", 4), ("ftps", 4)])
def test_f2_paper_random_structures_vs_oracle(P, ctx, kind, mb):
    """f2: the paper's random benchmark structures (U[-0.5, 1] entries, d = 3) at a
    small target bond, GPU vs oracle; eps^2 from ttn_op_norm2 vs the oracle's dense-free sweep."""
    import workloads.paper as WP
    from oracle import sandwich
    inst = WP.paper_random_instance(kind, mb, seed=1)
    op_g, st_g = gpu_pair(P, ctx, inst)
    out, rep = P.cbc_apply(ctx, op_g, st_g, mb)
    phi_g = to_oracle(P, out, inst.parent)
    op_o, psi_o = oracle_pair(inst)
    phi_o = oracle_cbc(op_o, psi_o, mb)
    assert phi_g.bonds() == phi_o.bonds()
    assert distances(phi_g, phi_o)[0] <= 1e-10
    assert abs(norm(phi_g) ** 2 - norm(phi_o) ** 2) <= 1e-10 * norm(phi_o) ** 2
    s = P.ttn_sandwich(ctx, out, op_g, st_g)                 # P2 on the GPU
    assert abs(s - rep["norm"] ** 2) <= 1e-11 * rep["norm"] ** 2


@pytest.mark.parametrize("kind", ["mps", "t3ns_chains", "t3ns_leaves"])
def test_f1_paper_circuit_matches_oracle_and_returns(P, ctx, kind):
    """f1 (§IV.B, reading A25): 27 qubits, N = 3 tree-like batches of
    CNOT (V1 x V2) gates, U then U^dagger, one TTNO per circuit level.  At D-bar = 10 (truncated)
    the GPU state after every level matches the oracle's (1 - cos <= 1e-10, same bonds) and
    both give the same Err; at D-bar = 200 the T3NS layouts return |0...0> to rounding (the
    paper's "converge to numerical error")."""
    import workloads.circuit_f1 as F
    from ._helpers import stable_distances
    st = F.structure_for(kind, 27)
    levels = F.full_circuit_levels(27, 3, seed=0)
    zero = TTN(st.parent, F.zero_state(st))
    for dbar in (10, 200):
        if dbar == 200 and kind == "mps":
            continue
        cur = P.ttn_create(ctx, P.TTN_STATE, st.parent, st.phys, [1] * st.n, F.zero_state(st))
        ref = zero.copy()
        for li, lev in enumerate(levels):
            o, b = F.level_operator(st, lev)
            oh = P.ttn_create(ctx, P.TTN_OPERATOR, st.parent, st.phys, b, o)
            cur, rep = P.cbc_apply(ctx, oh, cur, dbar)
            if dbar == 10:
                ref = oracle_cbc(TTN(st.parent, o, "operator"), ref, dbar)
                if li % 6 == 5 or li == len(levels) - 1:
                    g = to_oracle(P, cur, st.parent)
                    assert g.bonds() == ref.bonds(), (li, g.bonds(), ref.bonds())
                    assert stable_distances(g, ref)[0] <= 1e-10, li
        g = to_oracle(P, cur, st.parent)
        err = stable_distances(g, zero)[1]
        if dbar == 10:
            assert abs(err - stable_distances(ref, zero)[1]) <= 1e-8
            assert err > 1e-6                     # D-bar = 10 truncates
        else:
            assert err <= 1e-10, err
