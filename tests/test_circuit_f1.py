"""Pins of the f1 circuit workload (§IV.B, reading A25)
and of the oracle on it: the level TTNOs equal the dense tensor product of their gates, the
gates are CNOT (V1 x V2) with unitary V, the batch is a tree-like circuit (its gates span a
tree on the qubits), and the oracle's CBC of U then U^dagger returns |0...0> (Err = 0 at
an exact bond dimension, the paper's oracle-free check)."""
import numpy as np
import pytest

import workloads.circuit_f1 as F
from oracle import TTN, cbc_apply, to_dense_operator, to_dense_state

from ._helpers import distances

KINDS = ["mps", "t3ns_chains", "t3ns_leaves"]


def _apply_gate_dense(psi, n, pa, pb, g):
    """|psi> (2^n, qubit 0 most significant) -> (G on qubits pa, pb) |psi>."""
    t = psi.reshape([2] * n)
    t = np.moveaxis(t, [pa, pb], [0, 1]).reshape(4, -1)
    t = (g @ t).reshape([2, 2] + [2] * (n - 2))
    return np.moveaxis(t, [0, 1], [pa, pb]).reshape(-1)


def _positions(st):
    """dense position of each qubit: qubit nodes in node-id order (d = 1 nodes add nothing)."""
    qn = sorted(range(len(st.qubit_node)), key=lambda q: st.qubit_node[q])
    pos = [0] * len(qn)
    for p, q in enumerate(qn):
        pos[q] = p
    return pos


def test_gate_form_and_tree_like_batch():
    rng = np.random.default_rng(1)
    from workloads.circuit import haar_unitary
    v1, v2 = haar_unitary(rng, 2), haar_unitary(rng, 2)
    g = F.gate_cnot_v(v1, v2)
    assert np.allclose(g.conj().T @ g, np.eye(4), atol=1e-14)
    assert np.allclose(F.gate_cnot_v(np.eye(2), np.eye(2)), F.CNOT)
    for n in (3, 9, 27):
        levels = F.batch_levels_pairs(n)
        edges = [e for lev in levels for e in lev]
        assert len(edges) == n - 1                       # spanning tree: n - 1 edges, connected
        par = list(range(n))

        def find(x):
            while par[x] != x:
                x = par[x]
            return x
        for a, b in edges:
            ra, rb = find(a), find(b)
            assert ra != rb                               # acyclic
            par[ra] = rb
        for lev in levels:                                # disjoint supports per level
            qs = [q for e in lev for q in e]
            assert len(qs) == len(set(qs))


@pytest.mark.parametrize("kind", KINDS)
def test_level_ttno_equals_dense_gates(kind):
    n = 9
    st = F.structure_for(kind, n)
    pos = _positions(st)
    levels = F.circuit_gates(n, 1, seed=3)
    for lev in levels:
        ops, bond = F.level_operator(st, lev)
        M = to_dense_operator(TTN(st.parent, ops, "operator"))
        ref = np.eye(2 ** n, dtype=complex)
        for qa, qb, g in lev:
            ref = np.stack([_apply_gate_dense(ref[:, j], n, pos[qa], pos[qb], g) for j in range(2 ** n)], axis=1)
        assert np.linalg.norm(M - ref) <= 1e-12 * np.linalg.norm(ref)
        assert max(bond) == 2                             # operator Schmidt rank of CNOT (V1 x V2)


@pytest.mark.parametrize("kind", KINDS)
def test_oracle_u_then_udagger_returns_zero_state(kind):
    """Exact bond dimension: U^dagger U |0> = |0> to rounding, so Err ~ 1e-15; and the state
    after U alone equals the dense state vector."""
    n = 9
    st = F.structure_for(kind, n)
    pos = _positions(st)
    levels = F.full_circuit_levels(n, 2, seed=4)
    psi = TTN(st.parent, F.zero_state(st))
    zero = psi.copy()
    dense = np.zeros(2 ** n, dtype=complex)
    dense[0] = 1.0
    for li, lev in enumerate(levels):
        ops, _ = F.level_operator(st, lev)
        psi = cbc_apply(TTN(st.parent, ops, "operator"), psi, 64)
        if li < len(levels) // 2:
            for qa, qb, g in lev:
                dense = _apply_gate_dense(dense, n, pos[qa], pos[qb], g)
        if li == len(levels) // 2 - 1:
            v = to_dense_state(psi)
            assert np.linalg.norm(v - dense) <= 1e-12
    d_cos, d_rel = distances(psi, zero)
    assert d_rel <= 1e-12, d_rel
