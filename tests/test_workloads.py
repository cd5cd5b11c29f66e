"""Seeded input generators (workloads/): determinism, shapes, topology readings."""
import numpy as np
import pytest

import workloads as W


def test_configs_shapes_and_determinism():
    a = W.make_config(3, seed=5)
    b = W.make_config(3, seed=5)
    c = W.make_config(3, seed=6)
    assert len(a.parent) == 31 and a.parent == W.complete_binary(31)
    assert all(np.array_equal(x, y) for x, y in zip(a.state, b.state))
    assert not np.array_equal(a.state[0], c.state[0])
    assert a.state[0].shape == (2, 1, 32, 32) and a.op[0].shape == (2, 2, 1, 6, 6)
    assert a.state[30].shape == (2, 32) and a.op[30].shape == (2, 2, 6)


def test_config2_chain_and_config1():
    c2 = W.make_config(2)
    assert c2.parent == [-1] + list(range(31))
    assert c2.state[0].shape == (2, 1, 64) and c2.state[31].shape == (2, 64)
    assert c2.op[5].shape == (2, 2, 8, 8)
    c1 = W.make_config(1)
    assert c1.max_bond == 12 and W.make_config(1, max_bond=6).max_bond == 6


def test_config4_t3ns_reading():
    c4 = W.make_config(4)
    assert len(c4.parent) == 67
    ch = W.children_of(c4.parent)
    assert ch[0] == [1, 34]
    assert [c4.phys[j] for j in (1, 34)] == [1, 1]
    assert all(len(x) <= 2 for x in ch)
    assert max(W.depth_of(c4.parent)) == 17


def test_config5_circuit_layers():
    c5 = W.make_config(5, seed=0)
    assert all(t.shape == (2, 1) + (1,) * (t.ndim - 2) for t in c5.state)
    for layer in range(10):
        ops, bond, gates = W.circuit_layer_operator(c5.parent, 0, layer)
        used = [x for (cc, p, g) in gates for x in (cc, p)]
        assert len(used) == len(set(used))                 # disjoint supports
        assert 15 <= len(gates) <= 31
        assert all(bond[cc] == 4 for cc, _, _ in gates)


def test_topology_validation():
    with pytest.raises(ValueError):
        W.validate_parent([-1, -1])
    with pytest.raises(ValueError):
        W.validate_parent([1, 0])
    assert W.validate_parent(W.ftps(3)) == 0
    assert len(W.ftps(8)) == 72 and len(W.t_tree(20)) == 61
