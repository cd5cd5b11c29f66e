"""BASELINE.json configs (B:7-11) as seeded synthetic instances (readings: DESIGN.md §3).

cfg1  chain N=6, d=2, chi=4, D=3, max_bond 12 (exact) or 6                      (B:7)
cfg2  chain N=32, d=2, chi=64, D=8, max_bond 64                                 (B:8)
cfg3  complete binary 31 nodes, d=2 on every node, chi=32, D=6, max_bond 32     (B:9, A13)
cfg4  star-of-chains read as a 67-node T3NS: root d=2, junctions d=1,
      4 chains x 16 nodes d=2, chi=128, D=16, max_bond 128                      (B:10, A12)
cfg5  binary 63 qubits from |0...0>, 10 circuit layers, max_bond 256            (B:11, A15)
All entries complex128 (N(0,1)+iN(0,1))/sqrt(2); the state is NOT normalised here (A16).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import topology as topo
from .circuit import circuit_layer_operator
from .generators import operator_shapes, product_zero_state, random_tree_tensors, state_shapes


@dataclass
class Instance:
    name: str
    parent: List[int]
    phys: List[int]
    state_bond: List[int]
    op_bond: List[int]
    state: List[np.ndarray]
    op: List[np.ndarray]
    max_bond: int
    tol: float = 0.0
    seed: int = 0
    layers: int = 1
    extra: dict = field(default_factory=dict)


CONFIGS = {
    1: dict(kind="chain", n=6, d=2, chi=4, D=3, max_bond=12),
    2: dict(kind="chain", n=32, d=2, chi=64, D=8, max_bond=64),
    3: dict(kind="binary", n=31, d=2, chi=32, D=6, max_bond=32, batch=64),
    4: dict(kind="t3ns", n=67, d=2, chi=128, D=16, max_bond=128),
    5: dict(kind="circuit", n=63, d=2, chi=256, max_bond=256, layers=10, batch=64),
}


def _random_instance(name, parent, phys, chi, D, max_bond, seed, tol=0.0):
    n = len(parent)
    sb = [1 if parent[i] < 0 else chi for i in range(n)]
    ob = [1 if parent[i] < 0 else D for i in range(n)]
    rng = np.random.default_rng(seed)
    st = random_tree_tensors(rng, state_shapes(parent, phys, sb))
    op = random_tree_tensors(rng, operator_shapes(parent, phys, ob))
    return Instance(name, list(parent), list(phys), sb, ob, st, op, max_bond, tol, seed)


def random_instance(parent, phys, chi, D, max_bond, seed=0, tol=0.0, name="custom"):
    return _random_instance(name, parent, phys, chi, D, max_bond, seed, tol)


def make_config(k: int, seed: int = 0, max_bond: Optional[int] = None, layer: int = 0) -> Instance:
    c = CONFIGS[k]
    mb = c["max_bond"] if max_bond is None else max_bond
    if c["kind"] == "chain":
        parent = topo.chain(c["n"])
        return _random_instance(f"cfg{k}", parent, [c["d"]] * c["n"], c["chi"], c["D"], mb, seed)
    if c["kind"] == "binary":
        parent = topo.complete_binary(c["n"])
        return _random_instance(f"cfg{k}", parent, [c["d"]] * c["n"], c["chi"], c["D"], mb, seed)
    if c["kind"] == "t3ns":
        parent = topo.star_of_chains_t3ns(16)
        ch = topo.children_of(parent)
        phys = [1 if (parent[i] == 0) else 2 for i in range(len(parent))]  # junctions d=1
        assert all(len(ch[j]) == 2 for j in range(len(parent)) if phys[j] == 1)
        return _random_instance(f"cfg{k}", parent, phys, c["chi"], c["D"], mb, seed)
    if c["kind"] == "circuit":
        parent = topo.complete_binary(c["n"])
        phys = [2] * c["n"]
        st = product_zero_state(parent, phys)
        op, ob, gates = circuit_layer_operator(parent, seed, layer)
        inst = Instance(f"cfg{k}", parent, phys, [1] * c["n"], ob, st, op, mb, 0.0, seed, c["layers"])
        inst.extra["gates"] = gates
        return inst
    raise KeyError(k)
