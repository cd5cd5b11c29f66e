"""The paper's random benchmark (§IV.A) as seeded inputs.

Both real and imaginary parts of every TTNO and TTNS entry are iid U[-0.5, 1].
Structures (d = 3 on every physical leg):
  mps     tensor train, 50 sites, D_S = D_O = 40, target bonds D-bar = 2, 4, ..., 40
  ttree   T-tree: a central node with three chains of L = 20 (61 nodes), D = 10,
          D-bar = 2..10; the centre is a virtual junction, d = 1 (SPEC S:253 reading)
  binary  perfectly balanced binary tree of depth L = 6 (127 nodes), physical legs on the
          leaves only (d = 1 on inner nodes), D = 10, D-bar = 2..10
  ftps    fork tensor product: L = 8 virtual backbone nodes (d = 1), each with a chain of
          8 physical nodes (72 nodes), D = 10, D-bar = 2..10
The root is node 0 (first site / centre / apex / first backbone node).
"""
from __future__ import annotations

import numpy as np

from .configs import Instance
from .generators import operator_shapes, state_shapes
from .topology import chain, children_of, complete_binary, ftps, t_tree

PAPER_RANDOM = {
    "mps": dict(D=40, dbar=list(range(2, 41, 2))),
    "ttree": dict(D=10, dbar=list(range(2, 11, 2))),
    "binary": dict(D=10, dbar=list(range(2, 11, 2))),
    "ftps": dict(D=10, dbar=list(range(2, 11, 2))),
}


def paper_topology(kind: str):
    if kind == "mps":
        parent = chain(50)
        phys = [3] * 50
    elif kind == "ttree":
        parent = t_tree(20)
        phys = [1] + [3] * (len(parent) - 1)
    elif kind == "binary":
        parent = complete_binary(2 ** 7 - 1)
        ch = children_of(parent)
        phys = [3 if not ch[i] else 1 for i in range(len(parent))]
    elif kind == "ftps":
        parent = ftps(8)
        ch = children_of(parent)
        # backbone nodes are the ones whose parent is a backbone node or -1 and that start a
        # chain: node ids 0, 9, 18, ... (ftps() lays out backbone node, then its chain)
        backbone = set(range(0, len(parent), 9))
        phys = [1 if i in backbone else 3 for i in range(len(parent))]
    else:
        raise KeyError(kind)
    return parent, phys


def paper_random_instance(kind: str, max_bond: int, seed: int = 0, D: int | None = None) -> Instance:
    parent, phys = paper_topology(kind)
    D = PAPER_RANDOM[kind]["D"] if D is None else D
    n = len(parent)
    sb = [1 if parent[i] < 0 else D for i in range(n)]
    rng = np.random.default_rng(seed)
    u = lambda shp: rng.uniform(-0.5, 1.0, size=shp) + 1j * rng.uniform(-0.5, 1.0, size=shp)  # noqa: E731
    st = [u(s) for s in state_shapes(parent, phys, sb)]
    op = [u(s) for s in operator_shapes(parent, phys, sb)]
    return Instance(f"paper-{kind}", parent, phys, sb, list(sb), st, op, max_bond, 0.0, seed)
