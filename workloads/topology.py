"""Rooted tree topologies as parent arrays (§II.A; ABI in include/ttn_cbc.h).

`parent[i]` is the parent of node i, exactly one entry is -1 (the root).  Children of a
node are ordered by ascending node id, which fixes the leg order of
every site tensor: state [d_i, a_parent, a_c1, a_c2, ...], operator
[d_i(out), d_i(in), b_parent, b_c1, ...].
"""
from __future__ import annotations

from typing import List, Sequence


def validate_parent(parent: Sequence[int]) -> int:
    """Return the root id; raise ValueError unless `parent` is a single rooted tree."""
    n = len(parent)
    roots = [i for i, p in enumerate(parent) if p == -1]
    if n == 0 or len(roots) != 1:
        raise ValueError("topology: need exactly one root")
    for i, p in enumerate(parent):
        if p != -1 and not (0 <= p < n) or p == i:
            raise ValueError("topology: bad parent index")
    for i in range(n):  # every node must reach the root without cycles
        seen, j = 0, i
        while parent[j] != -1:
            j = parent[j]
            seen += 1
            if seen > n:
                raise ValueError("topology: cycle")
    return roots[0]


def children_of(parent: Sequence[int]) -> List[List[int]]:
    ch: List[List[int]] = [[] for _ in parent]
    for i, p in enumerate(parent):
        if p >= 0:
            ch[p].append(i)
    return ch  # ascending ids by construction


def depth_of(parent: Sequence[int]) -> List[int]:
    d = []
    for i in range(len(parent)):
        k, j = 0, i
        while parent[j] != -1:
            j = parent[j]
            k += 1
        d.append(k)
    return d


def chain(n: int) -> List[int]:
    """MPS / tensor train rooted at site 0: parent[i] = i-1."""
    return [-1] + list(range(n - 1))


def complete_binary(n_nodes: int) -> List[int]:
    """Heap-ordered binary tree: node 0 root, children of i are 2i+1, 2i+2 (B:9, B:11)."""
    return [-1] + [(i - 1) // 2 for i in range(1, n_nodes)]


def star_of_chains_t3ns(chain_len: int = 16) -> List[int]:
    """Config-4 T3NS reading: root 0 -> two junctions -> two chains each.

    Node ids: root 0, then for each junction J: J, its first chain (chain_len nodes,
    top first), its second chain.  67 nodes for chain_len=16.
    """
    parent = [-1]
    for _ in range(2):
        j = len(parent)
        parent.append(0)
        for _c in range(2):
            top = len(parent)
            parent.append(j)
            for k in range(1, chain_len):
                parent.append(top + k - 1)
    return parent


def star_of_chains_literal(n_chains: int = 4, chain_len: int = 16) -> List[int]:
    """Literal B:10 star: a root with `n_chains` child chains (65 nodes for 4 x 16)."""
    parent = [-1]
    for _ in range(n_chains):
        top = len(parent)
        parent.append(0)
        for k in range(1, chain_len):
            parent.append(top + k - 1)
    return parent


def t_tree(chain_len: int) -> List[int]:
    """T-tree: a central root with three chains of `chain_len` nodes."""
    return star_of_chains_literal(3, chain_len)


def ftps(L: int) -> List[int]:
    """Fork tensor product structure: backbone of L nodes, each with an L-chain."""
    parent = []
    backbone = []
    for b in range(L):
        idx = len(parent)
        parent.append(-1 if b == 0 else backbone[-1])
        backbone.append(idx)
        for k in range(L):
            parent.append(idx if k == 0 else len(parent) - 1)
    return parent
