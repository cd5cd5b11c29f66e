"""Config-5 circuit layers as TTNOs (B:11; reading A15 in DESIGN.md).

One layer: rng = numpy.random.default_rng([seed, layer]); the tree edges (identified by
their child id 1..n-1) are shuffled with rng.permutation; an edge is kept when neither
endpoint is already used (a greedy maximal matching, so the gates of one layer have
disjoint supports).  For every kept edge, in kept order, a Haar-random 4x4 unitary is
drawn (QR of a complex Ginibre matrix with the diagonal-phase fix), qubit order
(child, parent): G[(o_c, o_p), (i_c, i_p)].  The gate is split across its edge by an
SVD of M[(o_c, i_c), (o_p, i_p)] = U S V^H: the child's operator tensor is U sqrt(S) on
its parent leg and the parent's is sqrt(S) V^H on that child's leg (bond 4).  Every
other operator tensor is I_2 with bond 1.  This is input construction (the paper's own
TTNO construction, ref. Cakir2025 at P:334, is out of scope).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

from .generators import complex_gaussian, operator_shapes
from .topology import children_of, validate_parent


def haar_unitary(rng: np.random.Generator, n: int) -> np.ndarray:
    z = complex_gaussian(rng, (n, n))
    q, r = np.linalg.qr(z)
    ph = np.diag(r) / np.abs(np.diag(r))
    return q * ph[None, :]


def layer_matching(parent: Sequence[int], seed: int, layer: int) -> Tuple[np.random.Generator, List[int]]:
    rng = np.random.default_rng([seed, layer])
    edges = np.array([i for i in range(len(parent)) if parent[i] >= 0], dtype=np.int64)
    perm = rng.permutation(edges)
    used = set()
    kept = []
    for c in perm.tolist():
        p = parent[c]
        if c in used or p in used:
            continue
        used.add(c)
        used.add(p)
        kept.append(c)
    return rng, kept


def circuit_layer_operator(parent: Sequence[int], seed: int, layer: int, d: int = 2):
    """Return (op_tensors, op_bonds, gates) for one layer; gates = [(child, parent, G 4x4)]."""
    validate_parent(parent)
    assert d == 2
    n = len(parent)
    ch = children_of(parent)
    rng, kept = layer_matching(parent, seed, layer)
    bond = [1] * n
    gates = []
    for c in kept:
        gates.append((c, parent[c], haar_unitary(rng, 4)))
        bond[c] = 4
    shapes = operator_shapes(parent, [d] * n, bond)
    ops = []
    for i in range(n):
        t = np.zeros(shapes[i], dtype=np.complex128)
        for k in range(d):
            t[(k, k) + (0,) * (len(shapes[i]) - 2)] = 1.0
        ops.append(t)
    for c, p, g in gates:
        m = g.reshape(2, 2, 2, 2).transpose(0, 2, 1, 3).reshape(4, 4)
        u, s, vh = np.linalg.svd(m)
        a = (u * np.sqrt(s)[None, :]).reshape(2, 2, 4)        # [o_c, i_c, bond]
        b = (np.sqrt(s)[:, None] * vh).reshape(4, 2, 2)       # [bond, o_p, i_p]
        tc = np.zeros(shapes[c], dtype=np.complex128)
        tc[(slice(None), slice(None), slice(None)) + (0,) * (len(shapes[c]) - 3)] = a
        ops[c] = tc
        slot = 3 + ch[p].index(c)                             # leg index of child c in p's tensor
        tp = np.zeros(shapes[p], dtype=np.complex128)
        idx = [slice(None), slice(None)] + [0] * (len(shapes[p]) - 2)
        idx[slot] = slice(None)
        tp[tuple(idx)] = b.transpose(1, 2, 0)                 # [o_p, i_p, bond]
        ops[p] = tp
    return ops, bond, gates
