"""Seeded random TTNS/TTNO site tensors in the ABI leg order (B:7-10).

Shapes follow PAPER.md Eq. 2 and Eq. 4 with the leg convention of
P:66 (the parent leg first, extent 1 at the root):
  state node i    : [d_i, a_parent, a_c1, a_c2, ...]
  operator node i : [d_i (out, sigma'), d_i (in, sigma), b_parent, b_c1, ...]
Children are in ascending node id.  `bond[i]` is the extent of the edge (i, parent[i]);
it is ignored (treated as 1) for the root.

Draw order: rng = numpy.random.default_rng(seed); state
tensors for node 0..n-1 (each: re = standard_normal(shape), im = standard_normal(shape),
value = (re + i im)/sqrt(2)), then operator tensors for node 0..n-1.
No normalisation is applied here: each side normalises the state with its own norm
routine (A16), so no method arithmetic lives in this module.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

from .topology import children_of, validate_parent


def state_shapes(parent: Sequence[int], phys: Sequence[int], bond: Sequence[int]) -> List[Tuple[int, ...]]:
    validate_parent(parent)
    ch = children_of(parent)
    out = []
    for i in range(len(parent)):
        a0 = 1 if parent[i] < 0 else int(bond[i])
        out.append((int(phys[i]), a0) + tuple(int(bond[c]) for c in ch[i]))
    return out


def operator_shapes(parent: Sequence[int], phys: Sequence[int], bond: Sequence[int]) -> List[Tuple[int, ...]]:
    validate_parent(parent)
    ch = children_of(parent)
    out = []
    for i in range(len(parent)):
        b0 = 1 if parent[i] < 0 else int(bond[i])
        out.append((int(phys[i]), int(phys[i]), b0) + tuple(int(bond[c]) for c in ch[i]))
    return out


def complex_gaussian(rng: np.random.Generator, shape) -> np.ndarray:
    re = rng.standard_normal(shape)
    im = rng.standard_normal(shape)
    return (re + 1j * im) / np.sqrt(2.0)


def random_tree_tensors(rng: np.random.Generator, shapes: Sequence[Tuple[int, ...]]) -> List[np.ndarray]:
    return [np.ascontiguousarray(complex_gaussian(rng, s), dtype=np.complex128) for s in shapes]


def identity_operator(parent: Sequence[int], phys: Sequence[int]) -> List[np.ndarray]:
    """Identity TTNO with every operator bond 1."""
    shapes = operator_shapes(parent, phys, [1] * len(parent))
    out = []
    for s in shapes:
        t = np.zeros(s, dtype=np.complex128)
        d = s[0]
        for k in range(d):
            t[(k, k) + (0,) * (len(s) - 2)] = 1.0
        out.append(t)
    return out


def product_zero_state(parent: Sequence[int], phys: Sequence[int]) -> List[np.ndarray]:
    """|0...0> with every bond 1 (B:11)."""
    shapes = state_shapes(parent, phys, [1] * len(parent))
    out = []
    for s in shapes:
        t = np.zeros(s, dtype=np.complex128)
        t[(0,) * len(s)] = 1.0
        out.append(t)
    return out
