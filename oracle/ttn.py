"""TTN containers and exact contractions (oracle; test infrastructure only).

State node tensor  T^{[i]}[sigma, a_parent, a_c1, ...]          Eq. 2
Operator node      O^{[i]}[sigma', sigma, b_parent, b_c1, ...]   Eq. 4
Children in ascending node id; the root's parent leg has extent 1.
Dense ordering (A17): node id order, node 0 the most significant index.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence

import numpy as np


@dataclass
class TTN:
    parent: List[int]
    tensors: List[np.ndarray]
    kind: str = "state"  # "state" | "operator"

    def __post_init__(self):
        self.parent = [int(p) for p in self.parent]
        roots = [i for i, p in enumerate(self.parent) if p < 0]
        if len(roots) != 1:
            raise ValueError("topology mismatch: need exactly one root")
        self.root = roots[0]
        self.children = [[] for _ in self.parent]
        for i, p in enumerate(self.parent):
            if p >= 0:
                self.children[p].append(i)
        off = 1 if self.kind == "state" else 2
        for i, t in enumerate(self.tensors):
            if t.ndim != off + 1 + len(self.children[i]):
                raise ValueError(f"leg mismatch at node {i}")
            if i == self.root and t.shape[off] != 1:
                raise ValueError("root parent leg must have extent 1")
            for l, c in enumerate(self.children[i]):
                if self.tensors[c].shape[off] != t.shape[off + 1 + l]:
                    raise ValueError(f"leg mismatch on edge ({c},{i})")
        self.tensors = [np.asarray(t, dtype=np.complex128) for t in self.tensors]

    @property
    def n(self) -> int:
        return len(self.parent)

    def phys(self) -> List[int]:
        return [t.shape[0] for t in self.tensors]

    def bonds(self) -> List[int]:
        off = 1 if self.kind == "state" else 2
        return [t.shape[off] for t in self.tensors]

    def post_order(self) -> List[int]:
        out: List[int] = []

        def rec(i):
            for c in self.children[i]:
                rec(c)
            out.append(i)
        rec(self.root)
        return out

    def pre_order(self) -> List[int]:
        out: List[int] = []

        def rec(i):
            out.append(i)
            for c in self.children[i]:
                rec(c)
        rec(self.root)
        return out

    def copy(self) -> "TTN":
        return TTN(list(self.parent), [t.copy() for t in self.tensors], self.kind)


def _dense_generic(ttn: TTN, mats: Sequence[np.ndarray]) -> np.ndarray:
    """Contract site tensors mats[i][p, a_parent, a_c...] over all virtual legs.

    Returns an array with one axis per node in node-id order (extent mats[i].shape[0]).
    """
    def sub(i):
        cur = np.moveaxis(mats[i], 1, -1)          # [p_i, a_c1.., a_parent]
        nodes = [i]
        for c in ttn.children[i]:
            s, sn = sub(c)                          # [p(sn)..., a_c]
            k = len(nodes)                          # axis of this child's leg in cur
            cur = np.tensordot(cur, s, axes=([k], [s.ndim - 1]))
            # cur axes: [p(nodes)..., remaining child legs..., a_parent, p(sn)...]
            nrest = cur.ndim - k - len(sn)
            order = list(range(k)) + list(range(k + nrest, cur.ndim)) + list(range(k, k + nrest))
            cur = cur.transpose(order)
            nodes = nodes + sn
        return cur, nodes

    arr, nodes = sub(ttn.root)
    arr = arr[..., 0]                               # root parent leg, extent 1
    inv = np.argsort(nodes)
    return arr.transpose(inv)


def to_dense_state(psi: TTN) -> np.ndarray:
    """Eq. 2 as a dense vector."""
    assert psi.kind == "state"
    return _dense_generic(psi, psi.tensors).reshape(-1)


def to_dense_operator(op: TTN) -> np.ndarray:
    """Eq. 4 as a dense matrix; rows sigma', columns sigma."""
    assert op.kind == "operator"
    mats = [t.reshape((t.shape[0] * t.shape[1],) + t.shape[2:]) for t in op.tensors]
    arr = _dense_generic(op, mats)
    d = op.phys()
    arr = arr.reshape(sum(([di, di] for di in d), []))
    n = op.n
    arr = arr.transpose([2 * i for i in range(n)] + [2 * i + 1 for i in range(n)])
    D = int(np.prod(d))
    return arr.reshape(D, D)


def overlap(a: TTN, b: TTN) -> complex:
    """<a|b>, conjugate-linear in a, by a leaves-to-root environment sweep."""
    assert a.parent == b.parent
    env = {}
    for i in a.post_order():
        m = b.tensors[i]                            # [s, y0, y_c...]
        for c in a.children[i]:
            # contract the first remaining child leg (always axis 2) with E_c[x_c, y_c]
            m = np.tensordot(m, env[c], axes=([2], [1]))  # child leg replaced by x_c at the end
        ac = np.conj(a.tensors[i])                  # [s, x0, x_c...]
        nc = len(a.children[i])
        env[i] = np.tensordot(ac, m, axes=([0] + list(range(2, 2 + nc)), [0] + list(range(2, 2 + nc))))
    return complex(env[a.root][0, 0])


def norm(a: TTN) -> float:
    return float(np.sqrt(max(overlap(a, a).real, 0.0)))


def exact_apply(op: TTN, psi: TTN) -> TTN:
    """Uncompressed O|psi>: node tensors N[sigma', (a0 b0), (a_c b_c)...] (bond chi*D)."""
    out = []
    for i in range(psi.n):
        o, t = op.tensors[i], psi.tensors[i]
        nv = t.ndim - 1
        m = np.tensordot(o, t, axes=([1], [0]))     # [s', b0..b_{nv-1}, a0..a_{nv-1}]
        order = [0]
        for l in range(nv):
            order += [1 + nv + l, 1 + l]            # (a_l, b_l) with a major
        m = m.transpose(order)
        shp = (m.shape[0],) + tuple(m.shape[1 + 2 * l] * m.shape[2 + 2 * l] for l in range(nv))
        out.append(np.ascontiguousarray(m.reshape(shp)))
    return TTN(list(psi.parent), out, "state")


def sandwich(bra: TTN, op: TTN, ket: TTN) -> complex:
    """<bra| O |ket> (used for the projection identity P2)."""
    return overlap(bra, exact_apply(op, ket))
