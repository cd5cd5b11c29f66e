"""The paper's circuit experiment (§IV.B) as seeded inputs.

U_full = U U^dagger, U = prod_{i=1}^N U_i, each batch U_i a tree-like
circuit (Fig. 5, figure not in the container), every two-qubit gate G = CNOT (V1 x V2) with
Haar-random single-qubit V, every level of a batch one TTNO, start state
|0...0>, Err = || |psi0> - U_full |psi0> ||.  27 qubits, N = 3, three tree
structures: an MPS, a T3NS with MPS chains as subtrees (Fig. 6a) and a T3NS where
only leaves carry physical legs (Fig. 6b).

Readings (A25, the figures are missing):
  * batch: a ternary recursion over n = 3^L qubits.  Level l = 1..L groups the qubits into
    blocks of 3^l made of three sub-blocks; a block's representative is the representative of
    its middle sub-block (a 3-qubit block's is its middle qubit).  Each block chains its three
    sub-block representatives r0, r1, r2 with two gates, (r0, r1) in circuit level "a" and
    (r1, r2) in level "b".  Levels 1a, 1b, 2a, 2b, ..., La, Lb: 2L levels per batch, gates of a
    level have disjoint supports, and the 3^L - 1 gates of a batch form a spanning tree of
    the qubits (a tree-like circuit).  Control = the first qubit of the pair.
  * structures: "mps" = chain in qubit order; "t3ns_chains" = every 3-qubit block is a chain
    a - b - c attached to the tree at its middle qubit b, blocks joined by binary branching
    nodes without physical legs (d = 1), three sub-trees per level joined as
    B(x0, B'(x1, x2)); "t3ns_leaves" = the same binary branching pattern down to single
    qubits, qubits only at the leaves (every internal node d = 1).
  * level TTNO: each gate is split by an operator-Schmidt SVD (rank 2 for CNOT (V1 x V2)) and
    routed along the tree path between its qubits; path nodes carry identity on their
    physical leg times a delta between the two path edges.  Paths of one level never share an
    edge in these layouts (asserted), so every operator bond is 1 or the gate's rank.
  * U^dagger: the levels in reverse order with every gate conjugate-transposed.
Construction of inputs only: no CBC arithmetic here.
"""
from __future__ import annotations

import string
from typing import Dict, List, Sequence, Tuple

import numpy as np

from .circuit import haar_unitary
from .topology import children_of, validate_parent

CNOT = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=np.complex128)


def gate_cnot_v(v1: np.ndarray, v2: np.ndarray) -> np.ndarray:
    """G = CNOT (V1 x V2) on (control, target)."""
    return CNOT @ np.kron(v1, v2)


# ----------------------------------------------------------------------------- batch
def _rep(block_start: int, size: int) -> int:
    """Representative qubit of a block of `size` = 3^l qubits starting at block_start."""
    while size > 1:
        size //= 3
        block_start += size          # middle sub-block
    return block_start


def batch_levels_pairs(n_qubits: int) -> List[List[Tuple[int, int]]]:
    """Qubit pairs of the 2L levels of one batch (reading A25)."""
    L = int(round(np.log(n_qubits) / np.log(3)))
    if 3 ** L != n_qubits or L < 1:
        raise ValueError("tree-like batch needs 3^L qubits")
    levels = []
    for lev in range(1, L + 1):
        size, sub = 3 ** lev, 3 ** (lev - 1)
        a, b = [], []
        for s0 in range(0, n_qubits, size):
            r = [_rep(s0 + j * sub, sub) for j in range(3)]
            a.append((r[0], r[1]))
            b.append((r[1], r[2]))
        levels += [a, b]
    return levels


def circuit_gates(n_qubits: int, n_batches: int, seed: int):
    """Levels of U = U_N ... U_1 in application order: list of [(qa, qb, G 4x4)].  Haar V's
    drawn from default_rng([seed, batch]) in level / gate order, V1 then V2."""
    out = []
    pairs = batch_levels_pairs(n_qubits)
    for bi in range(n_batches):
        rng = np.random.default_rng([seed, bi])
        for lev in pairs:
            gl = []
            for qa, qb in lev:
                v1, v2 = haar_unitary(rng, 2), haar_unitary(rng, 2)
                gl.append((qa, qb, gate_cnot_v(v1, v2)))
            out.append(gl)
    return out


def full_circuit_levels(n_qubits: int, n_batches: int, seed: int):
    """U then U^dagger (levels reversed, gates conjugate-transposed): U_full = U^dagger U acts
    as the identity, the paper's check (U U^dagger and U^dagger U are both I)."""
    fwd = circuit_gates(n_qubits, n_batches, seed)
    back = [[(qa, qb, g.conj().T) for (qa, qb, g) in lev] for lev in reversed(fwd)]
    return fwd + back


# ----------------------------------------------------------------------------- structures
class Structure:
    def __init__(self, kind: str, parent: List[int], phys: List[int], qubit_node: List[int]):
        self.kind, self.parent, self.phys, self.qubit_node = kind, parent, phys, qubit_node

    @property
    def n(self):
        return len(self.parent)


def structure_for(kind: str, n_qubits: int) -> Structure:
    """Tree layouts of the circuit study (reading A25)."""
    L = int(round(np.log(n_qubits) / np.log(3)))
    if 3 ** L != n_qubits:
        raise ValueError("3^L qubits expected")
    if kind == "mps":
        return Structure(kind, [-1] + list(range(n_qubits - 1)), [2] * n_qubits, list(range(n_qubits)))
    parent: List[int] = []
    phys: List[int] = []
    qnode: Dict[int, int] = {}

    def new(p, d):
        parent.append(p)
        phys.append(d)
        return len(parent) - 1

    def block(p, start, size):
        """Subtree of the block [start, start + size) hanging below node p."""
        if kind == "t3ns_chains" and size == 3:      # chain a - b - c attached at b
            b = new(p, 2)
            qnode[start + 1] = b
            qnode[start] = new(b, 2)
            qnode[start + 2] = new(b, 2)
            return
        if size == 1:
            qnode[start] = new(p, 2)
            return
        sub = size // 3
        top = new(p, 1)                              # B(x0, B'(x1, x2))
        block(top, start, sub)
        mid = new(top, 1)
        block(mid, start + sub, sub)
        block(mid, start + 2 * sub, sub)

    if kind not in ("t3ns_chains", "t3ns_leaves"):
        raise ValueError(f"unknown structure {kind}")
    block(-1, 0, n_qubits)
    validate_parent(parent)
    return Structure(kind, parent, phys, [qnode[q] for q in range(n_qubits)])


# ----------------------------------------------------------------------------- level TTNO
def _path(parent: Sequence[int], a: int, b: int) -> List[int]:
    anc = []
    x = a
    while x != -1:
        anc.append(x)
        x = parent[x]
    pos = {v: i for i, v in enumerate(anc)}
    up_b = []
    y = b
    while y not in pos:
        up_b.append(y)
        y = parent[y]
    return anc[: pos[y] + 1] + up_b[::-1]


def level_operator(st: Structure, gates) -> Tuple[List[np.ndarray], List[int]]:
    """TTNO of one circuit level in the ABI leg order [d_out, d_in, b_parent, b_children...]
    (include/ttn_cbc.h); returns (tensors, bonds)."""
    parent, n = st.parent, st.n
    ch = children_of(parent)
    bond = [1] * n
    end: Dict[int, Tuple[np.ndarray, int]] = {}     # node -> (E[o, i, k], edge node) endpoint
    thru: Dict[int, List[Tuple[int, int]]] = {i: [] for i in range(n)}   # node -> [(edge1, edge2)]
    used_edges = set()
    for qa, qb, g in gates:
        na, nb = st.qubit_node[qa], st.qubit_node[qb]
        m = g.reshape(2, 2, 2, 2).transpose(0, 2, 1, 3).reshape(4, 4)   # [(oa, ia), (ob, ib)]
        u, s, vh = np.linalg.svd(m)
        r = int(np.sum(s > 1e-12 * s[0]))
        A = (u[:, :r] * np.sqrt(s[:r])[None, :]).reshape(2, 2, r)       # [oa, ia, k]
        B = (np.sqrt(s[:r])[:, None] * vh[:r]).reshape(r, 2, 2).transpose(1, 2, 0)   # [ob, ib, k]
        path = _path(parent, na, nb)
        # edge between consecutive path nodes, named by its child node
        edges = [(x if parent[x] == y else y) for x, y in zip(path[:-1], path[1:])]
        for e in edges:
            if e in used_edges:
                raise ValueError("two gates of one level share a tree edge")
            used_edges.add(e)
            bond[e] = r
        end[na] = (A, edges[0])
        end[nb] = (B, edges[-1])
        for j in range(1, len(path) - 1):
            thru[path[j]].append((edges[j - 1], edges[j]))
    ops = []
    letters = iter(string.ascii_letters)
    for i in range(n):
        d = st.phys[i]
        legs = ([i] if parent[i] >= 0 else [None]) + ch[i]        # edge of each virtual leg
        ext = [bond[e] if e is not None else 1 for e in legs]
        lab = [next(letters) for _ in legs]
        o, ii = "Y", "Z"
        terms, subs = [], []
        if i in end:
            E, e = end[i]
            terms.append(E)
            subs.append(o + ii + lab[legs.index(e)])
        else:
            terms.append(np.eye(d, dtype=np.complex128))
            subs.append(o + ii)
        for e1, e2 in thru[i]:
            r = bond[e1]
            terms.append(np.eye(r, dtype=np.complex128))
            subs.append(lab[legs.index(e1)] + lab[legs.index(e2)])
        covered = set("".join(subs))
        for l, x in zip(lab, ext):      # legs no path uses: extent 1
            if l not in covered:
                assert x == 1
                terms.append(np.ones(1, dtype=np.complex128))
                subs.append(l)
        t = np.einsum(",".join(subs) + "->" + o + ii + "".join(lab), *terms)
        ops.append(np.ascontiguousarray(t.reshape([d, d] + ext)))
        letters = iter(string.ascii_letters)
    return ops, bond


def zero_state(st: Structure) -> List[np.ndarray]:
    """|0...0> as a bond-1 TTNS in the ABI leg order."""
    ch = children_of(st.parent)
    out = []
    for i in range(st.n):
        t = np.zeros([st.phys[i], 1] + [1] * len(ch[i]), dtype=np.complex128)
        t.reshape(-1)[0] = 1.0
        out.append(t)
    return out
