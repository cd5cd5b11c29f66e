"""Direct method (§III.C) — oracle cross-check for pin P10.

"the TTNO is fully contracted with the TTNS, and the two virtual legs between every two
nodes are combined into one larger leg.  Then the compression is performed ... truncated
SVDs for each leg encountered during the sweep", here "recursively from the root to the
leaves with the root as the orthogonality center":
  1. exact product N = O|psi> with fused bonds (oracle.ttn.exact_apply);
  2. QR every non-root node toward its parent (leaves to root) -> root is the centre;
  3. at the centre i, truncate every child bond by an SVD of i split on that leg; then
     for each child: move the centre to the child (QR), recurse, move it back (QR).
"""
from __future__ import annotations

import numpy as np

from .cbc import _keep, SV_FLOOR, qr_pos
from .ttn import TTN, exact_apply


def _split(t: np.ndarray, leg: int):
    """Matrix view of t with `leg` as the column index: returns (matrix, permuted shape)."""
    m = np.moveaxis(t, leg, -1)
    return m.reshape(-1, m.shape[-1]), m.shape


def _unsplit(mat: np.ndarray, shp, leg: int):
    return np.moveaxis(mat.reshape(shp[:-1] + (mat.shape[1],)), -1, leg)


def _absorb(t: np.ndarray, leg: int, r: np.ndarray) -> np.ndarray:
    """t[..., x(leg), ...] -> sum_x r[y, x] t[..., x, ...] (new extent y on `leg`)."""
    return np.moveaxis(np.tensordot(r, t, axes=([1], [leg])), 0, leg)


def direct_apply(op: TTN, psi: TTN, max_bond: int, tol: float = 0.0) -> TTN:
    net = exact_apply(op, psi)
    N = [t.copy() for t in net.tensors]
    ch, par = net.children, net.parent

    def to_parent(i):  # make node i isometric toward its parent
        p = par[i]
        m, shp = _split(N[i], 1)
        q, r = qr_pos(m)
        N[i] = _unsplit(q, shp, 1)
        N[p] = _absorb(N[p], 2 + ch[p].index(i), r)

    def to_child(i, c):  # make node i isometric toward child c
        leg = 2 + ch[i].index(c)
        m, shp = _split(N[i], leg)
        q, r = qr_pos(m)
        N[i] = _unsplit(q, shp, leg)
        N[c] = _absorb(N[c], 1, r)

    for i in net.post_order():
        if par[i] >= 0:
            to_parent(i)

    def trunc(i):
        for c in ch[i]:
            leg = 2 + ch[i].index(c)
            m, shp = _split(N[i], leg)
            u, s, vh = np.linalg.svd(m, full_matrices=False)
            k = _keep(s, max_bond, tol, SV_FLOOR)
            N[i] = _unsplit(u[:, :k] * s[None, :k], shp, leg)
            N[c] = _absorb(N[c], 1, vh[:k])
        for c in ch[i]:
            to_child(i, c)
            trunc(c)
            to_parent(c)

    trunc(net.root)
    return TTN(list(net.parent), [np.ascontiguousarray(t) for t in N], "state")
