import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, workloads as W, paper_2601_19650_b200 as P
from oracle import TTN, cbc_apply, norm, overlap
from tests._helpers import distances
ctx = P.Context(0)
for d in (8, 64):
    parent = [-1, 0, 0]; rng = np.random.default_rng(5); eye = np.eye(d, dtype=complex)
    root = W.complex_gaussian(rng, (2, 1, d, d)); ops = W.identity_operator(parent, [2, d, d])
    for pert in (0.0, 1e-3):
        leaf = eye + pert * W.complex_gaussian(rng, (d, d))
        st = [root, leaf, leaf]
        psi = TTN(parent, st); op = TTN(parent, ops, "operator")
        hs = P.ttn_create(ctx, P.TTN_STATE, parent, [2, d, d], [1, d, d], st)
        ho = P.ttn_create(ctx, P.TTN_OPERATOR, parent, [2, d, d], [1, 1, 1], ops)
        out, rep = P.cbc_apply(ctx, ho, hs, d)
        g = TTN(parent, out.tensors())
        o = cbc_apply(op, psi, d)
        print(d, pert, "gpu vs psi", distances(g, psi), "oracle vs psi", distances(o, psi), g.bonds(), rep["norm"], norm(psi))
        for i in (1, 2):
            q = g.tensors[i].reshape(d, -1)
            print("   leaf", i, "isometry err", np.linalg.norm(q.conj().T @ q - np.eye(q.shape[1])))
