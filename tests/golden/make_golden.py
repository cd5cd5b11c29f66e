#!/usr/bin/env python
"""Write oracle-derived golden values for the full-size configs (calls only oracle/ and
workloads/; never the CUDA path).

  python tests/golden/make_golden.py 4      -> tests/golden/cfg4_seed0.json (+ .npz if --tensors)

Stored: output bond dims, ||phi||^2, the per-compress discarded weights (in the oracle's
sweep order: up post-order, then down pre-order), and the truncation error inputs.  These are
the values of the oracle AS IT STANDS (§III.B, Eqs. 10-14; readings A1-A21 of
DESIGN.md §3); tests/test_gpu_parity.py compares the GPU against them.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import workloads as W  # noqa: E402


def main():
    cfg = int(sys.argv[1])
    seed = int(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("-") else 0
    inst = W.make_config(cfg, seed=seed)
    psi = O.TTN(inst.parent, [t.copy() for t in inst.state])
    nrm = O.norm(psi)
    psi.tensors[psi.root] = psi.tensors[psi.root] / nrm          # A16
    op = O.TTN(inst.parent, inst.op, "operator")
    rec = {}
    t0 = time.time()
    phi = O.cbc_apply(op, psi, inst.max_bond, record=rec)
    dt = time.time() - t0
    out = {"config": cfg, "seed": seed, "max_bond": inst.max_bond, "oracle_seconds": dt,
           "psi_norm_raw": nrm, "bonds": phi.bonds(), "phi_norm2": rec["norm"] ** 2,
           "discarded": [dict(kind=c["kind"], node=c["node"], k=c["k"], w=c["w"]) for c in rec["compress"]],
           "source": "tests/golden/make_golden.py (oracle/cbc.py as it stands)"}
    base = os.path.join(ROOT, "tests", "golden", f"cfg{cfg}_seed{seed}")
    json.dump(out, open(base + ".json", "w"), indent=1)
    if "--tensors" in sys.argv:
        np.savez(base + "_phi.npz", *phi.tensors)
    print(json.dumps({k: out[k] for k in ("oracle_seconds", "phi_norm2", "bonds")}))


if __name__ == "__main__":
    main()
