#!/usr/bin/env python
"""The paper's circuit experiment on the GPU path (§IV.B; SURVEY §8 f1;
reading A25 in DESIGN.md): 27 qubits, N = 3 tree-like batches, U then U^dagger as one TTNO per
circuit level (36 applies), five seeds applied as one cbc_apply_batch per level, for the three
layouts (MPS, T3NS with MPS chains, T3NS with physical legs on the leaves only) and
D-bar = 10 .. 200.  Per point: Err = || |psi0> - U_full |psi0> || (computed from the
returned tensors by the QR-canonicalised difference of tests/_helpers, A18), the device time
of the 36 level applies (CUDA events, operators resident), and the maximum number of TTNS
entries during the run.  Tool.

  python tools/f1_circuit.py [--dbar 10,20,...] [--kinds mps,...] > profiles/f1_circuit_r02.jsonl
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2601_19650_b200 as P  # noqa: E402
import workloads.circuit_f1 as F  # noqa: E402
from oracle import TTN  # noqa: E402  (Err evaluation only, A18)
from tests._helpers import stable_distances  # noqa: E402


def run(ctx, stream, st, levels_ops, dbar, seeds):
    n = st.n
    cur = [P.ttn_create(ctx, P.TTN_STATE, st.parent, st.phys, [1] * n, F.zero_state(st)) for _ in seeds]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    peak = [0] * len(seeds)
    reps = None
    for ops in levels_ops:
        nxt, reps = P.cbc_apply_batch(ctx, ops, cur, dbar)
        for j, h in enumerate(nxt):
            peak[j] = max(peak[j], sum(int(np.prod(h.shape(i))) for i in range(n)))
        for h in cur:
            h.destroy()
        cur = nxt
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    zero = TTN(st.parent, F.zero_state(st))
    zh = P.ttn_create(ctx, P.TTN_STATE, st.parent, st.phys, [1] * n, F.zero_state(st))
    errs, how = [], []
    for h, rep in zip(cur, reps):
        b = h.bonds()
        big = max(b) > 128 and st.kind != "mps"
        if not big:   # stable: QR-canonicalised difference (A18)
            phi = TTN(st.parent, h.tensors())
            errs.append(stable_distances(phi, zero)[1])   # ||phi - psi0||, ||psi0|| = 1
            how.append("qr")
        else:         # large branching bonds: overlap form (floor ~1e-8)
            a = P.ttn_overlap(ctx, zh, h)
            e2 = 1.0 + rep["norm"] ** 2 - 2.0 * a.real
            errs.append(max(e2, 0.0) ** 0.5)
            how.append("overlap")
        h.destroy()
    zh.destroy()
    return ms, errs, peak, how


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dbar", default="10,20,30,40,50,75,100,150,200")
    ap.add_argument("--kinds", default="mps,t3ns_chains,t3ns_leaves")
    ap.add_argument("--seeds", type=int, default=5)
    ap.add_argument("--qubits", type=int, default=27)
    ap.add_argument("--batches", type=int, default=3)
    a = ap.parse_args()
    stream = torch.cuda.Stream(0)
    torch.cuda.set_stream(stream)
    ctx = P.Context(0, stream.cuda_stream)
    seeds = list(range(a.seeds))
    for kind in a.kinds.split(","):
        st = F.structure_for(kind, a.qubits)
        per_seed = [F.full_circuit_levels(a.qubits, a.batches, s) for s in seeds]
        levels_ops = []
        for li in range(len(per_seed[0])):
            ops = []
            for s in range(len(seeds)):
                o, b = F.level_operator(st, per_seed[s][li])
                ops.append(P.ttn_create(ctx, P.TTN_OPERATOR, st.parent, st.phys, b, o))
            levels_ops.append(ops)
        run(ctx, stream, st, levels_ops, 10, seeds)      # warm-up (plans, pools)
        for dbar in [int(x) for x in a.dbar.split(",")]:
            ms, errs, peak, how = run(ctx, stream, st, levels_ops, dbar, seeds)
            print(json.dumps({"structure": kind, "nodes": st.n, "qubits": a.qubits, "batches": a.batches,
                              "levels": len(levels_ops), "dbar": dbar, "seeds": len(seeds),
                              "err_mean": float(np.mean(errs)), "err_per_seed": errs,
                              "ms_per_circuit": ms / len(seeds), "ms_all_seeds": ms,
                              "max_entries_mean": float(np.mean(peak)), "max_entries": peak, "err_method": how,
                              "device": torch.cuda.get_device_name(0)}), flush=True)
        for ops in levels_ops:
            for h in ops:
                h.destroy()
    ctx.close()


if __name__ == "__main__":
    main()
