#!/usr/bin/env python
"""The paper's random benchmark (§IV.A, Fig. 4) on the GPU path:
for each structure and target bond dimension D-bar, the CBC runtime (CUDA events, median of
reps, inputs resident) and the relative error eps = ||phi - O psi|| / ||O psi|| =
sqrt(1 - ||phi||^2 / ||O psi||^2) (exact for CBC by the projection identity, A19), with
||O psi||^2 from ttn_op_norm2 -- no oracle and no dense vector involved.  Tool.

  python tools/paper_random.py [mps ttree binary ftps] > profiles/paper_random_r01.jsonl
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_19650_b200 as P  # noqa: E402
import workloads.paper as WP  # noqa: E402


def main():
    kinds = sys.argv[1:] or list(WP.PAPER_RANDOM)
    stream = torch.cuda.Stream(0)
    torch.cuda.set_stream(stream)
    ctx = P.Context(0, stream.cuda_stream)
    for kind in kinds:
        inst = WP.paper_random_instance(kind, 2, seed=0)
        st = P.ttn_create(ctx, P.TTN_STATE, inst.parent, inst.phys, inst.state_bond, inst.state)
        nrm = P.ttn_norm(ctx, st)
        tens = [t.copy() for t in inst.state]
        tens[0] = tens[0] / nrm
        st.destroy()
        st = P.ttn_create(ctx, P.TTN_STATE, inst.parent, inst.phys, inst.state_bond, tens)
        op = P.ttn_create(ctx, P.TTN_OPERATOR, inst.parent, inst.phys, inst.op_bond, inst.op)
        on2 = P.ttn_op_norm2(ctx, op, st)
        for dbar in WP.PAPER_RANDOM[kind]["dbar"]:
            out, rep = P.cbc_apply(ctx, op, st, dbar)   # warm-up
            out.destroy()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                out, rep = P.cbc_apply(ctx, op, st, dbar)
                e1.record(stream)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
                out.destroy()
            ts.sort()
            eps2 = max(1.0 - rep["norm"] ** 2 / on2, 0.0)
            print(json.dumps({"structure": kind, "nodes": len(inst.parent), "d": 3, "D": inst.state_bond[1],
                              "dbar": dbar, "ms_per_apply": ts[len(ts) // 2], "eps": eps2 ** 0.5,
                              "eps2": eps2, "max_bond": rep["max_bond"], "gflop": rep["flops_algorithmic"] / 1e9,
                              "device": torch.cuda.get_device_name(0)}), flush=True)
        st.destroy()
        op.destroy()
    ctx.close()


if __name__ == "__main__":
    main()
