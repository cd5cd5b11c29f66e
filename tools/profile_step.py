#!/usr/bin/env python
"""Exactly K steps of a bench config for ncu (no warm-up inside the profiled launches except
`--skip` untimed steps first): the launch list then holds K steps' kernels.  Tool.

  ncu ... python tools/profile_step.py --config 3 --steps 1 --skip 1 [--graphs]
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2601_19650_b200 as P  # noqa: E402
import workloads as W  # noqa: E402
from tests._helpers import gpu_pair  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--skip", type=int, default=1)
    ap.add_argument("--graphs", action="store_true")
    a = ap.parse_args()
    batch = {3: 64}.get(a.config, 1)
    insts = [W.make_config(a.config, seed=s) for s in range(batch)]
    stream = torch.cuda.Stream(0)
    torch.cuda.set_stream(stream)
    ctx = P.Context(0, stream.cuda_stream)
    P.ttn_ctx_set_schedule(ctx, True, a.graphs)
    pairs = [gpu_pair(P, ctx, i) for i in insts]
    ops, sts = [p[0] for p in pairs], [p[1] for p in pairs]
    mb = insts[0].max_bond
    for s in range(a.skip + a.steps):
        if s == a.skip:
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStart()
        outs, reps = P.cbc_apply_batch(ctx, ops, sts, mb)
        for h in outs:
            h.destroy()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("gemm flops/step algorithmic %.4e executed %.4e" % (sum(r["flops_gemm_min"] for r in reps),
                                                            sum(r["flops_gemm_exec"] for r in reps)))
    ctx.close()


if __name__ == "__main__":
    main()
