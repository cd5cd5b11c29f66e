import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2601_19650_b200 as P
import workloads as W
for cfg in (3, 4):
    insts = [W.make_config(cfg, seed=s) for s in range(64 if cfg == 3 else 1)]
    ctx = P.Context(0)
    st = [P.ttn_create(ctx, P.TTN_STATE, i.parent, i.phys, i.state_bond, i.state) for i in insts]
    op = [P.ttn_create(ctx, P.TTN_OPERATOR, i.parent, i.phys, i.op_bond, i.op) for i in insts]
    torch.cuda.reset_peak_memory_stats()
    free0, tot = torch.cuda.mem_get_info()
    outs, reps = P.cbc_apply_batch(ctx, op, st, insts[0].max_bond)
    free1, _ = torch.cuda.mem_get_info()
    print("cfg", cfg, "peak_entries", reps[0]["peak_entries"], "MB", reps[0]["peak_entries"] * 16 / 1e6, "device mem used by ctx after apply (GB)", (free0 - free1) / 1e9)
    ctx.close()
