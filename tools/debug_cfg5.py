"""Debug helper: run config 5 layer by layer through the C ABI and report the first non-finite layer."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
import paper_2601_19650_b200 as P
seeds = [int(x) for x in sys.argv[1:]] or [0, 1, 2]
ctx = P.Context(0)
insts = [W.make_config(5, seed=s) for s in seeds]
parent = insts[0].parent
cur = [P.ttn_create(ctx, P.TTN_STATE, parent, i.phys, i.state_bond, i.state) for i in insts]
for layer in range(10):
    ops = []
    for s in seeds:
        o, ob, _ = W.circuit_layer_operator(parent, s, layer)
        ops.append(P.ttn_create(ctx, P.TTN_OPERATOR, parent, [2] * 63, ob, o))
    try:
        cur, reps = P.cbc_apply_batch(ctx, ops, cur, 256)
    except Exception as e:
        print("layer", layer, "FAILED:", e); break
    print("layer", layer, [round(r["norm"], 14) for r in reps], [r["max_bond"] for r in reps], [r["rank_fallbacks"] for r in reps])
    bad = []
    for b, h in enumerate(cur):
        for i in range(63):
            t = h.get(i)
            if not np.all(np.isfinite(t)):
                bad.append((b, i, t.shape))
    if bad:
        print("  non-finite tensors after layer", layer, bad[:10])
        break
