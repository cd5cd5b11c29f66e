"""Does running the config-3 batch as S concurrent sub-batches (S contexts / streams / host
threads) beat one level-synchronous batch?  Tool."""
import os, sys, threading, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_19650_b200 as P
import workloads as W

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
B = 64
insts = [W.make_config(cfg, seed=s) for s in range(B)]
mb = insts[0].max_bond
for S in (1, 2, 4):
    streams = [torch.cuda.Stream(0) for _ in range(S)]
    ctxs = [P.Context(0, st.cuda_stream) for st in streams]
    parts = [list(range(i * B // S, (i + 1) * B // S)) for i in range(S)]
    hs = []
    for c, idx in zip(ctxs, parts):
        st = [P.ttn_create(c, P.TTN_STATE, insts[i].parent, insts[i].phys, insts[i].state_bond, insts[i].state) for i in idx]
        op = [P.ttn_create(c, P.TTN_OPERATOR, insts[i].parent, insts[i].phys, insts[i].op_bond, insts[i].op) for i in idx]
        hs.append((st, op))
    def work(j):
        outs, _ = P.cbc_apply_batch(ctxs[j], hs[j][1], hs[j][0], mb)
        for o in outs:
            o.destroy()
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        th = [threading.Thread(target=work, args=(j,)) for j in range(S)]
        for t in th: t.start()
        for t in th: t.join()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"S={S}: {1e3*dt:.1f} ms per {B} applies -> {B/dt:.1f} applies/s", flush=True)
    for st, op in hs:
        for h in st + op: h.destroy()
    for c in ctxs: c.close()
