"""Phase timing of bench.py's e2e path (host wall clock with syncs between phases). Tool."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_19650_b200 as P
import workloads as W

insts = [W.make_config(3, seed=s) for s in range(64)]
stream = torch.cuda.Stream(0)
torch.cuda.set_stream(stream)
ctx = P.Context(0, stream.cuda_stream)
def packed(tensors):
    flat = torch.from_numpy(np.concatenate([np.ascontiguousarray(t).ravel() for t in tensors])).pin_memory()
    views, off = [], 0
    for t in tensors:
        views.append(flat[off:off + t.size]); off += t.size
    return views
hs = [packed(i.state) for i in insts]
ho = [packed(i.op) for i in insts]
parent, phys, mb = insts[0].parent, insts[0].phys, 32
for rep in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    st = [P.ttn_create(ctx, P.TTN_STATE, parent, phys, i.state_bond, ts) for i, ts in zip(insts, hs)]
    op = [P.ttn_create(ctx, P.TTN_OPERATOR, parent, phys, i.op_bond, ts) for i, ts in zip(insts, ho)]
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    outs, reps = P.cbc_apply_batch(ctx, op, st, mb)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    bufs = [torch.empty(sum(int(np.prod(o.shape(j))) for j in range(o.n_nodes)), dtype=torch.complex128).pin_memory() for o in outs] if rep == 0 else bufs
    t4 = time.perf_counter()
    for o, b in zip(outs, bufs):
        P.ttn_get_data(ctx, o, b)
    t5 = time.perf_counter()
    for h in st + op + outs:
        h.destroy()
    torch.cuda.synchronize(); t6 = time.perf_counter()
    print(f"create enqueue {1e3*(t1-t0):.1f} ms, create drain {1e3*(t2-t1):.1f}, apply {1e3*(t3-t2):.1f}, "
          f"get_data {1e3*(t5-t4):.1f}, destroy {1e3*(t6-t5):.1f}", flush=True)
