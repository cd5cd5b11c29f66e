"""Two-lane e2e timeline probe (host timestamps per phase per lane). Tool."""
import os, sys, time, threading
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_19650_b200 as P
import workloads as W

insts = [W.make_config(3, seed=s) for s in range(64)]
def packed(tensors):
    flat = torch.from_numpy(np.concatenate([np.ascontiguousarray(t).ravel() for t in tensors])).pin_memory()
    views, off = [], 0
    for t in tensors:
        views.append(flat[off:off + t.size]); off += t.size
    return views
hs = [packed(i.state) for i in insts]
ho = [packed(i.op) for i in insts]
parent, phys, mb = insts[0].parent, insts[0].phys, 32
NL = int(os.environ.get("LANES", "2"))
gpu_lock = threading.Lock() if os.environ.get("LOCK") else None
NB = int(os.environ.get("BATCHES", "8"))
lanes = []
for _ in range(NL):
    ls = torch.cuda.Stream(0)
    lanes.append({"stream": ls, "ctx": P.Context(0, ls.cuda_stream), "bufs": None})
T0 = time.perf_counter()
log = []
def step(j, it):
    lane = lanes[j]; c = lane["ctx"]
    t0 = time.perf_counter()
    st = [P.ttn_create(c, P.TTN_STATE, parent, phys, i.state_bond, ts) for i, ts in zip(insts, hs)]
    op = [P.ttn_create(c, P.TTN_OPERATOR, parent, phys, i.op_bond, ts) for i, ts in zip(insts, ho)]
    t1 = time.perf_counter()
    if gpu_lock is not None:
        with gpu_lock:
            outs, reps = P.cbc_apply_batch(c, op, st, mb)
    else:
        outs, reps = P.cbc_apply_batch(c, op, st, mb)
    t2 = time.perf_counter()
    if lane["bufs"] is None:
        lane["bufs"] = [torch.empty(sum(int(np.prod(o.shape(q))) for q in range(o.n_nodes)), dtype=torch.complex128).pin_memory() for o in outs]
    P.ttn_get_data_batch(c, outs, lane["bufs"])
    t3 = time.perf_counter()
    for h in st + op + outs:
        h.destroy()
    t4 = time.perf_counter()
    log.append((j, it, *(1e3 * (x - T0) for x in (t0, t1, t2, t3, t4))))
for j in range(NL): step(j, -1)
torch.cuda.synchronize()
T0 = time.perf_counter(); log.clear()
started = [threading.Event() for _ in range(NL)]
def run(j):
    if j > 0:
        started[j - 1].wait()
    for it in range(j, NB, NL):
        step(j, it)
        started[j].set()
th = [threading.Thread(target=run, args=(j,)) for j in range(NL)]
[t.start() for t in th]; [t.join() for t in th]
torch.cuda.synchronize()
el = time.perf_counter() - T0
print("lanes", NL, "batches", NB, "total ms", 1e3 * el, "applies/s", NB * 64 / el)
for r in sorted(log, key=lambda x: x[2]):
    print("lane %d it %d  create %.1f-%.1f  apply -%.1f  get -%.1f  destroy -%.1f" % r)
