"""B200-native CBC (arXiv 2601.19650): Python binding of libttncbc.so.

Same names as the C ABI (include/ttn_cbc.h): ttn_ctx_create, ttn_create, cbc_apply,
cbc_apply_batch, ttn_overlap, ttn_norm, ttn_get_tensor, ...  The binding only marshals
arguments; every step of the hot path runs in the CUDA kernels of csrc/.  PyTorch is used
(optionally) for the CUDA stream and for device-resident inputs.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L
from ._lib import TTN_OPERATOR, TTN_STATE, TTNError

__all__ = ["Context", "TTN", "torch_allocator", "ttn_ctx_create", "ttn_create", "cbc_apply", "cbc_apply_batch", "ttn_overlap",
           "ttn_overlap_batch", "ttn_norm", "ttn_get_tensor", "ttn_get_data", "ttn_get_data_batch", "ttn_version", "TTN_STATE", "TTN_OPERATOR",
           "TTNError", "lib_path"]

lib_path = L.LIB_PATH


def ttn_version() -> str:
    return L.load().ttn_version().decode()


def torch_allocator(device: int):
    """ttn_allocator over PyTorch's caching allocator (torch.cuda.caching_allocator_alloc /
    caching_allocator_delete), so library workspaces and TTN handles share torch's memory.
    Returns (struct, keep-alive tuple)."""
    import torch

    def _alloc(state, nbytes, stream):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), device, int(stream or 0))
        except Exception:      # out of memory: NULL -> TTN_ERR_OOM
            return None

    def _free(state, ptr, stream):
        torch.cuda.caching_allocator_delete(int(ptr))

    fa, ff = L.ALLOC_FN(_alloc), L.FREE_FN(_free)
    return L.Allocator(fa, ff, None), (fa, ff)


class Context:
    """A ttn_ctx bound to one device and one CUDA stream (default: torch's current stream).
    allocator=None: the library's own stream-ordered pool; "torch": PyTorch's caching
    allocator (torch_allocator)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None, allocator: Optional[str] = None):
        lib = L.load()
        if stream is None:
            try:
                import torch
                if torch.cuda.is_available():
                    stream = torch.cuda.current_stream(device).cuda_stream
            except Exception:
                stream = None
        self.device = device
        self.stream = stream or 0
        self._alloc = None
        if allocator == "torch":
            self._alloc = torch_allocator(device)
        elif allocator is not None:
            raise ValueError("allocator must be None or 'torch'")
        h = C.c_void_p()
        L.check(None, lib.ttn_ctx_create(int(device), C.c_void_p(self.stream),
                                         C.byref(self._alloc[0]) if self._alloc else None, C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            L.load().ttn_ctx_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def ttn_ctx_create(device: int = 0, stream: Optional[int] = None, allocator: Optional[str] = None) -> Context:
    return Context(device, stream, allocator)


class TTN:
    """Handle of a device-resident TTNS / TTNO (immutable)."""

    def __init__(self, ctx: Context, h: C.c_void_p, kind: int, src=None):
        self.ctx, self.h, self.kind = ctx, h, kind
        # the caller's source buffers of an asynchronous (pinned / device) ttn_create: held
        # until the handle is destroyed, so a temporary cannot be recycled before the copy ran
        self._src = src

    def destroy(self):
        if self.h and self.ctx.h:      # a handle outliving its context is not freed (ctx owns the pool)
            L.load().ttn_destroy(self.h)
        self.h = None
        self._src = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    @property
    def n_nodes(self) -> int:
        v = C.c_int32()
        L.check(self.ctx.h, L.load().ttn_n_nodes(self.h, C.byref(v)))
        return v.value

    def shape(self, node: int):
        nd = C.c_int32()
        dims = (C.c_int64 * 16)()
        L.check(self.ctx.h, L.load().ttn_node_shape(self.h, node, C.byref(nd), dims))
        return tuple(dims[i] for i in range(nd.value))

    def bonds(self) -> List[int]:
        off = 1 if self.kind == TTN_STATE else 2
        return [self.shape(i)[off] for i in range(self.n_nodes)]

    def get(self, node: int) -> np.ndarray:
        return ttn_get_tensor(self.ctx, self, node)

    def tensors(self) -> List[np.ndarray]:
        return [self.get(i) for i in range(self.n_nodes)]


def node_sizes(kind: int, parent: Sequence[int], phys: Sequence[int], bond: Sequence[int]) -> List[int]:
    """Entries of every node tensor in the ABI leg order (include/ttn_cbc.h)."""
    n = len(parent)
    size = []
    for i in range(n):
        e = int(phys[i]) ** (2 if kind == TTN_OPERATOR else 1)
        e *= 1 if parent[i] < 0 else int(bond[i])
        for c in range(n):
            if parent[c] == i:
                e *= int(bond[c])
        size.append(e)
    return size


def ttn_create(ctx: Context, kind: int, parent: Sequence[int], phys: Sequence[int], bond: Sequence[int],
               tensors: Sequence, on_device: Optional[bool] = None) -> TTN:
    """tensors: numpy complex128 arrays (host) or torch complex128 tensors (pinned host or CUDA).
    Each tensor's size is checked against its ABI shape before the call."""
    n = len(parent)
    if len(tensors) != n or len(phys) != n or len(bond) != n:
        raise ValueError("one tensor, physical dimension and bond per node")
    want = node_sizes(kind, parent, phys, bond)
    for i, t in enumerate(tensors):
        got = t.numel() if hasattr(t, "numel") else int(np.size(t))
        if got != want[i]:
            raise ValueError(f"node {i}: tensor has {got} entries, its ABI shape needs {want[i]}")
    keep, tkeep = [], []
    ptrs = (C.c_void_p * n)()
    dev = on_device
    for i, t in enumerate(tensors):
        if hasattr(t, "data_ptr"):  # torch tensor
            import torch
            assert t.dtype == torch.complex128 and t.is_contiguous()
            ptrs[i] = t.data_ptr()
            dev = bool(t.is_cuda) if dev is None else dev
            tkeep.append(t)
        else:
            a = L.host_c128(t)
            keep.append(a)
            ptrs[i] = a.ctypes.data
            dev = False if dev is None else dev
    h = C.c_void_p()
    L.check(ctx.h, L.load().ttn_create(ctx.h, int(kind), n, L.as_i32(parent), L.as_i32(phys), L.as_i64(bond),
                                       ptrs, int(bool(dev)), C.byref(h)))
    # pageable numpy sources are fully copied when the call returns; torch tensors (pinned
    # host or device) are copied in stream order and stay referenced by the handle
    return TTN(ctx, h, kind, tkeep or None)


def ttn_get_tensor(ctx: Context, t: TTN, node: int) -> np.ndarray:
    shp = t.shape(node)
    out = np.empty(shp, dtype=np.complex128)
    L.check(ctx.h, L.load().ttn_get_tensor(ctx.h, t.h, node, C.c_void_p(out.ctypes.data), out.size))
    return out


def ttn_get_data_batch(ctx: Context, ts, outs):
    """ttn_get_data for several TTNs into the given buffers (numpy complex128 or pinned torch
    complex128 CPU tensors); one stream synchronisation for all copies."""
    n = len(ts)
    if len(outs) != n:
        raise ValueError("one output buffer per TTN")
    hs = (C.c_void_p * n)(*[t.h for t in ts])
    ptrs = (C.c_void_p * n)(*[(o.data_ptr() if hasattr(o, "data_ptr") else o.ctypes.data) for o in outs])
    caps = (C.c_size_t * n)(*[(o.numel() if hasattr(o, "numel") else o.size) for o in outs])
    L.check(ctx.h, L.load().ttn_get_data_batch(ctx.h, n, hs, ptrs, caps))
    return outs


def ttn_get_data(ctx: Context, t: TTN, out=None):
    """All nodes concatenated (node order, ABI leg order) into `out` (numpy complex128 or a
    pinned torch complex128 CPU tensor); one D2H copy."""
    total = sum(int(np.prod(t.shape(i))) for i in range(t.n_nodes))
    if out is None:
        out = np.empty(total, dtype=np.complex128)
    ptr = out.data_ptr() if hasattr(out, "data_ptr") else out.ctypes.data
    cap = out.numel() if hasattr(out, "numel") else out.size
    L.check(ctx.h, L.load().ttn_get_data(ctx.h, t.h, C.c_void_p(ptr), cap))
    return out


def cbc_apply(ctx: Context, op: TTN, state: TTN, max_bond: int, tol: float = 0.0):
    """Returns (new TTNS handle, report dict)."""
    out = C.c_void_p()
    rep = L.Report()
    L.check(ctx.h, L.load().cbc_apply(ctx.h, op.h, state.h, int(max_bond), float(tol), C.byref(out), C.byref(rep)))
    return TTN(ctx, out, TTN_STATE), rep.as_dict()


def cbc_apply_batch(ctx: Context, ops: Sequence[TTN], states: Sequence[TTN], max_bond: int, tol: float = 0.0):
    n = len(ops)
    po = (C.c_void_p * n)(*[o.h.value for o in ops])
    ps = (C.c_void_p * n)(*[s.h.value for s in states])
    outs = (C.c_void_p * n)()
    reps = (L.Report * n)()
    L.check(ctx.h, L.load().cbc_apply_batch(ctx.h, n, po, ps, int(max_bond), float(tol), outs, reps))
    return [TTN(ctx, C.c_void_p(outs[i]), TTN_STATE) for i in range(n)], [reps[i].as_dict() for i in range(n)]


def ttn_overlap(ctx: Context, a: TTN, b: TTN) -> complex:
    v = L.c128()
    L.check(ctx.h, L.load().ttn_overlap(ctx.h, a.h, b.h, C.byref(v)))
    return complex(v.re, v.im)


def ttn_overlap_batch(ctx: Context, a: Sequence[TTN], b: Sequence[TTN]) -> List[complex]:
    n = len(a)
    pa = (C.c_void_p * n)(*[x.h.value for x in a])
    pb = (C.c_void_p * n)(*[x.h.value for x in b])
    out = (L.c128 * n)()
    L.check(ctx.h, L.load().ttn_overlap_batch(ctx.h, n, pa, pb, out))
    return [complex(out[i].re, out[i].im) for i in range(n)]


def ttn_sandwich(ctx: Context, bra: TTN, op: TTN, ket: TTN) -> complex:
    """<bra| op |ket> (include/ttn_cbc.h)."""
    v = L.c128()
    L.check(ctx.h, L.load().ttn_sandwich(ctx.h, bra.h, op.h, ket.h, C.byref(v)))
    return complex(v.re, v.im)


def ttn_op_norm2(ctx: Context, op: TTN, ket: TTN) -> float:
    """||op |ket>||^2 = <ket| op^dagger op |ket>."""
    v = C.c_double()
    L.check(ctx.h, L.load().ttn_op_norm2(ctx.h, op.h, ket.h, C.byref(v)))
    return v.value


def ttn_profile_enable(on: bool = True) -> None:
    L.check(None, L.load().ttn_profile_enable(int(bool(on))))


def ttn_profile_read(family: str = "all") -> dict:
    ms, fl, by, n = C.c_double(), C.c_double(), C.c_double(), C.c_int64()
    L.check(None, L.load().ttn_profile_read(family.encode(), C.byref(ms), C.byref(fl), C.byref(by), C.byref(n)))
    return {"ms": ms.value, "flops": fl.value, "bytes": by.value, "launches": n.value}


def ttn_launch_count() -> int:
    v = C.c_int64()
    L.check(None, L.load().ttn_launch_count(C.byref(v)))
    return v.value


def ttn_test_heev(ctx: Context, a: np.ndarray, kmax: int, max_bond: int | None = None, tol: float = 0.0,
                  route: int = 0):
    """The compress eigensolver on host matrices a[nmat, n, n] (test hook, include/ttn_cbc.h):
    returns (lam[nmat, kmax], vt[nmat, kmax, n], k[nmat], w[nmat])."""
    a = L.host_c128(a)
    if a.ndim == 2:
        a = a[None]
    nmat, n, n2 = a.shape
    if n != n2:
        raise ValueError("square matrices expected")
    mb = kmax if max_bond is None else max_bond
    lam = np.zeros((nmat, kmax))
    vt = np.zeros((nmat, kmax, n), np.complex128)
    k = np.zeros(nmat, np.int32)
    w = np.zeros(nmat)
    L.check(ctx.h, L.load().ttn_test_heev(ctx.h, nmat, n, kmax, mb, float(tol), route, a.ctypes.data,
                                          lam.ctypes.data, vt.ctypes.data, k.ctypes.data, w.ctypes.data))
    return lam, vt, k, w


def ttn_norm(ctx: Context, a: TTN) -> float:
    v = C.c_double()
    L.check(ctx.h, L.load().ttn_norm(ctx.h, a.h, C.byref(v)))
    return v.value


def ttn_ctx_set_schedule(ctx: Context, speculate: bool = True, graphs: bool = True) -> None:
    """Speculative ranks / CUDA-graph replay of cbc_apply on ctx (include/ttn_cbc.h)."""
    L.check(ctx.h, L.load().ttn_ctx_set_schedule(ctx.h, int(bool(speculate)), int(bool(graphs))))


def ttn_ctx_set_workers(ctx: Context, n: int) -> None:
    """Concurrent sub-batches for cbc_apply_batch (include/ttn_cbc.h); n = 1 turns it off."""
    L.check(ctx.h, L.load().ttn_ctx_set_workers(ctx.h, int(n)))


# ---------------------------------------------------------------- multi-GPU (NCCL)
def ttn_comm_unique_id() -> bytes:
    """128-byte NCCL unique id (create on one rank, share the bytes with the others)."""
    buf = C.create_string_buffer(128)
    L.check(None, L.load().ttn_comm_unique_id(buf))
    return buf.raw


def ttn_ctx_set_comm(ctx: Context, unique_id: Optional[bytes], rank: int = 0, world: int = 1, parts: int = 1) -> None:
    """Make ctx one rank of a partitioned multi-GPU apply (include/ttn_cbc.h); None detaches."""
    if unique_id is None:
        L.check(ctx.h, L.load().ttn_ctx_set_comm(ctx.h, None, 0, 1, 1))
        return
    buf = C.create_string_buffer(bytes(unique_id), 128)
    L.check(ctx.h, L.load().ttn_ctx_set_comm(ctx.h, buf, int(rank), int(world), int(parts)))


class LoopbackGroup:
    """In-process loopback communicator group (include/ttn_cbc.h ttn_loopback_create): the
    partitioned multi-rank schedule with `world` contexts on one device, one host thread each."""

    def __init__(self, world: int):
        h = C.c_void_p()
        L.check(None, L.load().ttn_loopback_create(int(world), C.byref(h)))
        self.h, self.world = h, world

    def close(self):
        if self.h:
            L.load().ttn_loopback_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ttn_ctx_set_comm_loopback(ctx: Context, group: LoopbackGroup, rank: int, parts: int) -> None:
    L.check(ctx.h, L.load().ttn_ctx_set_comm_loopback(ctx.h, group.h, int(rank), int(parts)))


def ttn_partition_plan(parent: Sequence[int], parts: int) -> List[int]:
    """Subtree groups of a parts-way partitioned apply (-1: replicated top); host-only."""
    n = len(parent)
    out = (C.c_int32 * n)()
    L.check(None, L.load().ttn_partition_plan(n, L.as_i32(parent), int(parts), out))
    return list(out)


def share_bytes(payload: Optional[bytes], nbytes: int = 128, group=None) -> bytes:
    """Broadcast `nbytes` bytes from rank 0 of a torch.distributed group (gloo or nccl):
    the transport of the NCCL unique id (torch is plumbing only)."""
    import torch
    import torch.distributed as dist
    t = torch.zeros(nbytes, dtype=torch.uint8)
    if dist.get_rank(group) == 0:
        t[:] = torch.tensor(list(payload), dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        t = t.cuda(torch.cuda.current_device())
    dist.broadcast(t, src=0, group=group)
    return bytes(t.cpu().tolist())


def comm_bootstrap(ctx: Context, parts: Optional[int] = None, group=None) -> None:
    """Attach a NCCL communicator over the ranks of the initialised torch.distributed group."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = share_bytes(ttn_comm_unique_id() if rank == 0 else None, 128, group)
    ttn_ctx_set_comm(ctx, uid, rank, world, parts or world)
