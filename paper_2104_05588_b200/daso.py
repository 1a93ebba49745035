"""Thin Python binding of libdaso.so with the C ABI's names (include/daso.h).

Argument marshalling only: tensors become device pointers, torch's current CUDA
stream becomes a ``cudaStream_t``; every step of the hot path runs in the
library's sm_100a kernels and its NCCL communicators.  PyTorch supplies device
memory, streams and the ``torch.distributed`` rendezvous of the NCCL unique id.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Iterable, Optional

from . import _lib as L
from ._lib import DasoError, Record, check, lib  # noqa: F401

WIRES = {"bf16": L.WIRE_BF16, "fp32": L.WIRE_FP32}
EXCHANGES = {"nccl": L.EXCH_NCCL, "ce": L.EXCH_CE}
MODES = {"faithful": L.MODE_FAITHFUL, "sharded": L.MODE_SHARDED, "fused": L.MODE_FUSED}


def _torch():
    import torch
    return torch


def _stream(stream=None) -> C.c_void_p:
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream))


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(0 if t is None else int(t.data_ptr()))


def _dev_f32(t, name: str):
    torch = _torch()
    if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous float32 CUDA tensor")


def daso_padded_numel(n: int, gpus_per_node: int) -> int:
    return int(lib().daso_padded_numel(n, gpus_per_node))


# ------------------------------------------------------------------ schedule (host only)
class Schedule:
    """daso_sched_create / daso_sched_next / daso_sched_destroy."""

    def __init__(self, B_init: int, S_init: int = -1, warmup_epochs: int = 0, cooldown_epochs: int = 0,
                 total_epochs: int = 1, steps_per_epoch: int = 1 << 20, gpus_per_node: int = 1):
        cfg = L.SchedConfig(B_init, S_init, warmup_epochs, cooldown_epochs, total_epochs, steps_per_epoch,
                            gpus_per_node)
        h = C.c_void_p()
        check(lib().daso_sched_create(C.byref(cfg), C.byref(h)), "daso_sched_create")
        self._h = h

    def next(self, plateau: int = 0) -> dict:
        r = Record()
        check(lib().daso_sched_next(self._h, int(plateau), C.byref(r)), "daso_sched_next")
        return r.as_dict()

    def close(self):
        if getattr(self, "_h", None):
            lib().daso_sched_destroy(self._h)
            self._h = None

    __del__ = close


class PlateauDetector:
    """daso_plateau_*: one mean training loss per epoch -> plateau flag."""

    def __init__(self, patience: int = 5, threshold: float = 0.01):
        h = C.c_void_p()
        check(lib().daso_plateau_create(int(patience), float(threshold), C.byref(h)), "daso_plateau_create")
        self._h = h

    def update(self, loss: float) -> int:
        f = C.c_int(0)
        check(lib().daso_plateau_update(self._h, float(loss), C.byref(f)), "daso_plateau_update")
        return int(f.value)

    def close(self):
        if getattr(self, "_h", None):
            lib().daso_plateau_destroy(self._h)
            self._h = None

    __del__ = close


def daso_lr_at(step: int, steps_per_epoch: int, base_lr: float, world: int, warmup_epochs: int, factor: float,
               n_plateaus: int) -> float:
    out = C.c_double()
    check(lib().daso_lr_at(int(step), int(steps_per_epoch), float(base_lr), int(world), int(warmup_epochs),
                           float(factor), int(n_plateaus), C.byref(out)), "daso_lr_at")
    return float(out.value)


# ------------------------------------------------------------------ context
def daso_get_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().daso_get_unique_id(buf), "daso_get_unique_id")
    return buf.raw


def rendezvous_unique_id() -> bytes:
    """Rank 0 draws the NCCL unique id; torch.distributed broadcasts the 128 bytes."""
    import torch.distributed as dist
    obj = [daso_get_unique_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


class Ctx:
    """An initialised ``daso_ctx*``; methods are the ctx entry points of daso.h."""

    def __init__(self, handle: C.c_void_p, world: int, gpus_per_node: int, rank: int, mode: str, wire: str,
                 owned: bool = True):
        self._h = handle
        self._owned = owned
        self.world, self.G, self.rank = world, gpus_per_node, rank
        self.P = world // gpus_per_node
        self.node, self.local = rank // gpus_per_node, rank % gpus_per_node
        self.mode, self.wire = mode, wire
        self.n = 0

    # --- helpers
    def _check(self, status: int, where: str):
        check(status, where, self._h)

    # --- entry points
    def bind(self, x, g, v, n: Optional[int] = None):
        for t, nm in ((x, "x"), (g, "g"), (v, "v")):
            _dev_f32(t, nm)
        n = x.numel() if n is None else int(n)
        need = daso_padded_numel(n, self.G) if self.mode != "faithful" else n
        if min(x.numel(), g.numel(), v.numel()) < need:
            raise ValueError(f"buckets must hold {need} elements in {self.mode} mode")
        self._keep = (x, g, v)
        self.n = n
        self._check(lib().daso_bind(self._h, _ptr(x), _ptr(g), _ptr(v), n), "daso_bind")

    def alloc_bind(self, n: int):
        """daso_alloc_bind: library-owned (cudaMalloc) buckets; returns torch
        tensors x, g, v of daso_padded_numel(n, G) floats viewing them (valid until finalize)."""
        torch = _torch()
        px, pg, pv = C.c_void_p(), C.c_void_p(), C.c_void_p()
        self._check(lib().daso_alloc_bind(self._h, int(n), C.byref(px), C.byref(pg), C.byref(pv)), "daso_alloc_bind")
        self.n = int(n)
        n_pad = daso_padded_numel(n, self.G)
        dev = torch.device("cuda", torch.cuda.current_device())
        return tuple(torch.as_tensor(_DevBuf(p.value, n_pad, self), device=dev) for p in (px, pg, pv))

    def local_sync(self, stream=None):
        self._check(lib().daso_local_sync(self._h, _stream(stream)), "daso_local_sync")

    def local_update(self, lr: float, stream=None):
        self._check(lib().daso_local_update(self._h, float(lr), _stream(stream)), "daso_local_update")

    def global_send(self, group: int, S: int, stream=None):
        self._check(lib().daso_global_send(self._h, int(group), int(S), _stream(stream)), "daso_global_send")

    def global_merge(self, stream=None):
        self._check(lib().daso_global_merge(self._h, _stream(stream)), "daso_global_merge")

    def step(self, lr: float, plateau: int = 0, stream=None) -> dict:
        r = Record()
        self._check(lib().daso_step(self._h, float(lr), int(plateau), _stream(stream), C.byref(r)), "daso_step")
        return r.as_dict()

    def step_ex(self, lr: float, plateau: int = 0, grads_reduced: bool = False, stream=None) -> dict:
        r = Record()
        self._check(lib().daso_step_ex(self._h, float(lr), int(plateau), L.STEP_GRADS_REDUCED if grads_reduced else 0,
                                       _stream(stream), C.byref(r)), "daso_step_ex")
        return r.as_dict()

    def local_sync_bucket(self, offset: int, count: int, stream=None):
        self._check(lib().daso_local_sync_bucket(self._h, int(offset), int(count), _stream(stream)),
                    "daso_local_sync_bucket")

    def step_host(self, host_grads, lr: float, plateau: int = 0, stream=None) -> tuple[dict, int]:
        """host_grads: a (pinned) CPU float32 tensor of n elements."""
        torch = _torch()
        if host_grads.is_cuda or host_grads.dtype != torch.float32 or host_grads.numel() < self.n:
            raise ValueError("host_grads must be a CPU float32 tensor with >= n elements")
        r = Record()
        flag = C.c_uint32(0)
        self._check(lib().daso_step_host(self._h, _ptr(host_grads), float(lr), int(plateau), _stream(stream),
                                         C.byref(r), C.byref(flag)), "daso_step_host")
        return r.as_dict(), int(flag.value)

    def trace_enable(self, on: bool = True):
        self._check(lib().daso_trace_enable(self._h, int(on)), "daso_trace_enable")

    def trace_read(self, reset: bool = True) -> dict:
        t = L.Trace()
        self._check(lib().daso_trace_read(self._h, C.byref(t), int(reset)), "daso_trace_read")
        return t.as_dict()

    def set_exchange(self, enabled: bool) -> bool:
        """Timing knob (daso_set_exchange): False suppresses the group all-gather."""
        return bool(lib().daso_set_exchange(self._h, int(bool(enabled))))

    def exchange_alone(self, iters: int = 20) -> float:
        """daso_exchange_alone: mean ms of one group all-gather with nothing else running."""
        ms = C.c_double()
        self._check(lib().daso_exchange_alone(self._h, int(iters), C.byref(ms)), "daso_exchange_alone")
        return float(ms.value)

    def query(self) -> dict:
        r = Record()
        self._check(lib().daso_query(self._h, C.byref(r)), "daso_query")
        return r.as_dict()

    def check_finite(self, stream=None) -> bool:
        s = lib().daso_check_finite(self._h, _stream(stream))
        if s == L.ERR_NONFINITE:
            return False
        self._check(s, "daso_check_finite")
        return True

    def finalize(self):
        if not self._owned:
            raise RuntimeError("a virtual-cluster rank is finalized by VCluster.destroy()")
        if self._h:
            s = lib().daso_finalize(self._h)
            self._h = None
            check(s, "daso_finalize")


def daso_init(world: int, gpus_per_node: int, B: int, S: int, *, rank: int, uid: bytes,
              warmup_epochs: int = 0, cooldown_epochs: int = 0, total_epochs: int = 1,
              steps_per_epoch: int = 1 << 20, momentum: float = 0.9, weight_decay: float = 1e-4,
              wire: str = "bf16", mode: str = "faithful", check_finite: bool = True,
              nccl_max_ctas: int = 0, exchange: str = "nccl") -> Ctx:
    cfg = _config(rank, warmup_epochs, cooldown_epochs, total_epochs, steps_per_epoch, momentum, weight_decay, wire,
                  mode, check_finite, nccl_max_ctas, exchange)
    if len(uid) != 128:
        raise ValueError("uid must be 128 bytes")
    h = C.c_void_p()
    s = lib().daso_init(C.byref(h), world, gpus_per_node, B, S, C.byref(cfg), C.c_char_p(uid))
    if s != L.OK:
        msg = lib().daso_last_error(h).decode() if h.value else ""
        if h.value:
            lib().daso_finalize(h)
        raise DasoError(s, "daso_init", msg)
    return Ctx(h, world, gpus_per_node, rank, mode, wire)


def _config(rank, warmup_epochs, cooldown_epochs, total_epochs, steps_per_epoch, momentum, weight_decay, wire, mode,
            check_finite, nccl_max_ctas, exchange="nccl") -> L.Config:
    return L.Config(rank, warmup_epochs, cooldown_epochs, total_epochs, steps_per_epoch, momentum, weight_decay,
                    WIRES[wire], MODES[mode], int(check_finite), nccl_max_ctas, EXCHANGES[exchange])


class VCluster:
    """daso_vcluster_*: W = world virtual ranks of a P x G cluster on ONE GPU, each running the
    product batch (daso_step_ex and its kernels) with a loopback transport (include/daso.h).
    ``x(r)``, ``g(r)``, ``v(r)`` are torch views of rank r's cluster-owned buckets
    (daso_padded_numel(n, G) floats); ``rank(r)`` is its Ctx (trace / query / check_finite)."""

    def __init__(self, world: int, gpus_per_node: int, B: int, S: int, n: int, *, warmup_epochs: int = 0,
                 cooldown_epochs: int = 0, total_epochs: int = 1, steps_per_epoch: int = 1 << 20,
                 momentum: float = 0.9, weight_decay: float = 1e-4, wire: str = "bf16", mode: str = "fused",
                 check_finite: bool = True, exchange: str = "nccl"):
        """exchange="nccl": the group all-gather is emulated by loopback copies; "ce": the real
        copy-engine exchange (DASO_EXCH_CE) runs between the sibling ranks on this GPU."""
        torch = _torch()
        cfg = _config(0, warmup_epochs, cooldown_epochs, total_epochs, steps_per_epoch, momentum, weight_decay,
                      wire, mode, check_finite, 0, exchange)
        h = C.c_void_p()
        s = lib().daso_vcluster_create(C.byref(h), world, gpus_per_node, B, S, C.byref(cfg), int(n))
        if s != L.OK:
            msg = lib().daso_vcluster_last_error(h).decode() if h.value else ""
            if h.value:
                lib().daso_vcluster_destroy(h)
            raise DasoError(s, "daso_vcluster_create", msg)
        self._h = h
        self.world, self.G, self.n = world, gpus_per_node, int(n)
        self.P = world // gpus_per_node
        self.n_pad = daso_padded_numel(n, gpus_per_node)
        dev = torch.device("cuda", torch.cuda.current_device())
        self._bufs = []
        for r in range(world):
            px, pg, pv = C.c_void_p(), C.c_void_p(), C.c_void_p()
            check(lib().daso_vcluster_buffers(h, r, C.byref(px), C.byref(pg), C.byref(pv)), "daso_vcluster_buffers")
            self._bufs.append(tuple(torch.as_tensor(_DevBuf(p.value, self.n_pad, self), device=dev)
                                    for p in (px, pg, pv)))
        self._ranks = [Ctx(C.c_void_p(lib().daso_vcluster_rank(h, r)), world, gpus_per_node, r, mode, wire,
                           owned=False) for r in range(world)]
        for c in self._ranks:
            c.n = self.n

    def x(self, r: int):
        return self._bufs[r][0]

    def g(self, r: int):
        return self._bufs[r][1]

    def v(self, r: int):
        return self._bufs[r][2]

    def rank(self, r: int) -> Ctx:
        return self._ranks[r]

    def step(self, lr: float, plateau: int = 0, stream=None) -> list[dict]:
        recs = (Record * self.world)()
        s = lib().daso_vcluster_step(self._h, float(lr), int(plateau), _stream(stream), recs)
        if s != L.OK:
            raise DasoError(s, "daso_vcluster_step", lib().daso_vcluster_last_error(self._h).decode())
        return [r.as_dict() for r in recs]

    def destroy(self):
        if getattr(self, "_h", None):
            self._bufs = []
            s = lib().daso_vcluster_destroy(self._h)
            self._h = None
            check(s, "daso_vcluster_destroy")


class _DevBuf:
    """__cuda_array_interface__ over library-owned device memory (kept alive by `owner`)."""

    def __init__(self, ptr: int, numel: int, owner):
        self._owner = owner
        self.__cuda_array_interface__ = {"shape": (numel,), "typestr": "<f4", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def init_from_env(gpus_per_node: int, B: int, S: int, **kw) -> Ctx:
    """torchrun-style init: RANK / WORLD_SIZE / LOCAL_RANK from the environment;
    torch.distributed must already be initialised (any backend) for the id broadcast."""
    torch = _torch()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    uid = rendezvous_unique_id() if world > 1 else daso_get_unique_id()
    return daso_init(world, gpus_per_node, B, S, rank=rank, uid=uid, **kw)


# module-level aliases with the C names
def daso_bind(ctx: Ctx, x, g, v, n=None): return ctx.bind(x, g, v, n)
def daso_local_sync(ctx: Ctx, stream=None): return ctx.local_sync(stream)
def daso_local_update(ctx: Ctx, lr, stream=None): return ctx.local_update(lr, stream)
def daso_global_send(ctx: Ctx, group, S, stream=None): return ctx.global_send(group, S, stream)
def daso_global_merge(ctx: Ctx, stream=None): return ctx.global_merge(stream)
def daso_step(ctx: Ctx, lr, plateau=0, stream=None): return ctx.step(lr, plateau, stream)
def daso_step_host(ctx: Ctx, host_grads, lr, plateau=0, stream=None): return ctx.step_host(host_grads, lr, plateau, stream)
def daso_finalize(ctx: Ctx): return ctx.finalize()


# ------------------------------------------------------------------ kernel entry points
def daso_k_update(x, v, g, lr, mu, wd, gscale=1.0, pack_out=None, wire="bf16", flag=None, stream=None):
    for t, nm in ((x, "x"), (v, "v"), (g, "g")):
        _dev_f32(t, nm)
    check(lib().daso_k_update(_ptr(x), _ptr(v), _ptr(g), x.numel(), lr, mu, wd, gscale, _ptr(pack_out),
                              WIRES[wire], _ptr(flag), _stream(stream)), "daso_k_update")


def daso_k_update_merge(x, v, g, lr, mu, wd, gscale, slot, S, pack_out=None, wire="bf16", flag=None, stream=None):
    """slot: [P, stride] tensor (bf16 / int16 for the bf16 wire, float32 for fp32)."""
    for t, nm in ((x, "x"), (v, "v"), (g, "g")):
        _dev_f32(t, nm)
    check(lib().daso_k_update_merge(_ptr(x), _ptr(v), _ptr(g), x.numel(), lr, mu, wd, gscale, _ptr(slot),
                                    slot.shape[1], slot.shape[0], int(S), _ptr(pack_out), WIRES[wire], _ptr(flag),
                                    _stream(stream)), "daso_k_update_merge")


def daso_k_merge(x, slot, S, pack_out=None, wire="bf16", flag=None, stream=None):
    _dev_f32(x, "x")
    check(lib().daso_k_merge(_ptr(x), x.numel(), _ptr(slot), slot.shape[1], slot.shape[0], int(S), _ptr(pack_out),
                             WIRES[wire], _ptr(flag), _stream(stream)), "daso_k_merge")


def daso_k_average(x, slot, wire="bf16", flag=None, stream=None):
    _dev_f32(x, "x")
    check(lib().daso_k_average(_ptr(x), x.numel(), _ptr(slot), slot.shape[1], slot.shape[0], WIRES[wire],
                               _ptr(flag), _stream(stream)), "daso_k_average")


def daso_k_pack(x, pack_out, wire="bf16", stream=None):
    _dev_f32(x, "x")
    check(lib().daso_k_pack(_ptr(x), x.numel(), _ptr(pack_out), WIRES[wire], _stream(stream)), "daso_k_pack")


def daso_flat_layout(numels: Iterable[int], align: int = 64) -> tuple[list[int], int]:
    numels = list(numels)
    n = len(numels)
    arr = (C.c_size_t * max(n, 1))(*numels)
    offs = (C.c_size_t * max(n, 1))()
    tot = C.c_size_t()
    check(lib().daso_flat_layout(arr, n, align, offs, C.byref(tot)), "daso_flat_layout")
    return [int(offs[i]) for i in range(n)], int(tot.value)


def _is_dense(t) -> bool:
    """True if the tensor's elements exactly fill numel consecutive slots (any dim order)."""
    dims = sorted((st, sz) for st, sz in zip(t.stride(), t.shape) if sz != 1)
    expect = 1
    for st, sz in dims:
        if st != expect:
            return False
        expect *= sz
    return True


def _dense_f32(t, name: str):
    torch = _torch()
    if not (t.is_cuda and t.dtype == torch.float32 and _is_dense(t)):
        raise ValueError(f"{name} must be a dense (any memory format) float32 CUDA tensor")


def daso_k_gather(tensors, dst, offsets, stream=None):
    """Copy each tensor's memory block (numel floats in memory order) into dst[offset:]."""
    n = len(tensors)
    for t in tensors:
        _dense_f32(t, "tensor")
    src = (C.c_void_p * n)(*[t.data_ptr() for t in tensors])
    numel = (C.c_size_t * n)(*[t.numel() for t in tensors])
    offs = (C.c_size_t * n)(*offsets)
    check(lib().daso_k_gather(src, numel, offs, n, _ptr(dst), _stream(stream)), "daso_k_gather")


def daso_k_scatter(src, tensors, offsets, stream=None):
    n = len(tensors)
    dst = (C.c_void_p * n)(*[t.data_ptr() for t in tensors])
    numel = (C.c_size_t * n)(*[t.numel() for t in tensors])
    offs = (C.c_size_t * n)(*offsets)
    check(lib().daso_k_scatter(_ptr(src), dst, numel, offs, n, _stream(stream)), "daso_k_scatter")


def daso_kernel_impl(impl: int | str | None = None) -> int:
    """Select the fused-kernel data path: 0/"ldg", 1/"tma", 2/"auto"; returns the previous one."""
    code = {"ldg": 0, "tma": 1, "auto": 2, None: -1}.get(impl, impl)
    return int(lib().daso_kernel_impl(int(code)))


def daso_k_checksum(x, out_u64, stream=None):
    """out_u64: a 1-element int64 CUDA tensor receiving the checksum bits."""
    check(lib().daso_k_checksum(_ptr(x), x.numel(), _ptr(out_u64), _stream(stream)), "daso_k_checksum")


# ------------------------------------------------------------------ backward-overlapped local sync
def bucket_partition(offsets, numels, n, limit):
    """Split the flat gradient bucket into contiguous all-reduce buckets in reverse parameter
    order (the order backward produces gradients), each >= `limit` elements except the last.
    Returns (buckets: lists of parameter indices, ranges: (offset, count) per bucket); the
    ranges tile [0, offset_last + numel_last) exactly, inter-parameter padding included."""
    m = len(offsets)
    buckets, cur = [], []
    for i in range(m - 1, -1, -1):
        cur.append(i)
        lo = offsets[cur[-1]]
        hi = offsets[cur[0]] + numels[cur[0]]
        if hi - lo >= limit:
            buckets.append(cur)
            cur = []
    if cur:
        buckets.append(cur)
    ranges = []
    for b in buckets:
        lo = offsets[b[-1]]
        hi = offsets[b[0] + 1] if b[0] + 1 < m else offsets[b[0]] + numels[b[0]]
        ranges.append((lo, min(hi, n) - lo))
    return buckets, ranges


class OverlappedLocalSync:
    """Bucketed node all-reduce overlapped with backward (the DDP
    behaviour of the paper's local tier).  Buckets are contiguous ranges of the
    flat gradient bucket in reverse parameter order (~bucket_mb each); a post-accumulate
    grad hook launches a bucket's all-reduce (daso_local_sync_bucket) on a comm stream as
    soon as all its gradients exist.  Call ``step(lr)`` after backward: the compute stream
    waits for the buckets and runs daso_step_ex(..., grads_reduced=True)."""

    def __init__(self, ctx: Ctx, flat: "FlatParams", bucket_mb: float = 25.0):
        torch = _torch()
        self.ctx, self.flat = ctx, flat
        self.stream = torch.cuda.Stream(priority=-1)
        self.buckets, self.ranges = bucket_partition(flat.offsets, [p.numel() for p in flat.params], flat.n,
                                                     int(bucket_mb * (1 << 20) / 4))
        self.bucket_of = {i: k for k, b in enumerate(self.buckets) for i in b}
        self.pending = [len(b) for b in self.buckets]
        self.launched = 0
        self.handles = [p.register_post_accumulate_grad_hook(self._hook(i)) for i, p in enumerate(flat.params)]

    def _hook(self, i):
        def fn(_p):
            k = self.bucket_of[i]
            self.pending[k] -= 1
            if self.pending[k] == 0:
                torch = _torch()
                ev = torch.cuda.Event()
                ev.record(torch.cuda.current_stream())
                self.stream.wait_event(ev)
                self.ctx.local_sync_bucket(*self.ranges[k], stream=self.stream)
                self.launched += 1
        return fn

    def step(self, lr: float, plateau: int = 0) -> dict:
        torch = _torch()
        if self.launched != len(self.buckets):
            raise RuntimeError(f"only {self.launched} of {len(self.buckets)} gradient buckets became ready")
        ev = torch.cuda.Event()
        ev.record(self.stream)
        torch.cuda.current_stream().wait_event(ev)
        self.pending = [len(b) for b in self.buckets]
        self.launched = 0
        return self.ctx.step_ex(lr, plateau, grads_reduced=True)

    def remove(self):
        for h in self.handles:
            h.remove()


# ------------------------------------------------------------------ flat buckets for a torch model
class FlatParams:
    """Flatten a model's fp32 parameters into one contiguous bucket (K0, P:86
    "buffer packaging") and re-point every parameter and its ``.grad`` as views,
    so the per-step unpack is free.  Buckets x, g, v hold n_pad elements."""

    def __init__(self, params, gpus_per_node: int = 1, align: int = 64, ctx: "Ctx | None" = None,
                 buckets=None):
        """ctx given: the buckets are allocated and bound by the library (daso_alloc_bind —
        the fused mode's way around cuMem allocators such as expandable_segments);
        buckets=(x, g, v) given: adopt existing (e.g. VCluster-owned) float32 buckets of
        >= n_pad elements; otherwise torch allocates them and the caller binds."""
        torch = _torch()
        self.params = [p for p in params if p.requires_grad]
        if not self.params:
            raise ValueError("no trainable parameters")
        dev = self.params[0].device
        self.offsets, self.n = daso_flat_layout([p.numel() for p in self.params], align)
        self.n_pad = daso_padded_numel(self.n, gpus_per_node)
        if ctx is not None:
            self.x, self.g, self.v = ctx.alloc_bind(self.n)
        elif buckets is not None:
            for t, nm in zip(buckets, "xgv"):
                _dev_f32(t, nm)
                if t.numel() < self.n_pad:
                    raise ValueError(f"bucket {nm} holds {t.numel()} < {self.n_pad} elements")
            self.x, self.g, self.v = buckets
        else:
            self.x = torch.zeros(self.n_pad, dtype=torch.float32, device=dev)
            self.g = torch.zeros_like(self.x)
            self.v = torch.zeros_like(self.x)
        daso_k_gather([p.detach() for p in self.params], self.x, self.offsets)
        torch.cuda.current_stream().synchronize()
        # views keep each parameter's memory format (e.g. channels_last): the bucket holds
        # every tensor's memory block in memory order
        for p, o in zip(self.params, self.offsets):
            p.data = self.x.as_strided(p.shape, p.stride(), o)
            p.grad = self.g.as_strided(p.shape, p.stride(), o)
