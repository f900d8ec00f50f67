"""Multi-GPU plumbing.  The sharding, the exchanges of every dimension
(clearing-bitmap all-reduce or apparent-cofacet all-gather, residual-key all-gather + device
merge), rank 0's host residual with the deaths broadcast, and the result broadcast all run
inside libvr (include/vr.h "Multi-GPU"); this module only creates the communicators:

* `nccl_comm()` — one process per GPU (torchrun): rank 0 draws an NCCL unique id
  (vr_nccl_unique_id) and torch.distributed broadcasts its 128 bytes, then every rank opens
  its communicator (vr_comm_nccl);
* `local_comms(world)` — `world` ranks inside this process sharing the current GPU
  (vr_comm_local; each rank must be driven by its own thread): tests of the multi-rank logic
  on one device.

Argument marshalling only.
"""
from __future__ import annotations

import ctypes
import math
import threading

import numpy as np

from . import Barcode, _check, _collect, _options, load

__all__ = ["Comm", "nccl_comm", "local_comms", "barcodes_comm", "barcodes_sharded", "run_ranks"]


class Comm:
    """A vr_comm* owned by Python (freed with vr_comm_free)."""

    def __init__(self, ptr: ctypes.c_void_p, rank: int, world: int):
        self.ptr, self.rank, self.world = ptr, rank, world

    def close(self):
        if self.ptr:
            load().vr_comm_free(self.ptr)
            self.ptr = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(load().vr_nccl_unique_id(buf))
    return bytes(buf)


def share_unique_id(group=None) -> bytes:
    """Rank 0's NCCL unique id on every rank of the torch.distributed group."""
    import torch.distributed as dist
    obj = [unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def nccl_comm(device: int | None = None, group=None) -> Comm:
    """This process's rank of an NCCL communicator over the torch.distributed group."""
    import torch
    import torch.distributed as dist
    uid = share_unique_id(group)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.cuda.current_device() if device is None else device
    h = ctypes.c_void_p()
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    _check(load().vr_comm_nccl(buf, rank, world, dev, ctypes.byref(h)))
    return Comm(h, rank, world)


def local_comms(world: int) -> list:
    arr = (ctypes.c_void_p * world)()
    _check(load().vr_comm_local(world, arr))
    return [Comm(ctypes.c_void_p(arr[r]), r, world) for r in range(world)]


def barcodes_comm(dist_lower_tri, n: int, max_dim: int, threshold: float = math.inf, comm: Comm = None,
                  **opts) -> Barcode:
    """vr_barcodes_comm: this rank's part of a sharded computation (host input)."""
    lib = load()
    lt = np.ascontiguousarray(dist_lower_tri, dtype=np.float32)
    if lt.size != n * (n - 1) // 2:
        raise ValueError("dist_lower_tri must hold n(n-1)/2 values")
    h = ctypes.c_void_p()
    o = _options(**opts)
    _check(lib.vr_barcodes_comm(lt.ctypes.data if lt.size else None, n, max_dim, threshold, ctypes.byref(o), comm.ptr,
                                ctypes.byref(h)))
    try:
        return _collect(h)
    finally:
        lib.vr_free(h)


def barcodes_sharded(dist_lower_tri, n: int, max_dim: int, threshold: float = math.inf, comm: Comm = None,
                     **opts) -> Barcode:
    """Under torch.distributed (one process per GPU): the sharded computation, every rank
    returning the same barcode.  Opens (and closes) an NCCL communicator unless one is given."""
    own = comm is None
    if own:
        comm = nccl_comm()
    try:
        return barcodes_comm(dist_lower_tri, n, max_dim, threshold, comm, **opts)
    finally:
        if own:
            comm.close()


def run_ranks(world: int, fn):
    """Runs fn(comm) for the `world` ranks of a local group, one thread each (the ctypes calls
    release the GIL); returns the results in rank order, re-raising a rank's exception."""
    comms = local_comms(world)
    out, err = [None] * world, [None] * world

    def body(r):
        try:
            out[r] = fn(comms[r])
        except BaseException as e:  # pragma: no cover - re-raised below
            err[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for c in comms:
        c.close()
    for e in err:
        if e is not None:
            raise e
    return out
