"""ctypes mirror of include/strait_node.h and the record storage behind the
object-API views (pcie.PcieLinkState, runtime.AimdState / GpuRuntimeState /
RunningTaskEntry).

A record is one flat block: header, entry slots in running-list order, then
the pending-transfer ring.  On a CUDA box the block is page-locked host
memory, so ``strait_node_propose`` reads it in place (unified addressing);
without a device it is ordinary host memory and only the bookkeeping entry
points (host code of the same library) can run on it.
"""
from __future__ import annotations

import ctypes as C
import itertools

from ._abi import MAX_METRICS, STRAIT_OK, check, lib

STRAIT_ENOSPC = 5
_vp = C.c_void_p
_dp = C.POINTER(C.c_double)


class GpuHdr(C.Structure):
    _fields_ = [("gpu_id", C.c_int32), ("n_metrics", C.c_int32), ("concurrency_limit", C.c_int32),
                ("n_running", C.c_int32), ("slot_cap", C.c_int32), ("ring_cap", C.c_int32),
                ("ring_head", C.c_int32), ("ring_len", C.c_int32),
                ("t_available", C.c_double), ("cap_pct", C.c_double), ("aimd_floor", C.c_double),
                ("aimd_ceiling", C.c_double), ("aimd_increase", C.c_double), ("aimd_interval", C.c_double),
                ("aimd_last_tick", C.c_double), ("reserved", C.c_double),
                ("agg", C.c_double * MAX_METRICS)]


class NodeEntry(C.Structure):
    _fields_ = [("contrib", C.c_double * MAX_METRICS), ("tl_v", C.c_double * MAX_METRICS),
                ("tl_acc", C.c_double * MAX_METRICS),
                ("self_cmp", C.c_double), ("self_mem", C.c_double), ("t_kernel", C.c_double),
                ("deadline_abs", C.c_double), ("kstart_est", C.c_double), ("kernel_start", C.c_double),
                ("intf_pred", C.c_double), ("tl_t0", C.c_double), ("tl_tlast", C.c_double),
                ("prio", C.c_int32), ("started", C.c_int32), ("tl_n", C.c_int32), ("handle", C.c_int32)]


class ProposeOut(C.Structure):
    _fields_ = [("status", C.c_int32), ("size", C.c_int32), ("gpu_index", C.c_int32), ("err_gpu", C.c_int32),
                ("err_pos", C.c_int32), ("err_kind", C.c_int32), ("probes", C.c_int32), ("pad", C.c_int32),
                ("latency", C.c_double), ("intf", C.c_double)]


class ProposeArgs(C.Structure):
    _fields_ = [("n_metrics", C.c_int32), ("n_gpus", C.c_int32), ("k_max", C.c_int32), ("cand_prio", C.c_int32),
                ("use_violate", C.c_int32), ("use_meet", C.c_int32), ("fixed_size", C.c_int32),
                ("stage_stride", C.c_int32),
                ("now", C.c_double), ("effect_cap", C.c_double), ("deadline_ms", C.c_double),
                ("front_arrival", C.c_double),
                ("params", _vp), ("recs", _vp),
                ("cand_contrib", _vp), ("cand_self_cmp", _vp), ("cand_self_mem", _vp), ("cand_total", _vp),
                ("cand_kernel", _vp), ("pair_flags", _vp), ("pair_latency", _vp), ("pair_intf", _vp),
                ("seg_gpu", _vp), ("seg_latency", _vp), ("seg_intf", _vp), ("out", _vp)]


HDR_BYTES = C.sizeof(GpuHdr)
ENTRY_BYTES = C.sizeof(NodeEntry)
_declared = None


def nlib():
    """The product library with the node entry points declared."""
    global _declared
    L = lib()
    if _declared is not L:
        L.strait_node_record_bytes.restype = C.c_int64
        L.strait_node_record_bytes.argtypes = [C.c_int32, C.c_int32]
        L.strait_link_delay.restype = C.c_double
        L.strait_link_delay.argtypes = [_vp, C.c_double]
        L.strait_link_reserve.argtypes = [_vp, C.c_double, C.c_double, _dp, _dp]
        L.strait_link_calibrate.argtypes = [_vp, C.c_double]
        L.strait_aimd_advance.argtypes = [_vp, C.c_double]
        L.strait_aimd_reset.argtypes = [_vp]
        L.strait_aimd_reset.restype = None
        L.strait_entry_tl_record.argtypes = [C.POINTER(NodeEntry), C.c_int32, C.c_double, _dp]
        L.strait_entry_tl_twa.argtypes = [C.POINTER(NodeEntry), C.c_int32, C.c_double, _dp]
        L.strait_node_detach.argtypes = [_vp, C.c_int32, C.POINTER(NodeEntry)]
        L.strait_node_attach.argtypes = [_vp, C.POINTER(NodeEntry)]
        L.strait_node_excluding.argtypes = [_vp, C.c_int32, _dp]
        L.strait_node_lp_aggregate.argtypes = [_vp, _dp]
        L.strait_node_lp_aggregate.restype = None
        L.strait_node_add.argtypes = [_vp, C.POINTER(NodeEntry), C.c_double]
        L.strait_node_remove.argtypes = [_vp, C.c_int32, C.c_double, C.POINTER(NodeEntry)]
        L.strait_node_find.argtypes = [_vp, C.c_int32]
        L.strait_node_find.restype = C.c_int32
        L.strait_node_submit.argtypes = [_vp, C.POINTER(NodeEntry), C.c_double, C.c_double, _dp, _dp]
        L.strait_node_start.argtypes = [_vp, C.c_int32, C.c_double]
        L.strait_node_complete.argtypes = [_vp, C.c_int32, C.c_double, _dp, C.POINTER(NodeEntry)]
        L.strait_nodes_tick.argtypes = [_vp, C.c_int32, C.c_double]
        L.strait_node_propose.argtypes = [C.POINTER(ProposeArgs), _vp]
        L.strait_node_device_address.restype = _vp
        L.strait_node_device_address.argtypes = [_vp]
        _declared = L
    return L


def _cuda_ready() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


class Record:
    """Owner of one record block.  Views keep a reference to the Record (not
    to raw addresses), so growing the block is transparent to them."""

    __slots__ = ("_buf", "addr", "dev_addr", "hdr", "ents", "ring", "version", "__weakref__")

    def __init__(self, n_metrics: int, slot_cap: int, ring_cap: int, gpu_id: int = 0, concurrency_limit: int = 0):
        if not 1 <= n_metrics <= MAX_METRICS:
            raise ValueError(f"n_metrics {n_metrics} outside 1..{MAX_METRICS}")
        self.version = 0
        self._alloc(slot_cap, ring_cap)
        h = self.hdr
        h.slot_cap, h.ring_cap = slot_cap, ring_cap
        h.gpu_id, h.n_metrics, h.concurrency_limit = gpu_id, n_metrics, concurrency_limit
        h.cap_pct, h.aimd_floor, h.aimd_ceiling = 75.0, 75.0, 100.0  # AimdState defaults (runtime.py:23-28)
        h.aimd_increase, h.aimd_interval, h.aimd_last_tick = 0.25, 100.0, 0.0

    def _alloc(self, slot_cap: int, ring_cap: int, old: "Record | None" = None) -> None:
        n = int(nlib().strait_node_record_bytes(slot_cap, ring_cap))
        if _cuda_ready():
            import torch

            buf = torch.zeros(n, dtype=torch.uint8, pin_memory=True)  # page-locked: device-readable in place
            addr = buf.data_ptr()
            dev = nlib().strait_node_device_address(addr)
            if not dev:
                check(4)
        else:
            buf = (C.c_char * n)()
            addr, dev = C.addressof(buf), None
        if old is not None:  # header + live entries + the ring in FIFO order
            C.memmove(addr, old.addr, HDR_BYTES + ENTRY_BYTES * old.hdr.n_running)
        self._buf, self.addr, self.dev_addr = buf, addr, dev
        self.hdr = GpuHdr.from_address(addr)
        self.ents = (NodeEntry * slot_cap).from_address(addr + HDR_BYTES)
        self.ring = (C.c_double * max(ring_cap, 1)).from_address(addr + HDR_BYTES + ENTRY_BYTES * slot_cap)

    def grow(self, slot_cap: int | None = None, ring_cap: int | None = None) -> None:
        h = self.hdr
        slots = max(h.slot_cap, slot_cap or 0)
        rcap = max(h.ring_cap, ring_cap or 0)
        pending = [self.ring[(h.ring_head + i) % h.ring_cap] for i in range(h.ring_len)] if h.ring_cap else []
        snapshot = Record.__new__(Record)
        snapshot._buf, snapshot.addr, snapshot.hdr = self._buf, self.addr, self.hdr  # keeps the old block alive
        self._alloc(slots, rcap, old=snapshot)
        h = self.hdr
        h.slot_cap, h.ring_cap, h.ring_head = slots, rcap, 0
        for i, p in enumerate(pending):
            self.ring[i] = p
        self.version += 1

    def call(self, fn, *args, raise_errors: bool = True) -> int:
        """Run a mutator; on STRAIT_ENOSPC grow (slots x2 / ring x2) and retry.
        Returns the final status (after raising it unless ``raise_errors`` is False)."""
        while True:
            st = fn(self.addr, *args)
            if st != STRAIT_ENOSPC:
                if raise_errors:
                    check(st)
                return st
            h = self.hdr
            if h.ring_len == h.ring_cap:
                self.grow(ring_cap=max(8, 2 * h.ring_cap))
            else:
                self.grow(slot_cap=max(4, 2 * h.slot_cap, h.concurrency_limit))


make_record = Record


_handles = itertools.count(1)


def new_handle() -> int:
    return next(_handles) & 0x7FFFFFFF


def darr(values) -> C.Array:
    vals = list(values)
    return (C.c_double * max(len(vals), 1))(*vals)


__all__ = ["GpuHdr", "NodeEntry", "ProposeArgs", "ProposeOut", "Record", "make_record", "nlib", "new_handle",
           "darr", "HDR_BYTES", "ENTRY_BYTES", "STRAIT_OK"]
