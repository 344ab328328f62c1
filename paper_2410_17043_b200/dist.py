"""Multi-GPU bootstrap: one process per GPU, ``torch.distributed`` for the
plumbing, CUDA IPC mappings of every peer's receive / return buffers and
arrival counters so the engine stores straight into peer HBM over NVSwitch.

Rank layout: the layer's ``n`` expert-parallel ranks are split evenly over
the ``W`` processes; process p drives ranks ``[p*n/W, (p+1)*n/W)``. The
pointer tables the engine reads are indexed by global rank.
"""
from __future__ import annotations

import ctypes
from typing import Callable, Dict, List

from . import _lib

BUFFERS = ("recv", "ret", "ctr_d", "ctr_c", "counts2", "xflag")
OPTIONAL = ("meta_recv", "a_g", "cnt_e2", "ginfo",  # present when ranks host several experts
            "landed")  # one expert per rank: arrival credits of the arrival-driven expert GEMM


def _names(layer) -> tuple:
    return BUFFERS + tuple(b for b in OPTIONAL if getattr(layer, b, None) is not None)


def _strides(layer) -> Dict[str, int]:
    """Byte distance between consecutive ranks inside one process's buffer."""
    H = layer.cfg.hidden
    # counts2 / xflag: one per process (every rank of a process maps to its base)
    return {"recv": layer.cap * H * 2, "ret": layer.ret_stride * H * 2, "ctr_d": 8, "ctr_c": 8,
            "counts2": 0, "xflag": 0,
            "meta_recv": layer.cap * layer.meta_bytes, "a_g": 0, "cnt_e2": 0, "ginfo": 0,
            "landed": layer.n * 4}


def local_export(layer) -> dict:
    """IPC handles + offsets of this process's peer-visible buffers."""
    L = _lib.load()
    nb = L.aurora_ipc_handle_bytes()
    out = {"rank_base": layer.rank_base, "n_local": layer.n_local}
    for name in _names(layer):
        t = getattr(layer, name)
        h = ctypes.create_string_buffer(nb)
        off = ctypes.c_int64(0)
        _lib.check(L.aurora_ipc_get(t.data_ptr(), h, ctypes.byref(off)), "aurora_ipc_get")
        out[name] = (bytes(h.raw), int(off.value))
    return out


def assemble_peer_tables(exports: List[dict], my_process: int, n: int, strides: Dict[str, int],
                         local_ptrs: Dict[str, int], opener: Callable[[bytes, int], int]) -> Dict[str, list]:
    """Per buffer, the address of every global rank's region as seen from this
    process: local regions from ``local_ptrs``, remote ones through ``opener``
    (CUDA IPC in production; injectable for the CPU tests)."""
    names = [b for b in BUFFERS + OPTIONAL if b in exports[0]]
    tables = {name: [0] * n for name in names}
    covered = [False] * n
    for p, ex in enumerate(exports):
        for name in names:
            if p == my_process:
                base = local_ptrs[name]
            else:
                handle, off = ex[name]
                base = opener(handle, off)
            for r in range(ex["n_local"]):
                tables[name][ex["rank_base"] + r] = base + r * strides[name]
        for r in range(ex["n_local"]):
            if covered[ex["rank_base"] + r]:
                raise ValueError(f"rank {ex['rank_base'] + r} exported twice")
            covered[ex["rank_base"] + r] = True
    if not all(covered):
        raise ValueError("some ranks have no owner process")
    return tables


def connect_peers(layer, group=None) -> None:
    """Collective: exchange IPC handles and point the layer's engine tables at
    the peers' buffers. Call once after constructing the layer on every process."""
    import torch.distributed as dist

    L = _lib.load()
    mine = local_export(layer)
    world = dist.get_world_size(group)
    exports: List[dict] = [None] * world  # type: ignore[list-item]
    dist.all_gather_object(exports, mine, group=group)
    me = dist.get_rank(group)

    def opener(handle: bytes, off: int) -> int:
        out = ctypes.c_void_p(0)
        _lib.check(L.aurora_ipc_open(ctypes.create_string_buffer(handle, len(handle)), off, ctypes.byref(out)),
                   "aurora_ipc_open")
        return int(out.value)

    local = {name: getattr(layer, name).data_ptr() for name in _names(layer)}
    tables = assemble_peer_tables(exports, me, layer.n, _strides(layer), local, opener)
    layer._peers = tables
    layer._tables_for(layer.x, tables)
    dist.barrier(group)
