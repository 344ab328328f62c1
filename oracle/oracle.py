"""TEST INFRASTRUCTURE ONLY -- Python face of the CPU oracle.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (the
``cpu_baseline`` leg and the ``--impl reference`` arm) may import this module.
The product package never does; it fails loudly without its CUDA library.

* ``build_schedule_oracle``: ctypes over ``sched_oracle.c``, the C restatement
  of ``moeplan.build_schedule`` (reference ``pkg/src/moeplan/commsched.py:291-324``),
  pinned bit-exact against fixtures produced by the reference itself
  (``tests/golden/gen_golden.py``).
* ``router_oracle`` / ``pack_oracle``: the router, traffic matrix
  (``core.py:75-117``) and token permutation, in the arithmetic order the
  device kernels are defined by (see ``router_oracle.c``).
* ``moe_layer_oracle``: fp32 SwiGLU experts + gate-weighted aggregation, the
  numerics reference for the combined layer output (no reference analogue:
  the reference models the FFN as ``LayerProfile.ffn_work_per_token``).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

STATUS_OK, STATUS_VALUE, STATUS_OVERFLOW, STATUS_NOMATCH = 0, 1, 2, 3


def build() -> str:
    """Compile the oracle (gcc, seconds). Idempotent."""
    srcs = [os.path.join(_HERE, f) for f in ("sched_oracle.c", "router_oracle.c", "Makefile")]
    if os.path.exists(_LIB_PATH) and all(os.path.getmtime(s) <= os.path.getmtime(_LIB_PATH) for s in srcs):
        return _LIB_PATH
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int)
        L.oracle_build_schedule.argtypes = [dp, dp, ctypes.c_int, ip, dp, ip, ip, dp, ip, dp, dp]
        L.oracle_build_schedule.restype = ctypes.c_int
        L.oracle_row_sums.argtypes = [dp, ctypes.c_int, dp]
        L.oracle_col_sums.argtypes = [dp, ctypes.c_int, dp]
        L.oracle_router_logits.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.oracle_router_topk.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_void_p, ctypes.c_void_p]
        _lib = L
    return _lib


def _p(a, t=ctypes.c_double):
    return a.ctypes.data_as(ctypes.POINTER(t))


def raw_phase_cap(n: int) -> int:
    return n * n - 2 * n + 2


def phase_cap(n: int) -> int:
    return max(1, 2 * n * n - 3 * n + 2)


class OracleDecompositionError(RuntimeError):
    pass


def build_schedule_oracle(d, bandwidths=None) -> dict:
    """Restated build_schedule. Returns a plain dict:
    ``raw``: list of (perm tuple, duration); ``phases``: list of
    (transfers tuple, duration); ``makespan`` (math.fsum, commsched.py:323);
    ``b_max``; ``t`` (the time-normalised matrix)."""
    d = np.ascontiguousarray(np.asarray(d, dtype=np.float64))
    n = d.shape[0]
    bw = np.ones(n) if bandwidths is None else np.ascontiguousarray(np.asarray(bandwidths, dtype=np.float64))
    R, P = raw_phase_cap(n), phase_cap(n)
    raw_perm = np.zeros(R * n, dtype=np.int32)
    raw_dur = np.zeros(R)
    phase_recv = np.zeros(P * n, dtype=np.int32)
    phase_dur = np.zeros(P)
    t = np.zeros((n, n))
    n_raw, n_ph = ctypes.c_int(0), ctypes.c_int(0)
    bmax = ctypes.c_double(0)
    st = lib().oracle_build_schedule(_p(d), _p(bw), n, _p(raw_perm, ctypes.c_int), _p(raw_dur),
                                     ctypes.byref(n_raw), _p(phase_recv, ctypes.c_int), _p(phase_dur),
                                     ctypes.byref(n_ph), _p(t), ctypes.byref(bmax))
    if st == STATUS_VALUE:
        raise ValueError("oracle: invalid traffic/time matrix")
    if st in (STATUS_OVERFLOW, STATUS_NOMATCH):
        raise OracleDecompositionError(f"oracle: decomposition failed ({st})")
    raw = [(tuple(int(v) for v in raw_perm[r * n:(r + 1) * n]), float(raw_dur[r])) for r in range(n_raw.value)]
    phases = []
    for k in range(n_ph.value):
        row = phase_recv[k * n:(k + 1) * n]
        phases.append((tuple((i, int(j)) for i, j in enumerate(row) if j >= 0), float(phase_dur[k])))
    return {
        "n": n,
        "raw": raw,
        "phases": phases,
        "phase_recv": phase_recv[: n_ph.value * n].reshape(-1, n).copy(),
        "makespan": math.fsum(p[1] for p in phases),
        "b_max": float(bmax.value),
        "t": t,
    }


def numpy_row_sums(m):
    m = np.ascontiguousarray(m, dtype=np.float64)
    out = np.zeros(m.shape[0])
    lib().oracle_row_sums(_p(m), m.shape[0], _p(out))
    return out


# ------------------------------ router / pack ------------------------------

def bf16_bits(t) -> np.ndarray:
    """torch bf16 tensor -> numpy uint16 bit pattern (host copy)."""
    import torch
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def router_oracle(x_bits: np.ndarray, w_bits: np.ndarray, bias: np.ndarray, k: int):
    """-> (logits f32 [T,E], topk_idx i32 [T,k], topk_w f32 [T,k])"""
    x_bits = np.ascontiguousarray(x_bits, dtype=np.uint16)
    w_bits = np.ascontiguousarray(w_bits, dtype=np.uint16)
    bias = np.ascontiguousarray(bias, dtype=np.float32)
    T, H = x_bits.shape
    E = w_bits.shape[0]
    assert H % 256 == 0
    logits = np.zeros((T, E), dtype=np.float32)
    lib().oracle_router_logits(x_bits.ctypes.data, w_bits.ctypes.data, bias.ctypes.data, T, H, E, logits.ctypes.data)
    idx = np.zeros((T, k), dtype=np.int32)
    wts = np.zeros((T, k), dtype=np.float32)
    lib().oracle_router_topk(logits.ctypes.data, T, E, k, idx.ctypes.data, wts.ctypes.data)
    return logits, idx, wts


def pack_oracle(topk_idx: np.ndarray, gpu_of_expert, n: int):
    """Traffic matrix and token permutation from the routing decisions.

    Token t lives on rank ``t // (T/n)`` (workload.py:59-61: one batch shard
    per GPU). A token goes to each distinct GPU among its k experts once
    (dedupe), in k-slot order. Returns ``counts[n,n]`` (diagonal = local
    tokens; TrafficMatrix drops it, core.py:95), ``lists[i][j]`` = ascending
    global token ids rank i sends to rank j, and ``pos[T,k]`` = index of the
    token inside ``lists[src][dst(slot)]``.
    """
    T, k = topk_idx.shape
    g = np.asarray(gpu_of_expert, dtype=np.int64)
    Tr = T // n
    counts = np.zeros((n, n), dtype=np.int64)
    lists = [[[] for _ in range(n)] for _ in range(n)]
    pos = np.zeros((T, k), dtype=np.int32)
    for t in range(T):
        i = t // Tr
        seen = {}
        for s in range(k):
            j = int(g[topk_idx[t, s]])
            if j not in seen:
                seen[j] = len(lists[i][j])
                lists[i][j].append(t)
                counts[i, j] += 1
            pos[t, s] = seen[j]
    return counts, lists, pos


def _f32(w):
    if hasattr(w, "detach"):  # torch tensor (e.g. bf16 weights kept compact on the host)
        return w.detach().float().numpy()
    return np.asarray(w, dtype=np.float32)


def bf16_round(a) -> np.ndarray:
    """fp32 -> nearest bf16 (ties to even), returned as fp32: the rounding the
    kernels apply when they store h and y (``__float2bfloat16_rn``)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    out = r.astype(np.uint32).view(np.float32)
    return np.where(np.isnan(a), a, out)


def moe_layer_oracle(x: np.ndarray, topk_idx, topk_w, w1, w3, w2, emulate_bf16: bool = False,
                     gpu_of_expert=None) -> np.ndarray:
    """fp32 SwiGLU MoE: out[t] = sum_s w[t,s] * W2_e (silu(W1_e x) * W3_e x).
    x [T,H] float32; w1/w3 [E][F,H], w2 [E][H,F]: arrays or per-expert
    sequences (numpy or torch, converted to fp32 one expert at a time).

    ``emulate_bf16``: round where the device path stores bf16 -- the SwiGLU
    intermediate h, the expert output y, and (with ``gpu_of_expert`` and
    several experts per rank) the per-(token, rank) pre-reduced row
    ``bf16(sum_s w_s y_s)`` the expert rank returns (arithmetic
    contracts); the final sum stays fp32 in slot order, rounded to bf16."""
    T, H = x.shape
    E = len(w1)
    k = topk_idx.shape[1]
    y_slot = np.zeros((T, k, H), dtype=np.float32) if emulate_bf16 else None
    out = np.zeros((T, H), dtype=np.float32)
    for e in range(E):
        rows, slots = np.nonzero(topk_idx == e)
        if rows.size == 0:
            continue
        xe = x[rows]
        g = xe @ _f32(w1[e]).T
        u = xe @ _f32(w3[e]).T
        h = (g / (1.0 + np.exp(-g))) * u
        if emulate_bf16:
            y_slot[rows, slots] = bf16_round(bf16_round(h) @ _f32(w2[e]).T)
        else:
            out[rows] += topk_w[rows, slots][:, None] * (h @ _f32(w2[e]).T)
    if not emulate_bf16:
        return out
    return aggregate_oracle(y_slot, topk_idx, topk_w, gpu_of_expert)


def aggregate_oracle(y_slot, topk_idx, topk_w, gpu_of_expert=None) -> np.ndarray:
    """Combine + aggregation of bf16 expert outputs ``y_slot[T,k,H]`` (one per
    (token, slot)) in the device path's order: one expert per rank -> fp32
    ``sum_s w_s y_s`` in slot order; several experts per rank -> each expert
    rank first pre-reduces its slots to ``bf16(sum w_s y_s)``, the sender sums
    those rows (first-slot order). Rounded to bf16."""
    y_slot = np.asarray(y_slot, dtype=np.float32)
    T, k, H = y_slot.shape
    w = np.asarray(topk_w, dtype=np.float32)
    out = np.zeros((T, H), dtype=np.float32)
    E = None if gpu_of_expert is None else len(gpu_of_expert)
    G = 1 if gpu_of_expert is None else E // len(set(int(g) for g in gpu_of_expert))
    if G == 1:
        for s in range(k):
            out += w[:, s:s + 1] * y_slot[:, s]
        return bf16_round(out)
    rank = np.asarray(gpu_of_expert)[np.asarray(topk_idx)]   # [T, k]
    for t in range(T):
        acc = np.zeros(H, dtype=np.float32)
        for r in dict.fromkeys(rank[t].tolist()):             # ranks in first-slot order
            part = np.zeros(H, dtype=np.float32)
            for s in range(k):
                if rank[t, s] == r:
                    part += w[t, s] * y_slot[t, s]
            acc += bf16_round(part)
        out[t] = acc
    return bf16_round(out)


def row_errors(got, ref):
    """Per-row relative L2 error ||got_t - ref_t|| / ||ref_t|| and the max
    elementwise error over max|ref| (the two bounds the layer tests assert)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    num = np.linalg.norm(got - ref, axis=1)
    den = np.maximum(np.linalg.norm(ref, axis=1), 1e-30)
    return num / den, float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))
