"""Multi-process host logic of the multi-GPU layer on CPU (gloo, world size 2):
the IPC-handle exchange and the per-rank peer pointer tables the engine reads."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    import torch.distributed as dist
    from paper_2410_17043_b200.dist import BUFFERS, assemble_peer_tables
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n_local = n // world
    # fake "exports": handle bytes encode (process, buffer); offsets are per buffer
    mine = {"rank_base": rank * n_local, "n_local": n_local}
    for b, name in enumerate(BUFFERS):
        mine[name] = (bytes([rank, b]) * 32, 64 * (b + 1))
    exports = [None] * world
    dist.all_gather_object(exports, mine)
    strides = {"recv": 1 << 20, "ret": 1 << 16, "ctr_d": 4, "ctr_c": 4, "counts2": 0, "xflag": 0}
    local = {name: 0x7000_0000 + rank * 0x100_0000 + b * 0x10_0000 for b, name in enumerate(BUFFERS)}

    def opener(handle, off):
        p, b = handle[0], handle[1]
        return 0x9000_0000 + p * 0x100_0000 + b * 0x10_0000 + off

    tables = assemble_peer_tables(exports, rank, n, strides, local, opener)
    q.put((rank, tables))
    dist.barrier()
    dist.destroy_process_group()


def test_peer_tables_two_processes():
    n, world = 8, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2410_17043_b200.dist import BUFFERS
    strides = {"recv": 1 << 20, "ret": 1 << 16, "ctr_d": 4, "ctr_c": 4, "counts2": 0, "xflag": 0}
    for me in range(world):
        t = got[me]
        for b, name in enumerate(BUFFERS):
            for g in range(n):
                owner, r = divmod(g, n // world)
                if owner == me:
                    base = 0x7000_0000 + me * 0x100_0000 + b * 0x10_0000
                else:
                    base = 0x9000_0000 + owner * 0x100_0000 + b * 0x10_0000 + 64 * (b + 1)
                assert t[name][g] == base + r * strides[name], (me, name, g)


def test_assemble_rejects_gaps_and_overlaps():
    from paper_2410_17043_b200.dist import BUFFERS, assemble_peer_tables
    mk = lambda base, nl: {"rank_base": base, "n_local": nl, **{b: (b"\0" * 64, 0) for b in BUFFERS}}
    strides = {b: 4 for b in BUFFERS}
    local = {b: 0 for b in BUFFERS}
    with pytest.raises(ValueError):
        assemble_peer_tables([mk(0, 2), mk(3, 1)], 0, 4, strides, local, lambda h, o: 0)
    with pytest.raises(ValueError):
        assemble_peer_tables([mk(0, 2), mk(1, 2)], 0, 4, strides, local, lambda h, o: 0)
