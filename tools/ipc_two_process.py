"""The multi-GPU path through real CUDA IPC on one device: two (or P) processes
(gloo for the host collectives), each driving 8 / P of the 8 ranks (P = 8: one
rank per process, the N = 8 deployment's shape), peer tables
from dist.connect_peers (cudaIpcGetMemHandle / OpenMemHandle), system-scope
flags. Without MPS the two processes' kernels time-slice, so the engines
progress only across context switches: this checks correctness, not speed.
Output compared with a single-process loopback run of the same layer.
Usage: python tools/ipc_two_process.py [e8|e16] [P]"""
import os, socket, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.multiprocessing as mp

CFG = dict(hidden=256, ffn=256, experts=8, top_k=2, tokens=1024, ranks=8, skew=1.0, seed=3)
if len(sys.argv) > 1 and sys.argv[1] == "e16":  # several experts per rank: the metadata plane crosses too
    CFG.update(experts=16, top_k=4)
NPROC = int(sys.argv[2]) if len(sys.argv) > 2 else 2


def _port():
    s = socket.socket(); s.bind(("127.0.0.1", 0)); p = s.getsockname()[1]; s.close(); return p


def worker(rank, world, port, q, stream_schedule):
    import torch.distributed as dist
    from paper_2410_17043_b200 import dist as adist
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    cfg = MoEConfig(**CFG)
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
    nl = cfg.ranks // world
    layer = AuroraMoELayer(cfg, rank_base=nl * rank, n_local=nl, spin_limit=1 << 24)
    layer.stream_schedule = stream_schedule
    adist.connect_peers(layer)
    xs = x[rank * cfg.tokens // world:(rank + 1) * cfg.tokens // world].contiguous()
    t0 = time.time()
    outs = []
    for _ in range(2):  # twice: counters rearmed across processes
        outs.append(layer(xs).clone())
        torch.cuda.synchronize()
        layer.check_status()
    assert torch.equal(outs[0], outs[1])
    # by value (numpy bytes): a shared-memory tensor handle would need this process alive
    # until the parent has opened it
    q.put((rank, outs[1].cpu().view(torch.int16).numpy().tobytes(), time.time() - t0))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    cfg = MoEConfig(**CFG)
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
    ref = AuroraMoELayer(cfg)(x).cpu()
    torch.cuda.synchronize()
    ctx = mp.get_context("spawn")
    ok = True
    for stream_schedule in (False, True):
        q = ctx.Queue()
        port = _port()
        ps = [ctx.Process(target=worker, args=(r, NPROC, port, q, stream_schedule)) for r in range(NPROC)]
        for p_ in ps:
            p_.start()
        res = dict((r, (o, t)) for r, o, t in (q.get(timeout=300) for _ in range(NPROC)))
        for p_ in ps:
            p_.join(timeout=60)
        import numpy as np
        part = [torch.from_numpy(np.frombuffer(res[r][0], dtype=np.int16).copy()).view(torch.bfloat16)
                .view(cfg.tokens // NPROC, cfg.hidden) for r in range(NPROC)]
        out = torch.cat(part)
        same = torch.equal(out, ref)
        ok &= same
        print(f"{NPROC} processes via CUDA IPC (K2 {'overlapped' if stream_schedule else 'serial'}, E={cfg.experts}): "
              f"identical to loopback: {same} | seconds per process: {[round(res[r][1], 2) for r in range(NPROC)]}",
              flush=True)
    sys.exit(0 if ok else 1)
