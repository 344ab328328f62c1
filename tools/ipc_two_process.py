"""The multi-GPU path through real CUDA IPC on one device: two processes
(gloo for the host collectives), each driving 4 of the 8 ranks, peer tables
from dist.connect_peers (cudaIpcGetMemHandle / OpenMemHandle), system-scope
flags. Without MPS the two processes' kernels time-slice, so the engines
progress only across context switches: this checks correctness, not speed.
Output compared with a single-process loopback run of the same layer.
Usage: python tools/ipc_two_process.py"""
import os, socket, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.multiprocessing as mp

CFG = dict(hidden=256, ffn=256, experts=8, top_k=2, tokens=1024, ranks=8, skew=1.0, seed=3)
if len(sys.argv) > 1 and sys.argv[1] == "e16":  # several experts per rank: the metadata plane crosses too
    CFG.update(experts=16, top_k=4)


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
    layer = AuroraMoELayer(cfg, rank_base=4 * rank, n_local=4, spin_limit=1 << 24)
    layer.stream_schedule = stream_schedule
    adist.connect_peers(layer)
    xs = x[rank * cfg.tokens // 2:(rank + 1) * cfg.tokens // 2].contiguous()
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
        ps = [ctx.Process(target=worker, args=(r, 2, port, q, stream_schedule)) for r in range(2)]
        for p_ in ps:
            p_.start()
        res = dict((r, (o, t)) for r, o, t in (q.get(timeout=300) for _ in range(2)))
        for p_ in ps:
            p_.join(timeout=60)
        import numpy as np
        half = [torch.from_numpy(np.frombuffer(res[r][0], dtype=np.int16).copy()).view(torch.bfloat16)
                .view(cfg.tokens // 2, cfg.hidden) for r in (0, 1)]
        out = torch.cat(half)
        same = torch.equal(out, ref)
        ok &= same
        print(f"two processes via CUDA IPC (K2 {'overlapped' if stream_schedule else 'serial'}, E={cfg.experts}): "
              f"identical to loopback: {same} | seconds per process: {[round(res[r][1], 2) for r in (0, 1)]}",
              flush=True)
    sys.exit(0 if ok else 1)
